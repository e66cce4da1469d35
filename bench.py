#!/usr/bin/env python
"""Benchmark: GAN train images/sec (full G+D step, whole box), weak scaling.

Workload (BASELINE.json configs[4], the sweep the metric is quoted on): the
64x64x3 architecture (c4), 125 labels per GPU, per-label batch 32, 1280
cosine-field images per label (synthetic), Adam 2e-4.  One
step advances every resident label by one train_step (reference
gan.cpp:136-182); one "image" is one real image through that step.

  python bench.py [--gpus N --steps K --warmup W]           # our arm
  python bench.py --impl reference [...]                    # CPU reference arm (oracle port)
Multi-GPU: launched by torchrun, one rank per GPU; labels are sharded in
contiguous blocks of 125 per rank, no collective inside the training loop,
one NCCL gather of 64 generated samples per label + loss statistics at the end.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MATH = {"fp32": 0, "tf32x3": 1, "tf32": 2, "bf16": 3}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--cfg", type=int, default=4)
    p.add_argument("--labels-per-gpu", type=int, default=125)
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--per-label", type=int, default=1280)
    p.add_argument("--math", choices=list(MATH), default="tf32x3")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-steps", type=int, default=1)
    p.add_argument("--gather-samples", type=int, default=64)
    return p.parse_args()


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def measured_peaks() -> dict:
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def cpu_baseline_run(cfg: int, batch: int, steps: int, cores: int) -> dict:
    """The reference algorithm (oracle port, f64 = the reference precision) on
    the host cores: `cores` labels, one worker thread each, `steps` steps."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    lib = oracle_lib.lib()
    secs = lib.or_bench_steps(cfg, 64, cores, batch, steps, cores)
    if secs <= 0:
        raise RuntimeError("cpu baseline failed: " + lib.or_last_error().decode())
    imgs = cores * batch * steps
    return {"value": imgs / secs, "unit": "images/s", "cores": cores, "kind": "port",
            "sample": f"{cores} labels x {steps} step(s) x batch {batch} of config c{cfg} (f64, oracle port of the "
                      f"reference per-sample im2col+GEMM path, one worker thread per label)",
            "seconds": secs}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = cpu_cores()
    for _ in range(args.warmup):
        cpu_baseline_run(args.cfg, args.batch, 1, cores)
    times = []
    for _ in range(args.steps):
        r = cpu_baseline_run(args.cfg, args.batch, 1, cores)
        times.append(r["seconds"])
    imgs = cores * args.batch * args.steps
    value = imgs / sum(times)
    from paper_2102_10485_b200.archs import baseline_arch
    line = {
        "impl": "reference", "metric": "GAN train images/sec (G+D step, whole box)", "value": value,
        "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * sum(times) / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (cosine fields)",
        # the same workload as our arm's line; the CPU times a bounded sample of it per step
        "config": {"workload": f"c{args.cfg} arch sweep: {args.labels_per_gpu} labels/GPU, per-label batch "
                               f"{args.batch}, {'x'.join(map(str, baseline_arch(args.cfg).image))}",
                   "labels_per_gpu": args.labels_per_gpu, "global_batch": args.gpus * args.labels_per_gpu * args.batch,
                   "per_label": args.per_label, "math": "f64 (reference CPU algorithm)",
                   "parallelism": f"one worker thread per label, {cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": f"{cores} labels x 1 step x batch {args.batch} per timed step (of the "
                                   f"{args.labels_per_gpu} labels/GPU workload; the f64 oracle port of the "
                                   f"reference per-sample im2col+GEMM path, one worker thread per label)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run directly (no WORLD_SIZE in the environment):
    launch N ranks, one per GPU, through torch.distributed.run on 127.0.0.1
    exactly as the driver would, with NCCL_DEBUG=INFO (INIT) so the rank count
    NCCL brings up is visible.  Rank 0's JSON line is the output."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2102_10485_b200 import GroupSpec, LabelGroup, _native as N, algorithmic_flops_per_image, baseline_arch
    from paper_2102_10485_b200.build import build
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    lib = N.lib()

    arch = baseline_arch(args.cfg)
    Lg = args.labels_per_gpu
    labels = list(range(rank * Lg, (rank + 1) * Lg))
    steps_per_epoch = -(-args.per_label // args.batch)
    total_steps = args.warmup + args.steps + 2
    epochs = -(-total_steps // steps_per_epoch) + 1
    threads = max(1, min(16, cpu_cores() // max(1, world)))
    grp = LabelGroup(GroupSpec(arch=arch, class_ids=labels, batch=args.batch, epochs=epochs,
                               per_label=args.per_label, base_seed=1, math=MATH[args.math], threads=threads,
                               device=local))
    t0 = time.time()
    grp.generate_dataset(2024)
    gen_s = time.time() - t0

    # warm-up
    grp.train_steps(args.warmup)
    grp.sync()

    # timed region: barrier + sync on both sides, device time from CUDA events
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.pg_launch_count()
    sampler.start()
    w0 = time.time()
    ran = grp.train_steps(args.steps)
    dev_ms = grp.last_device_ms()
    wall_ms = (time.time() - w0) * 1000
    clocks = sampler.stop()
    launches = lib.pg_launch_count() - launches0
    torch.cuda.synchronize()
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    # exact images in the timed steps: an epoch ends with a partial tail batch
    # when per_label is not a multiple of the batch (run_worker, partition.cpp:92-96)
    imgs = world * Lg * images_in_steps(args.warmup, ran, args.per_label, args.batch)
    value = imgs / (max_ms / 1000.0)

    # per-kernel timing pass (separate from the headline): implicit-GEMM share,
    # per-layer tensor classes and per-kernel HBM classes (CUDA events around
    # every launch of one step)
    lib.pg_kernel_timing(1)
    grp.train_steps(1)
    grp.sync()
    gemm_ms = C_double_out(lib.pg_kernel_timing_read)
    import ctypes as C
    n_rep = lib.pg_kernel_timing_report(None, 0)
    rep_buf = C.create_string_buffer(n_rep + 1)
    lib.pg_kernel_timing_report(rep_buf, n_rep + 1)
    lib.pg_kernel_timing(0)
    timing_lines = rep_buf.value.decode().splitlines()
    flops_img = algorithmic_flops_per_image(arch)
    step_flops = Lg * images_in_steps(args.warmup + ran, 1, args.per_label, args.batch) * flops_img
    peaks = measured_peaks()
    achieved = step_flops / (gemm_ms / 1000.0) / 1e12 if gemm_ms > 0 else None
    # denominator: this GPU's tcgen05 kind::tf32 dense rate, measured live by
    # the pair-MMA probe (the driver's MEASURED_PEAKS.json holds a bf16 figure)
    import ctypes as C
    tf32_peak = C.c_double(0.0)
    N.check(lib.pg_tc_tf32_peak(1 << 16, C.byref(tf32_peak)))
    tf32_peak = tf32_peak.value
    x3 = args.math == "tf32x3"
    # DRAM bytes of the step's implicit-GEMM launches, from the committed ncu launch list
    traffic = None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("gemm_dram_bytes_per_step")
    tensor_classes, hbm_classes = kernel_classes(timing_lines, tf32_peak, peaks["hbm_gbs"])
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": (achieved / tf32_peak) if achieved else None, "traffic": traffic,
                "traffic_unit": "bytes per step (all implicit-GEMM launches, ncu dram__bytes_read + write)",
                # 3xTF32 issues three MMAs per product: tensor-pipe occupancy is 3x the algorithmic fraction
                "pipe_frac": (achieved * (3 if x3 else 1) / tf32_peak) if achieved else None,
                "kernel": "implicit-GEMM (conv/convT/dense fwd, dgrad, wgrad), all launches of one step",
                "peak_basis": "measured live: pg_tc_tf32_peak (cta_group::2 M256 N256 K8 kind::tf32 MMAs "
                              "back to back on every SM pair)",
                "bf16_dense_driver": peaks["bf16_tflops"],
                "gemm_ms_per_step": gemm_ms, "gemm_share_of_step": gemm_ms / (max_ms / ran) if ran else None,
                "algorithmic_flop_per_image": flops_img,
                # per GEMM shape (all launches of one step): algorithmic TFLOP/s (padded channel
                # counts, e.g. RGB as 4) and its fraction of the tf32 peak; pipe_frac = 3x for 3xTF32
                "tensor_classes": tensor_classes,
                # HBM-bound kernels: algorithmic bytes / time vs the measured copy bandwidth
                "hbm_classes": hbm_classes, "hbm_peak_gbs": peaks["hbm_gbs"],
                "hbm_peak_basis": "MEASURED_PEAKS.json hbm_gbs (" + peaks["source"] + ")"}

    # e2e through the public API: host batch (pinned) -> train_step -> reports
    e2e = None
    if args.e2e_steps > 0:
        c, h, w = arch.image
        pinned = torch.empty((Lg, args.batch, c, h, w), dtype=torch.float32, pin_memory=True)
        host = pinned.numpy()
        rng = np.random.default_rng(rank)
        host[:] = rng.uniform(0, 1, host.shape).astype(np.float32)
        grp.train_step(host)  # warm the path
        if world > 1:
            dist.barrier()
        e0 = time.time()
        for _ in range(args.e2e_steps):
            grp.train_step(host)
        e_ms = (time.time() - e0) * 1000
        te = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = float(te.item())
        h2d = host.nbytes + 2 * Lg * args.batch * arch.d_z * 4
        e2e = {"value": world * Lg * args.batch * args.e2e_steps / (e_ms / 1000.0), "unit": "images/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": Lg * 4 * 8}

    # final gather: 64 generated samples per label + per-label loss statistics
    g0 = time.time()
    samples = torch.from_numpy(grp.generate(args.gather_samples, seed=99)).cuda()
    stats = torch.from_numpy(np.stack([grp.reports(l)[-1] for l in range(Lg)])).cuda()
    if world > 1:
        gs = [torch.empty_like(samples) for _ in range(world)] if rank == 0 else None
        gl = [torch.empty_like(stats) for _ in range(world)] if rank == 0 else None
        dist.gather(samples, gs, dst=0)
        dist.gather(stats, gl, dst=0)
        torch.cuda.synchronize()
    gather_s = time.time() - g0
    failed = int(grp.failed().sum())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_run(args.cfg, args.batch, args.cpu_steps, cpu_cores())

    if rank == 0:
        line = {
            "metric": "GAN train images/sec (G+D step, whole box)", "value": value, "unit": "images/s",
            "n_gpus": world, "steps": ran, "warmup": args.warmup, "ms_per_step": max_ms / max(ran, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"fp32": "fp32", "tf32x3": "fp32 (3xTF32 split on tcgen05)", "tf32": "tf32",
                      "bf16": "bf16 GEMM operands, fp32 accumulation"}[args.math],
            "data": "synthetic (per-label cosine fields + N(0,0.1^2) noise, 1280/label)",
            "config": {"workload": f"c{args.cfg} arch sweep: {Lg} labels/GPU, per-label batch {args.batch}, "
                                   f"{'x'.join(map(str, arch.image))}", "labels_per_gpu": Lg,
                       "global_batch": world * Lg * args.batch, "per_label": args.per_label, "math": args.math,
                       "parallelism": f"label-sharded x{world}",
                       "l2": "per-step working set (tens of GB) far exceeds the 126 MB L2; no flush needed"},
            "clocks": clocks, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "wall_ms": wall_ms, "dataset_gen_s": gen_s, "final_gather_s": gather_s, "failed_labels": failed,
        }
        print(json.dumps(line), flush=True)
    grp.close()
    if world > 1:
        dist.destroy_process_group()


def images_in_steps(first: int, n: int, per_label: int, batch: int) -> int:
    """images one label consumes in steps [first, first + n) of the worker protocol"""
    spe = -(-per_label // batch)
    total = 0
    for s in range(first, first + n):
        pos = s % spe
        total += min(batch, per_label - pos * batch)
    return total


def kernel_classes(lines, tf32_peak, hbm_gbs):
    """Aggregate the per-launch timing report of one step: implicit GEMMs by
    shape (algorithmic FLOP = 2 L M N K x phases), HBM-bound kernels by name
    (tag bytes = algorithmic bytes moved)."""
    gemm, hbm = {}, {}
    for line in lines:
        parts = line.split()
        if not parts:
            continue
        ms = float(parts[-1])
        kv = dict(x.split("=", 1) for x in parts[1:-1] if "=" in x)
        if parts[0] == "hbm":
            c = hbm.setdefault(parts[1], [0, 0.0, 0.0])
            c[0] += 1
            c[1] += ms
            c[2] += float(kv.get("bytes", 0))
        else:
            key = f"{parts[0]} M={kv['M']} N={kv['N']} K={kv['K']}" + (f" x{kv['phases']}" if kv.get("phases", "1") != "1" else "")
            flops = 2.0 * int(kv["L"]) * int(kv["M"]) * int(kv["N"]) * int(kv["K"]) * int(kv.get("phases", 1))
            c = gemm.setdefault(key, [0, 0.0, 0.0])
            c[0] += 1
            c[1] += ms
            c[2] += flops
    tc = [{"class": k, "launches": n, "ms_per_step": ms, "tflops": f / ms / 1e9 if ms else None,
           "frac": f / ms / 1e9 / tf32_peak if ms else None} for k, (n, ms, f) in gemm.items()]
    hc = [{"class": k, "launches": n, "ms_per_step": ms, "gbs": b / ms / 1e6 if ms else None,
           "frac": b / ms / 1e6 / hbm_gbs if ms else None} for k, (n, ms, b) in hbm.items()]
    tc.sort(key=lambda r: -r["ms_per_step"])
    hc.sort(key=lambda r: -r["ms_per_step"])
    return tc, hc


def C_double_out(fn) -> float:
    import ctypes as C
    out = C.c_double()
    fn(C.byref(out))
    return out.value


if __name__ == "__main__":
    main()
