"""`python -m paper_2102_10485_b200 {train,sample,bench}` — the reference
driver's train / sample / bench commands (src/run.cpp:363-444 cmd_train,
531-556 cmd_sample, 516-529 cmd_bench) on the device path, writing the same
artifacts:

  train   <out>/checkpoints/class_<k>.bin   (reference checkpoint format)
          <out>/losses.csv                  mode,class_id,step,j_d,j_g,d_real_mean,d_fake_mean (%.17g)
          <out>/manifest.json               format "partgan-manifest": k, priors, base_seed, config, workers
  sample  <out>.npz                         mixture_sample over the manifest's checkpoints (partition.cpp:182-227)
  bench   <out>/scaling.csv                 k,wall_clock_s,max_worker_s,cores_used,oversubscribed (weak scaling
                                            over K labels at a fixed per-label workload, bench_weak_scaling)
`train --config run.json` reads the reference's JSON RunConfig (runconfig.py:
unknown keys rejected, the reference's validation messages; ConfigError exits 2).

Distributed mode only (one independent pair per label, the paper's method);
datasets are the seeded cosine-field synthetic sets of BASELINE.json (no
MNIST / CIFAR files exist in this environment).  Labels shard over ranks as
contiguous blocks when launched under torchrun (one process per GPU); rank 0
writes the losses and the manifest after gathering the per-rank rows.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from . import _native as N
from .archs import baseline_arch, with_bn
from .runconfig import ConfigError, load_config_file
from .trainer import AdamConfig, GroupSpec, LabelGroup, derive_seed, estimate_priors

MATH = {"fp32": N.MATH_FP32_SIMT, "tf32x3": N.MATH_TF32X3, "tf32": N.MATH_TF32, "bf16": N.MATH_BF16}


def _rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def apply_config(a: argparse.Namespace) -> None:
    """RunConfig (JSON) -> the train arguments (run.cpp:363-404 reads the same fields)"""
    cfg = load_config_file(a.config)
    syn = cfg.dataset.synthetic
    a.arch, a.labels, a.per_label, a.epochs, a.batch = cfg.resolved_arch(), syn.k, syn.per_class_n, cfg.epochs, cfg.batch_size
    a.lr, a.beta1, a.beta2, a.adam_eps, a.seed, a.data_seed = cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps, cfg.seed, syn.seed
    a.clamp, a.init_std, a.bn_eps, a.bn_momentum, a.d_z = cfg.clamp, cfg.init_std, cfg.bn_eps, cfg.bn_momentum, cfg.d_z
    if a.out is None:
        a.out = cfg.out_dir


def cmd_train(a: argparse.Namespace) -> int:
    if a.config:
        apply_config(a)
    if a.out is None:
        raise ConfigError("train: --out (or out_dir in --config) is required")
    rank, world, local = _rank_world()
    arch = with_bn(baseline_arch(a.arch, a.d_z), a.bn_eps, a.bn_momentum)
    lo, hi = a.labels * rank // world, a.labels * (rank + 1) // world
    labels = list(range(lo, hi))
    grp = LabelGroup(GroupSpec(arch=arch, class_ids=labels, batch=a.batch, epochs=a.epochs, per_label=a.per_label,
                               base_seed=a.seed,
                               adam=AdamConfig(lr=a.lr, beta1=a.beta1, beta2=a.beta2, eps=a.adam_eps),
                               clamp=a.clamp, init_std=a.init_std, math=MATH[a.math], device=local))
    grp.generate_dataset(a.data_seed)
    t0 = time.time()
    while grp.train_steps(64) > 0:
        pass
    dur = time.time() - t0
    os.makedirs(os.path.join(a.out, "checkpoints"), exist_ok=True)
    rows, workers = [], []
    for i, k in enumerate(labels):
        rel = f"checkpoints/class_{k}.bin"
        grp.save_checkpoint(i, os.path.join(a.out, rel))
        reps = grp.reports(i)
        workers.append({"class_id": k, "seed": derive_seed(a.seed, k), "checkpoint": rel, "steps": len(reps),
                        "duration_s": dur, "start_s": 0.0, "end_s": dur, "rank": rank})
        for s, r in enumerate(reps):
            rows.append(f"distributed_cgan,{k},{s},{r[0]:.17g},{r[1]:.17g},{r[2]:.17g},{r[3]:.17g}\n")
    grp.close()
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("gloo")
        gathered = [None] * world
        dist.all_gather_object(gathered, (rows, workers))
        rows = [r for g in gathered for r in g[0]]
        workers = [w for g in gathered for w in g[1]]
    if rank == 0:
        with open(os.path.join(a.out, "losses.csv"), "w") as f:
            f.write("mode,class_id,step,j_d,j_g,d_real_mean,d_fake_mean\n")
            f.writelines(rows)
        counts, probs = estimate_priors((k, range(a.per_label)) for k in range(a.labels))
        manifest = {
            "format": "partgan-manifest", "mode": "distributed_cgan", "k": a.labels, "base_seed": a.seed,
            "priors": {"counts": counts.tolist(), "probabilities": probs.tolist()},
            "config": {"arch": f"c{a.arch}", "epochs": a.epochs, "batch_size": a.batch, "per_label": a.per_label,
                       "lr": a.lr, "beta1": a.beta1, "beta2": a.beta2, "d_z": arch.d_z, "data_seed": a.data_seed,
                       "dataset": "synthetic cosine fields (BASELINE.json)", "math": a.math, "world_size": world},
            "workers": sorted(workers, key=lambda w: w["class_id"]), "coordinator_duration_s": dur,
        }
        with open(os.path.join(a.out, "manifest.json"), "w") as f:
            f.write(json.dumps(manifest, indent=2) + "\n")
        print(f"trained {a.labels} worker(s) in {dur:.17g} s; manifest: {os.path.join(a.out, 'manifest.json')}")
    return 0


def cmd_sample(a: argparse.Namespace) -> int:
    with open(a.manifest) as f:
        man = json.load(f)
    if man.get("format") != "partgan-manifest":
        raise SystemExit(f"{a.manifest} is not a partgan manifest")
    cfg = man["config"]
    arch = baseline_arch(int(cfg["arch"].lstrip("c")))
    root = os.path.dirname(os.path.abspath(a.manifest))
    ws = man["workers"]
    grp = LabelGroup(GroupSpec(arch=arch, class_ids=[w["class_id"] for w in ws], batch=cfg["batch_size"],
                               per_label=cfg["per_label"], math=MATH[cfg.get("math", "tf32x3")]))
    for i, w in enumerate(ws):
        grp.load_checkpoint(i, os.path.join(root, w["checkpoint"]))
    samples, ids = grp.mixture_sample(np.asarray(man["priors"]["probabilities"]), a.n, a.seed)
    grp.close()
    np.savez(a.out, samples=samples, class_ids=np.asarray([ws[i]["class_id"] for i in ids]))
    print(f"wrote {a.n} samples to {a.out}")
    return 0


def cmd_bench(a: argparse.Namespace) -> int:
    """cmd_bench / bench_weak_scaling (run.cpp:516-529, partition.cpp:229-271) on
    the device path: for each K, K labels of the BASELINE architecture train a
    fixed per-label workload (per_label images, epochs, batch) as one label
    group; wall clock of the training loop (device-synchronised).  The group
    runs every label in lockstep, so max_worker_s = wall_clock_s; cores_used
    is the GPU count; nothing is oversubscribed."""
    import torch
    arch = baseline_arch(a.arch)
    rows = []
    for k in [int(x) for x in a.k.split(",")]:
        if k < 1:
            raise ConfigError("bench_weak_scaling: K must be >= 1")
        grp = LabelGroup(GroupSpec(arch=arch, class_ids=list(range(k)), batch=a.batch, epochs=a.epochs,
                                   per_label=a.per_label, base_seed=a.seed, math=MATH[a.math]))
        grp.generate_dataset(derive_seed(a.seed, k))
        grp.sync()
        torch.cuda.synchronize()
        t0 = time.time()
        while grp.train_steps(64) > 0:
            pass
        grp.sync()
        wall = time.time() - t0
        grp.close()
        rows.append((k, wall, wall, 1, 0))
        print(f"K={k} wall={wall:.17g}s max_worker={wall:.17g}s")
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "scaling.csv"), "w") as f:
        f.write("k,wall_clock_s,max_worker_s,cores_used,oversubscribed\n")
        for r in rows:
            f.write(f"{r[0]},{r[1]:.17g},{r[2]:.17g},{r[3]},{r[4]}\n")
    return 0


def main(argv: list[str] | None = None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_2102_10485_b200")
    sub = p.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("train", help="train one (G, D) pair per label (run.cpp:363-444)")
    t.add_argument("--arch", type=int, default=1, choices=[1, 2, 3, 4], help="BASELINE.json config c1..c4")
    t.add_argument("--labels", type=int, default=10)
    t.add_argument("--per-label", type=int, default=256)
    t.add_argument("--epochs", type=int, default=1)
    t.add_argument("--batch", type=int, default=64)
    t.add_argument("--lr", type=float, default=2e-4)
    t.add_argument("--beta1", type=float, default=0.5)
    t.add_argument("--beta2", type=float, default=0.999)
    t.add_argument("--seed", type=int, default=1, help="base seed: worker seed = derive_seed(seed, class_id)")
    t.add_argument("--data-seed", type=int, default=2024)
    t.add_argument("--math", choices=list(MATH), default="tf32x3")
    t.add_argument("--out", default=None)
    t.add_argument("--config", default=None, help="the reference's JSON RunConfig (unknown keys rejected)")
    t.set_defaults(adam_eps=1e-8, clamp=1e-7, init_std=0.02, bn_eps=1e-5, bn_momentum=0.1, d_z=100)
    b = sub.add_parser("bench", help="weak scaling over K labels -> scaling.csv (run.cpp:516-529)")
    b.add_argument("--out", required=True)
    b.add_argument("--k", default="1,2,4,8")
    b.add_argument("--arch", type=int, default=4, choices=[1, 2, 3, 4])
    b.add_argument("--per-label", type=int, default=64)
    b.add_argument("--batch", type=int, default=32)
    b.add_argument("--epochs", type=int, default=1)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--math", choices=list(MATH), default="tf32x3")
    s = sub.add_parser("sample", help="mixture samples from a trained run (run.cpp:531-556)")
    s.add_argument("--manifest", required=True)
    s.add_argument("--n", type=int, default=64)
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--out", required=True)
    a = p.parse_args(argv)
    try:
        return {"train": cmd_train, "sample": cmd_sample, "bench": cmd_bench}[a.cmd](a)
    except ConfigError as e:  # tools/main.cpp: ConfigError -> exit 2
        print(f"config error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
