"""`python -m paper_2102_10485_b200 {train,sample}` — the reference driver's
train / sample commands (src/run.cpp:363-444 cmd_train, 531-556 cmd_sample)
on the device path, writing the same artifacts:

  train   <out>/checkpoints/class_<k>.bin   (reference checkpoint format)
          <out>/losses.csv                  mode,class_id,step,j_d,j_g,d_real_mean,d_fake_mean (%.17g)
          <out>/manifest.json               format "partgan-manifest": k, priors, base_seed, config, workers
  sample  <out>.npz                         mixture_sample over the manifest's checkpoints (partition.cpp:182-227)

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
from .archs import baseline_arch
from .trainer import AdamConfig, GroupSpec, LabelGroup, derive_seed

MATH = {"fp32": N.MATH_FP32_SIMT, "tf32x3": N.MATH_TF32X3, "tf32": N.MATH_TF32}


def _rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def cmd_train(a: argparse.Namespace) -> int:
    rank, world, local = _rank_world()
    arch = baseline_arch(a.arch)
    lo, hi = a.labels * rank // world, a.labels * (rank + 1) // world
    labels = list(range(lo, hi))
    grp = LabelGroup(GroupSpec(arch=arch, class_ids=labels, batch=a.batch, epochs=a.epochs, per_label=a.per_label,
                               base_seed=a.seed, adam=AdamConfig(lr=a.lr, beta1=a.beta1, beta2=a.beta2),
                               math=MATH[a.math], device=local))
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
        total = a.labels * a.per_label
        manifest = {
            "format": "partgan-manifest", "mode": "distributed_cgan", "k": a.labels, "base_seed": a.seed,
            "priors": {"counts": [a.per_label] * a.labels, "probabilities": [a.per_label / total] * a.labels},
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
    t.add_argument("--out", required=True)
    s = sub.add_parser("sample", help="mixture samples from a trained run (run.cpp:531-556)")
    s.add_argument("--manifest", required=True)
    s.add_argument("--n", type=int, default=64)
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--out", required=True)
    a = p.parse_args(argv)
    return cmd_train(a) if a.cmd == "train" else cmd_sample(a)


if __name__ == "__main__":
    sys.exit(main())
