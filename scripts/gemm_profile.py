"""Per-GEMM-launch device times of one training step (CUDA events around each
implicit-GEMM launch), with achieved TFLOP/s per launch.
  python scripts/gemm_profile.py [--labels 125] [--batch 32] [--cfg 4] [--math tf32x3]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10485_b200 import GroupSpec, LabelGroup, _native as N, baseline_arch

p = argparse.ArgumentParser()
p.add_argument("--labels", type=int, default=125)
p.add_argument("--batch", type=int, default=32)
p.add_argument("--cfg", type=int, default=4)
p.add_argument("--math", default="tf32x3")
args = p.parse_args()
math = {"fp32": 0, "tf32x3": 1, "tf32": 2}[args.math]
lib = N.lib()
grp = LabelGroup(GroupSpec(arch=baseline_arch(args.cfg), class_ids=list(range(args.labels)), batch=args.batch,
                           per_label=args.batch * 4, epochs=4, math=math))
grp.generate_dataset(1)
grp.train_steps(2)
grp.sync()
lib.pg_kernel_timing(1)
grp.train_steps(1)
grp.sync()
n = lib.pg_kernel_timing_report(None, 0)
buf = C.create_string_buffer(n + 1)
lib.pg_kernel_timing_report(buf, n + 1)
lib.pg_kernel_timing(0)
step_ms = None
grp.train_steps(1)
step_ms = grp.last_device_ms()
total = 0.0
rows = []
for line in buf.value.decode().splitlines():
    parts = line.split()
    ms = float(parts[-1])
    kv = dict(x.split("=") for x in parts[1:-1] if "=" in x)
    L, M, Nn, K, ph = (int(kv[k]) for k in ("L", "M", "N", "K", "phases"))
    flops = 2.0 * L * ph * M * Nn * K
    total += ms
    rows.append((ms, parts[0], line.rsplit(" ", 1)[0], flops / ms / 1e9))
print(f"step {step_ms:.2f} ms, GEMM total {total:.2f} ms ({100 * total / step_ms:.0f}%)")
for ms, kind, tag, tf in sorted(rows, reverse=True):
    print(f"{ms:8.3f} ms {tf:7.1f} TF/s  {tag}")
