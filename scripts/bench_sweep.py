"""BASELINE.json configs[1..4] sweep on one GPU: bench.py lines for the
per-label batch sweep 16/32/64/128 at 125 labels (c4 architecture) and for
the c1 / c2 / c3 configurations at their per-GPU label counts (c1, c2: all 10
labels on the GPU, B = 64; c3: 13 labels = the 8-GPU share of 100, B = 32).
Writes one JSON line per run to the output file.
    python scripts/bench_sweep.py [--out profiles/r02_sweep.jsonl] [--steps 10]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = [
    ("c4 sweep B=16", ["--cfg", "4", "--labels-per-gpu", "125", "--batch", "16"]),
    ("c4 sweep B=32", ["--cfg", "4", "--labels-per-gpu", "125", "--batch", "32"]),
    ("c4 sweep B=64", ["--cfg", "4", "--labels-per-gpu", "125", "--batch", "64"]),
    ("c4 sweep B=128", ["--cfg", "4", "--labels-per-gpu", "125", "--batch", "128"]),
    # the small configurations are launch-latency scale: 300 timed steps so the clock sampler sees the run
    ("c1 (10 labels, B=64)", ["--cfg", "1", "--labels-per-gpu", "10", "--batch", "64", "--per-label", "6000",
                             "--steps", "300"]),
    ("c2 (10 labels, B=64)", ["--cfg", "2", "--labels-per-gpu", "10", "--batch", "64", "--per-label", "5000",
                             "--steps", "300"]),
    ("c3 (13 labels/GPU, B=32)", ["--cfg", "3", "--labels-per-gpu", "13", "--batch", "32", "--per-label", "500",
                                 "--steps", "300"]),
]

p = argparse.ArgumentParser()
p.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweep.jsonl"))
p.add_argument("--steps", type=int, default=10)
p.add_argument("--only", default="")
args = p.parse_args()
with open(args.out, "a") as f:
    for name, extra in RUNS:
        if args.only and args.only not in name:
            continue
        steps = [] if "--steps" in extra else ["--steps", str(args.steps)]
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), *steps, "--warmup", "3", "--no-cpu-baseline", *extra]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        line = next((ln for ln in reversed(r.stdout.splitlines()) if ln.startswith("{")), None)
        rec = {"run": name, "rc": r.returncode}
        if line:
            d = json.loads(line)
            rec.update(value=d["value"], ms_per_step=d["ms_per_step"], e2e=d["e2e"]["value"] if d.get("e2e") else None,
                       clocks=d["clocks"], config=d["config"], roofline_frac=d["roofline"]["frac"],
                       pipe_frac=d["roofline"]["pipe_frac"], gpu_launches=d["gpu_launches"])
        else:
            rec["stderr"] = r.stderr[-2000:]
        print(json.dumps(rec), flush=True)
        f.write(json.dumps(rec) + "\n")
