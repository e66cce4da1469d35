"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`)
per kernel: launches, total time, share.  Usage:
    python scripts/summarize_launches.py gpurun_out/launches.csv [steps]
`steps` = training steps covered by the capture (to print per-step times)."""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = re.sub(r"\(.*\)$", "", name)  # drop the argument list
    return name.replace("pg::", "")


def main():
    path = sys.argv[1]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        t = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        t_ns = t * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), r["Grid Size"], t_ns))
    agg = defaultdict(lambda: [0, 0.0])
    for k, _, t in rows:
        agg[k][0] += 1
        agg[k][1] += t
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total / 1e6:.2f} ms total ({total / 1e6 / steps:.2f} ms per step over {steps:g} steps)")
    print(f"| kernel | launches | total ms | ms/step | share |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t / 1e6:.3f} | {t / 1e6 / steps:.3f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    main()
