"""Top warp-stall SASS lines of an ncu --page source --csv export (.csv or .csv.gz)."""
import csv, gzip, sys
f = sys.argv[1]
rows = list(csv.reader((gzip.open if f.endswith(".gz") else open)(f, "rt")))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
si, ei = idx["Warp Stall Sampling (All Samples)"], idx["Instructions Executed"]
data = []
for r in rows[2:]:
    try:
        data.append((float(r[si] or 0), float(r[ei] or 0), r[idx["Source"]].strip(), r[0]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0] / tot * 100:5.1f}% exec={d[1]:>10.0f} {d[3][-5:]} {d[2][:100]}")
print("total instructions executed", sum(d[1] for d in data))
