"""DRAM bytes of the implicit-GEMM launches per training step, from an ncu
launch list with dram__bytes_read.sum / dram__bytes_write.sum
(scripts/round_evidence.sh), written to profiles/gemm_traffic.json for
bench.py's roofline `traffic` field.
    python scripts/traffic_from_launches.py gpurun_out/launches.csv <steps in capture> <round tag>"""
import csv
import json
import sys
from collections import defaultdict

path, steps, tag = sys.argv[1], float(sys.argv[2]), sys.argv[3]
GEMM = ("gemm_pair_kernel", "gemm_tc_kernel", "gemm_tma_kernel", "gemm_simt_kernel", "thin_", "dense_wide",
        "dense_fprop", "dense_dgrad", "dense_wgrad", "col2im4", "im2col4", "wt_transpose4", "tf32_lo",
        "fprop4_kernel", "wgrad4_kernel", "dgrad4_kernel")
with open(path) as f:
    rows = list(csv.DictReader(ln for ln in f if ln.startswith('"')))
per = defaultdict(float)
for r in rows:
    if r["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    per[r["Kernel Name"]] += v
total = sum(v for k, v in per.items() if any(g in k for g in GEMM))
out = {"gemm_dram_bytes_per_step": total / steps,
       "source": f"{path}: dram__bytes_read.sum + dram__bytes_write.sum of every implicit-GEMM launch "
                 f"(gemm_* / thin_* / dense_* kernels and the lowered path's helpers) / {steps:g} training steps",
       "round": tag}
json.dump(out, open("profiles/gemm_traffic.json", "w"), indent=1)
print(json.dumps(out))
