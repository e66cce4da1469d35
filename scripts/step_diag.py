"""Diagnostic: one c1 training step per math mode vs the f64 oracle; for each
parameter-gradient tensor print the relative max error and how concentrated
the error is (elements above 10% of the max error)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle_lib
from paper_2102_10485_b200 import GroupSpec, LabelGroup, _native as N, baseline_arch
from parity import layer_tensors

cfg, L, per_label, B = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1, 2, 128, 64)))
arch = baseline_arch(cfg)
orc = oracle_lib.OracleGroup(64, cfg, L, per_label, B, data_seed=3, base_seed=7)
orc.step(1)
for math in (0, 1):
    grp = LabelGroup(GroupSpec(arch=arch, class_ids=list(range(L)), batch=B, per_label=per_label, base_seed=7,
                               math=math))
    grp.generate_dataset(3)
    grp.train_steps(1)
    print(f"=== math {math}: reports", grp.reports(0)[-1], orc.get(0, 10)[-4:])
    for lab in range(L):
     print(f"  -- label {lab}: reports", grp.reports(lab)[-1], orc.get(lab, 10)[-4:])
     for net, gcode, spec, ish in (("D", N.F_DISC_GRADS, arch.disc, arch.image), ("G", N.F_GEN_GRADS, arch.gen, (100,))):
        g, r = grp.get(lab, gcode), orc.get(lab, gcode)
        for name, off, n, fb in layer_tensors(spec, ish):
            a, b = g[off:off + n], r[off:off + n]
            e = np.abs(a - b)
            scale = np.abs(b).max()
            big = int((e > 0.1 * e.max()).sum())
            print(f"  {net}.{name:16s} rel {e.max() / scale:.2e} elems>10%max {big:7d}/{n}  median {np.median(e) / scale:.1e}"
                  f"{'  (feeds BN)' if fb else ''}")
    grp.close()
