"""The oracle's MaskTape (parity instrumentation, oracle/oracle.hpp): replaying
a step's own activation masks is the identity, and an fp32 restatement that
replays the f64 masks agrees with f64 to the 1e-4 bar the GPU parity tests
use (so that bar is attainable by an fp32 implementation once the kink
discontinuities are pinned).  CPU only."""
import numpy as np

from parity import layer_tensors, rel_max, update_err
from paper_2102_10485_b200 import baseline_arch


def _seed(o, rng):
    for f in (6, 7, 8, 9):
        n = o.get(0, f).size
        v = 1e-3 * rng.standard_normal(n) if f in (6, 8) else 1e-6 * (1 + np.abs(rng.standard_normal(n)))
        o.set(0, f, v.astype(np.float32).astype(np.float64))
    o.set(0, 12, np.array([10.0, 10.0, 0.0]))


def test_mask_tape_replay_and_fp32_bar(oracle):
    arch = baseline_arch(1)
    mk = lambda prec: oracle.OracleGroup(prec, 1, 1, 64, 32, data_seed=3, base_seed=7)
    ref = mk(64)
    _seed(ref, np.random.default_rng(1))
    ref.record_masks(0)
    ref.step(1)
    m = ref.recorded_masks(0)
    # G z1 + D real + D fake + G z2 + D fake, each activation layer [B][C][H][W]
    g_act = 128 * 7 * 7 + 64 * 14 * 14
    d_act = 64 * 14 * 14 + 128 * 7 * 7
    assert m.size == 32 * (2 * g_act + 3 * d_act)
    assert 0.2 < m.mean() < 0.8
    # replaying its own masks reproduces the f64 step bit for bit
    rep = mk(64)
    _seed(rep, np.random.default_rng(1))
    rep.set_masks(0, m)
    rep.step(1)
    assert rep.mask_flips(0) == 0
    for f in (0, 1, 2, 3, 4, 5, 10):
        assert np.array_equal(rep.get(0, f), ref.get(0, f)), f
    # a wrong-length tape is rejected
    bad = mk(64)
    bad.set_masks(0, m[:-1])
    try:
        bad.step(1)
        raise AssertionError("short tape accepted")
    except RuntimeError as e:
        assert "mask tape" in str(e)
    # fp32 replaying the f64 masks: every gradient and update within 1e-4
    f32 = mk(32)
    _seed(f32, np.random.default_rng(1))
    p0 = {0: f32.get(0, 0), 1: f32.get(0, 1)}
    f32.set_masks(0, m)
    f32.step(1)
    for gcode, pcode, spec, ish in ((4, 0, arch.gen, (arch.d_z,)), (5, 1, arch.disc, arch.image)):
        for name, off, n, feeds_bn in layer_tensors(spec, ish):
            if feeds_bn:
                continue
            sl = slice(off, off + n)
            assert rel_max(f32.get(0, gcode)[sl], ref.get(0, gcode)[sl]) < 1e-4, name
            assert update_err(f32.get(0, pcode)[sl], ref.get(0, pcode)[sl], p0[pcode][sl]) < 1e-4, name
