"""Full training-step parity: the device label group vs the CPU oracle's
run_worker protocol on identical seeds (same cosine-field data, same
per-label streams, same init).  North-star bars:
  - minibatch indices bit-exact;
  - single-step losses / parameter gradients / updated weights within 1e-4
    relative (fp32-accurate modes);
  - 10-step loss trajectories within 1e-3.
Metrics (tests/parity.py): losses and gradients per tensor max|a-b|/max|ref|;
updated weights and BN running buffers per tensor ||a-b||/||ref||.  Biases of
layers that feed a train-mode BatchNorm have an exact gradient of zero (BN
removes the per-channel mean), so both sides hold rounding noise there; they
are checked as |g| <= 1e-5 max|g_W| instead and their updates as |dp| <= 2 lr.
"""
import numpy as np
import pytest

from paper_2102_10485_b200 import GroupSpec, LabelGroup, _native as N, baseline_arch
from parity import layer_tensors, rel_l2, rel_max

pytestmark = pytest.mark.gpu

# oracle field codes match pg_group_get codes 0..12
OR = dict(gp=0, dp=1, gb=2, db=3, gg=4, dg=5, reports=10, batch=11)


def make_pair(cfg, n_labels, per_label, batch, math, epochs=1, first_label=0, threads=8):
    arch = baseline_arch(cfg)
    grp = LabelGroup(GroupSpec(arch=arch, class_ids=list(range(first_label, first_label + n_labels)), batch=batch,
                               epochs=epochs, per_label=per_label, base_seed=7, math=math, threads=threads))
    grp.generate_dataset(3)
    return arch, grp


def frac_outside(a, ref, tol):
    """fraction of elements with |a - ref| > tol * max|ref|"""
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    return float(np.mean(np.abs(a - ref) > tol * scale))


def compare_pair_state(grp, orc, arch, n_labels, tol=1e-4, kink_frac=1e-3, lr=2e-4):
    """Per parameter tensor (reference flat layout):
      gradients: all but a `kink_frac` fraction of elements within `tol` of
                 max|ref| (relative), and ||g - ref|| / ||ref|| <= 10 tol;
      weights:   the same element criterion, and every element within 2 lr
                 per step of the reference (one Adam step moves a weight by
                 at most ~lr);
      BN running buffers: ||b - ref|| / ||ref|| <= tol.
    The fraction allowance exists for activation kinks: a ReLU / LeakyReLU
    whose pre-activation lies within ~1e-6 of zero can switch side under a
    different (equally valid) fp32 rounding; that concentrates an error on the
    few elements it touches (tests/test_gpu_step.py docstring)."""
    report, bad = {}, []
    steps = max(1, grp_steps(grp, 0))
    for l in range(n_labels):
        for net, pcode, gcode, bcode, spec, ishape in (
                ("G", N.F_GEN_PARAMS, N.F_GEN_GRADS, N.F_GEN_BUFFERS, arch.gen, (arch.d_z,)),
                ("D", N.F_DISC_PARAMS, N.F_DISC_GRADS, N.F_DISC_BUFFERS, arch.disc, arch.image)):
            gp, rp = grp.get(l, pcode), orc.get(l, pcode)
            gg, rg = grp.get(l, gcode), orc.get(l, gcode)
            assert gp.shape == rp.shape and gg.shape == rg.shape
            tensors = layer_tensors(spec, ishape)
            wscale = {name.split(".")[0]: np.abs(rg[off:off + n]).max()
                      for name, off, n, _ in tensors if name.endswith(".w")}
            for name, off, n, feeds_bn in tensors:
                sl = slice(off, off + n)
                key = f"{l}.{net}.{name}"
                if feeds_bn:
                    # gauge direction: exact gradient is zero, both sides hold rounding noise
                    scale = wscale[name.split(".")[0]]
                    if np.abs(gg[sl]).max() > 1e-5 * scale + 1e-12 or np.abs(gp[sl] - rp[sl]).max() > 2 * lr * steps:
                        bad.append(key + " (gauge bias)")
                    continue
                fg, eg = frac_outside(gg[sl], rg[sl], tol), rel_l2(gg[sl], rg[sl])
                fw = frac_outside(gp[sl], rp[sl], tol)
                dw = np.abs(gp[sl] - rp[sl]).max()
                report[key] = (fg, eg, fw)
                if fg > kink_frac or eg > 10 * tol:
                    bad.append(f"{key}.grad frac={fg:.2e} l2={eg:.2e}")
                if fw > kink_frac or dw > 2 * lr * steps + tol * np.abs(rp[sl]).max():
                    bad.append(f"{key}.param frac={fw:.2e} maxdiff={dw:.2e}")
            gb, rb = grp.get(l, bcode), orc.get(l, bcode)
            if rb.size and rel_l2(gb, rb) > tol:
                bad.append(f"{l}.{net}.buffers l2={rel_l2(gb, rb):.2e}")
    assert not bad, bad
    return report


def grp_steps(grp, l):
    return int(grp.get(l, N.F_COUNTERS)[2])


@pytest.mark.parametrize("math", [0, 1])
@pytest.mark.parametrize("cfg,n_labels,per_label,batch", [(1, 2, 128, 64), (2, 2, 64, 16), (4, 2, 8, 4)])
def test_single_step_parity(oracle, cfg, n_labels, per_label, batch, math):
    arch, grp = make_pair(cfg, n_labels, per_label, batch, math)
    orc = oracle.OracleGroup(64, cfg, n_labels, per_label, batch, data_seed=3, base_seed=7)
    # initial state identical to build_network's draws (cast to fp32)
    for l in range(n_labels):
        assert rel_max(grp.get(l, N.F_GEN_PARAMS), orc.get(l, OR["gp"])) < 1e-7
        assert rel_max(grp.get(l, N.F_DISC_PARAMS), orc.get(l, OR["dp"])) < 1e-7
    assert grp.train_steps(1) == 1
    orc.step(1)
    for l in range(n_labels):
        # minibatch indices: bit-exact.  The device group reports positions in
        # the label's shard; the oracle reports rows of its label-blocked
        # dataset (row = l * per_label + position).
        assert np.array_equal(grp.get(l, N.F_LAST_BATCH) + l * per_label, orc.get(l, OR["batch"]))
        r, q = grp.reports(l)[-1], orc.get(l, OR["reports"]).reshape(-1, 4)[-1]
        assert abs(r[0] - q[0]) <= 1e-4 * abs(q[0]), (r, q)   # J_D
        assert abs(r[1] - q[1]) <= 1e-4 * abs(q[1]), (r, q)   # J_G
        assert abs(r[2] - q[2]) <= 1e-4 * abs(q[2])
        assert abs(r[3] - q[3]) <= 1e-4 * abs(q[3])
    # both fp32-accurate modes (SIMT fp32 and 3xTF32, whose GEMMs are within
    # 1.2e-6 of f64 at any K: scripts/tc_accuracy.py) are held to the 1e-4 bar
    compare_pair_state(grp, orc, arch, n_labels)
    assert not grp.failed().any()


@pytest.mark.parametrize("math", [0, 1])
def test_indices_bit_exact_over_epochs_with_ragged_tail(oracle, math):
    """10 steps of c1 over two epochs with a partial tail batch (per_label 80,
    batch 16 -> 5 steps per epoch; per_label 72 -> 4 full + 1 of 8): the
    shuffle / batching protocol is bit-exact at every step and the epoch
    budget is honoured."""
    for per_label in (80, 72):
        arch, grp = make_pair(1, 2, per_label, 16, math, epochs=2)
        orc = oracle.OracleGroup(64, 1, 2, per_label, 16, data_seed=3, base_seed=7, epochs=2)
        for s in range(10):
            assert grp.train_steps(1) == 1
            orc.step(1)
            for l in range(2):
                assert np.array_equal(grp.get(l, N.F_LAST_BATCH) + l * per_label, orc.get(l, OR["batch"])), \
                    (per_label, s)
        assert grp.train_steps(5) == 0


@pytest.mark.parametrize("math", [0, 1])
def test_ten_step_loss_trajectory(oracle, math):
    """10-step J_D / J_G trajectories (c1, batch 64, one epoch) vs the f64
    oracle.  Bar: 1e-3 relative, or four times the divergence of the oracle's
    own f32 restatement from f64 at that step, whichever is larger.  The second
    clause exists because the GAN/Adam dynamics amplify rounding: the f32
    oracle (identical algorithm and summation order, only the precision
    differs) itself drifts from f64 by up to ~3e-3 within 10 steps here
    (DESIGN.md §parity)."""
    arch, grp = make_pair(1, 2, 640, 64, math)
    orc = oracle.OracleGroup(64, 1, 2, 640, 64, data_seed=3, base_seed=7)
    o32 = oracle.OracleGroup(32, 1, 2, 640, 64, data_seed=3, base_seed=7)
    assert grp.train_steps(10) == 10
    orc.step(10)
    o32.step(10)
    for l in range(2):
        r = grp.reports(l)[:, :2]
        q = orc.get(l, OR["reports"]).reshape(-1, 4)[:, :2]
        f = o32.get(l, OR["reports"]).reshape(-1, 4)[:, :2]
        err = (np.abs(r - q) / np.abs(q)).max(1)
        env = (np.abs(f - q) / np.abs(q)).max(1)
        tol = np.maximum(1e-3, 4 * env)
        assert (err <= tol).all(), (err, env)
        print(f"label {l}: device-vs-f64 {np.array2string(err, precision=1)}; "
              f"f32-oracle-vs-f64 {np.array2string(env, precision=1)}")


def test_host_batch_step_matches_explicit_inputs(oracle):
    """The reference train_step call shape: real batch from host memory with
    explicit latents, vs the oracle's step on the same inputs."""
    arch, grp = make_pair(1, 2, 64, 32, 0)
    orc = oracle.OracleGroup(64, 1, 2, 64, 32, data_seed=3, base_seed=7)
    rng = np.random.default_rng(0)
    real = rng.uniform(0, 1, (2, 32) + arch.image)
    z1, z2 = rng.normal(size=(2, 32, 100)), rng.normal(size=(2, 32, 100))
    rep = grp.train_step_inputs(real, z1, z2)
    for l in range(2):
        q = orc.step_inputs(l, real[l], z1[l], z2[l])
        assert np.all(np.abs(rep[l] - q) <= 1e-4 * np.abs(q)), (rep[l], q)
        # real images were passed in as float32: compare against what the oracle saw
    compare_pair_state(grp, orc, arch, 2)


def test_generate_eval_mode(oracle):
    """generate(): eval-mode BN, (v+1)/2 range, deterministic per seed."""
    arch, grp = make_pair(1, 2, 64, 32, 0)
    grp.train_steps(1)
    a, b = grp.generate(40, seed=5), grp.generate(40, seed=5)
    assert a.shape == (2, 40, 1, 28, 28)
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() <= 1
    assert a.std() > 0
