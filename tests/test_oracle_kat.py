"""The oracle is trusted only after it passes the reference's own known-answer
tests: oracle/kat.cpp ports test_optim, test_gan, test_nn and
test_partition cases, plus pins for the BASELINE additions (ConvTranspose2d,
c1..c4 parameter counts, cosine dataset)."""
import subprocess

import pytest


def test_oracle_known_answer_tests(oracle):
    r = subprocess.run([str(oracle.KAT)], capture_output=True, text=True, timeout=600)
    lines = r.stdout.splitlines()
    failed = [l for l in lines if l.startswith("FAIL")]
    passed = [l for l in lines if l.startswith("PASS")]
    assert not failed, "\n".join(failed)
    assert r.returncode == 0
    # every ported suite is represented
    for suite in ("optim.", "gan.", "nn.", "partition.", "new."):
        assert any(suite in l for l in passed), suite
    assert len(passed) >= 45


@pytest.mark.parametrize("cfg,gen,disc", [(1, 766017, 138817), (2, 1073219, 663745), (4, 3585347, 2766529)])
def test_baseline_param_counts(oracle, cfg, gen, disc):
    from paper_2102_10485_b200.archs import baseline_arch
    a = baseline_arch(cfg)
    assert oracle.net_info(a.gen, str(a.d_z))[0] == gen
    assert oracle.net_info(a.disc, " ".join(map(str, a.image)))[0] == disc
