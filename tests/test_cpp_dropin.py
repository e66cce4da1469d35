"""A compiled C++ caller of the library through the reference-API mirror
include/partgan_b200.hpp (over include/pg_network.h + pg_trainer.h):
tests/cpp/dropin_test.cpp.  CPU: it compiles and links against
libpartgan_b200.so with only the public headers.  GPU: it runs, executing
ports of the reference's own API tests (test_optim / test_nn / test_gan /
test_partition) through the C-ABI."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "dropin_test.cpp"
OUT = ROOT / "tests" / "cpp" / "_build" / "dropin_test"


def build_dropin() -> Path:
    from paper_2102_10485_b200 import build
    lib = build.build()
    OUT.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-Wno-unused-parameter", f"-I{ROOT / 'include'}",
           str(SRC), f"-L{lib.parent}", "-lpartgan_b200", f"-Wl,-rpath,{lib.parent}", "-o", str(OUT)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return OUT


def test_dropin_compiles_against_public_headers():
    exe = build_dropin()
    assert exe.exists()
    # the binary links the product library itself (not the oracle)
    deps = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
    assert "libpartgan_b200.so" in deps and "liboracle" not in deps


@pytest.mark.gpu
def test_dropin_runs_reference_api_tests():
    exe = build_dropin()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and r.stdout.count("PASS") >= 15
