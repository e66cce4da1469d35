"""The C-ABI library loads without a GPU and exports every symbol the public
headers declare; host-only entry points agree with the reference protocol."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(pg_[a-zA-Z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol(native):
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in sorted(names) if not hasattr(native, n)]
    assert not missing, missing


def test_no_gpu_needed_for_loading(native):
    # pg_device_count works (returns 0 here) and never raises
    assert native.pg_device_count() >= 0


def test_errors_surface_through_last_error(native):
    import ctypes as C
    from paper_2102_10485_b200 import _native as N
    d = N.ConvDesc(B=1, Cin=3, H=8, W=8, Cout=4, OH=5, OW=4, k=4, s=2, p=1)  # wrong OH
    rc = native.pg_conv2d_fwd(C.byref(d), 1, None, None, 0, None, 0, 0, 0.0, None, 0, None)
    assert rc == N.PG_EINVAL
    assert b"output extent" in native.pg_last_error()


def test_workspace_query_errors_and_detach(native):
    """pg_workspace_size reports invalid input as (size_t)-1 with the reason in
    pg_last_error; pg_set_workspace rejects misaligned buffers and detaching
    needs no device."""
    import ctypes as C
    from paper_2102_10485_b200 import _native as N
    bad = N.ConvDesc(B=1, Cin=3, H=8, W=8, Cout=4, OH=5, OW=4, k=4, s=2, p=1)
    assert native.pg_workspace_size(N.PG_OP_CONV2D_FWD, C.byref(bad), 1, N.MATH_TF32X3) == 2**64 - 1
    assert b"output extent" in native.pg_last_error()
    ok = N.ConvDesc(B=1, Cin=3, H=8, W=8, Cout=4, OH=4, OW=4, k=4, s=2, p=1)
    assert native.pg_workspace_size(99, C.byref(ok), 1, N.MATH_TF32X3) == 2**64 - 1
    assert b"unknown operator" in native.pg_last_error()
    assert native.pg_workspace_size(N.PG_OP_CONV2D_FWD, C.byref(ok), 1, 7) == 2**64 - 1
    assert native.pg_set_workspace(None, C.c_void_p(0x1008), 4096) == N.PG_EINVAL
    assert b"256-byte aligned" in native.pg_last_error()
    assert native.pg_set_workspace(None, None, 0) == N.PG_OK
