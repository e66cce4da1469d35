"""ctypes binding of libpartgan_b200.so (include/pg_kernels.h, include/pg_trainer.h).

The library is built in-tree by ``paper_2102_10485_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or does not load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("PG_LIB", "")) if os.environ.get("PG_LIB") else \
    Path(__file__).resolve().parent / "_lib" / "libpartgan_b200.so"  # PG_LIB: tuning-variant builds only

PG_OK, PG_EINVAL, PG_ECUDA, PG_ENONFINITE, PG_EUNSUPPORTED = 0, -1, -2, -3, -4
MATH_FP32_SIMT, MATH_TF32X3, MATH_TF32, MATH_BF16 = 0, 1, 2, 3
ACT_NONE, ACT_RELU, ACT_LRELU, ACT_TANH, ACT_SIGMOID = 0, 1, 2, 3, 4
(PG_OP_CONV2D_FWD, PG_OP_CONV2D_BWD_DATA, PG_OP_CONV2D_BWD_FILTER, PG_OP_CONVT2D_FWD, PG_OP_CONVT2D_BWD_DATA,
 PG_OP_CONVT2D_BWD_FILTER, PG_OP_DENSE_FWD, PG_OP_DENSE_BWD_DATA, PG_OP_DENSE_BWD_FILTER) = range(9)

(F_GEN_PARAMS, F_DISC_PARAMS, F_GEN_BUFFERS, F_DISC_BUFFERS, F_GEN_GRADS, F_DISC_GRADS, F_GEN_ADAM_M,
 F_GEN_ADAM_V, F_DISC_ADAM_M, F_DISC_ADAM_V, F_REPORTS, F_LAST_BATCH, F_COUNTERS) = range(13)


class PgError(RuntimeError):
    pass


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("B", "Cin", "H", "W", "Cout", "OH", "OW", "k", "s", "p")]


class GroupConfig(C.Structure):
    _fields_ = [
        ("gen_spec", C.c_char_p), ("disc_spec", C.c_char_p),
        ("C", C.c_int), ("H", C.c_int), ("W", C.c_int), ("d_z", C.c_int),
        ("n_labels", C.c_int), ("class_ids", C.POINTER(C.c_int)), ("base_seed", C.c_uint64),
        ("batch", C.c_int), ("epochs", C.c_int), ("per_label", C.c_long),
        ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
        ("clamp", C.c_double), ("init_std", C.c_double),
        ("math", C.c_int), ("threads", C.c_int), ("device", C.c_int),
        ("seeds", C.POINTER(C.c_uint64)),
    ]


_P = C.c_void_p
_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_LL = C.c_longlong

_SIGNATURES = {
    "pg_last_error": (C.c_char_p, []),
    "pg_device_count": (C.c_int, []),
    "pg_launch_count": (C.c_longlong, []),
    "pg_kernel_timing": (C.c_int, [C.c_int]),
    "pg_kernel_timing_read": (C.c_int, [C.POINTER(C.c_double)]),
    "pg_kernel_timing_report": (C.c_long, [C.c_char_p, C.c_long]),
    "pg_tc_tf32_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "pg_conv2d_fwd": (C.c_int, [C.POINTER(ConvDesc), C.c_int, _P, _P, _LL, _P, _LL, C.c_int, C.c_float, _P, C.c_int, _P]),
    "pg_conv2d_bwd_data": (C.c_int, [C.POINTER(ConvDesc), C.c_int, _P, _P, _LL, _P, C.c_int, _P]),
    "pg_conv2d_bwd_filter": (C.c_int, [C.POINTER(ConvDesc), C.c_int, _P, _P, _P, _LL, C.c_int, C.c_int, _P]),
    "pg_convT2d_fwd": (C.c_int, [C.POINTER(ConvDesc), C.c_int, _P, _P, _LL, _P, _LL, C.c_int, C.c_float, _P, C.c_int, _P]),
    "pg_convT2d_bwd_data": (C.c_int, [C.POINTER(ConvDesc), C.c_int, _P, _P, _LL, _P, C.c_int, _P]),
    "pg_convT2d_bwd_filter": (C.c_int, [C.POINTER(ConvDesc), C.c_int, _P, _P, _P, _LL, C.c_int, C.c_int, _P]),
    "pg_dense_fwd": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _LL, _P, _LL, C.c_int, C.c_float, _P, C.c_int, _P]),
    "pg_dense_bwd_data": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _LL, _P, C.c_int, _P]),
    "pg_dense_bwd_filter": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, _LL, C.c_int, C.c_int, _P]),
    "pg_bn_workspace_floats": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "pg_workspace_size": (C.c_size_t, [C.c_int, C.POINTER(ConvDesc), C.c_int, C.c_int]),
    "pg_set_workspace": (C.c_int, [_P, _P, C.c_size_t]),
    "pg_bn_fwd": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _LL, _P, _LL, C.c_float, C.c_float, C.c_int,
                            C.c_int, C.c_float, _P, _P, _P, _P, _P]),
    "pg_bn_bwd": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, _P, _P, _LL, C.c_int, C.c_float, _P, _P,
                            _LL, C.c_int, _P, _P]),
    "pg_act_bwd": (C.c_int, [_LL, _P, _P, C.c_int, C.c_float, _P, _P]),
    "pg_gan_losses": (C.c_int, [C.c_int, C.c_int, _P, _P, C.c_int, C.c_double, _P, _P, _P, _P]),
    "pg_gen_loss": (C.c_int, [C.c_int, C.c_int, _P, C.c_int, C.c_double, _P, _P, _P]),
    "pg_adam_step": (C.c_int, [C.c_int, _LL, _P, _P, _P, _P, _P, _P, C.c_double, C.c_double, C.c_double, C.c_double,
                               _P]),
    "pg_gather_real": (C.c_int, [C.c_int, C.c_int, _P, _P, _LL, _LL, C.c_int, C.c_int, _P, _P]),
    "pg_group_create": (C.c_int, [C.POINTER(GroupConfig), C.POINTER(_P)]),
    "pg_group_destroy": (None, [_P]),
    "pg_group_set_dataset": (C.c_int, [_P, _F]),
    "pg_group_generate_dataset": (C.c_int, [_P, C.c_uint64]),
    "pg_group_train_steps": (C.c_int, [_P, C.c_int]),
    "pg_group_train_step": (C.c_int, [_P, _F, C.c_int, _D]),
    "pg_group_train_step_inputs": (C.c_int, [_P, _F, _F, _F, C.c_int, _D]),
    "pg_group_get": (C.c_long, [_P, C.c_int, C.c_int, _D, C.c_long]),
    "pg_group_set": (C.c_int, [_P, C.c_int, C.c_int, _D, C.c_long]),
    "pg_group_failed": (C.c_int, [_P, _I]),
    "pg_group_generate": (C.c_int, [_P, C.c_long, C.c_uint64, _F]),
    "pg_group_generate_latents": (C.c_int, [_P, _F, C.c_long, _F]),
    "pg_net_create": (C.c_int, [C.c_char_p, C.POINTER(C.c_long), C.c_int, C.c_uint64, C.c_double, C.c_int, C.c_int,
                                C.POINTER(_P)]),
    "pg_net_destroy": (None, [_P]),
    "pg_net_param_count": (C.c_long, [_P]),
    "pg_net_buffer_count": (C.c_long, [_P]),
    "pg_net_out_shape": (C.c_int, [_P, C.POINTER(C.c_long), _I]),
    "pg_net_get_params": (C.c_int, [_P, _D]),
    "pg_net_set_params": (C.c_int, [_P, _D]),
    "pg_net_get_buffers": (C.c_int, [_P, _D]),
    "pg_net_set_buffers": (C.c_int, [_P, _D]),
    "pg_net_forward": (C.c_int, [_P, _D, C.c_int, C.c_int, _D, C.POINTER(_P)]),
    "pg_net_backward": (C.c_int, [_P, _P, _D, C.c_int, _D, _D]),
    "pg_trace_destroy": (None, [_P]),
    "pg_adam_step_host": (C.c_int, [C.c_long, _D, _D, _D, _D, C.POINTER(C.c_long), C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_int]),
    "pg_softmax_rows": (C.c_int, [C.POINTER(C.c_double), C.c_long, C.c_long, C.POINTER(C.c_double)]),
    "pg_inception_score": (C.c_int, [C.POINTER(C.c_double), C.c_long, C.c_long, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "pg_anova_f": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_long), C.c_long, C.POINTER(C.c_double)]),
    "pg_anova_per_channel": (C.c_int, [_F, C.POINTER(C.c_int), C.c_long, C.c_long, C.c_long, C.c_long, C.c_long,
                                       C.POINTER(C.c_double)]),
    "pg_group_save_checkpoint": (C.c_int, [_P, C.c_int, C.c_char_p]),
    "pg_group_load_checkpoint": (C.c_int, [_P, C.c_int, C.c_char_p]),
    "pg_group_mixture_sample": (C.c_int, [_P, C.POINTER(C.c_double), C.c_long, C.c_uint64, _F, C.POINTER(C.c_int)]),
    "pg_group_capture_masks": (C.c_int, [_P, C.c_int]),
    "pg_group_get_masks": (C.c_long, [_P, C.c_int, C.POINTER(C.c_uint8), C.c_long]),
    "pg_group_last_ms": (C.c_float, [_P]),
    "pg_group_sync": (C.c_int, [_P]),
    "pg_group_sizes": (C.c_int, [_P, C.POINTER(C.c_longlong)]),
    "pg_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "pg_shard_begin": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "pg_cosine_label": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_long, C.c_uint64, C.c_int, _D]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise PgError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(rc: int, what: str = "") -> int:
    if rc < 0:
        msg = lib().pg_last_error().decode(errors="replace")
        raise PgError(f"{what}: {msg} (code {rc})")
    return rc
