"""ctypes loader for libtpipe.so (the C-ABI of include/tpipe.h and
include/tpipe_kernels.h). Argument marshalling only: every step of the hot
path runs in the library's sm_100a kernels. There is no fallback — a missing
library is an error."""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtpipe.so")

vp, i32, i64, u32, u64, f32 = C.c_void_p, C.c_int, C.c_long, C.c_uint32, C.c_uint64, C.c_float

_lib = None


class TPipeError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TPipeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().tpipe_last_error().decode()
        raise TPipeError(f"{what}: rc={rc}: {msg}")
    return rc


def _declare(L):
    L.tpipe_last_error.restype = C.c_char_p
    L.tpipe_last_error.argtypes = []
    gemm_args = [i32, i32, i32, i32, vp, i64, i32, vp, i64, i32, i32, vp, i64, vp, vp, i64, vp, i64,
                 vp, i64, vp]
    L.tpipe_k_gemm.argtypes = gemm_args
    L.tpipe_k_gemm_simt.argtypes = gemm_args
    L.tpipe_k_gemm_dot.argtypes = [i32, i32, i32, vp, i64, i32, vp, i64, i32, vp, i64, vp, i64, vp, i32, i32, vp]
    L.tpipe_k_gemm_set_pair.argtypes = [i32]
    L.tpipe_k_gemm_set_pair.restype = None
    L.tpipe_k_gemm_set_pair_min_tiles.argtypes = [i32]
    L.tpipe_k_gemm_set_pair_min_tiles.restype = None
    for knob in ("tpipe_k_gemm_set_wide_choice", "tpipe_k_ln_set_rows_bwd"):
        if hasattr(L, knob):   # (absent from older builds used in A/B runs)
            getattr(L, knob).argtypes = [i32]
            getattr(L, knob).restype = None
    L.tpipe_k_ln_fwd.argtypes = [i32, vp, vp, vp, vp, vp, vp, i32, i32, vp]
    L.tpipe_k_ln_bwd.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp]
    L.tpipe_k_ln_bwd_rsum.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp]
    L.tpipe_k_ln_bwd_partials.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, vp]
    L.tpipe_k_attn_fwd.argtypes = [i32, vp, vp, vp, i32, i32, i32, i32, vp]
    L.tpipe_k_attn_bwd.argtypes = [i32, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, vp]
    L.tpipe_k_embed_fwd.argtypes = [i32, vp, vp, vp, vp, i32, i32, i32, vp]
    L.tpipe_k_embed_bwd.argtypes = [i32, vp, vp, vp, vp, vp, i32, i32, i32, vp]
    L.tpipe_k_ce_fwd.argtypes = [vp, vp, vp, vp, f32, i32, i32, vp]
    L.tpipe_k_ce_bwd.argtypes = [i32, vp, vp, vp, vp, f32, i32, i32, vp]
    L.tpipe_k_head_ce.argtypes = [vp, vp, vp, vp, vp, vp, f32, i32, i32, i32, vp, vp]
    L.tpipe_k_colsum.argtypes = [i32, vp, vp, vp, i32, i32, vp]
    L.tpipe_k_adamw.argtypes = [i32, vp, vp, vp, vp, vp, i64, i32, f32, f32, f32, f32, f32, f32,
                                f32, vp]
    L.tpipe_host_adamw.argtypes = [vp, vp, vp, vp, vp, i64, i32, f32, f32, f32, f32, f32, f32, f32]
    L.tpipe_host_adamw.restype = None
    for name in ("tpipe_plan_create", "tpipe_plan_destroy", "tpipe_runtime_create"):
        if hasattr(L, name):
            pass
    try:
        from . import _decl_plan  # noqa: F401  (plan/runtime prototypes)
        _decl_plan.declare(L)
    except ImportError:
        pass
