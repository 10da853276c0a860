"""ctypes declaration of include/tfdp.h.  Argument marshalling only — every step of the
path runs in libtfdp.so's kernels.  Loading fails loudly if the library is missing."""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# TFDP_LIB_PATH: developer A/B runs against a variant build (build.py defines/out)
LIB_PATH = os.environ.get("TFDP_LIB_PATH") or os.path.join(HERE, "libtfdp.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "tfdp.h")

TFDP_OK = 0
STATUS = {0: "TFDP_OK", 1: "TFDP_ERR_ARG", 2: "TFDP_ERR_CUDA", 3: "TFDP_ERR_OOM",
          4: "TFDP_ERR_DIVERGED", 5: "TFDP_ERR_STATE", 6: "TFDP_ERR_NCCL",
          7: "TFDP_ERR_UNSUPPORTED"}
EXACT, IBFFT = 0, 1
COOL_LINEAR, COOL_CONSTANT = 0, 1
DIST_SPREAD_ALL, DIST_GRID_ALLREDUCE, DIST_SLAB = 0, 1, 2
WARN_ALPHA_BETA, WARN_GAMMA, WARN_NINT_CAPPED = 1, 2, 4


class tfdp_params(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("alpha", C.c_double), ("beta", C.c_double),
        ("gamma", C.c_double), ("rho", C.c_double), ("solver", C.c_int32),
        ("k", C.c_int32), ("n_int_min", C.c_int32), ("n_int_fixed", C.c_int32),
        ("fft_size", C.c_int32), ("step0", C.c_double), ("iterations", C.c_int32),
        ("t0", C.c_int32), ("cooling", C.c_int32), ("dist_mode", C.c_int32),
        ("node_order", C.c_int32), ("interval_rule", C.c_int32),
    ]


class tfdp_dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
                ("nccl_uid", C.c_void_p)]


_P = C.c_void_p
_SIGS = {
    "tfdp_params_default": (C.c_int, [C.POINTER(tfdp_params)]),
    "tfdp_csr_build": (C.c_int, [C.c_int64, C.c_int64, _P, _P, _P, _P, C.POINTER(C.c_int64)]),
    "tfdp_shard_range": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]),
    "tfdp_init": (C.c_int, [C.POINTER(_P), C.c_int64, _P, _P, _P, C.POINTER(tfdp_params),
                            C.POINTER(tfdp_dist), _P]),
    "tfdp_step": (C.c_int, [_P, C.c_int32]),
    "tfdp_forces": (C.c_int, [_P, _P, _P]),
    "tfdp_group_step": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "tfdp_group_forces": (C.c_int, [_P, C.c_int32, _P, _P]),
    "tfdp_slab_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _P, _P]),
    "tfdp_layout": (C.c_int, [_P, _P]),
    "tfdp_set_layout": (C.c_int, [_P, _P]),
    "tfdp_set_iteration": (C.c_int, [_P, C.c_int32]),
    "tfdp_iteration": (C.c_int32, [_P]),
    "tfdp_set_params": (C.c_int, [_P, C.POINTER(tfdp_params)]),
    "tfdp_global_refine": (C.c_int, [_P, C.c_double, C.c_double, C.c_int32]),
    "tfdp_np1": (C.c_int, [_P, C.POINTER(C.c_double), _P]),
    "tfdp_pivot_mds": (C.c_int, [_P, C.c_int32, C.c_uint64, _P]),
    "tfdp_set_focus": (C.c_int, [_P, _P, C.c_int64, C.c_double, C.c_double, C.c_double]),
    "tfdp_local_refine": (C.c_int, [_P, _P, C.c_int64, C.c_double, C.c_double, C.c_double,
                                    C.c_int32]),
    "tfdp_shard": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tfdp_fft_geometry": (C.c_int, [_P, _P, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32)]),
    "tfdp_fft_plan": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "tfdp_profile": (C.c_int, [_P, C.c_int32]),
    "tfdp_profile_mask": (C.c_int, [_P, C.c_uint32]),
    "tfdp_profile_select": (C.c_int, [_P, C.c_uint32]),
    "tfdp_profile_read": (C.c_int32, [_P, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), C.c_int32]),
    "tfdp_launch_count": (C.c_int64, [_P]),
    "tfdp_warnings": (C.c_uint32, [_P]),
    "tfdp_last_error": (C.c_char_p, [_P]),
    "tfdp_status_string": (C.c_char_p, [C.c_int]),
    "tfdp_destroy": (None, [_P]),
    "tfdp_nccl_unique_id": (C.c_int, [_P]),
}

_lib = None


def declared_symbols() -> list[str]:
    """Every function include/tfdp.h declares (parsed from the header)."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tfdp_[a-z0-9_]+)\s*\(", text)) - {"tfdp_ctx"})


def lib() -> C.CDLL:
    """Load libtfdp.so (built by __graft_entry__.build()).  No fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " — there is no CPU fallback")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class TfdpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status: int, ctx=None):
    if status != TFDP_OK:
        m = lib().tfdp_last_error(ctx)
        raise TfdpError(status, m.decode() if m else "")
