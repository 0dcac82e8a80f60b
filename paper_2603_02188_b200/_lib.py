"""ctypes binding of libmlra_b200.so (include/mlra_b200.h).

The shared library is built in-tree by ``paper_2603_02188_b200.build``. There is no
fallback: if the library is missing or a call fails, the caller gets an exception.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import AttnKitError, ConfigError, CudaError, NumericError, ShapeMismatchError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmlra_b200.so")

_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float

#: exported symbol -> (restype, argtypes); mirrors include/mlra_b200.h one-to-one
SIGNATURES = {
    "mlra_version": (_I, []),
    "mlra_last_error": (ctypes.c_char_p, []),
    "mlra_num_sms": (_I, []),
    "mlra_cache_append": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P]),
    "mlra_cache_append_latent": (_I, [_P] * 5 + [_I] * 8 + [_F, _F, _F, _I, _I, _I, _I, _P, _P]),
    "mlra_absorb_query": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _F, _P]),
    "mlra_workspace_bytes": (ctypes.c_size_t, [_I, _I, _I, _I, _I, _I]),
    "mlra_default_splits": (_I, [_I, _I, _I, _I]),
    "mlra_default_splits_heads": (_I, [_I, _I, _I, _I, _I]),
    "mlra_decode_partials": (_I, [_P] * 7 + [_I] * 10 + [_P]),
    "mlra_combine": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _F, _I, _P, _P]),
    "mlra_check_status": (_I, [_P, _I, _P]),
    "mlra_decode_step": (_I, [_P] * 9 + [_I] * 11 + [_F, _F, _P]),
    "mlra_gqa_default_splits": (_I, [_I, _I, _I]),
    "mlra_gqa_workspace_bytes": (ctypes.c_size_t, [_I, _I, _I, _I, _I]),
    "mlra_gqa_decode_partials": (_I, [_P] * 6 + [_I] * 8 + [_F, _P]),
    "mlra_gqa_decode_step": (_I, [_P] * 6 + [_I] * 8 + [_F, _P]),
    "mlra_outproj_comm_bytes": (ctypes.c_size_t, [_I, _I, _I]),
    "mlra_outproj_workspace_bytes": (ctypes.c_size_t, [_I, _I]),
    "mlra_outproj": (_I, [_P] * 5 + [_I] * 5 + [_P, _P, _P]),
    "mlra_outproj_sim": (_I, [_P] * 5 + [_I] * 4 + [_P, _P, _P]),
    "mlra_allreduce_comm_bytes": (ctypes.c_size_t, [_I, _I]),
    "mlra_decode_step_tp": (_I, [_P] * 9 + [_I] * 11 + [_F, _F, _I, _I, _P, _P]),
    "mlra_allreduce": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "mlra_allreduce_sim": (_I, [_P, _P, _I, _I, _P, _P]),
    "mlra_comm_alloc": (_I, [ctypes.c_size_t, _P]),
    "mlra_comm_free": (_I, [_P]),
    "mlra_ipc_handle": (_I, [_P, _P]),
    "mlra_ipc_open": (_I, [_P, _P]),
    "mlra_ipc_close": (_I, [_P]),
    "mlra_prefill_attention": (_I, [_P] * 6 + [_I] * 11 + [_F, _P]),
    "mlra_rows_split": (_I, [_P] + [_I] * 4 + [_F, _F, _P, _P, _I, _P]),
    "mlra_query_epilogue": (_I, [_P] + [_I] * 7 + [_F, _F, _F, _P, _P, _P]),
    "mlra_decode_plan": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _I, _I, _P]),
    "mlra_decode_step_ragged": (_I, [_P] * 9 + [_I] * 11 + [_F, _F, _P]),
    "mlra_proj_down": (_I, [_P, _P] + [_I] * 5 + [_P] * 5),
    "mlra_proj_query": (_I, [_P, _P, _F, _F, _P] + [_I] * 6 + [_P, _I, _F, _F, _F, _P, _P, _P]),
}

_CODES = {-1: ShapeMismatchError, -2: ConfigError, -3: NumericError, -4: CudaError}


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or LIB_PATH
        if not os.path.exists(path):
            raise CudaError(
                f"CUDA extension {path} not built; run `python -m paper_2603_02188_b200.build` "
                "(there is no CPU fallback for the decode path)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = load().mlra_last_error().decode(errors="replace")
    raise _CODES.get(rc, AttnKitError)(f"{what}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
