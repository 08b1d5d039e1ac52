"""ctypes binding of libtinyserve.so (include/tinyserve.h).  Argument marshalling only.

Every compute step runs in the CUDA kernels of the library; this module passes
`tensor.data_ptr()` and the current CUDA stream, and raises on a non-zero status.  There
is no CPU fallback: a missing library or a non-CUDA tensor raises immediately.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# the release library; TS_DEV_LIB=1 (development / test child processes only) loads the dev
# build of the same source instead (A/B knobs, timestamp hooks, TS_DEBUG error word)
LIB_PATH = os.path.join(HERE, "libtinyserve_dev.so" if os.environ.get("TS_DEV_LIB") == "1"
                        else "libtinyserve.so")

TS_F32, TS_BF16, TS_FP8E4M3 = 0, 1, 2
_STATUS = {0: "TS_OK", 1: "TS_ERR_CONFIG", 2: "TS_ERR_SHAPE", 3: "TS_ERR_ALIGN",
           4: "TS_ERR_UNSUPPORTED", 5: "TS_ERR_CUDA", 6: "TS_ERR_WORKSPACE"}

# every symbol include/tinyserve.h declares
SYMBOLS = ["ts_meta_append", "ts_meta_build", "ts_score_pages", "ts_select_topk",
           "ts_sparse_decode_attn", "ts_decode_step", "ts_decode_step_append", "ts_decode_step_prefetch", "ts_select_merge", "ts_lse_merge", "ts_workspace_bytes",
           "ts_attn_workspace_bytes", "ts_status_str", "ts_version", "ts_last_launch_count",
           "ts_profile_events", "ts_dense_decode_attn", "ts_dense_workspace_bytes",
           "ts_kv_quantize", "ts_pool_bytes", "ts_select_candidates", "ts_shard_attend"]


class TinyServeError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed: {msg}")
        self.status = status
        self.name = _STATUS.get(status, str(status))


class Layout(ctypes.Structure):
    """ts_layout (include/tinyserve.h)."""
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("max_pages", ctypes.c_int32),
                ("num_blocks", ctypes.c_int32), ("shard_stride", ctypes.c_int32),
                ("shard_offset", ctypes.c_int32), ("kv_dtype", ctypes.c_int32)]

    def __repr__(self):
        return "Layout(" + ", ".join(f"{n}={getattr(self, n)}" for n, _ in self._fields_) + ")"


_lib = None


def lib() -> ctypes.CDLL:
    """Load libtinyserve.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (nvcc, sm_100a)")
        L = ctypes.CDLL(LIB_PATH)
        P, I, F, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_size_t
        LP = ctypes.POINTER(Layout)
        sig = {
            "ts_meta_append": [LP, P, P, P, I, P, P, P, P, P],
            "ts_meta_build": [LP, P, P, P, P, P],
            "ts_score_pages": [LP, P, P, P, P, P, P],
            "ts_select_topk": [P, I, I, P, P, I, I, I, P, P, P, P],
            "ts_sparse_decode_attn": [LP, P, P, P, P, P, P, P, I, F, P, P, P, SZ, P],
            "ts_decode_step": [LP, P, P, P, P, P, P, I, F, P, P, P, P, P, SZ, P],
            "ts_decode_step_append": [LP, P, P, P, P, P, P, P, P, I, F, P, P, P, P, P, SZ, P],
            "ts_decode_step_prefetch": [LP, P, P, P, P, P, P, I, F, P, P, P, P, P, SZ, P],
            "ts_select_merge": [P, P, I, ctypes.c_int64, I, I, I, P, P, P, P],
            "ts_lse_merge": [I, I, I, P, P, ctypes.c_int64, P, P, P],
            "ts_dense_decode_attn": [LP, P, P, P, P, P, F, P, P, P, SZ, P],
            "ts_kv_quantize": [ctypes.c_int64, I, P, P, P],
            "ts_select_candidates": [LP, P, P, P, P, I, P, P, P, P],
            "ts_shard_attend": [LP, P, P, P, P, P, P, P, I, ctypes.c_int64, I, F, P, P, P, P, P, SZ, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.ts_workspace_bytes.argtypes = [LP, I]
        L.ts_workspace_bytes.restype = SZ
        L.ts_attn_workspace_bytes.argtypes = [LP, I]
        L.ts_attn_workspace_bytes.restype = SZ
        L.ts_dense_workspace_bytes.argtypes = [LP]
        L.ts_dense_workspace_bytes.restype = SZ
        L.ts_pool_bytes.argtypes = [LP]
        L.ts_pool_bytes.restype = SZ
        L.ts_status_str.argtypes = [ctypes.c_int]
        L.ts_status_str.restype = ctypes.c_char_p
        L.ts_version.restype = ctypes.c_char_p
        L.ts_last_launch_count.restype = ctypes.c_int32
        L.ts_profile_events.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32]
        L.ts_profile_events.restype = None
        _lib = L
    return _lib


def check(fn: str, status: int) -> None:
    if status != 0:
        raise TinyServeError(fn, status, lib().ts_status_str(status).decode())


def exported_symbols() -> list:
    L = lib()
    return [s for s in SYMBOLS if hasattr(L, s)]
