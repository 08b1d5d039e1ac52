"""float64 CPU oracle for the TinyServe decode hot path (§3.5, Alg. 1).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product package
paper_2509_12211_b200 never imports it, and the two share no code.

The arithmetic lives in tinyserve_oracle.c (plain C, double precision, no -ffast-math);
this module only builds it with gcc and marshals numpy arrays through ctypes.  Every
function cites the paper passage it follows in the C source.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tinyserve_oracle.c")
_LIB = os.path.join(_HERE, "libtsoracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -fopenmp (IEEE double, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Layout(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("max_pages", ctypes.c_int32),
                ("num_blocks", ctypes.c_int32), ("dtype", ctypes.c_int32)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32 = ctypes.c_int
            L.or_meta_build.argtypes = [P, P, P, P, P, P, i32]
            L.or_meta_append.argtypes = [P, P, P, P, P, P, P, P, P]
            L.or_score_pages.argtypes = [P, P, P, P, P, P, i32]
            L.or_select_topk.argtypes = [P, i32, i32, P, P, i32, P, P, P, i32]
            L.or_sparse_attn.argtypes = [P, P, P, P, P, P, P, P, i32, ctypes.c_double, P, P, i32]
            L.or_decode_step.argtypes = [P, P, P, P, P, P, i32, ctypes.c_double, P, P, P, P, P, i32]
            L.or_lse_merge.argtypes = [i32, i32, i32, P, P, P, P]
            L.or_relevance.argtypes = [P, P, P, i32]
            L.or_relevance.restype = ctypes.c_double
            L.or_e4m3_value.argtypes = [ctypes.c_uint8]
            L.or_e4m3_value.restype = ctypes.c_double
            L.or_e4m3_round.argtypes = [ctypes.c_double]
            L.or_e4m3_round.restype = ctypes.c_uint8
            L.or_kv_exponent.argtypes = [ctypes.c_double]
            L.or_kv_exponent.restype = ctypes.c_int
            L.or_kv_quantize.argtypes = [ctypes.c_longlong, i32, P, P, P]
            L.or_kv_dequantize.argtypes = [ctypes.c_longlong, i32, P, P, P]
            L.or_num_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def num_threads() -> int:
    return lib().or_num_threads()


# ---------------------------------------------------------------- marshalling helpers
def _raw(t):
    """Host numpy view of the raw element bits of a torch tensor / numpy array.

    bf16 tensors are passed as uint16 bit patterns; fp32 as float32.  Returns
    (array, dtype_code) with dtype_code 1 = bf16, 0 = fp32.
    """
    try:
        import torch
        if isinstance(t, torch.Tensor):
            t = t.detach().to("cpu").contiguous()
            if t.dtype == torch.bfloat16:
                return t.view(torch.int16).numpy().view(np.uint16), 1
            if t.dtype == torch.float32:
                return t.numpy(), 0
            raise TypeError(t.dtype)
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(t)
    if a.dtype == np.uint16:
        return a, 1
    if a.dtype == np.float32:
        return a, 0
    raise TypeError(a.dtype)


def _i32(t):
    try:
        import torch
        if isinstance(t, torch.Tensor):
            t = t.detach().to("cpu")
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(t), dtype=np.int32)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def layout(B, Hq, Hkv, d, S, max_pages, num_blocks, dtype_code) -> _Layout:
    assert Hq % Hkv == 0 and (Hq // Hkv) * d <= 2048 and d <= 256
    return _Layout(B, Hq, Hkv, d, S, max_pages, num_blocks, dtype_code)


def _case_layout(q, k_pool, page_table):
    B, Hq, d = q.shape
    nb, Hkv, S, d2 = k_pool.shape
    assert d2 == d
    mp = page_table.shape[1]
    return B, Hq, Hkv, d, S, mp, nb


# ---------------------------------------------------------------- public oracle API
def meta_build(k_pool, page_table, seq_lens, threads: int = 0):
    """Eq. 1: (m, M) per logical page; returns (mmin, mmax) [B][Hkv][max_pages][d] f64."""
    kr, dc = _raw(k_pool)
    pt, sl = _i32(page_table), _i32(seq_lens)
    nb, Hkv, S, d = kr.shape
    B, mp = pt.shape
    L = layout(B, Hkv, Hkv, d, S, mp, nb, dc)
    mmin = np.zeros((B, Hkv, mp, d), np.float64)
    mmax = np.zeros((B, Hkv, mp, d), np.float64)
    lib().or_meta_build(ctypes.byref(L), _p(kr), _p(pt), _p(sl), _p(mmin), _p(mmax), threads)
    return mmin, mmax


def meta_append(k_new, v_new, seq_lens_before, page_table, k_pool_raw, v_pool_raw, mmin, mmax):
    """SPEC.md:56-59 incremental append; mutates the raw pools and the f64 metadata."""
    kn, dc = _raw(k_new)
    vn, _ = _raw(v_new)
    pt, sl = _i32(page_table), _i32(seq_lens_before)
    nb, Hkv, S, d = k_pool_raw.shape
    B, mp = pt.shape
    L = layout(B, Hkv, Hkv, d, S, mp, nb, dc)
    rc = lib().or_meta_append(ctypes.byref(L), _p(kn), _p(vn), _p(sl), _p(pt), _p(k_pool_raw),
                              _p(v_pool_raw), _p(mmin), _p(mmax))
    if rc:
        raise ValueError("or_meta_append: no page for the new token (shape error)")


def relevance(q, m, M) -> float:
    """Eq. 2 for one query and one page's (m, M), float64 inputs."""
    q = np.ascontiguousarray(q, np.float64)
    m = np.ascontiguousarray(m, np.float64)
    M = np.ascontiguousarray(M, np.float64)
    return lib().or_relevance(_p(q), _p(m), _p(M), q.shape[0])


def score_pages(q, mmin, mmax, seq_lens, page_size, threads: int = 0):
    """Eq. 2 + GQA max (reading R9); returns scores [B][Hkv][max_pages] f64 (-inf past P_b)."""
    qr, dc = _raw(q)
    sl = _i32(seq_lens)
    B, Hq, d = qr.shape
    _, Hkv, mp, _ = mmin.shape
    L = layout(B, Hq, Hkv, d, page_size, mp, 0, dc)
    mmin = np.ascontiguousarray(mmin, np.float64)
    mmax = np.ascontiguousarray(mmax, np.float64)
    sc = np.zeros((B, Hkv, mp), np.float64)
    lib().or_score_pages(ctypes.byref(L), _p(qr), _p(mmin), _p(mmax), _p(sl), _p(sc), threads)
    return sc


def select_topk(scores, row_len, k, ids_in=None, threads: int = 0):
    """Top-K per row, ties -> lower id, ids ascending (reading R6).

    scores [rows][stride] (any float dtype, widened to f64); returns (ids [rows][k] int32
    padded with -1, sel_scores [rows][k] f64, count [rows] int32).
    """
    sc = np.ascontiguousarray(scores, np.float64)
    rows, stride = sc.shape
    rl = None if row_len is None else _i32(row_len)
    ids = None if ids_in is None else _i32(ids_in)
    out = np.zeros((rows, k), np.int32)
    oscore = np.zeros((rows, k), np.float64)
    cnt = np.zeros(rows, np.int32)
    rc = lib().or_select_topk(_p(sc), rows, stride, _p(rl), _p(ids), k, _p(out), _p(oscore),
                              _p(cnt), threads)
    if rc:
        raise ValueError("k must be >= 1")
    return out, oscore, cnt


def sparse_attn(q, k_pool, v_pool, page_table, seq_lens, sel_ids, sel_count, scale,
                threads: int = 0):
    """SparseAttn over the selected pages; returns (o [B][Hq][d] f64, lse [B][Hq] f64)."""
    qr, dc = _raw(q)
    kr, _ = _raw(k_pool)
    vr, _ = _raw(v_pool)
    pt, sl = _i32(page_table), _i32(seq_lens)
    B, Hq, Hkv, d, S, mp, nb = _case_layout(qr, kr, pt)
    L = layout(B, Hq, Hkv, d, S, mp, nb, dc)
    ids = _i32(sel_ids).reshape(B, Hkv, -1)
    cnt = _i32(sel_count).reshape(B, Hkv)
    o = np.zeros((B, Hq, d), np.float64)
    lse = np.zeros((B, Hq), np.float64)
    lib().or_sparse_attn(ctypes.byref(L), _p(qr), _p(kr), _p(vr), _p(pt), _p(sl), _p(ids),
                         _p(cnt), ids.shape[2], float(scale), _p(o), _p(lse), threads)
    return o, lse


def decode_step(q, k_pool, v_pool, page_table, seq_lens, budget_tokens, scale,
                threads: int = 0, want_scores: bool = False):
    """Alg. 1 end to end (metadata recomputed from K).  Returns dict o, lse, sel_ids,
    sel_count (and scores if asked)."""
    qr, dc = _raw(q)
    kr, _ = _raw(k_pool)
    vr, _ = _raw(v_pool)
    pt, sl = _i32(page_table), _i32(seq_lens)
    B, Hq, Hkv, d, S, mp, nb = _case_layout(qr, kr, pt)
    L = layout(B, Hq, Hkv, d, S, mp, nb, dc)
    kmax = max(1, budget_tokens // S)
    o = np.zeros((B, Hq, d), np.float64)
    lse = np.zeros((B, Hq), np.float64)
    ids = np.zeros((B, Hkv, kmax), np.int32)
    cnt = np.zeros((B, Hkv), np.int32)
    sc = np.zeros((B, Hkv, mp), np.float64) if want_scores else None
    rc = lib().or_decode_step(ctypes.byref(L), _p(qr), _p(kr), _p(vr), _p(pt), _p(sl),
                              int(budget_tokens), float(scale), _p(o), _p(lse), _p(ids), _p(cnt),
                              _p(sc), threads)
    if rc:
        raise ValueError("configuration error (budget < 1, S < 1 or d < 1)")
    out = {"o": o, "lse": lse, "sel_ids": ids, "sel_count": cnt}
    if want_scores:
        out["scores"] = sc
    return out


def lse_merge(o_parts, lse_parts):
    """Merge partial attentions over disjoint token sets: o_parts [parts][rows][d]."""
    op = np.ascontiguousarray(o_parts, np.float64)
    lp = np.ascontiguousarray(lse_parts, np.float64)
    parts, rows, d = op.shape
    o = np.zeros((rows, d), np.float64)
    lse = np.zeros(rows, np.float64)
    lib().or_lse_merge(parts, rows, d, _p(op), _p(lp), _p(o), _p(lse))
    return o, lse


def widen(t) -> np.ndarray:
    """Exact float64 copy of a bf16/fp32 tensor (for assembling test inputs)."""
    a, dc = _raw(t)
    if dc == 1:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


# ---------------------------------------------------------------- FP8 KV (reading R21)
def e4m3_value(code: int) -> float:
    """Value of one OCP FP8 E4M3 code (format definition)."""
    return lib().or_e4m3_value(int(code))


def e4m3_round(x: float) -> int:
    """Nearest E4M3 code (ties to even, saturating at 448)."""
    return int(lib().or_e4m3_round(float(x)))


def kv_exponent(amax: float) -> int:
    """Smallest e in [-64, 64] with amax <= 448 * 2^e."""
    return int(lib().or_kv_exponent(float(amax)))


def kv_quantize(x):
    """Quantise bf16 rows [..., d] -> (codes uint8 [..., d], exps int8 [...]) (reading R21)."""
    xr, dc = _raw(x)
    assert dc == 1, "FP8 KV quantisation takes bf16 rows"
    d = xr.shape[-1]
    rows = int(np.prod(xr.shape[:-1]))
    codes = np.zeros(xr.shape, np.uint8)
    exps = np.zeros(xr.shape[:-1], np.int8)
    lib().or_kv_quantize(rows, d, _p(np.ascontiguousarray(xr)), _p(codes), _p(exps))
    return codes, exps


def kv_dequantize(codes, exps) -> np.ndarray:
    """codes [..., d] uint8, exps [...] int8 -> exact fp32 values [..., d]."""
    codes = np.ascontiguousarray(codes, np.uint8)
    exps = np.ascontiguousarray(exps, np.int8)
    d = codes.shape[-1]
    rows = int(np.prod(codes.shape[:-1]))
    out = np.zeros(codes.shape, np.float32)
    lib().or_kv_dequantize(rows, d, _p(codes), _p(exps), _p(out))
    return out


def decode_step_fp8(q, k_codes, k_exps, v_codes, v_exps, page_table, seq_lens, budget_tokens,
                    scale, threads: int = 0, want_scores: bool = False):
    """Alg. 1 over an FP8 cache (reading R21): the K / V pools are dequantised exactly to
    fp32 ([NB][Hkv][S][d] codes with [NB][Hkv][S] exponents), q (bf16) is widened exactly,
    and the float64 decode_step runs unchanged on those values — metadata over the
    dequantised keys (Eq. 1), scores (Eq. 2), top-K, attention."""
    import torch
    kd = torch.from_numpy(kv_dequantize(k_codes, k_exps))
    vd = torch.from_numpy(kv_dequantize(v_codes, v_exps))
    qf = torch.from_numpy(widen(q).astype(np.float32))
    return decode_step(qf, kd, vd, page_table, seq_lens, budget_tokens, scale, threads=threads,
                       want_scores=want_scores)
