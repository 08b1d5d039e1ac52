"""TinyServe decode hot path on B200 (sm_100a): query-aware page selection + sparse attention.

Thin Python binding over libtinyserve.so (include/tinyserve.h).  PyTorch is used only for
device memory, streams and process groups; every step of the path runs in the library's
CUDA kernels.  Names follow the C ABI:

  meta_append, meta_build, score_pages, select_topk, sparse_decode_attn, decode_step,
  lse_merge, workspace_bytes, attn_workspace_bytes

Tensors: q [B][Hq][d], k_pool / v_pool [NB][Hkv][S][d], meta
[B][Hkv][max_pages][2][d] (logical page order; kv dtype: bf16 or fp32), page_table
[B][max_pages] int32, seq_lens [B] int32; o [B][Hq][d] fp32, lse [B][Hq] fp32.
"""
from __future__ import annotations

import torch

from ._lib import Layout, TinyServeError, TS_BF16, TS_F32, TS_FP8E4M3, check, exported_symbols, lib

__all__ = ["Layout", "TinyServeError", "make_layout", "meta_append", "meta_build",
           "score_pages", "select_topk", "sparse_decode_attn", "decode_step", "decode_step_append", "decode_step_prefetch", "select_merge", "lse_merge",
           "workspace_bytes", "attn_workspace_bytes", "dense_decode_attn", "dense_workspace_bytes", "new_workspace", "new_meta", "kmax", "launch_count",
           "profile_events", "kv_quantize", "fp8_pool", "fp8_views", "fp8_split", "pool_bytes",
           "select_candidates", "shard_attend",
           "exported_symbols", "PagedKV"]


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return TS_BF16
    if dt == torch.float32:
        return TS_F32
    raise TypeError(f"kv dtype must be bfloat16 or float32, got {dt}")


def _cuda(*ts):
    for t in ts:
        if t is not None and (not isinstance(t, torch.Tensor) or not t.is_cuda):
            raise TypeError("tinyserve: every tensor must be a CUDA tensor (no CPU fallback)")
        if t is not None and not t.is_contiguous():
            raise ValueError("tinyserve: tensors must be contiguous")


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def make_layout(q: torch.Tensor, k_pool: torch.Tensor, page_table: torch.Tensor,
                shard_stride: int = 1, shard_offset: int = 0, pool_shape=None) -> Layout:
    """Layout of a cache.  An FP8 cache (reading R21) is a flat uint8 pool (codes, then row
    exponents; see fp8_pool) and needs pool_shape = (num_blocks, Hkv, S, d); q stays bf16."""
    B, Hq, d = q.shape
    if k_pool.dtype == torch.uint8:
        if pool_shape is None:
            raise ValueError("an FP8 pool needs pool_shape=(num_blocks, Hkv, S, d)")
        nb, Hkv, S, d2 = pool_shape
        if d2 != d or q.dtype != torch.bfloat16 or k_pool.numel() < nb * Hkv * S * (d + 1):
            raise ValueError("FP8 cache: q must be bf16 and the pool hold num_blocks*Hkv*S*(d+1) bytes")
        return Layout(B, Hq, Hkv, d, S, page_table.shape[1], nb, shard_stride, shard_offset,
                      TS_FP8E4M3)
    nb, Hkv, S, d2 = k_pool.shape
    if d2 != d or q.dtype != k_pool.dtype:
        raise ValueError("q and k_pool disagree on head_dim or dtype")
    return Layout(B, Hq, Hkv, d, S, page_table.shape[1], nb, shard_stride, shard_offset,
                  _dtype_code(k_pool.dtype))


def kmax(layout: Layout, budget_tokens: int) -> int:
    """K = floor(budget / S) clipped to [1, max_pages] (reading R4); per row clipped to P_b."""
    return min(layout.max_pages, max(1, budget_tokens // layout.page_size))


def workspace_bytes(layout: Layout, budget_tokens: int) -> int:
    return lib().ts_workspace_bytes(layout, budget_tokens)


def attn_workspace_bytes(layout: Layout, sel_stride: int) -> int:
    return lib().ts_attn_workspace_bytes(layout, sel_stride)


def new_workspace(nbytes: int, device) -> torch.Tensor:
    """Zero-filled workspace (the split-K tickets must start at zero; the library re-arms them)."""
    return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def profile_events(events) -> None:
    """Make ts_decode_step record the given torch.cuda.Events (4: before score, after score,
    after select, after attention) on its stream; None clears.  Events must be created with
    external=True and recorded once beforehand (lazy creation)."""
    if not events:
        lib().ts_profile_events(None, 0)
        return
    import ctypes
    arr = (ctypes.c_void_p * len(events))(*[(e.cuda_event if e is not None else None)
                                             for e in events])
    lib().ts_profile_events(arr, len(events))


def launch_count() -> int:
    """Kernel launches enqueued by the last library call on this thread."""
    return lib().ts_last_launch_count()


def meta_append(layout, k_new, v_new, seq_lens, page_table, k_pool, v_pool, meta,
                advance=True, stream=None):
    """Append one token per sequence (k_new, v_new [B][Hkv][d]) at position seq_lens[b];
    with advance=True the kernel also increments seq_lens."""
    _cuda(k_new, v_new, seq_lens, page_table, k_pool, v_pool, meta)
    check("ts_meta_append", lib().ts_meta_append(
        layout, _ptr(k_new), _ptr(v_new), _ptr(seq_lens), int(bool(advance)), _ptr(page_table),
        _ptr(k_pool), _ptr(v_pool), _ptr(meta), _stream(stream)))


def new_meta(layout, dtype, device) -> torch.Tensor:
    """Zeroed metadata [B][Hkv][max_pages][2][d] (logical page order; bf16 for FP8 caches)."""
    if layout.kv_dtype == TS_FP8E4M3:
        dtype = torch.bfloat16
    return torch.zeros((layout.batch, layout.num_kv_heads, layout.max_pages, 2, layout.head_dim),
                       dtype=dtype, device=device)


def meta_build(layout, k_pool, page_table, seq_lens, meta=None, stream=None):
    if meta is None:
        meta = new_meta(layout, k_pool.dtype, k_pool.device)
    _cuda(k_pool, page_table, seq_lens, meta)
    check("ts_meta_build", lib().ts_meta_build(layout, _ptr(k_pool), _ptr(page_table),
                                               _ptr(seq_lens), _ptr(meta), _stream(stream)))
    return meta


def pool_bytes(layout) -> int:
    return lib().ts_pool_bytes(layout)


def fp8_pool(num_blocks, num_kv_heads, page_size, head_dim, device) -> torch.Tensor:
    """A zeroed FP8 pool (reading R21): 1040-byte sub-page records of 16 rows (codes [16][64]
    then the 16 row exponents), NB*Hkv*S*65 bytes."""
    return torch.zeros(num_blocks * num_kv_heads * page_size * (head_dim + 1), dtype=torch.uint8,
                       device=device)


def fp8_views(pool, num_blocks, num_kv_heads, page_size, head_dim=64):
    """(codes [NB][Hkv][S/16][16][64] uint8, exps [NB][Hkv][S/16][16] int8): writable views of
    an FP8 pool's sub-page records (token slot s of a block is [s // 16][s % 16])."""
    rec = pool.view(num_blocks, num_kv_heads, page_size // 16, 16 * head_dim + 16)
    codes = rec[..., : 16 * head_dim].unflatten(-1, (16, head_dim))
    exps = rec[..., 16 * head_dim:].view(torch.int8)
    return codes, exps


def fp8_split(pool, num_blocks, num_kv_heads, page_size, head_dim=64):
    """Contiguous copies (codes [NB][Hkv][S][64] uint8, exps [NB][Hkv][S] int8) of an FP8 pool."""
    c, e = fp8_views(pool, num_blocks, num_kv_heads, page_size, head_dim)
    return (c.reshape(num_blocks, num_kv_heads, page_size, head_dim).contiguous(),
            e.reshape(num_blocks, num_kv_heads, page_size).contiguous())


def kv_quantize(src: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """bf16 rows [..., d] (a pool [NB][Hkv][S][d]; rows a multiple of 16) -> FP8 pool
    (ts_kv_quantize)."""
    d = src.shape[-1]
    rows = src.numel() // d
    if out is None:
        out = torch.empty(rows * (d + 1), dtype=torch.uint8, device=src.device)
    _cuda(src, out)
    check("ts_kv_quantize", lib().ts_kv_quantize(rows, d, _ptr(src), _ptr(out), _stream(stream)))
    return out


def score_pages(layout, q, meta, page_table, seq_lens, scores=None, stream=None):
    if scores is None:
        scores = torch.empty((layout.batch, layout.num_kv_heads, layout.max_pages),
                             dtype=torch.float32, device=q.device)
    _cuda(q, meta, page_table, seq_lens, scores)
    check("ts_score_pages", lib().ts_score_pages(layout, _ptr(q), _ptr(meta), _ptr(page_table),
                                                 _ptr(seq_lens), _ptr(scores), _stream(stream)))
    return scores


def select_topk(scores, k, row_len=None, ids_in=None, id_stride=1, id_offset=0,
                sel_ids=None, sel_scores=None, sel_count=None, want_scores=True, stream=None):
    """scores [rows][stride] fp32 -> (sel_ids [rows][k], sel_scores [rows][k], sel_count [rows])."""
    s2 = scores.reshape(-1, scores.shape[-1])
    rows, stride = s2.shape
    dev = scores.device
    if sel_ids is None:
        sel_ids = torch.empty((rows, k), dtype=torch.int32, device=dev)
    if sel_scores is None and want_scores:
        sel_scores = torch.empty((rows, k), dtype=torch.float32, device=dev)
    if sel_count is None:
        sel_count = torch.empty((rows,), dtype=torch.int32, device=dev)
    _cuda(s2, row_len, ids_in, sel_ids, sel_scores, sel_count)
    check("ts_select_topk", lib().ts_select_topk(
        _ptr(s2), rows, stride, _ptr(row_len), _ptr(ids_in), id_stride, id_offset, k,
        _ptr(sel_ids), _ptr(sel_scores), _ptr(sel_count), _stream(stream)))
    return sel_ids, sel_scores, sel_count


def sparse_decode_attn(layout, q, k_pool, v_pool, page_table, seq_lens, sel_ids, sel_count,
                       scale, o=None, lse=None, ws=None, want_lse=True, stream=None):
    dev = q.device
    sel_stride = sel_ids.shape[-1]
    if o is None:
        o = torch.empty((layout.batch, layout.num_q_heads, layout.head_dim), dtype=torch.float32,
                        device=dev)
    if lse is None and want_lse:
        lse = torch.empty((layout.batch, layout.num_q_heads), dtype=torch.float32, device=dev)
    if ws is None:
        ws = new_workspace(attn_workspace_bytes(layout, sel_stride), dev)
    _cuda(q, k_pool, v_pool, page_table, seq_lens, sel_ids, sel_count, o, lse, ws)
    check("ts_sparse_decode_attn", lib().ts_sparse_decode_attn(
        layout, _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(page_table), _ptr(seq_lens),
        _ptr(sel_ids), _ptr(sel_count), sel_stride, float(scale), _ptr(o), _ptr(lse), _ptr(ws),
        ws.numel(), _stream(stream)))
    return o, lse


def dense_decode_attn(layout, q, k_pool, v_pool, page_table, seq_lens, scale, o=None, lse=None,
                      ws=None, want_lse=True, stream=None):
    """FullCache baseline: attention over every valid token (ts_dense_decode_attn)."""
    dev = q.device
    if o is None:
        o = torch.empty((layout.batch, layout.num_q_heads, layout.head_dim), dtype=torch.float32,
                        device=dev)
    if lse is None and want_lse:
        lse = torch.empty((layout.batch, layout.num_q_heads), dtype=torch.float32, device=dev)
    if ws is None:
        ws = new_workspace(lib().ts_dense_workspace_bytes(layout), dev)
    _cuda(q, k_pool, v_pool, page_table, seq_lens, o, lse, ws)
    check("ts_dense_decode_attn", lib().ts_dense_decode_attn(
        layout, _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(page_table), _ptr(seq_lens),
        float(scale), _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream(stream)))
    return o, lse


def dense_workspace_bytes(layout) -> int:
    return lib().ts_dense_workspace_bytes(layout)


def decode_step(layout, q, k_pool, v_pool, meta, page_table, seq_lens, budget_tokens, scale,
                o=None, lse=None, sel_ids=None, sel_count=None, ws=None, want_lse=True,
                want_selection=True, stream=None):
    """Alg. 1 end to end: score -> select -> sparse attention.  Returns (o, lse, sel_ids, sel_count)."""
    dev = q.device
    K = kmax(layout, budget_tokens)
    rows = layout.batch * layout.num_kv_heads
    if o is None:
        o = torch.empty((layout.batch, layout.num_q_heads, layout.head_dim), dtype=torch.float32,
                        device=dev)
    if lse is None and want_lse:
        lse = torch.empty((layout.batch, layout.num_q_heads), dtype=torch.float32, device=dev)
    if want_selection:
        if sel_ids is None:
            sel_ids = torch.empty((layout.batch, layout.num_kv_heads, K), dtype=torch.int32, device=dev)
        if sel_count is None:
            sel_count = torch.empty((layout.batch, layout.num_kv_heads), dtype=torch.int32, device=dev)
    if ws is None:
        ws = new_workspace(workspace_bytes(layout, budget_tokens), dev)
    _cuda(q, k_pool, v_pool, meta, page_table, seq_lens, o, lse, sel_ids, sel_count, ws)
    check("ts_decode_step", lib().ts_decode_step(
        layout, _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(meta), _ptr(page_table), _ptr(seq_lens),
        int(budget_tokens), float(scale), _ptr(o), _ptr(lse), _ptr(sel_ids), _ptr(sel_count),
        _ptr(ws), ws.numel(), _stream(stream)))
    return o, lse, sel_ids, sel_count


def decode_step_prefetch(layout, q, k_pool, v_pool, meta, page_table, seq_lens, budget_tokens,
                         scale, sel_ids, sel_count, o=None, lse=None, ws=None, want_lse=True,
                         stream=None):
    """Alg. 1 with cross-step reuse (NEXT-2): sel_ids / sel_count hold the previous step's
    selection on entry (prefetched into L2 while the pages are scored) and this step's on
    return.  Results equal decode_step.  Returns (o, lse, sel_ids, sel_count)."""
    dev = q.device
    if o is None:
        o = torch.empty((layout.batch, layout.num_q_heads, layout.head_dim), dtype=torch.float32,
                        device=dev)
    if lse is None and want_lse:
        lse = torch.empty((layout.batch, layout.num_q_heads), dtype=torch.float32, device=dev)
    if ws is None:
        ws = new_workspace(workspace_bytes(layout, budget_tokens), dev)
    _cuda(q, k_pool, v_pool, meta, page_table, seq_lens, o, lse, sel_ids, sel_count, ws)
    check("ts_decode_step_prefetch", lib().ts_decode_step_prefetch(
        layout, _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(meta), _ptr(page_table), _ptr(seq_lens),
        int(budget_tokens), float(scale), _ptr(o), _ptr(lse), _ptr(sel_ids), _ptr(sel_count),
        _ptr(ws), ws.numel(), _stream(stream)))
    return o, lse, sel_ids, sel_count


def decode_step_append(layout, q, k_new, v_new, k_pool, v_pool, meta, page_table, seq_lens,
                       budget_tokens, scale, o=None, lse=None, sel_ids=None, sel_count=None, ws=None,
                       want_lse=True, want_selection=True, stream=None):
    """Serving-loop step: append the newest token (slot seq_lens - 1: seq_lens already counts
    it) into k_pool / v_pool / meta, then Alg. 1 — one launch on the bf16 cluster path.
    Returns (o, lse, sel_ids, sel_count)."""
    dev = q.device
    K = kmax(layout, budget_tokens)
    if o is None:
        o = torch.empty((layout.batch, layout.num_q_heads, layout.head_dim), dtype=torch.float32,
                        device=dev)
    if lse is None and want_lse:
        lse = torch.empty((layout.batch, layout.num_q_heads), dtype=torch.float32, device=dev)
    if want_selection:
        if sel_ids is None:
            sel_ids = torch.empty((layout.batch, layout.num_kv_heads, K), dtype=torch.int32, device=dev)
        if sel_count is None:
            sel_count = torch.empty((layout.batch, layout.num_kv_heads), dtype=torch.int32, device=dev)
    if ws is None:
        ws = new_workspace(workspace_bytes(layout, budget_tokens), dev)
    _cuda(q, k_new, v_new, k_pool, v_pool, meta, page_table, seq_lens, o, lse, sel_ids, sel_count, ws)
    check("ts_decode_step_append", lib().ts_decode_step_append(
        layout, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(k_pool), _ptr(v_pool), _ptr(meta),
        _ptr(page_table), _ptr(seq_lens), int(budget_tokens), float(scale), _ptr(o), _ptr(lse),
        _ptr(sel_ids), _ptr(sel_count), _ptr(ws), ws.numel(), _stream(stream)))
    return o, lse, sel_ids, sel_count


def select_merge(cand_scores, cand_ids, k, parts=None, rows=None, k_part=None, part_stride=0,
                 sel_ids=None, sel_scores=None, sel_count=None, want_scores=True, stream=None):
    """Global top-k over per-part candidate lists ([parts][rows][k_part] unless part_stride
    and explicit sizes are given).  Returns (sel_ids [rows][k], sel_scores, sel_count)."""
    if parts is None:
        parts, rows, k_part = cand_scores.shape
    dev = cand_scores.device
    if sel_ids is None:
        sel_ids = torch.empty((rows, k), dtype=torch.int32, device=dev)
    if sel_scores is None and want_scores:
        sel_scores = torch.empty((rows, k), dtype=torch.float32, device=dev)
    if sel_count is None:
        sel_count = torch.empty((rows,), dtype=torch.int32, device=dev)
    _cuda(sel_ids, sel_scores, sel_count)
    check("ts_select_merge", lib().ts_select_merge(
        cand_scores.data_ptr(), cand_ids.data_ptr(), parts, part_stride, rows, k_part, k,
        _ptr(sel_ids), _ptr(sel_scores), _ptr(sel_count), _stream(stream)))
    return sel_ids, sel_scores, sel_count


def select_candidates(layout, q, meta, page_table, seq_lens, k, cand_scores=None, cand_ids=None,
                      cand_count=None, stream=None):
    """One rank's local half of the sequence-sharded step (ts_select_candidates): the k owned
    pages with the largest scores per row, GLOBAL ids ascending.  Returns (scores, ids, count)."""
    rows, dev = layout.batch * layout.num_kv_heads, q.device
    if cand_scores is None:
        cand_scores = torch.empty((rows, k), dtype=torch.float32, device=dev)
    if cand_ids is None:
        cand_ids = torch.empty((rows, k), dtype=torch.int32, device=dev)
    if cand_count is None:
        cand_count = torch.empty((rows,), dtype=torch.int32, device=dev)
    _cuda(q, meta, page_table, seq_lens, cand_scores, cand_ids, cand_count)
    check("ts_select_candidates", lib().ts_select_candidates(
        layout, _ptr(q), _ptr(meta), _ptr(page_table), _ptr(seq_lens), int(k), _ptr(cand_scores),
        _ptr(cand_ids), _ptr(cand_count), _stream(stream)))
    return cand_scores, cand_ids, cand_count


def shard_attend(layout, q, k_pool, v_pool, page_table, seq_lens, cand_scores, cand_ids, parts, k,
                 scale, part_stride=0, o=None, lse=None, sel_ids=None, sel_count=None, ws=None,
                 stream=None):
    """Candidate merge + partial attention over the owned selected pages (ts_shard_attend).
    cand_scores / cand_ids: `parts` lists of [rows][k] (part_stride elements apart; 0 =
    contiguous).  Returns (o, lse, sel_ids, sel_count)."""
    dev = q.device
    if o is None:
        o = torch.empty((layout.batch, layout.num_q_heads, layout.head_dim), dtype=torch.float32, device=dev)
    if lse is None:
        lse = torch.empty((layout.batch, layout.num_q_heads), dtype=torch.float32, device=dev)
    if ws is None:
        ws = new_workspace(attn_workspace_bytes(layout, k), dev)
    _cuda(q, k_pool, v_pool, page_table, seq_lens, o, lse, sel_ids, sel_count, ws)
    check("ts_shard_attend", lib().ts_shard_attend(
        layout, _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(page_table), _ptr(seq_lens),
        cand_scores.data_ptr(), cand_ids.data_ptr(), int(parts), int(part_stride), int(k),
        float(scale), _ptr(o), _ptr(lse), _ptr(sel_ids), _ptr(sel_count), _ptr(ws), ws.numel(),
        _stream(stream)))
    return o, lse, sel_ids, sel_count


def lse_merge(o_parts, lse_parts, o=None, lse=None, parts=None, rows=None, d=None,
              part_stride=0, stream=None):
    """o_parts [parts][rows][d], lse_parts [parts][rows] -> (o [rows][d], lse [rows]).
    With part_stride != 0, parts/rows/d must be given and both arrays are strided views."""
    if parts is None:
        parts, rows, d = o_parts.shape
    dev = o_parts.device
    if o is None:
        o = torch.empty((rows, d), dtype=torch.float32, device=dev)
    if lse is None:
        lse = torch.empty((rows,), dtype=torch.float32, device=dev)
    _cuda(o, lse)
    check("ts_lse_merge", lib().ts_lse_merge(parts, rows, d, o_parts.data_ptr(),
                                             lse_parts.data_ptr(), part_stride, _ptr(o), _ptr(lse),
                                             _stream(stream)))
    return o, lse


class PagedKV:
    """A paged KV cache on one GPU (vLLM-style block pool + page table) with its metadata.

    Convenience owner of the device tensors for one attention layer; all compute goes
    through the C ABI.  `append` = ts_meta_append + seq_lens += 1 (SPEC.md:388 order:
    append, then select); `step` = ts_decode_step.
    """

    def __init__(self, k_pool, v_pool, page_table, seq_lens, num_q_heads, meta=None,
                 shard_stride=1, shard_offset=0):
        _cuda(k_pool, v_pool, page_table, seq_lens)
        self.k_pool, self.v_pool = k_pool, v_pool
        self.page_table, self.seq_lens = page_table, seq_lens
        B = page_table.shape[0]
        q_like = torch.empty((B, num_q_heads, k_pool.shape[-1]), dtype=k_pool.dtype, device="meta")
        self.layout = make_layout(q_like, k_pool, page_table, shard_stride, shard_offset)
        self.meta = meta if meta is not None else meta_build(self.layout, k_pool, page_table, seq_lens)
        self._ws = {}

    def workspace(self, budget_tokens):
        if budget_tokens not in self._ws:
            self._ws[budget_tokens] = new_workspace(workspace_bytes(self.layout, budget_tokens),
                                                    self.k_pool.device)
        return self._ws[budget_tokens]

    def append(self, k_new, v_new, stream=None):
        meta_append(self.layout, k_new, v_new, self.seq_lens, self.page_table, self.k_pool,
                    self.v_pool, self.meta, advance=True, stream=stream)

    def step(self, q, budget_tokens, scale, **kw):
        return decode_step(self.layout, q, self.k_pool, self.v_pool, self.meta, self.page_table,
                           self.seq_lens, budget_tokens, scale, ws=self.workspace(budget_tokens), **kw)
