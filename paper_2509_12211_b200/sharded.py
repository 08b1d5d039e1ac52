"""Sequence-sharded decode step over G ranks.

Block-cyclic ownership: global page j lives on rank j % G at local index j // G
(ts_layout.shard_stride = G, shard_offset = rank).  One step is

  1. ts_score_pages       local pages (scores bit-identical to the unsharded ones)
  2. ts_select_topk       local top-K with GLOBAL ids (id = jl * G + rank)
  3. all-gather #1        candidates [2][rows][K] int32 words (fp32 score bits | ids)
  4. ts_select_merge      global top-K over the G*K candidates — identical on every rank
                          and equal to the unsharded selection
  5. ts_sparse_decode_attn  partial (o, lse) over the OWNED selected pages
  6. all-gather #2        partials [B*Hq*d | B*Hq] fp32
  7. ts_lse_merge         o = sum_r exp(lse_r - lse) o_r

With the bf16 tensor-core layouts the rank's kernels are fused to two launches: steps 1-2 are
ts_select_candidates and steps 4-5 are ts_shard_attend (candidate merge in the attention
kernel's prologue), so one step is 3 launches + 2 all-gathers; other layouts (or an `ops`
object without the fused calls, e.g. the CPU tests') run the composed sequence above.

Every arithmetic step runs in libtinyserve.so; this module only sequences the calls and
moves bytes (torch.distributed all_gather_into_tensor over NCCL on GPUs).  The protocol is
written against an `ops` object with the binding's signatures so the same sequencing is
exercised by the CPU (gloo) tests with a test-side implementation of the ops.
"""
from __future__ import annotations

import torch


class ShardStep:
    """Buffers and phases of one rank's sequence-sharded decode step."""

    def __init__(self, ops, layout, world: int, rank: int, budget_tokens: int, device):
        assert layout.shard_stride == world and layout.shard_offset == rank
        self.ops, self.L, self.G, self.r = ops, layout, world, rank
        # K = floor(budget / S) clipped to the GLOBAL page count (as ts.kmax unsharded)
        self.K = min(layout.max_pages * world, max(1, budget_tokens // layout.page_size))
        B, Hkv, Hq, d = layout.batch, layout.num_kv_heads, layout.num_q_heads, layout.head_dim
        self.rows = B * Hkv
        self.nq = B * Hq * d
        self.cand = torch.empty((2, self.rows, self.K), dtype=torch.int32, device=device)
        self.cand_g = torch.empty((world, 2, self.rows, self.K), dtype=torch.int32, device=device)
        self.part = torch.empty((self.nq + B * Hq,), dtype=torch.float32, device=device)
        self.part_g = torch.empty((world, self.nq + B * Hq), dtype=torch.float32, device=device)
        self.sel_ids = torch.empty((B, Hkv, self.K), dtype=torch.int32, device=device)
        self.sel_count = torch.empty((B, Hkv), dtype=torch.int32, device=device)
        self.scores = torch.empty((B, Hkv, layout.max_pages), dtype=torch.float32, device=device)
        self.o = torch.empty((B, Hq, d), dtype=torch.float32, device=device)
        self.lse = torch.empty((B, Hq), dtype=torch.float32, device=device)
        self.ws = None
        # fused two-launch form when the ops provide it (decided on first use: a layout the
        # fused kernels do not cover raises TS_ERR_UNSUPPORTED and falls back)
        self.fused = hasattr(ops, "select_candidates") and hasattr(ops, "shard_attend")

    def _unsupported(self, ex) -> bool:
        return getattr(ex, "name", "") == "TS_ERR_UNSUPPORTED"

    # -- phase 1: local scores + local candidates ------------------------------------------
    def local_candidates(self, q, meta, page_table, seq_lens):
        ops, L = self.ops, self.L
        if self.fused:
            try:
                ops.select_candidates(L, q, meta, page_table, seq_lens, self.K,
                                      cand_scores=self.cand[0].view(torch.float32),
                                      cand_ids=self.cand[1], cand_count=self.sel_count.view(-1))
                return self.cand
            except Exception as ex:  # noqa: BLE001
                if not self._unsupported(ex):
                    raise
                self.fused = False
        ops.score_pages(L, q, meta, page_table, seq_lens, scores=self.scores)
        cs = self.cand[0].view(torch.float32)
        ci = self.cand[1]
        ops.select_topk(self.scores.view(self.rows, L.max_pages), self.K, id_stride=self.G,
                        id_offset=self.r, sel_ids=ci, sel_scores=cs,
                        sel_count=self.sel_count.view(-1))
        return self.cand

    # -- phase 2: global selection (identical on all ranks) + partial attention -------------
    def partial_attention(self, cand_g, q, k_pool, v_pool, page_table, seq_lens, scale):
        ops, L = self.ops, self.L
        flat = cand_g.view(-1)
        o_r = self.part[: self.nq].view(L.batch, L.num_q_heads, L.head_dim)
        lse_r = self.part[self.nq:].view(L.batch, L.num_q_heads)
        if self.ws is None:
            self.ws = ops.new_workspace(ops.attn_workspace_bytes(L, self.K), q.device)
        if self.fused:
            try:
                ops.shard_attend(L, q, k_pool, v_pool, page_table, seq_lens, flat.view(torch.float32),
                                 flat[self.rows * self.K:], self.G, self.K, scale,
                                 part_stride=2 * self.rows * self.K, o=o_r, lse=lse_r,
                                 sel_ids=self.sel_ids, sel_count=self.sel_count, ws=self.ws)
                return self.part
            except Exception as ex:  # noqa: BLE001
                if not self._unsupported(ex):
                    raise
                self.fused = False
        ops.select_merge(flat.view(torch.float32), flat[self.rows * self.K:], self.K,
                         parts=self.G, rows=self.rows, k_part=self.K,
                         part_stride=2 * self.rows * self.K,
                         sel_ids=self.sel_ids.view(self.rows, self.K), want_scores=False,
                         sel_count=self.sel_count.view(-1))
        ops.sparse_decode_attn(L, q, k_pool, v_pool, page_table, seq_lens, self.sel_ids,
                               self.sel_count, scale, o=o_r, lse=lse_r, ws=self.ws)
        return self.part

    # -- phase 3: merge the partials ---------------------------------------------------------
    def merge(self, part_g):
        L = self.L
        rows_q = L.batch * L.num_q_heads
        flat = part_g.view(-1)
        self.ops.lse_merge(flat, flat[self.nq:], o=self.o.view(rows_q, L.head_dim),
                           lse=self.lse.view(rows_q), parts=self.G, rows=rows_q, d=L.head_dim,
                           part_stride=self.nq + rows_q)
        return self.o, self.lse

    # -- one rank's step with the exchanges emulated (bench.py --slice: per-GPU work) -------
    def step_local(self, q, k_pool, v_pool, meta, page_table, seq_lens, scale):
        """This rank's kernels of one step, each all-gather replaced by replicating the local
        buffer G times (same bytes and shapes as the real exchange; no collective)."""
        cand = self.local_candidates(q, meta, page_table, seq_lens)
        self.cand_g.copy_(cand.unsqueeze(0).expand_as(self.cand_g))
        part = self.partial_attention(self.cand_g, q, k_pool, v_pool, page_table, seq_lens, scale)
        self.part_g.copy_(part.unsqueeze(0).expand_as(self.part_g))
        return self.merge(self.part_g)

    # -- one step with torch.distributed (NCCL on GPUs, gloo on CPU) -----------------------
    def step(self, q, k_pool, v_pool, meta, page_table, seq_lens, scale, group=None):
        import torch.distributed as dist
        cand = self.local_candidates(q, meta, page_table, seq_lens)
        dist.all_gather_into_tensor(self.cand_g.view(-1), cand.view(-1), group=group)
        part = self.partial_attention(self.cand_g, q, k_pool, v_pool, page_table, seq_lens, scale)
        dist.all_gather_into_tensor(self.part_g.view(-1), part, group=group)
        return self.merge(self.part_g)


def shard_page_table(page_table: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """Local page table of `rank`: local index jl <-> global page jl * world + rank."""
    B, mp = page_table.shape
    mpl = -(-mp // world)
    out = torch.zeros((B, mpl), dtype=page_table.dtype, device=page_table.device)
    loc = page_table[:, rank::world]
    out[:, : loc.shape[1]] = loc
    return out.contiguous()


def emulate(ops, layout_global, world, q, k_pool, v_pool, page_table, seq_lens, budget_tokens,
            scale, metas=None, fused=True):
    """Run the G-rank protocol in one process on one device (shard emulation):
    the exchanges are concatenations.  Every rank reads the same global pool through its
    local page table.  Returns (o, lse, sel_ids, sel_count) of rank 0 plus every rank's
    selection (all must agree)."""
    from . import Layout, meta_build
    steps, pts = [], []
    for r in range(world):
        pt = shard_page_table(page_table, world, r)
        L = Layout(layout_global.batch, layout_global.num_q_heads, layout_global.num_kv_heads,
                   layout_global.head_dim, layout_global.page_size, pt.shape[1],
                   layout_global.num_blocks, world, r, layout_global.kv_dtype)
        steps.append(ShardStep(ops, L, world, r, budget_tokens, q.device))
        steps[-1].fused = steps[-1].fused and fused
        pts.append(pt)
    if metas is None:
        metas = [meta_build(s.L, k_pool, pts[r], seq_lens) for r, s in enumerate(steps)]
    cands = [s.local_candidates(q, metas[r], pts[r], seq_lens).clone() for r, s in enumerate(steps)]
    cand_g = torch.stack(cands)
    parts = [s.partial_attention(cand_g, q, k_pool, v_pool, pts[r], seq_lens, scale).clone()
             for r, s in enumerate(steps)]
    part_g = torch.stack(parts)
    o, lse = steps[0].merge(part_g)
    return o, lse, [s.sel_ids for s in steps], [s.sel_count for s in steps]
