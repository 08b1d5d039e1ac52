"""Sequence-sharded decode step over REAL torch.distributed process groups
on CPU: world_size 2 (and 3), gloo backend, one process per rank.

`paper_2509_12211_b200.sharded.ShardStep` sequences the per-rank calls (local score,
local top-K with global ids, all-gather #1, candidate merge, partial attention over owned
pages, all-gather #2, LSE merge).  On a GPU box the ops are the C ABI; here they are a
test-side adapter over the float64 oracle, so this checks the host protocol — block-cyclic
ownership, candidate packing, all-gather layouts, part strides — against the unsharded
oracle: the global selection must equal the unsharded one exactly and o must agree to
float64 merge rounding.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2509_12211_b200 import sharded
from paper_2509_12211_b200._lib import Layout, TS_BF16, TS_F32


class OracleOps:
    """The binding's signatures, computed by the oracle on host tensors (test-only)."""

    def __init__(self, k_pool_global, page_table_global):
        self.k_pool = k_pool_global
        self.pt = page_table_global

    # metadata of the local pages: global page jl * G + r, logical order
    def meta_local(self, L, seq_lens):
        mmin, mmax = oracle.meta_build(self.k_pool, self.pt, seq_lens)
        G, r = L.shard_stride, L.shard_offset
        lo = np.zeros(mmin.shape[:2] + (L.max_pages,) + mmin.shape[3:])
        hi = np.zeros_like(lo)
        n = mmin[:, :, r::G].shape[2]
        lo[:, :, :n], hi[:, :, :n] = mmin[:, :, r::G], mmax[:, :, r::G]
        return lo, hi

    def score_pages(self, L, q, meta, page_table, seq_lens, scores):
        G, r = L.shard_stride, L.shard_offset
        lo, hi = meta
        # score the local records; a local page exists iff its global id < P_b
        sc = np.full(scores.shape, -np.inf)
        P = [(-(-int(x) // L.page_size)) for x in seq_lens]
        every = torch.full_like(seq_lens, L.max_pages * L.page_size)  # score every record
        full = oracle.score_pages(q, lo, hi, every, L.page_size)
        for b in range(L.batch):
            for jl in range(L.max_pages):
                if jl * G + r < P[b]:
                    sc[b, :, jl] = full[b, :, jl]
        scores.copy_(torch.from_numpy(sc).to(torch.float32))

    def select_topk(self, scores2d, k, id_stride, id_offset, sel_ids, sel_scores, sel_count):
        rows, n = scores2d.shape
        ids_in = np.tile(np.arange(n, dtype=np.int32) * id_stride + id_offset, (rows, 1))
        ids, sc, cnt = oracle.select_topk(scores2d.numpy(), None, k, ids_in=ids_in)
        sel_ids.copy_(torch.from_numpy(ids))
        sel_scores.copy_(torch.from_numpy(sc).to(torch.float32))
        sel_count.copy_(torch.from_numpy(cnt))

    def select_merge(self, flat_scores, flat_ids, k, parts, rows, k_part, part_stride, sel_ids,
                     want_scores, sel_count):
        s = np.empty((rows, parts * k_part))
        i = np.empty((rows, parts * k_part), np.int32)
        fs, fi = flat_scores.numpy(), flat_ids.numpy()
        for p in range(parts):
            for r in range(rows):
                a = p * part_stride + r * k_part
                s[r, p * k_part:(p + 1) * k_part] = fs[a:a + k_part]
                i[r, p * k_part:(p + 1) * k_part] = fi[a:a + k_part]
        ids, _, cnt = oracle.select_topk(s, None, k, ids_in=i)
        sel_ids.copy_(torch.from_numpy(ids))
        sel_count.copy_(torch.from_numpy(cnt))

    def new_workspace(self, nbytes, device):
        return torch.zeros(max(1, nbytes), dtype=torch.uint8)

    def attn_workspace_bytes(self, L, sel_stride):
        return 256

    def sparse_decode_attn(self, L, q, k_pool, v_pool, page_table, seq_lens, sel_ids, sel_count,
                           scale, o, lse, ws):
        G, r = L.shard_stride, L.shard_offset
        B, Hkv, K = sel_ids.shape
        # owned selected pages only, through a global-index view of the local page table
        mp_g = L.max_pages * G
        pt_g = torch.zeros((B, mp_g), dtype=torch.int32)
        pt_g[:, r::G] = page_table[:, : pt_g[:, r::G].shape[1]]
        own = np.full((B, Hkv, K), -1, np.int32)
        cnt = np.zeros((B, Hkv), np.int32)
        ids, c = sel_ids.numpy(), sel_count.numpy()
        for b in range(B):
            for g in range(Hkv):
                mine = [int(x) for x in ids[b, g, :c[b, g]] if x % G == r]
                own[b, g, :len(mine)] = mine
                cnt[b, g] = len(mine)
        oo, ll = oracle.sparse_attn(q, k_pool, v_pool, pt_g, seq_lens, own, cnt, scale)
        o.copy_(torch.from_numpy(oo).to(torch.float32))
        lse.copy_(torch.from_numpy(ll).to(torch.float32))

    def lse_merge(self, flat_o, flat_lse, o, lse, parts, rows, d, part_stride):
        fo, fl = flat_o.numpy().astype(np.float64), flat_lse.numpy().astype(np.float64)
        op = np.stack([fo[p * part_stride: p * part_stride + rows * d].reshape(rows, d)
                       for p in range(parts)])
        lp = np.stack([fl[p * part_stride: p * part_stride + rows] for p in range(parts)])
        oo, ll = oracle.lse_merge(op, lp)
        o.copy_(torch.from_numpy(oo).to(torch.float32))
        lse.copy_(torch.from_numpy(ll).to(torch.float32))


def _case(cname):
    cfg = synth.config(cname, batch=2, ctx=700, budget_tokens=96) if cname == "c3" else \
        synth.config(cname, batch=2, ctx=900, budget_tokens=128)
    case = synth.make_case(cfg, seed=7, ragged=True)
    import oracle.margin
    ref = oracle.margin.enforce(case, cfg.budget_tokens)
    return cfg, case, ref


def _worker(rank, world, port, cname, q_bits, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, case, _ = _case(cname)
        case["q"] = q_bits.clone()  # the margin-enforced q from the parent
        pt_l = sharded.shard_page_table(case["page_table"], world, rank)
        dt = TS_BF16 if cfg.dtype == "bf16" else TS_F32
        L = Layout(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.page_size,
                   pt_l.shape[1], case["num_blocks"], world, rank, dt)
        ops = OracleOps(case["k_pool"], case["page_table"])
        st = sharded.ShardStep(ops, L, world, rank, cfg.budget_tokens, torch.device("cpu"))
        meta = ops.meta_local(L, case["seq_lens"])
        o, lse = st.step(case["q"], case["k_pool"], case["v_pool"], meta, pt_l, case["seq_lens"],
                         cfg.scale)
        out[rank] = (o.clone(), lse.clone(), st.sel_ids.clone(), st.sel_count.clone())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cname,world", [("c3", 2), ("c2", 2), ("c3", 3)])
def test_sharded_step_gloo_matches_unsharded_oracle(orc, cname, world):
    cfg, case, ref = _case(cname)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as man:
        out = man.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, cname, case["q"], out))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(240)
            assert p.exitcode == 0, f"rank process failed (exit {p.exitcode})"
        res = dict(out)
    for r in range(world):
        o, lse, ids, cnt = res[r]
        # the global selection is identical on every rank and equals the unsharded one
        assert np.array_equal(cnt.numpy(), ref["sel_count"])
        assert np.array_equal(ids.numpy(), ref["sel_ids"])
        # partial attentions merged across ranks == attention over the whole selection
        assert np.abs(o.numpy() - ref["o"]).max() < 1e-5
        lr, lo = ref["lse"], lse.numpy()
        fin = np.isfinite(lr)
        assert np.array_equal(fin, np.isfinite(lo))
        assert np.abs(lo[fin] - lr[fin]).max() < 1e-5
