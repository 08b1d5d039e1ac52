"""Sequence-sharded step over NCCL, 2 ranks on 2 GPUs: the selection is
bit-identical to the unsharded step and o matches it within fp32 merge rounding.  Skips on
boxes with fewer than 2 GPUs (this run's gpurun / driver tiers have one)."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, out):
    import numpy as np
    import torch.distributed as dist

    import synth
    import paper_2509_12211_b200 as ts
    from paper_2509_12211_b200 import sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    cfg = synth.config("c5", batch=2, ctx=20000, budget_tokens=1024)
    case = synth.make_case(cfg, seed=33, device=dev, ragged=True)
    L = ts.make_layout(case["q"], case["k_pool"], case["page_table"])
    meta = ts.meta_build(L, case["k_pool"], case["page_table"], case["seq_lens"])
    o1, l1, i1, c1 = ts.decode_step(L, case["q"], case["k_pool"], case["v_pool"], meta,
                                    case["page_table"], case["seq_lens"], cfg.budget_tokens, cfg.scale)
    pt = sharded.shard_page_table(case["page_table"], world, rank)
    Ls = ts.Layout(L.batch, L.num_q_heads, L.num_kv_heads, L.head_dim, L.page_size, pt.shape[1],
                   L.num_blocks, world, rank, L.kv_dtype)
    ms = ts.meta_build(Ls, case["k_pool"], pt, case["seq_lens"])
    st = sharded.ShardStep(ts, Ls, world, rank, cfg.budget_tokens, dev)
    o, lse = st.step(case["q"], case["k_pool"], case["v_pool"], ms, pt, case["seq_lens"], cfg.scale)
    torch.cuda.synchronize()
    ok = torch.equal(st.sel_ids, i1) and torch.equal(st.sel_count, c1)
    err = float((o - o1).abs().max())
    out[rank] = (bool(ok), err)
    dist.destroy_process_group()


def test_sequence_sharded_nccl_two_ranks():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        ok, err = out[r]
        assert ok, f"rank {r}: sharded selection differs from the unsharded one"
        assert err <= 5e-4, f"rank {r}: max |o_sharded - o| = {err}"
