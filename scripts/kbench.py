#!/usr/bin/env python
"""Per-entry-point timing breakdown (development tool, not the bench contract).

Times each C-ABI call on cold rotating replicas inside CUDA graphs:
  score_pages | select_topk | sparse_decode_attn (given selection) | decode_step
usage: python scripts/kbench.py [c2|c3|c5] [reps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2509_12211_b200 as ts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = synth.config(name)
dev = torch.device("cuda:0")
R = int(os.environ.get("R", "6"))
reps = []
for r in range(R):
    c = synth.make_case(cfg, seed=100 + r, device=dev)
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
    meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
    K = ts.kmax(L, cfg.budget_tokens)
    o, lse, ids, cnt = ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"],
                                      c["seq_lens"], cfg.budget_tokens, cfg.scale)
    scores = ts.score_pages(L, c["q"], meta, c["page_table"], c["seq_lens"])
    c.update(L=L, meta=meta, ids=ids, cnt=cnt, o=o, lse=lse, scores=scores,
             ws=ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev),
             aws=ts.new_workspace(ts.attn_workspace_bytes(L, K), dev),
             sids=torch.empty_like(ids.view(-1, K)), ssc=torch.empty(ids.numel(), device=dev),
             scnt=torch.empty_like(cnt.view(-1)))
    reps.append(c)
torch.cuda.synchronize()
s = torch.cuda.Stream()


def calls(c):
    L = c["L"]
    return {
        "score_pages": lambda: ts.score_pages(L, c["q"], c["meta"], c["page_table"], c["seq_lens"],
                                              scores=c["scores"], stream=s),
        "select_topk": lambda: ts.select_topk(c["scores"].view(-1, L.max_pages), c["ids"].shape[-1],
                                              sel_ids=c["sids"], sel_scores=None, want_scores=False,
                                              sel_count=c["scnt"], stream=s),
        "sparse_attn": lambda: ts.sparse_decode_attn(L, c["q"], c["k_pool"], c["v_pool"],
                                                     c["page_table"], c["seq_lens"], c["ids"],
                                                     c["cnt"], cfg.scale, o=c["o"], lse=c["lse"],
                                                     ws=c["aws"], stream=s),
        "decode_step": lambda: ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], c["meta"],
                                              c["page_table"], c["seq_lens"], cfg.budget_tokens,
                                              cfg.scale, o=c["o"], lse=c["lse"], sel_ids=c["ids"],
                                              sel_count=c["cnt"], ws=c["ws"], stream=s),
    }


KEYS = os.environ.get("ONLY", "score_pages,select_topk,sparse_attn,decode_step").split(",")
for key in KEYS:
    gs = []
    for c in reps:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            calls(c)[key]()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                calls(c)[key]()
        gs.append(g)
    torch.cuda.synchronize()
    for i in range(10):
        gs[i % R].replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for i in range(iters):
            gs[i % R].replay()
        b.record(s)
    torch.cuda.synchronize()
    print(f"{name} {key:12s} {a.elapsed_time(b) / iters * 1e3:8.2f} us", flush=True)
