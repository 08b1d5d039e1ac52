#!/usr/bin/env python
"""synthetic page-size x budget-ratio sweep (PAPER.md:474-484, 688-707 ablations,
reproduced on synthetic TinyLLaMA-shaped caches, no model): per (S, K/P) the decode step time,
the FullCache (dense) time, the speedup, and the accuracy proxy = relative L2 error of the sparse
output against dense attention over the same cache (SPEC.md:236-244 output_error idea).
Writes one JSON line per point.  usage: python scripts/sweep_next4.py [out.jsonl]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2509_12211_b200 as ts  # noqa: E402

dev = torch.device("cuda:0")
s = torch.cuda.Stream()
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout


def timed(fns, iters=100):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for f in fns:
            f()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for f in fns:
                f()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, iters // len(fns))
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(n):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (n * len(fns)) * 1e3


for S in (16, 32, 64):
    base = synth.config("c3", page_size=S)
    reps = []
    for r in range(4):
        c = synth.make_case(base, seed=300 + r, device=dev)
        L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
        c.update(L=L, meta=ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"]),
                 dws=ts.new_workspace(ts.dense_workspace_bytes(L), dev))
        reps.append(c)
    dense_o = [ts.dense_decode_attn(c["L"], c["q"], c["k_pool"], c["v_pool"], c["page_table"],
                                    c["seq_lens"], base.scale, ws=c["dws"])[0] for c in reps]
    dense_us = timed([lambda c=c: ts.dense_decode_attn(c["L"], c["q"], c["k_pool"], c["v_pool"],
                                                       c["page_table"], c["seq_lens"], base.scale,
                                                       ws=c["dws"], stream=s) for c in reps])
    for ratio in (0.1, 0.2, 0.3, 0.5):
        budget = int(ratio * base.ctx)
        for c in reps:
            c["ws"] = ts.new_workspace(ts.workspace_bytes(c["L"], budget), dev)
        outs = [ts.decode_step(c["L"], c["q"], c["k_pool"], c["v_pool"], c["meta"], c["page_table"],
                               c["seq_lens"], budget, base.scale, ws=c["ws"])[0] for c in reps]
        torch.cuda.synchronize()
        err = torch.stack([((o - d).norm(dim=-1) / d.norm(dim=-1)).mean() for o, d in zip(outs, dense_o)]).mean()
        us = timed([lambda c=c: ts.decode_step(c["L"], c["q"], c["k_pool"], c["v_pool"], c["meta"],
                                               c["page_table"], c["seq_lens"], budget, base.scale,
                                               ws=c["ws"], stream=s) for c in reps])
        line = {"config": "c3 shape (TinyLLaMA 32q/4kv, d 64, B 16, 32k ctx)", "page_size": S,
                "budget_ratio": ratio, "budget_tokens": budget, "sparse_us": us, "dense_us": dense_us,
                "speedup": dense_us / us, "rel_l2_err_vs_dense": float(err),
                "data": "synthetic clustered keys (synth.make_case), random q"}
        print(json.dumps(line), file=out, flush=True)
