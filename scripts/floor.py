"""Replay-overhead floor vs kernel time (development tool)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, paper_2509_12211_b200 as ts
dev = torch.device("cuda:0"); s = torch.cuda.Stream()
def timeit(fns, iters=200, per_graph=1):
    gs = []
    for k in range(0, len(fns), per_graph):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for f in fns[k:k + per_graph]: f()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for f in fns[k:k + per_graph]: f()
        gs.append(g)
    torch.cuda.synchronize()
    for i in range(10): gs[i % len(gs)].replay()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    n = iters // per_graph
    with torch.cuda.stream(s):
        a.record(s)
        for i in range(n): gs[i % len(gs)].replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (n * per_graph) * 1e3
x = torch.zeros(1, device=dev)
print(f"tiny add, 1/graph: {timeit([lambda: x.add_(1)]*4):.2f} us; 8/graph: {timeit([lambda: x.add_(1)]*8, per_graph=8):.2f} us")
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = synth.config(name)
reps = []
for r in range(4):
    c = synth.make_case(cfg, seed=100 + r, device=dev)
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
    meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
    o, lse, ids, cnt = ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale)
    c.update(L=L, ids=ids, cnt=cnt, o=o, lse=lse, cnt1=torch.ones_like(cnt),
             aws=ts.new_workspace(ts.attn_workspace_bytes(L, ids.shape[-1]), dev))
    reps.append(c)
torch.cuda.synchronize()
def attn(c, key="cnt"):
    return lambda: ts.sparse_decode_attn(c["L"], c["q"], c["k_pool"], c["v_pool"], c["page_table"], c["seq_lens"], c["ids"], c[key], cfg.scale, o=c["o"], lse=c["lse"], ws=c["aws"], stream=s)
for key in ["cnt1", "cnt"]:
    print(f"{name} attn {key}: 1/graph {timeit([attn(c, key) for c in reps]):.2f} us; 4/graph {timeit([attn(c, key) for c in reps], per_graph=4):.2f} us")
