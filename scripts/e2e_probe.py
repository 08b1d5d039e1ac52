"""Where does the e2e step time go? (development tool) decode only / + append / + copies."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, paper_2509_12211_b200 as ts
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c2"); dev = torch.device("cuda:0")
s = torch.cuda.Stream()
reps = []
for r in range(6):
    c = synth.make_case(cfg, seed=r, device=dev)
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
    c.update(L=L, meta=ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"]),
             ws=ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev),
             pos=(c["seq_lens"] - 1).contiguous())
    reps.append(c)
B, Hq, Hkv, d = cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
hq = torch.randn(B, Hq, d).to(torch.bfloat16).pin_memory(); hk = torch.randn(B, Hkv, d).to(torch.bfloat16).pin_memory()
dq = hq.to(dev); dk = hk.to(dev); dv = hk.to(dev)
o = torch.empty(B, Hq, d, device=dev); lse = torch.empty(B, Hq, device=dev)
ho = torch.empty(B, Hq, d).pin_memory()
def timed(fn, n=300):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s): fn()
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(n // 6): g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (n // 6 * 6) * 1e3
def dec(c): ts.decode_step(c["L"], dq, c["k_pool"], c["v_pool"], c["meta"], c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale, o=o, lse=lse, ws=c["ws"], stream=s)
def app(c): ts.meta_append(c["L"], dk, dv, c["pos"], c["page_table"], c["k_pool"], c["v_pool"], c["meta"], advance=False, stream=s)
print("decode only      ", round(timed(lambda: [dec(c) for c in reps]), 2), "us/step")
print("append only      ", round(timed(lambda: [app(c) for c in reps]), 2), "us/step")
print("append + decode  ", round(timed(lambda: [(app(c), dec(c)) for c in reps]), 2), "us/step")
print("H2D q only       ", round(timed(lambda: [dq.copy_(hq, non_blocking=True) for c in reps]), 2), "us/step")
print("D2H o only       ", round(timed(lambda: [ho.copy_(o, non_blocking=True) for c in reps]), 2), "us/step")
print("h2d+app+dec+d2h  ", round(timed(lambda: [(dq.copy_(hq, non_blocking=True), app(c), dec(c), ho.copy_(o, non_blocking=True)) for c in reps]), 2), "us/step")
