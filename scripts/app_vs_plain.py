"""Device time of ts_decode_step vs ts_decode_step_append in a PDL-chained graph (development)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, bench, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.config(name); dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
stream = torch.cuda.Stream()
R = 6
reps = [bench.build_replica(ts, cfg, seed=r, device=dev) for r in range(R)]
kn = torch.randn(cfg.batch, cfg.num_kv_heads, cfg.head_dim, device=dev).to(torch.bfloat16)
st = {"i": 0}
def plain():
    r = reps[st["i"] % R]; st["i"] += 1
    bench.step_fn(ts, cfg, r, stream)
def app():
    r = reps[st["i"] % R]; st["i"] += 1
    ts.decode_step_append(r["layout"], r["q"], kn, kn, r["k_pool"], r["v_pool"], r["meta"], r["page_table"],
                          r["seq_lens"], cfg.budget_tokens, cfg.scale, o=r["o"], lse=r["lse"], sel_ids=r["ids"],
                          sel_count=r["cnt"], ws=r["ws"], stream=stream)
for nm, fn in (("plain", plain), ("append", app), ("plain", plain)):
    print(name, nm, round(bench.time_graph(fn, 60 * R, stream), 2), "us")
