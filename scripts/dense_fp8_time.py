"""FullCache (dense) attention time over bf16 and FP8 caches (development: consumer cost)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, bench, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = synth.config(name); dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
stream = torch.cuda.Stream()
for kv in ("bf16", "fp8"):
    reps = [bench.build_replica(ts, cfg, seed=r, device=dev, kv="fp8" if kv == "fp8" else "") for r in range(3)]
    ws = [ts.new_workspace(ts.dense_workspace_bytes(r["layout"]), dev) for r in reps]
    st = {"i": 0}
    def f():
        r = reps[st["i"] % 3]; w = ws[st["i"] % 3]; st["i"] += 1
        ts.dense_decode_attn(r["layout"], r["q"], r["k_pool"], r["v_pool"], r["page_table"], r["seq_lens"],
                             cfg.scale, o=r["o"], lse=r["lse"], ws=w, stream=stream)
    print(name, kv, "dense", round(bench.time_graph(f, 30, stream), 1), "us")
    del reps, ws
    torch.cuda.empty_cache()
