"""Run a few ts_decode_step calls of one config (development: ncu target).
usage: python scripts/one_step.py c2 [bf16|fp8] [steps]"""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1]; kv = sys.argv[2] if len(sys.argv) > 2 else "bf16"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = synth.config(name); dev = torch.device("cuda:0")
c = synth.make_case(cfg, seed=5, device=dev)
shape = tuple(c["k_pool"].shape)
if kv == "fp8":
    c["k_pool"], c["v_pool"] = ts.kv_quantize(c["k_pool"]), ts.kv_quantize(c["v_pool"])
L = ts.make_layout(c["q"], c["k_pool"], c["page_table"], pool_shape=shape if kv == "fp8" else None)
meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
ws = ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev)
for _ in range(n):
    ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"],
                   cfg.budget_tokens, cfg.scale, ws=ws)
torch.cuda.synchronize()
print("ok", name, kv)
