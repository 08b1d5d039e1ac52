"""Per-CTA timeline of the attention kernel (development tool)."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.config(name); dev = torch.device("cuda:0")
c = synth.make_case(cfg, seed=5, device=dev)
L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
o, lse, ids, cnt = ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale)
buf = torch.zeros(512 * 8, dtype=torch.int64, device=dev)
lib = ts._lib.lib(); lib.ts_debug_timestamps.argtypes = [ctypes.c_void_p]
ws = ts.new_workspace(ts.attn_workspace_bytes(L, ids.shape[-1]), dev)
for it in range(3):
    torch.cuda.synchronize()
    buf.zero_()
    lib.ts_debug_timestamps(buf.data_ptr() if it == 2 else None)
    ts.sparse_decode_attn(L, c["q"], c["k_pool"], c["v_pool"], c["page_table"], c["seq_lens"], ids, cnt, cfg.scale, ws=ws)
    torch.cuda.synchronize()
lib.ts_debug_timestamps(None)
t = buf.cpu().numpy().reshape(512, 8)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
rel[t == 0] = np.nan
names = ["start", "grab1", "desc1", "tma1", "data1", "cons_end", "tma_end", "merge_end"]
print(name, "CTAs", len(t))
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{n:10s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f} us")
