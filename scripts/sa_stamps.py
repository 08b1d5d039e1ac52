"""Timeline of sparse_attn_kernel (development tool): per-CTA globaltimer stamps."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
os.environ["TS_DEV_LIB"] = "1"  # the timestamp hooks exist in the dev build only
from paper_2509_12211_b200 import _build; _build.build(dev=True)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
one = len(sys.argv) > 2 and sys.argv[2] == "cnt1"
cfg = synth.config(name); dev = torch.device("cuda:0")
reps = []
for r in range(3):
    c = synth.make_case(cfg, seed=5 + r, device=dev)
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
    meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
    o, lse, ids, cnt = ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale)
    if one: cnt.fill_(1)
    c.update(L=L, o=o, lse=lse, ids=ids, cnt=cnt, aws=ts.new_workspace(ts.attn_workspace_bytes(L, ids.shape[-1]), dev))
    reps.append(c)
buf = torch.zeros(2048 * 8, dtype=torch.int64, device=dev)
lib = ts._lib.lib(); lib.ts_debug_timestamps.argtypes = [ctypes.c_void_p]
for it in range(7):
    c = reps[it % 3]
    torch.cuda.synchronize(); buf.zero_(); torch.cuda.synchronize()
    lib.ts_debug_timestamps(buf.data_ptr() if it == 6 else None)
    ts.sparse_decode_attn(c["L"], c["q"], c["k_pool"], c["v_pool"], c["page_table"], c["seq_lens"], c["ids"], c["cnt"], cfg.scale, o=c["o"], lse=c["lse"], ws=c["aws"])
    torch.cuda.synchronize()
lib.ts_debug_timestamps(None)
a = buf.cpu().numpy().reshape(2048, 8).astype(np.float64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
rel = (a - t0) / 1e3
names = (["start", "flag", "pages", "consumed", "-", "-", "-", "end"] if os.environ.get("TS_SA_TMA", "1") != "0" else ["start", "q", "pages", "loop_end", "cta_merged", "cl_sync1", "out", "cl_sync2"])
print(name, "cnt1" if one else "", "CTAs", len(a))
for i, n in enumerate(names):
    col = rel[:, i]
    if n == "-" or not np.isfinite(col).any() or (a[:, i] == 0).all():
        continue
    print(f"{n:10s} min {col.min():7.2f} p10 {np.percentile(col,10):7.2f} med {np.median(col):7.2f} p90 {np.percentile(col,90):7.2f} max {col.max():7.2f} us")
