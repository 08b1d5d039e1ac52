"""Timeline of the one-launch decode step (development tool): per-CTA globaltimer stamps of
decode_cluster_kernel phases (start, scored, exchanged, selected, listed, consumed, end) in one
ts_decode_step; dev build only (TS_DEV_LIB=1).  usage: python scripts/step_stamps.py c3 [bf16|fp8]"""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
os.environ["TS_DEV_LIB"] = "1"  # the timestamp hooks exist in the dev build only
from paper_2509_12211_b200 import _build; _build.build(dev=True)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
kv = sys.argv[2] if len(sys.argv) > 2 else "bf16"  # bf16 | fp8
cfg = synth.config(name); dev = torch.device("cuda:0")
reps = []
for r in range(4):
    c = synth.make_case(cfg, seed=5 + r, device=dev)
    shape = tuple(c["k_pool"].shape)
    if kv == "fp8":
        c["k_pool"], c["v_pool"] = ts.kv_quantize(c["k_pool"]), ts.kv_quantize(c["v_pool"])
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"], pool_shape=shape if kv == "fp8" else None)
    meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
    c.update(L=L, meta=meta, ws=ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev))
    reps.append(c)
b1 = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
b2 = torch.zeros(2048 * 8, dtype=torch.int64, device=dev)
lib = ts._lib.lib()
lib.ts_debug_timestamps.argtypes = [ctypes.c_void_p]; lib.ts_debug_ss_timestamps.argtypes = [ctypes.c_void_p]
warm = os.environ.get("STAMP_WARM") == "1"  # every call on replica 0 (L2-resident bytes)
for it in range(9):
    c = reps[0 if warm else it % 4]
    torch.cuda.synchronize(); b1.zero_(); b2.zero_(); torch.cuda.synchronize()
    on = it == 8
    lib.ts_debug_ss_timestamps(b1.data_ptr() if on else None)
    lib.ts_debug_timestamps(b2.data_ptr() if on else None)
    ts.decode_step(c["L"], c["q"], c["k_pool"], c["v_pool"], c["meta"], c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale, ws=c["ws"])
    torch.cuda.synchronize()
lib.ts_debug_ss_timestamps(None); lib.ts_debug_timestamps(None)
a1 = b1.cpu().numpy().reshape(4096, 8).astype(np.float64); a1 = a1[a1[:, 0] > 0]
a2 = b2.cpu().numpy().reshape(2048, 8).astype(np.float64); a2 = a2[a2[:, 0] > 0]
t0 = a1[:, 0].min()
def show(a, names, title):
    print(title, "CTAs", len(a))
    for i, n in enumerate(names):
        if n == "-": continue
        col = a[:, i]; col = col[col > 0]
        if len(col) == 0: continue
        col = (col - t0) / 1e3
        print(f"  {n:11s} n {len(col):5d} min {col.min():7.2f} p10 {np.percentile(col,10):7.2f} med {np.median(col):7.2f} p90 {np.percentile(col,90):7.2f} max {col.max():7.2f} us")
if os.environ.get("TS_TWO_KERNELS", "0") == "0":
    show(a1, ["start", "scored", "selected", "listed", "consumed", "gathered", "keys", "end"], f"{name} decode_cluster_kernel ({kv} KV)")
    # per-CTA phase durations (us): score = 0->1, exchange = 1->5, select = 6->2, attend = 3->4, merge = 4->7
    for nm, (i, j) in (("score", (0, 1)), ("exchange", (1, 5)), ("ptwait", (5, 6)), ("select", (6, 2)), ("attend", (3, 4)), ("merge", (4, 7))):
        d = (a1[:, j] - a1[:, i]) / 1e3
        d = d[(a1[:, i] > 0) & (a1[:, j] > 0)]
        if len(d):
            print(f"  per-CTA {nm:9s} p10 {np.percentile(d,10):6.2f} med {np.median(d):6.2f} p90 {np.percentile(d,90):6.2f} us")
    sys.exit(0)
show(a1, ["start", "scored", "gathered", "selected", "keys", "pass0", "thresh", "compacted"], f"{name} K1 score_select")
show(a2, ["start", "flag", "pages", "consumed", "-", "-", "-", "end"] if os.environ.get("TS_SA_TMA", "1") != "0" else ["start", "q", "pages", "loop_end", "cta_merged", "cl_sync1", "out", "cl_sync2"], f"{name} K2 sparse_attn")
