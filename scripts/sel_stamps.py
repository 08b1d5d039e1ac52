"""Phase durations inside cta_topk (development tool; needs TS_NVCC_EXTRA=-DTS_SEL_PROF build):
per leader CTA of decode_cluster_kernel, median / p90 of each phase of the exact top-K."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
os.environ["TS_DEV_LIB"] = "1"  # the timestamp hooks exist in the dev build only
from paper_2509_12211_b200 import _build; _build.build(dev=True)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = synth.config(name); dev = torch.device("cuda:0")
reps = []
for r in range(4):
    c = synth.make_case(cfg, seed=5 + r, device=dev)
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
    meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
    c.update(L=L, meta=meta, ws=ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev))
    reps.append(c)
buf = torch.zeros(3 * 4096 * 8, dtype=torch.int64, device=dev)
lib = ts._lib.lib(); lib.ts_debug_ss_timestamps.argtypes = [ctypes.c_void_p]
for it in range(12):
    c = reps[it % 4]
    torch.cuda.synchronize(); buf.zero_(); torch.cuda.synchronize()
    lib.ts_debug_ss_timestamps(buf.data_ptr() if it == 11 else None)
    ts.decode_step(c["L"], c["q"], c["k_pool"], c["v_pool"], c["meta"], c["page_table"], c["seq_lens"],
                   cfg.budget_tokens, cfg.scale, ws=c["ws"])
    torch.cuda.synchronize()
lib.ts_debug_ss_timestamps(None)
a = buf.cpu().numpy().reshape(3, 4096, 8).astype(np.float64)
names = ["start", "hist", "binsearch", "cands", "threshold", "scan", "emit", "listed(7)"]
for reg, title in ((1, "leader select"), (2, "chunk select (two-level)")):
    x = a[reg]; x = x[x[:, 0] > 0]
    if len(x) == 0: continue
    print(f"{name} {title}: CTAs {len(x)}  (us since cta_topk start; phase delta)")
    prev = np.zeros(len(x))
    for i, n in enumerate(names):
        col = x[:, i]; ok = col > 0
        if not ok.any(): continue
        d = (col - x[:, 0]) / 1e3
        print(f"  {n:10s} n {ok.sum():4d} med {np.median(d[ok]):6.2f} p90 {np.percentile(d[ok], 90):6.2f}")
