"""Timeline of the pipelined decode step (development tool): per-CTA globaltimer stamps of
decode_pipe_kernel in one ts_decode_step (cold replicas rotated before the stamped call)."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
over = dict(kv.split("=") for kv in sys.argv[2:])
over = {k: int(v) for k, v in over.items()}
cfg = synth.config(name, **over); dev = torch.device("cuda:0")
reps = []
for r in range(4):
    c = synth.make_case(cfg, seed=5 + r, device=dev)
    L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
    meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
    c.update(L=L, meta=meta, ws=ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev))
    reps.append(c)
buf = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
lib = ts._lib.lib()
lib.ts_debug_ss_timestamps.argtypes = [ctypes.c_void_p]
for it in range(9):
    c = reps[it % 4]
    torch.cuda.synchronize(); buf.zero_(); torch.cuda.synchronize()
    lib.ts_debug_ss_timestamps(buf.data_ptr() if it == 8 else None)
    ts.decode_step(c["L"], c["q"], c["k_pool"], c["v_pool"], c["meta"], c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale, ws=c["ws"])
    torch.cuda.synchronize()
lib.ts_debug_ss_timestamps(None)
a = buf.cpu().numpy().reshape(4096, 16).astype(np.float64); a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
names = ["start", "scoredA", "selectedA", "scoredB", "selectedB", "attendedA", "attendedB", "-",
         "P:meta_issued", "P:selA_seen", "P:kvA_issued", "P:selB_seen", "P:kvB_issued", "endA", "endB"]
print(name, over, "CTAs", len(a))
for i, n in enumerate(names):
    if n == "-": continue
    col = a[:, i]; col = col[col > 0]
    if len(col) == 0: continue
    col = (col - t0) / 1e3
    print(f"  {n:13s} n {len(col):5d} min {col.min():7.2f} p10 {np.percentile(col,10):7.2f} med {np.median(col):7.2f} p90 {np.percentile(col,90):7.2f} max {col.max():7.2f} us")
