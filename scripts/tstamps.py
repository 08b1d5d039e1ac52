"""Timeline of the pipeline kernel (development tool): per-CTA stamps + per-row publish."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import synth, paper_2509_12211_b200 as ts
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "step"
cfg = synth.config(name); dev = torch.device("cuda:0")
c = synth.make_case(cfg, seed=5, device=dev)
L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
ws = ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), dev)
o, lse, ids, cnt = ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale, ws=ws)
buf = torch.zeros(16384 + 8192, dtype=torch.int64, device=dev)
lib = ts._lib.lib(); lib.ts_debug_timestamps.argtypes = [ctypes.c_void_p]
aws = ts.new_workspace(ts.attn_workspace_bytes(L, ids.shape[-1]), dev)
for it in range(3):
    torch.cuda.synchronize(); buf.zero_()
    lib.ts_debug_timestamps(buf.data_ptr() if it == 2 else None)
    if mode == "step":
        ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"], cfg.budget_tokens, cfg.scale, o=o, lse=lse, sel_ids=ids, sel_count=cnt, ws=ws)
    else:
        ts.sparse_decode_attn(L, c["q"], c["k_pool"], c["v_pool"], c["page_table"], c["seq_lens"], ids, cnt, cfg.scale, ws=aws)
    torch.cuda.synchronize()
lib.ts_debug_timestamps(None)
a = buf.cpu().numpy()
t = a[:4096].reshape(512, 8); t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3; rel[t == 0] = np.nan
names = ["start", "grab1", "desc1", "tma1", "data1", "cons_end", "tma_end", "merge_end"]
print(name, mode, "CTAs", len(t))
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{n:10s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f} us")
rows = a[4096:4096 + 8192]; rows = rows[rows > 0]
if len(rows):
    r = (rows - t0) / 1e3
    print(f"row publish: n {len(r)} first {r.min():.2f} p10 {np.percentile(r,10):.2f} med {np.median(r):.2f} p90 {np.percentile(r,90):.2f} last {r.max():.2f} us")

st = a[12288:16384].reshape(1024, 4).astype(np.float64)
st[st == 0] = np.nan
st = (st - t0) / 1e3
ok = ~np.isnan(st[:, 0])
if ok.any():
    s = st[ok]
    for e, nm in enumerate(["merge start", "chunk topk done", "cands loaded", "final topk done"]):
        col = s[:, e]
        if np.isfinite(col).any():
            print(f"score item {nm:16s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f} us")
    d1 = s[:, 1] - s[:, 0]
    print(f"chunk topk duration med {np.nanmedian(d1):.2f} max {np.nanmax(d1):.2f} us")
    if np.isfinite(s[:, 3]).any():
        d3 = s[:, 3] - s[:, 2]
        d2 = s[:, 2] - s[:, 1]
        print(f"ticket->cands loaded med {np.nanmedian(d2):.2f}; final topk med {np.nanmedian(d3):.2f} max {np.nanmax(d3):.2f} us")
tr = a[16384:16384 + 4096].reshape(4, 512, 2)
arr = a[16384 + 4096:16384 + 4096 + 1024].reshape(4, 256)
for c in range(2):
    print(f"--- CTA {c}: i, flags, issue, data, done (us)")
    for i in range(0, 256, 1):
        iss, done, dat = tr[c, i, 0], tr[c, i, 1], arr[c, i]
        if iss == 0 and done == 0:
            continue
        fl = (int(iss) >> 52) & 0xfff
        ti = ((int(iss) & ((1 << 52) - 1)) - t0) / 1e3 if iss else float('nan')
        print(f"{i:4d} {fl:4x} {ti:7.2f} {(dat - t0) / 1e3 if dat else float('nan'):7.2f} {(done - t0) / 1e3 if done else float('nan'):7.2f}")
