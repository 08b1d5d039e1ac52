#!/usr/bin/env python
"""Top stall reasons and hottest SASS lines (with CUDA source line) of an ncu report
(development tool).  usage: python scripts/ncu_stalls.py <report> [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
if not hi:
    hi = [i for i, r in enumerate(rows) if r and "Source" in r]
h = rows[hi[0]]
body = rows[hi[0] + 1:(hi[1] - 1 if len(hi) > 1 else len(rows))]
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ix[S]] or 0) for r in body if len(r) > ix[S] and r[ix[S]].isdigit())
print("total samples", tot)
agg = {k: sum(int(r[ix[k]] or 0) for r in body if len(r) > ix[k] and r[ix[k]].isdigit()) for k in stalls}
for k, v in sorted(agg.items(), key=lambda a: -a[1])[:10]:
    print(f"  {k:28s} {v:7d} {100 * v / max(1, tot):5.1f}%")
body = [r for r in body if len(r) > ix[S] and r[ix[S]].isdigit()]
body.sort(key=lambda r: -int(r[ix[S]]))
for r in body[:n]:
    top = sorted(((int(r[ix[k]] or 0), k) for k in stalls), reverse=True)[:2]
    print(f"{int(r[ix[S]]):6d} {r[ix['Source']].strip()[:70]:70s} {top}")
