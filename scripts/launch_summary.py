"""Median duration per kernel of an ncu launch list (--metrics gpu__time_duration.sum --csv)
(development tool).  usage: python scripts/launch_summary.py <launches.csv>"""
import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
hdr=rows[0]; ix={h:i for i,h in enumerate(hdr)}
d=collections.defaultdict(list)
for r in rows[1:]:
    if r[ix["Metric Name"]]=="gpu__time_duration.sum": d[r[ix["Kernel Name"]][:80]].append(float(r[ix["Metric Value"]]))
for k,v in d.items(): print(len(v), "median ns", sorted(v)[len(v)//2], k)
