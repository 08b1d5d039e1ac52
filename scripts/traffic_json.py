#!/usr/bin/env python
"""DRAM traffic per launch of each kernel from ncu --set full reports -> profiles/traffic.json,
which bench.py reports as roofline.traffic (development tool).

usage: python scripts/traffic_json.py c2=gpurun_out/prof_c2_X.ncu-rep c3=... [-o profiles/traffic.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}


def kernel_traffic(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").strip()
        name = name.split("<")[0].split("::")[-1]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[ix[m]].replace(",", "")) * UNIT[units[ix[m]].lower()]
        acc.setdefault(name, []).append(b)
    return {k: sum(v) / len(v) for k, v in acc.items()}


def main():
    outp = "profiles/traffic.json"
    args = sys.argv[1:]
    if "-o" in args:
        outp = args[args.index("-o") + 1]
        args = args[:args.index("-o")]
    data = json.load(open(outp)) if os.path.exists(outp) else {}
    for a in args:
        cfg, rep = a.split("=", 1)
        data[cfg] = {"per_launch_bytes": kernel_traffic(rep), "report": os.path.basename(rep)}
    with open(outp, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
