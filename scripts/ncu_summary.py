#!/usr/bin/env python
"""Summarise an ncu report (--set full) into a few lines for profiles/ (development tool).

usage: python scripts/ncu_summary.py <report.ncu-rep> [algorithmic_bytes_per_launch]
"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print(f"kernel: {r[idx['Kernel Name']][:90]}")
        vals = {}
        for w in WANT:
            if w in idx:
                vals[w] = r[idx[w]]
                print(f"  {w:66s} {r[idx[w]]:>14s} {units[idx[w]]}")
        try:
            def tob(w):
                u = units[idx[w]].lower()
                f = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}[u]
                return float(vals[w].replace(",", "")) * f
            traffic = tob("dram__bytes_read.sum") + tob("dram__bytes_write.sum")
            t_us = float(vals["gpu__time_duration.sum"].replace(",", ""))
            tu = units[idx["gpu__time_duration.sum"]]
            t_s = t_us * {"usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9, "msecond": 1e-3, "ms": 1e-3}[tu]
            print(f"  traffic (dram read+write) per launch: {traffic:.0f} B; "
                  f"{traffic / t_s / 1e9:.0f} GB/s over the launch")
            if alg:
                print(f"  algorithmic bytes {alg:.0f} B; traffic/algorithmic = {traffic / alg:.3f}; "
                      f"algorithmic GB/s = {alg / t_s / 1e9:.0f}")
        except Exception as e:  # noqa: BLE001
            print("  (traffic summary unavailable:", e, ")")


if __name__ == "__main__":
    main()
