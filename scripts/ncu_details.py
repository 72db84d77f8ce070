"""Key metrics from an ncu details CSV: python scripts/ncu_details.py gpurun_out/details_<tag>.csv"""
import csv
import sys

WANT = ("Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "L2 Hit Rate",
        "Registers Per Thread", "Achieved Occupancy", "Issue Slots Busy", "No Eligible",
        "Executed Ipc Active", "Mem Busy", "Max Bandwidth", "Dynamic Shared Memory Per Block")
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ki, gi, bi, si, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Grid Size", "Block Size", "Section Name",
                                                          "Metric Name", "Metric Unit", "Metric Value"))
    print("==", path, rows[1][ki][:70], rows[1][gi], rows[1][bi])
    seen = set()
    for r in rows[1:]:
        if len(r) > vi and r[mi] in WANT and r[mi] not in seen:
            seen.add(r[mi])
            print(f"   {r[mi]:34s} {r[vi]:>14s} {r[ui]}")
