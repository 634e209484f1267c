#!/usr/bin/env python
"""Summarise an .ncu-rep (ncu --set full capture) into a short text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/r1_xxx.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
    "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
    "Achieved Occupancy", "Theoretical Occupancy", "Block Size", "Grid Size",
    "Dynamic Shared Memory Per Block", "Avg. Active Threads Per Warp",
    "Warp Cycles Per Issued Instruction", "Executed Instructions", "L2 Hit Rate", "L1/TEX Hit Rate",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__average_warp_latency_issue_stalled_barrier", "launch__registers_per_thread"]


def main(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    if not rows:
        print("no data")
        return
    hdr = rows[0]
    ik, iname, iunit, ival = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                              hdr.index("Metric Unit"), hdr.index("Metric Value"))
    seen = set()
    for r in rows[1:]:
        if len(r) <= ival:
            continue
        if r[iname] in KEYS and (r[ik], r[iname]) not in seen:
            seen.add((r[ik], r[iname]))
            print(f"{r[ik][:40]:40s} {r[iname]:40s} {r[ival]:>16s} {r[iunit]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        h = rr[0]
        for data in rr[2:]:
            name = data[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            for m in RAW:
                if m in h:
                    print(f"{name[:40]:40s} {m:60s} {data[h.index(m)]:>16s} {rr[1][h.index(m)]}")


if __name__ == "__main__":
    main(sys.argv[1])
