#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) into a short text file for profiles/: duration,
issue / occupancy figures, DRAM and L1/XBAR traffic, the busiest memory interface, and the SASS
instructions with the most warp-stall samples (needs -lineinfo builds and --import-source on).

    python tools/ncu_summary.py gpurun_out/x/prof.ncu-rep [--title "..."] [--algo-bytes N] > profiles/r02/x.txt
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess

DETAILS = ["Duration", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy", "Issued Instructions",
           "No Eligible", "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Registers Per Thread",
           "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "L1/TEX Cache Throughput",
           "DRAM Throughput", "Memory Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__m_l1tex2xbar_write_bytes.sum",
       "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_req_cycles_active.max.pct_of_peak_sustained_elapsed",
       "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "smsp__inst_executed.sum",
       "lts__t_sectors_srcunit_tex_aperture_sysmem_op_read.sum", "lts__t_sectors_srcunit_tex_aperture_sysmem_op_write.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--title", default="")
    ap.add_argument("--algo-bytes", type=float, default=0.0, help="algorithmic bytes of the profiled launch")
    ap.add_argument("--top", type=int, default=10)
    a = ap.parse_args()
    if a.title:
        print(a.title)
    rows = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "details", "--csv"))))
    h = rows[0]
    dur_ms = None
    kernel = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        kernel = kernel or d.get("Kernel Name")
        if d["Metric Name"] in DETAILS:
            print(f"  {d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
            if d["Metric Name"] == "Duration":
                v = float(d["Metric Value"].replace(",", ""))
                dur_ms = {"ms": v, "us": v / 1e3, "ns": v / 1e6, "s": v * 1e3}.get(d["Metric Unit"].strip(), v)
    print(f"  kernel: {kernel}")
    raw = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "raw", "--csv"))))
    if len(raw) >= 3:
        for name, unit, val in zip(raw[0], raw[1], raw[2]):
            if name in RAW:
                print(f"  {name}: {val} {unit}")
    if a.algo_bytes and dur_ms:
        print(f"  => {a.algo_bytes / 2**20:.0f} MiB algorithmic in {dur_ms:.3f} ms = {a.algo_bytes / dur_ms / 1e6:.2f} GB/s (under ncu)")
    src = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        idx = {k: i for i, k in enumerate(h)}
        col = idx.get("Warp Stall Sampling (All Samples)")
        if col is not None:
            data = [r for r in src[2:] if len(r) > col]
            tot = sum(int(r[col]) for r in data)
            print(f"  warp-stall samples by SASS instruction (top {a.top} of {tot}):")
            for r in sorted(data, key=lambda r: -int(r[col]))[: a.top]:
                print(f"    {r[col]:>6}  {r[idx['Instructions Executed']]:>9} exec  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
