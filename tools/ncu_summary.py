#!/usr/bin/env python
"""Summarise an ncu --set full report: key raw metrics + hottest source lines.

usage: python tools/ncu_summary.py REPORT.ncu-rep [label] > profiles/<name>.md
(needs the ncu CLI; reads the report offline, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__block_size",
    "launch__grid_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: {label}\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"## kernel `{name}`\n\n| metric | unit | value |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {units[i]} | {r[i]} |")
        print()
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    cur, hdr2, lines = None, None, []
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 and r[0] and len(r) > 7 and r[2] == "-":
            try:
                lines.append((cur, int(r[0]), r[1].strip()[:80], int(r[4] or 0), int(r[7] or 0)))
            except ValueError:
                pass
    ts = sum(x[3] for x in lines) or 1
    ti = sum(x[4] for x in lines) or 1
    print("## hottest source lines (warp-stall samples / executed instructions)\n")
    print("| samples % | inst % | line | source |\n|---|---|---|---|")
    for f, ln, s, a, b in sorted(lines, key=lambda x: -x[3])[:25]:
        print(f"| {100 * a / ts:.1f} | {100 * b / ti:.1f} | {f}:{ln} | `{s.replace('|', '/')}` |")


if __name__ == "__main__":
    main()
