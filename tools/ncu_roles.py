"""Per-line / per-role breakdown of an ncu --set full report of the split-bf16
kernel: instructions, warp-stall samples and top stall reasons, grouped by
source file / line range.  usage: python tools/ncu_roles.py REPORT [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = "?", None
rows = collections.defaultdict(lambda: collections.Counter())
src = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit():
        continue
    k = (fname, int(r[0]))
    src[k] = r[1].strip()[:70]
    for h, i in hdr.items():
        if h in ("Instructions Executed", "Warp Stall Sampling (All Samples)") or (
                h.startswith("stall_") and "Not Issued" not in h):
            try:
                rows[k][h] += int(float(r[i]))
            except ValueError:
                pass
ti = sum(v["Instructions Executed"] for v in rows.values()) or 1
ts = sum(v["Warp Stall Sampling (All Samples)"] for v in rows.values()) or 1
print(f"total instructions {ti}, samples {ts}")
for k, v in sorted(rows.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"])[:N]:
    st = sorted(((c, h[6:]) for h, c in v.items() if h.startswith("stall_")), reverse=True)[:3]
    print(f"{100 * v['Warp Stall Sampling (All Samples)'] / ts:5.1f}% smp {100 * v['Instructions Executed'] / ti:5.1f}% ins "
          f"{k[0]}:{k[1]:<4} {src[k]:70s} {[f'{h}:{100 * c / ts:.1f}' for c, h in st if c]}")
