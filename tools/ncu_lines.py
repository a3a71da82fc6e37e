"""Per-CUDA-source-line summary of an ncu report (warp-stall samples, top
stall reasons, instructions, shared-memory wavefronts actual/ideal).
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, res = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        names = r
        continue
    if hdr is None or not r[0]:
        continue
    def g(name):
        try:
            return int(float(r[hdr[name]])) if hdr[name] < len(r) else 0
        except (KeyError, ValueError):
            return 0
    stalls = sorted(((g(h), h[6:]) for h in hdr if h.startswith("stall_") and "Not Issued" not in h), reverse=True)[:3]
    res.append((g("Warp Stall Sampling (All Samples)"), f"{fname}:{r[0]}", r[1].strip()[:60], g("Instructions Executed"),
                g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Ideal"), stalls))
tot = sum(x[0] for x in res) or 1
print("total samples", tot)
for s, loc, src, inst, wf, wfi, st in sorted(res, key=lambda x: -x[0])[:N]:
    print(f"{100 * s / tot:5.1f}% {loc:22s} inst {inst:>9} wf {wf:>8}/{wfi:<8} {src:60s} {[f'{h}:{v}' for v, h in st if v]}")
