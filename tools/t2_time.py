"""Quick device timing of one workload through the batched Detector (inputs
synthesized on the GPU, two input copies alternated past L2).  Study tool:
with DBP_LIB pointing at a study build, DBP_ABLATE selects timing ablations.
usage: python tools/t2_time.py [config] [reps] [key=value options...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1808_04473_b200 as dbp  # noqa: E402
from paper_1808_04473_b200 import _lib  # noqa: E402
from paper_1808_04473_b200.synth import synth_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
opts = dict(kv.split("=") for kv in sys.argv[3:])
wl = bench.WORKLOADS[name]
W, T = bench.W, bench.T
const = dbp.make_constellation(bench.CONST[wl["bits"]])
n = wl["frames"] * W
counts = [wl["B"] // wl["C"]] * wl["C"]
lp = {"t_max": wl["t_max"]} if wl["kind"] == "lama" else None
det = dbp.Detector(wl["arch"], wl["kind"], n, wl["B"], wl["U"], T, counts, const, lama_params=lp)
copies = [synth_device(s, n, wl["B"], wl["U"], T, const, n0=0.05) for s in (1, 2)]
with _lib.options(**{k: int(v) for k, v in opts.items()}):
    for k in range(3):
        det.run(*copies[k % 2], 0.05)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        det.run(*copies[k % 2], 0.05)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
frac = bench.algorithmic_bytes(wl, n) / (ms * 1e-3) / 1e9 / 6551.4
print(f"{name} {opts} ablate={os.environ.get('DBP_ABLATE', '0')} kernel={_lib.lib().dbp_last_kernel()}: "
      f"{ms:.4f} ms  {bench.bits_per_step(wl) / (ms * 1e-3) / 1e9:.1f} Gb/s  frac {frac:.3f}")
