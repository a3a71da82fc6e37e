"""Throughput of on-device frame synthesis (dbp_synthesize) on the cfg5
shapes: bytes of H + Y written per second vs the measured HBM copy
bandwidth (its roofline: the kernel writes each output byte once and reads
nothing but a few symbols).  Prints one JSON line per shape."""

import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1808_04473_b200 as dbp  # noqa: E402
import numpy as np  # noqa: E402

from paper_1808_04473_b200 import _lib  # noqa: E402
from paper_1808_04473_b200.synth import synth_device  # noqa: E402

peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
const = dbp.make_constellation("qam64")
for b, u, frames in ((512, 64, 64), (1024, 64, 64), (128, 16, 11)):
    n = frames * 1200
    H, Y = synth_device(1, n, b, u, 14, const, n0=0.01)  # warm-up + allocation
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 3
    syms = np.ascontiguousarray(np.stack([const.symbols.real, const.symbols.imag], -1).astype(np.float32))
    for r in range(reps):  # kernel only, into the preallocated buffers
        _lib.check(_lib.lib().dbp_synthesize(2 + r, n, 0, b, u, 14, syms.ctypes.data, const.size, 0.01, None, 1,
                                             _lib.ptr(H), _lib.ptr(Y), None, _lib.stream_ptr()))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nbytes = (H.numel() + Y.numel()) * 8
    print(json.dumps({"shape": f"B={b} U={u} T=14 items={n}", "bytes": nbytes, "ms": ms,
                      "GB_per_s": nbytes / ms / 1e6, "frac_of_hbm": nbytes / ms / 1e6 / peak}))
    del H, Y
    torch.cuda.empty_cache()
