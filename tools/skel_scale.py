"""Stream-only skeleton (DBP_ABLATE=132) of the cfg2 tensor-core kernel vs
batch size: separates a per-launch fixed cost from the streaming rate."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04473_b200 as dbp
from paper_1808_04473_b200.synth import synth_device

const = dbp.make_constellation("qam16")
for mult in (1, 2, 4, 8):
    n = 13200 * mult
    H, Y = synth_device(1, n, 128, 16, 14, const, n0=0.05)
    for _ in range(3):
        out = dbp.detect("pd", "lmmse", H, Y, 0.05, [32] * 4, const, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        out = dbp.detect("pd", "lmmse", H, Y, 0.05, [32] * 4, const, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = (H.numel() + Y.numel()) * 8
    print(json.dumps({"items": n, "ms": round(ms, 4), "input_GBps": round(nbytes / ms / 1e6, 1)}), flush=True)
    del H, Y, out
