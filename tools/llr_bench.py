"""Throughput of the bit-LLR kernel (dbp_llr, soft.llr) on the cfg2 output
shape (13200 items x T=14 x U=16, 64-QAM -> 6 bits per symbol): algorithmic
bytes = 8 (x-hat) + 4 (sigma2 per UE, amortised over T) + 4 * 6 (LLRs) per
symbol, vs the measured HBM copy bandwidth.  Prints one JSON line per
(mode, shape)."""

import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1808_04473_b200 as dbp  # noqa: E402

peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
for name, n in (("qam64", 13200), ("qam64", 13200 * 16), ("qam16", 13200 * 16)):
    const = dbp.make_constellation(name)
    nb = 2 * (len(const.pam_levels).bit_length() - 1)
    x = torch.randn(n, 14, 16, dtype=torch.complex64, device="cuda")
    s2 = torch.rand(n, 16, device="cuda") * 0.1 + 0.01
    for exact in (False, True):
        for _ in range(3):
            out = dbp.llr(x, s2, const, exact=exact)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            out = dbp.llr(x, s2, const, exact=exact)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        nbytes = x.numel() * 8 + s2.numel() * 4 + out.numel() * 4
        print(json.dumps({"constellation": name, "exact": exact, "shape": f"items={n} T=14 U=16",
                          "bytes": nbytes, "ms": ms, "GB_per_s": nbytes / ms / 1e6,
                          "frac_of_hbm": nbytes / ms / 1e6 / peak}), flush=True)
        del out
