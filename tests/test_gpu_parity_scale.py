"""Parity at the BASELINE sizes (VERDICT r1 task 1).

Every BASELINE configuration runs through the batched detector at its full
frame size (W = 1200 subcarriers x T = 14 OFDM symbols x all clusters; cfg2 with
all 11 SNR frames; cfg5 with 2 of its 64 frames, the same kernel path the bench
times), and a random sample of subcarriers of every frame -- at least 64 per
frame, and enough for >= 1e5 detected symbols per configuration -- is checked
against the vectorized oracle (oracle.run_batch_vec, pinned to the per-vector
restatement and the reference's golden vectors by tests/test_oracle_vec.py)
fed the same complex64 inputs.

Bars (tests/parity.py, BASELINE.json north star): max normwise relative error
<= 1e-4 on x-hat (per vector ||x - x_ref||_inf / ||x_ref||_inf), entrywise
<= 1e-4 on sigma2 and on the fusion weights nu, decision mismatches <= 1e-5 of
the symbols (at least 1 allowed), each at a decision boundary.  The observed
figures are printed (pytest -s) and, with DBP_PARITY_OUT=<file>, written as JSON.
"""

import json
import os

import numpy as np
import pytest
import torch

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O
from paper_1808_04473_b200.synth import snr_to_n0, synth_device
from parity import DEC_RATE, NU_TOL, SIGMA2_TOL, XHAT_TOL, check_decisions, entry_rel

pytestmark = pytest.mark.gpu

W, T = 1200, 14
CONST = {2: "qpsk", 4: "qam16", 6: "qam64"}
# name: arch, kind, B, C, U, bits, SNR per frame (dB), t_max, subcarriers sampled per frame
WORKLOADS = {
    "cfg1": ("fd", "lmmse", 64, 2, 8, 4, [10.0], 0, 1200),
    "cfg2": ("pd", "lmmse", 128, 4, 16, 4, [float(s) for s in range(0, 21, 2)], 0, 64),
    "cfg3-zf": ("fd", "zf", 256, 8, 16, 6, [15.0], 0, 512),
    "cfg3-mrc": ("fd", "mrc", 256, 8, 16, 6, [15.0], 0, 512),
    "cfg4-fd": ("fd", "lama", 256, 8, 32, 4, [8.0], 10, 256),
    "cfg4-pd": ("pd", "lama", 256, 8, 32, 4, [8.0], 10, 256),
    "cfg5-pd512": ("pd", "lmmse", 512, 8, 64, 6, [20.0, 20.0], 0, 64),
    "cfg5-fd512": ("fd", "lmmse", 512, 8, 64, 6, [20.0, 20.0], 0, 64),
    "cfg5-pd1024": ("pd", "lmmse", 1024, 8, 64, 6, [20.0, 20.0], 0, 64),
    "cfg5-fd1024": ("fd", "lmmse", 1024, 8, 64, 6, [20.0, 20.0], 0, 64),
}


def _normwise(x, ref):
    num = np.max(np.abs(x - ref), axis=-1)
    den = np.maximum(np.max(np.abs(ref), axis=-1), 1e-30)
    return num / den


def run_parity(name, seed=2024):
    arch, kind, b, c, u, bits, snrs, t_max, per_frame = WORKLOADS[name]
    const = dbp.make_constellation(CONST[bits])
    frames = len(snrs)
    n = frames * W
    n0 = snr_to_n0(snrs, const.es)
    n0_dev = torch.tensor(np.asarray(n0, dtype=np.float32), device="cuda")
    H, Y = synth_device(seed, n, b, u, T, const, n0_dev=n0_dev, n0_group=W)
    counts = [b // c] * c
    lp = {"t_max": t_max} if kind == "lama" else None
    det = dbp.Detector(arch, kind, n, b, u, T, counts, const, lama_params=lp)
    out = det.run(H, Y, 0.0, n0_dev, W, check=True)
    rng = np.random.default_rng(seed)
    items = np.concatenate([f * W + np.sort(rng.choice(W, min(per_frame, W), replace=False)) for f in range(frames)])
    idx = torch.from_numpy(items).cuda()
    Hs = H.index_select(0, idx).cpu().numpy().astype(np.complex128)
    Ys = Y.index_select(0, idx).cpu().numpy().astype(np.complex128)
    n0s = np.repeat(np.asarray(n0, dtype=np.float32), W)[items].astype(float)
    ref = O.run_batch_vec(arch, kind, Hs, Ys, O.uniform_offsets(b, c), n0s, 1.0, const.symbols, lama_params=lp)
    xh = out.xhat.index_select(0, idx).cpu().numpy().astype(np.complex128)
    dec = out.decisions.index_select(0, idx).cpu().numpy()
    s2 = out.sigma2.index_select(0, idx).cpu().numpy().astype(float)
    if kind == "lama":  # tau per symbol, broadcast over UEs
        s2 = np.broadcast_to(s2[:, :, None], ref["sigma2"].shape)
    else:
        s2 = np.broadcast_to(s2[:, None, :], ref["sigma2"].shape)
    nw = _normwise(xh, ref["z"])
    nbad, ntot, at_boundary = check_decisions(dec, ref["dec"], ref["z"], xh, const.pam_levels)
    res = {"config": name, "arch": arch, "kind": kind, "B": b, "C": c, "U": u, "frames": frames,
           "items_detected": n, "items_checked": int(items.size), "vectors_checked": int(items.size * T),
           "symbols_checked": int(ntot), "xhat_normwise_max": float(nw.max()),
           "xhat_normwise_p999": float(np.quantile(nw, 0.999)), "sigma2_entry_max": entry_rel(s2, ref["sigma2"]),
           "decision_mismatches": int(nbad), "mismatch_rate": nbad / ntot, "mismatches_at_boundary": bool(at_boundary),
           "kernel": dbp._lib.lib().dbp_last_kernel()}
    if arch == "fd":
        nu = out.nu.index_select(0, idx).cpu().numpy().astype(float)
        if kind == "lama":  # [n][C][T] -> [n][T][C][U]
            nu = np.broadcast_to(np.transpose(nu, (0, 2, 1))[:, :, :, None], ref["nu"].shape)
        else:               # [n][C][U] -> [n][T][C][U]
            nu = np.broadcast_to(nu[:, None], ref["nu"].shape)
        res["nu_entry_max"] = entry_rel(nu, ref["nu"])
    return res


@pytest.mark.parametrize("name", list(WORKLOADS))
def test_parity_at_baseline_size(name):
    res = run_parity(name)
    print(json.dumps(res))
    out = os.environ.get("DBP_PARITY_OUT")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps(res) + "\n")
    assert res["symbols_checked"] >= 100_000 or res["items_checked"] == res["items_detected"]
    assert res["xhat_normwise_max"] < XHAT_TOL, res
    assert res["sigma2_entry_max"] < SIGMA2_TOL, res
    if "nu_entry_max" in res:
        assert res["nu_entry_max"] < NU_TOL, res
    assert res["mismatches_at_boundary"], res
    assert res["decision_mismatches"] <= max(1, int(np.ceil(DEC_RATE * res["symbols_checked"]))), res
