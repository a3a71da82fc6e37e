"""The vectorized oracle (oracle.run_batch_vec, used for parity at the
BASELINE sizes) equals the per-vector restatement (oracle.run_batch, pinned to
the reference's golden vectors by test_oracle_golden.py) on every
architecture / equalizer, and reproduces the reference's golden outputs."""

import numpy as np
import pytest

from oracle import dbp_oracle as O

CASES = [("pd", k) for k in ("mrc", "zf", "lmmse", "lama")] + [("fd", k) for k in ("mrc", "zf", "lmmse", "lama")]


@pytest.mark.parametrize("arch,kind", CASES)
def test_vec_equals_per_vector(arch, kind):
    rng = np.random.default_rng(3)
    n, b, c, u, t = 4, 64, 4, 8, 3
    H = (rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / np.sqrt(2 * b)
    syms, _ = O.square_qam(4)
    s = syms[rng.integers(0, 16, (n, t, u))]
    Y = np.einsum("nbu,ntu->ntb", H, s) + 0.2 * (rng.standard_normal((n, t, b)) + 1j * rng.standard_normal((n, t, b)))
    n0 = rng.uniform(0.02, 0.2, n)
    lp = {"t_max": 6} if kind == "lama" else None
    off = O.uniform_offsets(b, c)
    a = O.run_batch(arch, kind, H, Y, off, n0, 1.0, syms, lama_params=lp)
    v = O.run_batch_vec(arch, kind, H, Y, off, n0, 1.0, syms, lama_params=lp)
    np.testing.assert_allclose(v["z"], a["z"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(v["sigma2"], a["sigma2"], rtol=1e-10, atol=1e-14)
    np.testing.assert_array_equal(v["dec"], a["dec"])
    if arch == "fd":
        np.testing.assert_allclose(v["nu"], a["nu"], rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_vec_reproduces_reference_golden(golden, cfg):
    g = golden(cfg)
    b, c = int(g["B"]), int(g["C"])
    syms, _ = O.square_qam(int(g["bits"]))
    for key in sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_dec")}):
        arch, kind = key.split("_")
        lp = {"t_max": int(g["t_max"])} if kind == "lama" else None
        v = O.run_batch_vec(arch, kind, g["H"].astype(complex), g["Y"].astype(complex), O.uniform_offsets(b, c),
                            g["n0"], 1.0, syms, lama_params=lp)
        np.testing.assert_allclose(v["z"], g[f"{key}_z"], rtol=1e-9, atol=1e-11)
        np.testing.assert_array_equal(v["dec"], g[f"{key}_dec"])
