"""Pin the CPU oracle (oracle/dbp_oracle.py) to the reference's own outputs
(tests/golden/*.npz, produced by running /root/reference via make_golden.py).
CPU only."""

import numpy as np
import pytest

from oracle import dbp_oracle as O

TOL = 1e-10


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1e-300, np.max(np.abs(b)))


@pytest.mark.parametrize("i", range(6))
def test_linear_units(golden, i):
    g = golden("units")
    h, y, n0 = g[f"lin{i}_h"], g[f"lin{i}_y"], float(g[f"lin{i}_n0"])
    gram, ym = O.gram_mrc(h, y)
    assert rel(gram, g[f"lin{i}_gram"]) < TOL and rel(ym, g[f"lin{i}_ymrc"]) < TOL
    for kind in ("mrc", "zf", "lmmse"):
        z, s2, gain = O.linear_equalize(kind, gram, ym, n0)
        assert rel(z, g[f"lin{i}_{kind}_z"]) < TOL
        assert rel(s2, g[f"lin{i}_{kind}_sigma2"]) < TOL
        if gain is not None:
            assert rel(gain, g[f"lin{i}_{kind}_gain"]) < TOL
            zu, su = O.unbias(z, s2, gain)
            assert rel(zu, g[f"lin{i}_{kind}_uz"]) < TOL
            assert rel(su, g[f"lin{i}_{kind}_usigma2"]) < TOL


@pytest.mark.parametrize("name,bits", [("qpsk", 2), ("qam16", 4), ("qam64", 6)])
def test_lama_units(golden, name, bits):
    g = golden("units")
    syms, _ = O.square_qam(bits)
    gram, ym = O.gram_mrc(g[f"lama_{name}_h"], g[f"lama_{name}_y"])
    z, s2, tr = O.lama_equalize(gram, ym, syms, 1.0, 0.05, 16 / 64, t_max=6, want_trace=True)
    assert rel(z, g[f"lama_{name}_z"]) < TOL
    assert rel(s2, g[f"lama_{name}_sigma2"]) < TOL
    assert rel([t[1] for t in tr], g[f"lama_{name}_trace_z"]) < TOL
    assert rel([t[4] for t in tr], g[f"lama_{name}_trace_phi"]) < TOL
    zd, _, _ = O.lama_equalize(gram, ym, syms, 1.0, 0.05, 16 / 64, t_max=6, damping=0.7)
    assert rel(zd, g[f"lama_{name}_damped_z"]) < TOL


def test_lama_receive_domain_equals_gram_domain():
    """Acceptance criterion 3 (test_acceptance.py:99-113) in float64: the
    receive-domain recursion (oracle.lama_receive_domain) and the pinned
    Gram-domain oracle give the same iterates on 20 instances."""
    rng = np.random.default_rng(99)
    syms, _ = O.square_qam(2)
    b, u, n0 = 64, 16, 0.05
    for _ in range(20):
        h = (rng.standard_normal((b, u)) + 1j * rng.standard_normal((b, u))) / np.sqrt(2 * b)
        s0 = syms[rng.integers(0, syms.size, u)]
        y = h @ s0 + (rng.standard_normal(b) + 1j * rng.standard_normal(b)) * np.sqrt(n0 / 2)
        gram, ym = O.gram_mrc(h, y)
        _, _, tr = O.lama_equalize(gram, ym, syms, 1.0, n0, u / b, t_max=5, want_trace=True)
        ref = O.lama_receive_domain(y, h, syms, n0, u / b, 5)
        for st, (z, phi) in zip(tr, ref):
            assert np.max(np.abs(st[1] - z)) < TOL and abs(st[4] - phi) < TOL


def test_posterior_and_hard_units(golden):
    g = golden("units")
    for name, bits in (("qpsk", 2), ("qam16", 4), ("qam64", 6)):
        syms, _ = O.square_qam(bits)
        for k, tau in enumerate((1e-3, 0.1, 1.0, 10.0)):
            f, gv = O.posterior_mean_var(g["post_z"], tau, syms)
            assert np.max(np.abs(f - g[f"post_{name}_{k}_f"])) < 1e-12
            assert np.max(np.abs(gv - g[f"post_{name}_{k}_g"])) < 1e-12
        assert np.array_equal(O.hard_detect_index(g["hard_z"], syms), g[f"hard_{name}_idx"])
    assert list(O.message_volume(16, 1200, 14, 4)) == list(g["vol_16_1200_14_4"])


@pytest.mark.parametrize("c", [1, 2, 4, 8])
def test_fd_units(golden, c):
    g = golden("units")
    syms, _ = O.square_qam(4)
    h, y = g[f"fd{c}_h"], g[f"fd{c}_y"]
    off = O.uniform_offsets(64, c)
    for kind in ("mrc", "zf", "lmmse", "lama"):
        if f"fd{c}_{kind}_z" not in g:
            continue
        r = O.fd_equalize(kind, h, y, off, 0.1, 1.0, syms, {"t_max": 5} if kind == "lama" else None)
        assert rel(r["z"], g[f"fd{c}_{kind}_z"]) < TOL
        assert rel(r["sigma2"], g[f"fd{c}_{kind}_sigma2"]) < TOL
        assert rel(r["nu"], g[f"fd{c}_{kind}_nu"]) < TOL


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5a"])
def test_config_samples(golden, cfg):
    g = golden(cfg)
    syms, _ = O.square_qam(int(g["bits"]))
    b, c = int(g["B"]), int(g["C"])
    off = O.uniform_offsets(b, c)
    H = g["H"].astype(np.complex128)
    Y = g["Y"].astype(np.complex128)
    t_max = int(g["t_max"])
    keys = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_dec")})
    # keep the CPU suite fast: first item, a few OFDM symbols
    items, tsel = [0], [0, 7, 13]
    for key in keys:
        arch, kind = key.split("_")
        lp = {"t_max": t_max} if kind == "lama" else None
        r = O.run_batch(arch, kind, H[:1][:, :, :], Y[:1][:, tsel], off, g["n0"][:1], 1.0, syms, lp,
                        items=items)
        assert rel(r["z"][0], g[f"{key}_z"][0][tsel]) < 1e-9
        assert rel(r["sigma2"][0], g[f"{key}_sigma2"][0][tsel]) < 1e-9
        assert np.array_equal(r["dec"][0], g[f"{key}_dec"][0][tsel])
        if arch == "fd":
            assert rel(r["nu"][0], g[f"{key}_nu"][0][tsel]) < 1e-9


def test_oracle_error_contract():
    with pytest.raises(O.OracleError) as e:
        O.linear_equalize("zf", np.ones((3, 3)) * 4, np.ones(3), 0.1)
    assert e.value.code == "SingularGramError"
    with pytest.raises(O.OracleError) as e:
        O.lama_equalize(np.eye(2) * 1e160, np.ones(2), O.square_qam(2)[0], 1.0, 0.1, 0.5, t_max=8)
    assert e.value.code == "DivergenceError" and e.value.iteration is not None
    with pytest.raises(O.OracleError):
        O.optimal_fusion_weights(np.array([[0.0], [1.0]]))
