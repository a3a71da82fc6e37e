"""The oracle's Gauss-Hermite quadratures (oracle.dbp_oracle: lama_mse_pam,
lama_mse, mi_awgn) against the reference's own
kernels (tests/golden/golden_quad.npz, tests/golden/make_golden_quad.py)."""

import os

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_quad.npz"))


def close(a, b, rtol=1e-11, atol=1e-15):
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol)


@pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
def test_oracle_quadratures_match_reference(name):
    c = dbp.make_constellation(name)
    close([O.lama_mse_pam(s, c.pam_levels) for s in G["sigma2"]], G[f"{name}_mse_pam"])
    close([O.lama_mse_pam(s, c.pam_levels, 64) for s in G["sigma2"]], G[f"{name}_mse_pam_o64"])
    close([O.lama_mse(s, c.symbols, 16) for s in G["sigma2"]], G[f"{name}_mse_2d_o16"])
    close([O.mi_awgn(c.es / s, c.symbols, 16) for s in G["sinr"][1:]], G[f"{name}_mi_o16"])


@pytest.mark.parametrize("tag,beta,c", [("small", 8 / 64, 2), ("crit8", 16 / 256, 8)])
def test_linear_asymptotic_sinr_matches_reference(tag, beta, c):
    """The closed-form large-system SINRs (host arithmetic, no GPU) equal the
    reference's for MRC / ZF / L-MMSE in every architecture."""
    from paper_1808_04473_b200 import asymptotics as A

    q16 = dbp.make_constellation("qam16")
    w = np.full(c, 1.0 / c)
    for kind in ("mrc", "zf", "lmmse"):
        for arch in ("pd", "fd", "centralized"):
            got = [A.asymptotic_sinr(kind, arch, q16, 10.0 ** (x / 10.0), beta, weights=w) for x in G[f"sinr_{tag}_snr"]]
            close(got, G[f"sinr_{tag}_{kind}_{arch}"], rtol=1e-13)
