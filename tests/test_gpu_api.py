"""The reference's own unit tests for the hot path (pkg/tests/test_equalize.py,
test_fusion.py, test_kernels.py posterior part), re-run against the drop-in
API on the GPU with fp32 tolerances, plus the golden known-answer cases that
the reference produced (tests/golden/golden_units.npz)."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from paper_1808_04473_b200 import (ClusterPartition, ConfigError, DivergenceError, FusedStats, SingularGramError,
                                   SystemConfig)
from paper_1808_04473_b200.equalize import EqualizerOutput
from paper_1808_04473_b200.fusion import ClusterOutput, FusionWeights
from oracle import dbp_oracle as O

pytestmark = pytest.mark.gpu

QPSK = dbp.make_constellation("qpsk")
QAM16 = dbp.make_constellation("qam16")
QAM64 = dbp.make_constellation("qam64")
F32 = 2e-5  # fp32 tolerance for O(1) quantities (reference uses 1e-10..1e-12 in fp64)


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1e-30, np.max(np.abs(b)))


def random_setup(rng, b=64, u=16, n0=0.05, c=4, const=QAM16):
    cfg = SystemConfig(b=b, u=u, n0=n0)
    part = ClusterPartition.uniform(b, c)
    ch = dbp.sample_rayleigh_channel(cfg, rng, part)
    s0 = dbp.sample_symbols(const, u, rng)
    y = dbp.transmit(ch, s0, n0, rng)
    return cfg, ch, s0, y


# ----------------------------------------------------- test_equalize.py ----
class TestPreprocess:
    def test_identity_channel(self):
        y = np.arange(1, 5) + 1j * np.arange(4)
        p = dbp.local_preprocess(np.eye(4, dtype=complex), y)
        assert np.allclose(p.gram, np.eye(4), atol=1e-6)
        assert np.allclose(p.y_mrc, y, atol=1e-6)

    def test_zero_channel(self):
        p = dbp.local_preprocess(np.zeros((6, 3), dtype=complex), np.ones(6, dtype=complex))
        assert np.allclose(p.gram, 0) and np.allclose(p.y_mrc, 0)

    def test_matches_golden_triple_loop_shapes(self, golden):
        g = golden("units")
        for i in range(6):
            p = dbp.local_preprocess(g[f"lin{i}_h"], g[f"lin{i}_y"])
            assert rel(p.gram, g[f"lin{i}_gram"]) < F32
            assert rel(p.y_mrc, g[f"lin{i}_ymrc"]) < F32

    def test_gram_is_hermitian_psd(self):
        rng = np.random.default_rng(4)
        h = rng.standard_normal((10, 5)) + 1j * rng.standard_normal((10, 5))
        g = dbp.local_preprocess(h, np.zeros(10, dtype=complex)).gram
        assert np.max(np.abs(g - g.conj().T)) < 1e-6
        assert np.min(np.linalg.eigvalsh(g)) > -1e-4

    def test_batched_with_symbols(self):
        rng = np.random.default_rng(5)
        h = (rng.standard_normal((3, 20, 6)) + 1j * rng.standard_normal((3, 20, 6))) / 5
        y = rng.standard_normal((3, 14, 20)) + 1j * rng.standard_normal((3, 14, 20))
        p = dbp.local_preprocess(h, y)
        for n in range(3):
            gr, _ = O.gram_mrc(h[n], y[n, 0])
            assert rel(p.gram[n], gr) < F32
            for t in range(14):
                assert rel(p.y_mrc[n, t], O.gram_mrc(h[n], y[n, t])[1]) < F32

    def test_dimension_mismatch(self):
        with pytest.raises(dbp.DimensionMismatchError):
            dbp.local_preprocess(np.ones((4, 2)), np.ones(5))


class TestFusePartials:
    def test_single_part_passthrough(self):
        rng = np.random.default_rng(0)
        h = rng.standard_normal((8, 3)) + 0j
        y = rng.standard_normal(8) + 0j
        p = dbp.local_preprocess(h, y)
        f = dbp.fuse_partials([p])
        assert np.array_equal(f.gram, p.gram) and np.array_equal(f.y_mrc, p.y_mrc)

    def test_matches_unpartitioned(self):
        rng = np.random.default_rng(1)
        _, ch, _, y = random_setup(rng)
        parts = [dbp.local_preprocess(h_c, y[sl]) for h_c, sl in zip(ch.cluster_views, ch.partition.slices())]
        fused = dbp.fuse_partials(parts)
        whole = dbp.centralized_stats(ch.h, y)
        assert rel(fused.gram, whole.gram) < F32 and rel(fused.y_mrc, whole.y_mrc) < F32

    def test_negated_parts_cancel(self):
        g = np.eye(2, dtype=complex)
        p1 = dbp.PartialStats(gram=g, y_mrc=np.ones(2, dtype=complex))
        p2 = dbp.PartialStats(gram=-g, y_mrc=-np.ones(2, dtype=complex))
        assert np.allclose(dbp.fuse_partials([p1, p2]).gram, 0)

    def test_empty_list_rejected(self):
        with pytest.raises(ConfigError):
            dbp.fuse_partials([])


class TestLinearEqualize:
    def test_identity_gram_estimates(self):
        y_mrc = np.array([0.3 + 1j, -0.5 - 0.2j, 1.1 + 0j])
        stats = FusedStats(gram=np.eye(3, dtype=complex), y_mrc=y_mrc)
        n0 = 0.2
        assert np.allclose(dbp.linear_equalize("mrc", stats, n0).z, y_mrc, atol=1e-6)
        assert np.allclose(dbp.linear_equalize("zf", stats, n0).z, y_mrc, atol=1e-6)
        assert np.allclose(dbp.linear_equalize("lmmse", stats, n0).z, y_mrc / 1.2, atol=1e-6)

    def test_noiseless_zf_recovers_symbols(self):
        rng = np.random.default_rng(5)
        h = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        s0 = dbp.sample_symbols(QPSK, 4, rng)
        out = dbp.linear_equalize("zf", dbp.centralized_stats(h, h @ s0), 0.0)
        assert np.max(np.abs(out.z - s0)) < 1e-3
        assert np.max(out.sigma2) == 0.0

    def test_golden_units(self, golden):
        g = golden("units")
        for i in range(6):
            st = FusedStats(gram=g[f"lin{i}_gram"], y_mrc=g[f"lin{i}_ymrc"])
            n0 = float(g[f"lin{i}_n0"])
            for kind in ("mrc", "zf", "lmmse"):
                o = dbp.linear_equalize(kind, st, n0)
                assert rel(o.z, g[f"lin{i}_{kind}_z"]) < 1e-4, (i, kind)
                assert rel(o.sigma2, g[f"lin{i}_{kind}_sigma2"]) < 1e-4, (i, kind)
                if kind == "lmmse":
                    assert rel(o.signal_gain, g[f"lin{i}_{kind}_gain"]) < 1e-4
                    ub = dbp.unbiased_output(o)
                    assert rel(ub.z, g[f"lin{i}_{kind}_uz"]) < 1e-4
                    assert rel(ub.sigma2, g[f"lin{i}_{kind}_usigma2"]) < 1e-4

    def test_zf_singular_gram(self):
        stats = dbp.centralized_stats(np.ones((4, 3), dtype=complex), np.ones(4, dtype=complex))
        with pytest.raises(SingularGramError):
            dbp.linear_equalize("zf", stats, 0.1)

    @pytest.mark.parametrize("u", [16, 40, 64])
    def test_zf_rank_deficient_batch(self, u):
        """B = u / 2 antennas: every item's Gram has rank u / 2 (ZF singular,
        the solvers of u <= 16, 17..32 and the blocked 64-wide sweep), while
        L-MMSE on the same statistics stays regular."""
        rng = np.random.default_rng(u)
        b = u // 2
        h = (rng.standard_normal((5, b, u)) + 1j * rng.standard_normal((5, b, u))) / np.sqrt(2 * b)
        y = (rng.standard_normal((5, b)) + 1j * rng.standard_normal((5, b))) * 0.1
        stats = dbp.centralized_stats(h, y)
        with pytest.raises(SingularGramError):
            dbp.linear_equalize("zf", stats, 0.1)
        out = dbp.linear_equalize("lmmse", stats, 0.1)
        for i in range(5):
            g, m = O.gram_mrc(h[i], y[i])
            z, s2, _ = O.linear_equalize("lmmse", g, m, 0.1)
            assert rel(out.z[i], z) < 1e-4 and rel(out.sigma2[i], s2) < 1e-4

    def test_mrc_zero_diagonal(self):
        stats = FusedStats(gram=np.zeros((2, 2), dtype=complex), y_mrc=np.zeros(2, dtype=complex))
        with pytest.raises(SingularGramError):
            dbp.linear_equalize("mrc", stats, 0.1)

    @pytest.mark.parametrize("c", [1, 2, 4, 8])
    def test_pd_equals_centralized(self, c):
        rng = np.random.default_rng(10 + c)
        cfg, ch, _, y = random_setup(rng, c=c)
        parts = [dbp.local_preprocess(h_c, y[sl]) for h_c, sl in zip(ch.cluster_views, ch.partition.slices())]
        fused = dbp.fuse_partials(parts)
        whole = dbp.centralized_stats(ch.h, y)
        for kind in ("mrc", "zf", "lmmse"):
            a = dbp.linear_equalize(kind, fused, cfg.n0)
            b = dbp.linear_equalize(kind, whole, cfg.n0)
            assert rel(a.z, b.z) < 1e-5 and rel(a.sigma2, b.sigma2) < 1e-5

    def test_lmmse_tends_to_zf(self):
        rng = np.random.default_rng(20)
        cfg, ch, _, y = random_setup(rng, n0=0.0)
        stats = dbp.centralized_stats(ch.h, y)
        zf = dbp.linear_equalize("zf", stats, 1e-12)
        lm = dbp.linear_equalize("lmmse", stats, 1e-12)
        assert np.max(np.abs(zf.z - lm.z)) < 1e-4

    def test_lmmse_unbiased_form(self):
        y_mrc = np.array([1 + 1j, -2j, 0.5 + 0j])
        stats = FusedStats(gram=np.eye(3, dtype=complex), y_mrc=y_mrc)
        out = dbp.linear_equalize("lmmse", stats, 0.25)
        assert np.allclose(out.signal_gain, 0.8, atol=1e-6)
        fixed = dbp.unbiased_output(out)
        assert np.allclose(fixed.z, y_mrc, atol=1e-6)
        assert np.allclose(fixed.sigma2, 0.25, atol=1e-6)
        zf = dbp.linear_equalize("zf", stats, 0.25)
        assert dbp.unbiased_output(zf) is zf


class TestPosterior:
    def test_symmetric_point(self):
        f, g = dbp.posterior_stats(0j, 0.4, QPSK)
        assert abs(f) < 1e-7 and g == pytest.approx(1.0, abs=1e-6)

    def test_requires_positive_tau(self):
        with pytest.raises(ConfigError):
            dbp.posterior_stats(0.1 + 0.1j, 0.0, QPSK)

    def test_hard_limit(self):
        target = QAM16.symbols[5]
        f, g = dbp.posterior_stats(complex(target + 0.02), 1e-9, QAM16)
        assert abs(f - target) < 1e-6 and g < 1e-6

    def test_golden_grid(self, golden):
        g = golden("units")
        for name, const in (("qpsk", QPSK), ("qam16", QAM16), ("qam64", QAM64)):
            for k, tau in enumerate((1e-3, 0.1, 1.0, 10.0)):
                f, gv = dbp.kernels.posterior_mean_var(g["post_z"], tau, const.symbols)
                assert np.max(np.abs(f - g[f"post_{name}_{k}_f"])) < 2e-4, (name, tau)
                assert np.max(np.abs(gv - g[f"post_{name}_{k}_g"])) < 2e-4, (name, tau)

    def test_tiny_tau_no_nan(self):
        f, g = dbp.kernels.posterior_mean_var(np.array([100.0 + 100.0j, 0j]), 1e-300 + 1e-30, QPSK.symbols)
        assert np.all(np.isfinite(f)) and np.all(np.isfinite(g))


class TestLama:
    def test_first_iteration_is_mrc_vector(self):
        rng = np.random.default_rng(30)
        _, ch, _, y = random_setup(rng)
        stats = dbp.centralized_stats(ch.h, y)
        out, trace = dbp.lama_equalize(stats, QAM16, n0=0.1, beta=0.25, t_max=1)
        assert trace[0].phi == pytest.approx(1.0)
        assert rel(out.z, stats.y_mrc) < 1e-6
        assert np.allclose(out.sigma2, 0.1 + 0.25, atol=1e-6)

    def test_orthogonal_noiseless_single_step(self):
        rng = np.random.default_rng(31)
        s0 = dbp.sample_symbols(QPSK, 8, rng)
        stats = FusedStats(gram=np.eye(8, dtype=complex), y_mrc=s0.copy())
        out, _ = dbp.lama_equalize(stats, QPSK, n0=0.0, beta=0.125, t_max=1)
        assert np.max(np.abs(out.z - s0)) < 1e-6

    @pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
    def test_golden_traces(self, golden, name):
        g = golden("units")
        const = dbp.make_constellation(name)
        stats = dbp.centralized_stats(g[f"lama_{name}_h"], g[f"lama_{name}_y"])
        out, tr = dbp.lama_equalize(stats, const, 0.05, 16 / 64, t_max=6)
        assert rel(out.z, g[f"lama_{name}_z"]) < 1e-4
        assert rel(out.sigma2, g[f"lama_{name}_sigma2"]) < 1e-4
        for k, st in enumerate(tr):
            assert rel(st.z, g[f"lama_{name}_trace_z"][k]) < 1e-4
            assert abs(st.phi - g[f"lama_{name}_trace_phi"][k]) < 1e-4
        out2, _ = dbp.lama_equalize(stats, const, 0.05, 16 / 64, t_max=6, damping=0.7)
        assert rel(out2.z, g[f"lama_{name}_damped_z"]) < 1e-4

    def test_matches_receive_domain_recursion(self):
        """acceptance criterion 3 (test_acceptance.py:99-113) at fp32."""
        rng = np.random.default_rng(99)
        for _ in range(5):
            cfg, ch, _, y = random_setup(rng, const=QPSK)
            stats = dbp.centralized_stats(ch.h, y)
            _, trace = dbp.lama_equalize(stats, QPSK, cfg.n0, cfg.beta, t_max=5)
            g64, m64 = O.gram_mrc(ch.h, y)
            _, _, ref = O.lama_equalize(g64, m64, QPSK.symbols, 1.0, cfg.n0, cfg.beta, t_max=5, want_trace=True)
            for st, r in zip(trace, ref):
                assert rel(st.z, r[1]) < 1e-4 and abs(st.phi - r[4]) < 1e-4

    def test_divergence_reports_iteration(self):
        stats = FusedStats(gram=np.eye(2, dtype=complex) * 1e30, y_mrc=np.ones(2, dtype=complex))
        with pytest.raises(DivergenceError) as err:
            dbp.lama_equalize(stats, QPSK, n0=0.1, beta=0.5, t_max=8)
        assert err.value.iteration is not None

    def test_rejects_bad_params(self):
        stats = FusedStats(gram=np.eye(2, dtype=complex), y_mrc=np.zeros(2, dtype=complex))
        with pytest.raises(ConfigError):
            dbp.lama_equalize(stats, QPSK, 0.1, 0.5, t_max=0)
        with pytest.raises(ConfigError):
            dbp.lama_equalize(stats, QPSK, 0.1, 0.5, damping=0.0)


class TestHardDetect:
    def test_exact_symbol(self):
        z = QAM16.symbols[[3, 7, 11]]
        assert np.allclose(dbp.hard_detect(z, QAM16), z)

    def test_tie_breaks_to_first_symbol(self):
        assert dbp.hard_detect(np.array([0j]), QPSK)[0] == QPSK.symbols[0]

    def test_golden(self, golden):
        g = golden("units")
        for name, const in (("qpsk", QPSK), ("qam16", QAM16), ("qam64", QAM64)):
            assert np.array_equal(dbp.hard_detect_index(g["hard_z"], const), g[f"hard_{name}_idx"])


# ------------------------------------------------------- test_fusion.py ----
def make_system(rng, b=64, u=16, n0=0.1, c=4, const=QAM16):
    return random_setup(rng, b=b, u=u, n0=n0, c=c, const=const)


class TestClusterEqualize:
    def test_single_cluster_equals_centralized(self):
        rng = np.random.default_rng(0)
        cfg, ch, _, y = make_system(rng, c=1)
        for kind in ("mrc", "zf", "lmmse"):
            local = dbp.cluster_equalize(kind, ch.h, y, cfg.n0, total_antennas=cfg.b)
            central = dbp.linear_equalize(kind, dbp.fuse_partials([dbp.local_preprocess(ch.h, y)]), cfg.n0)
            assert rel(local.z, central.z) < 1e-5 and rel(local.sigma2, central.sigma2) < 1e-5

    def test_single_cluster_lama_equals_pd(self):
        rng = np.random.default_rng(1)
        cfg, ch, _, y = make_system(rng, c=1, const=QPSK)
        local = dbp.cluster_equalize("lama", ch.h, y, cfg.n0, total_antennas=cfg.b, constellation=QPSK,
                                     lama_params={"t_max": 6})
        pd, _ = dbp.lama_equalize(dbp.fuse_partials([dbp.local_preprocess(ch.h, y)]), QPSK, cfg.n0, cfg.beta,
                                  t_max=6)
        assert rel(local.z, pd.z) < 1e-5

    def test_zf_underdetermined_cluster(self):
        rng = np.random.default_rng(2)
        h_c = rng.standard_normal((8, 16)) + 1j * rng.standard_normal((8, 16))
        with pytest.raises(SingularGramError):
            dbp.cluster_equalize("zf", h_c, np.zeros(8, dtype=complex), 0.1)

    def test_zf_sigma2_matches_dense_inverse(self):
        rng = np.random.default_rng(3)
        h_c = (rng.standard_normal((32, 16)) + 1j * rng.standard_normal((32, 16))) / 8
        y_c = rng.standard_normal(32) + 1j * rng.standard_normal(32)
        out = dbp.cluster_equalize("zf", h_c, y_c, n0=0.1)
        ref = np.real(np.diag(np.linalg.inv(h_c.conj().T @ h_c))) * 0.1
        assert rel(out.sigma2, ref) < 1e-4

    def test_linear_kinds_invariant_to_rescaling(self):
        rng = np.random.default_rng(4)
        h_c = (rng.standard_normal((24, 6)) + 1j * rng.standard_normal((24, 6))) / 10
        y_c = rng.standard_normal(24) + 1j * rng.standard_normal(24)
        for kind in ("mrc", "zf", "lmmse"):
            raw = dbp.cluster_equalize(kind, h_c, y_c, n0=0.07)
            scaled = dbp.cluster_equalize(kind, h_c, y_c, n0=0.07, total_antennas=96)
            assert rel(raw.z, scaled.z) < 1e-6 and rel(raw.sigma2, scaled.sigma2) < 1e-6


class TestFusionWeights:
    def test_equal_variances_give_uniform_weights(self):
        assert np.allclose(dbp.optimal_fusion_weights(np.full((4, 3), 0.2)).nu, 0.25)

    def test_two_cluster_hand_value(self):
        nu = dbp.optimal_fusion_weights(np.array([[1.0], [3.0]])).nu
        assert nu[:, 0] == pytest.approx([0.75, 0.25], abs=1e-6)

    def test_vanishing_variance_takes_all_weight(self):
        nu = dbp.optimal_fusion_weights(np.array([[1e-12], [1.0]])).nu
        assert nu[0, 0] == pytest.approx(1.0, abs=1e-6)

    def test_rejects_nonpositive(self):
        with pytest.raises(ConfigError):
            dbp.optimal_fusion_weights(np.array([[0.0], [1.0]]))
        with pytest.raises(ConfigError):
            dbp.optimal_fusion_weights(np.array([[-1.0], [1.0]]))

    def test_columns_sum_to_one(self):
        rng = np.random.default_rng(5)
        nu = dbp.optimal_fusion_weights(10.0 ** rng.uniform(-3, 1, (6, 9))).nu
        assert np.max(np.abs(nu.sum(axis=0) - 1.0)) < 1e-6


class TestFuseEstimates:
    def _outputs(self, z_rows, s2_rows):
        return [ClusterOutput(cluster_id=i, z=np.asarray(z, dtype=complex), sigma2=np.asarray(s, dtype=float),
                              equalizer="zf") for i, (z, s) in enumerate(zip(z_rows, s2_rows))]

    def test_single_cluster_passthrough(self):
        outs = self._outputs([[1 + 1j, 2]], [[0.5, 0.25]])
        fused = dbp.fuse_estimates(outs, FusionWeights(nu=np.ones((1, 2))))
        assert np.allclose(fused.z, outs[0].z) and np.allclose(fused.sigma2, outs[0].sigma2)

    def test_hand_worked_two_cluster_case(self):
        outs = self._outputs([[1 + 0j], [2 + 0j]], [[1.0], [3.0]])
        fused = dbp.fuse_estimates(outs, dbp.optimal_fusion_weights(np.array([[1.0], [3.0]])))
        assert fused.z[0] == pytest.approx(1.25, abs=1e-6)
        assert fused.sigma2[0] == pytest.approx(0.75, abs=1e-6)

    def test_dimension_mismatch(self):
        outs = self._outputs([[1 + 0j], [2 + 0j]], [[1.0], [3.0]])
        with pytest.raises(dbp.DimensionMismatchError):
            dbp.fuse_estimates(outs, FusionWeights(nu=np.ones((3, 1)) / 3))


class TestNegativeVariance:
    """equalize.py:115-120 on the device: unbiased_output's variance
    (sigma2 - (1 - c)^2 Es) / c^2 below -1e-9 raises NegativeVarianceError
    (status ST_NEGVAR of dbp_unbias), rounding-level negatives clamp to 0."""

    def test_unbias_negative_variance_raises(self):
        out = EqualizerOutput(z=np.array([1 + 0j, 0.5j]), sigma2=np.array([0.3, 0.01]), equalizer=dbp.Equalizer.LMMSE,
                              signal_gain=np.array([0.9, 0.5]))
        with pytest.raises(dbp.NegativeVarianceError):
            dbp.unbiased_output(out)

    def test_unbias_rounding_negative_clamps(self):
        c = 0.5
        out = EqualizerOutput(z=np.array([1 + 0j]), sigma2=np.array([np.nextafter(np.float32((1 - c) ** 2), np.float32(0))]), equalizer=dbp.Equalizer.LMMSE,
                              signal_gain=np.array([c]))
        res = dbp.unbiased_output(out)
        assert res.sigma2[0] == 0.0


class TestFdPipeline:
    def test_golden_units(self, golden):
        g = golden("units")
        for c in (1, 2, 4, 8):
            part = ClusterPartition.uniform(64, c)
            ch = dbp.ChannelRealization(g[f"fd{c}_h"], part)
            # MRC, L-MMSE (regularized: kappa(G_c + rho I) <= 1 + ||G_c|| / rho)
            # and LAMA (no inverse) are held to the fixed 1e-4 of the north
            # star.  Only unregularized ZF on a square local system (B_c = U =
            # 16 at C = 4: kappa(G_c) ~ 4e4) gets an allowance proportional to
            # kappa; C = 8 (B_c < U) has no ZF case (SingularGramError).
            hh = g[f"fd{c}_h"]
            kappa = max(np.linalg.cond(hh[sl].conj().T @ hh[sl]) for sl in part.slices())
            for kind in ("mrc", "zf", "lmmse", "lama"):
                if f"fd{c}_{kind}_z" not in g:
                    continue
                lp = {"t_max": 5} if kind == "lama" else None
                fd = dbp.fd_equalize(kind, ch, g[f"fd{c}_y"], 0.1, constellation=QAM16, lama_params=lp,
                                     return_weights=True)
                tol = max(1e-4, 2e-6 * kappa) if (kind == "zf" and 64 // c <= 16) else 1e-4
                assert rel(fd.z, g[f"fd{c}_{kind}_z"]) < tol, (c, kind)
                assert rel(fd.sigma2, g[f"fd{c}_{kind}_sigma2"]) < tol, (c, kind)
                assert rel(fd.nu, g[f"fd{c}_{kind}_nu"]) < tol, (c, kind)

    def test_mrc_fd_equals_pd_exactly(self):
        for c in (1, 2, 4, 8):
            rng = np.random.default_rng(100 + c)
            cfg, ch, _, y = make_system(rng, c=c)
            fd = dbp.fd_equalize("mrc", ch, y, cfg.n0)
            parts = [dbp.local_preprocess(h_c, y[sl]) for h_c, sl in zip(ch.cluster_views, ch.partition.slices())]
            pd = dbp.linear_equalize("mrc", dbp.fuse_partials(parts), cfg.n0)
            assert rel(fd.z, pd.z) < 1e-5

    def test_fused_variance_below_cluster_minimum(self):
        rng = np.random.default_rng(7)
        cfg, ch, _, y = make_system(rng, c=4)
        fd = dbp.fd_equalize("lmmse", ch, y, cfg.n0)
        per = [dbp.cluster_equalize("lmmse", h_c, y[sl], cfg.n0, total_antennas=cfg.b).sigma2
               for h_c, sl in zip(ch.cluster_views, ch.partition.slices())]
        assert np.all(fd.sigma2 <= np.min(per, axis=0) * (1 + 1e-5))

    def test_lama_fd_sigma2_is_running_estimate(self):
        rng = np.random.default_rng(8)
        cfg, ch, _, y = make_system(rng, c=2, const=QPSK)
        out = dbp.cluster_equalize("lama", ch.cluster_views[0], y[ch.partition.slices()[0]], cfg.n0,
                                   total_antennas=cfg.b, constellation=QPSK, lama_params={"t_max": 4})
        assert np.ptp(out.sigma2) == 0.0

    def test_fd_detects_at_moderate_noise(self):
        rng = np.random.default_rng(9)
        cfg, ch, s0, y = make_system(rng, b=128, u=8, n0=0.02, c=4, const=QPSK)
        for kind in ("zf", "lmmse", "lama"):
            fd = dbp.fd_equalize(kind, ch, y, cfg.n0, constellation=QPSK,
                                 lama_params={"t_max": 8} if kind == "lama" else None)
            assert np.array_equal(dbp.hard_detect(fd, QPSK), s0)

    def test_ragged_partition_and_odd_sizes(self):
        """Uneven cluster sizes (odd counts) and odd U go through the host
        padding path and still match the oracle."""
        rng = np.random.default_rng(11)
        b, u = 45, 5
        part = ClusterPartition(b, (13, 20, 12))
        h = (rng.standard_normal((b, u)) + 1j * rng.standard_normal((b, u))) / np.sqrt(2 * b)
        y = rng.standard_normal(b) + 1j * rng.standard_normal(b)
        ch = dbp.ChannelRealization(h, part)
        for kind in ("mrc", "zf", "lmmse", "lama"):
            lp = {"t_max": 4} if kind == "lama" else None
            fd = dbp.fd_equalize(kind, ch, y, 0.05, constellation=QPSK, lama_params=lp, return_weights=True)
            ref = O.fd_equalize(kind, ch.h.astype(np.complex64).astype(complex),
                                y.astype(np.complex64).astype(complex), list(part.offsets), 0.05, 1.0,
                                QPSK.symbols, lp)
            assert rel(fd.z, ref["z"]) < 1e-4, kind
            assert rel(fd.nu, ref["nu"]) < 1e-4, kind


def test_backend_name():
    assert dbp.kernels.backend() == "cuda-sm_100a"


def test_torch_tensors_stay_on_device():
    import torch

    rng = np.random.default_rng(12)
    h = torch.as_tensor((rng.standard_normal((4, 32, 8)) + 1j * rng.standard_normal((4, 32, 8))).astype(np.complex64),
                        device="cuda")
    y = torch.as_tensor((rng.standard_normal((4, 14, 32)) + 1j * rng.standard_normal((4, 14, 32))).astype(np.complex64),
                        device="cuda")
    p = dbp.local_preprocess(h, y)
    assert p.gram.is_cuda and p.gram.shape == (4, 8, 8) and p.y_mrc.shape == (4, 14, 8)
    out = dbp.linear_equalize("zf", dbp.FusedStats(p.gram, p.y_mrc), 0.1)
    assert out.z.is_cuda and out.z.shape == (4, 14, 8)
