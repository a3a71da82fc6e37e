"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package itself (``/root/reference/pkg/src/dbp``, pure-NumPy kernel backend)
on seeded complex64-rounded inputs.

Run in the build container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed):
  golden_cfg*.npz  -- per-BASELINE-config samples: inputs H [n][B][U] and
                      Y [n][T][B] (complex64), n0 per item, and the reference
                      outputs exactly as montecarlo._equalize produces them
                      (PD: local_preprocess -> fuse_partials -> linear_equalize
                      -> unbiased_output, or lama_equalize(beta=U/B); FD:
                      fd_equalize plus the fusion weights replicated from its
                      internals, fusion.py:141-153), and hard decisions as
                      symbol indices.
  golden_units.npz -- small known-answer cases for every hot-path function.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
os.environ.setdefault("DBP_PURE_PYTHON", "1")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import dbp as ref  # noqa: E402  (the reference package)
from dbp import fusion as ref_fusion  # noqa: E402

from paper_1808_04473_b200.synth import synth_frames  # noqa: E402

CONFIGS = {
    # name: (archs, kinds, B, C, U, bits, snr list, items per snr, t_max)
    "cfg1": (("fd",), ("lmmse",), 64, 2, 8, 4, (10.0,), 6, None),
    "cfg2": (("pd",), ("lmmse",), 128, 4, 16, 4, (0.0, 10.0, 20.0), 2, None),
    "cfg3": (("fd",), ("zf", "mrc"), 256, 8, 16, 6, (15.0,), 3, None),
    "cfg4": (("pd", "fd"), ("lama",), 256, 8, 32, 4, (8.0,), 2, 10),
    "cfg5a": (("pd", "fd"), ("lmmse",), 512, 8, 64, 6, (20.0,), 1, None),
    "cfg5b": (("pd", "fd"), ("lmmse",), 1024, 8, 64, 6, (20.0,), 1, None),
}
T = 14
CONST = {4: ref.make_constellation("qam16"), 6: ref.make_constellation("qam64"),
         2: ref.make_constellation("qpsk")}


def sym_index(values, const):
    return np.argmin(np.abs(np.asarray(values)[:, None] - const.symbols[None, :]), axis=1)


def ref_pd(kind, h, y, part, n0, const, t_max):
    parts = [ref.local_preprocess(h[sl], y[sl]) for sl in part.slices()]
    fused = ref.fuse_partials(parts)
    if kind == "lama":
        out, _ = ref.lama_equalize(fused, const, n0, h.shape[1] / h.shape[0], t_max=t_max)
        return out.z, out.sigma2, None
    out = ref.linear_equalize(kind, fused, n0, es=const.es)
    unb = ref.unbiased_output(out, es=const.es)
    return unb.z, unb.sigma2, None


def ref_fd(kind, h, y, part, n0, const, t_max):
    ch = ref.ChannelRealization(h, part)
    lp = {"t_max": t_max} if kind == "lama" else None
    fd = ref.fd_equalize(kind, ch, y, n0, es=const.es, constellation=const, lama_params=lp)
    outs = [ref.cluster_equalize(kind, hc, y[sl], n0, es=const.es, total_antennas=ch.b,
                                 constellation=const, lama_params=lp, cluster_id=i)
            for i, (hc, sl) in enumerate(zip(ch.cluster_views, part.slices()))]
    outs = [ref_fusion._unbias_cluster(o, const.es) for o in outs]
    if kind == "mrc":
        g = np.stack([o.mrc_gains for o in outs])
        nu = g / g.sum(axis=0, keepdims=True)
    else:
        nu = ref.optimal_fusion_weights(np.stack([o.sigma2 for o in outs])).nu
    return fd.z, fd.sigma2, nu


def make_config(name, spec, seed):
    archs, kinds, b, c, u, bits, snrs, items, t_max = spec
    const = CONST[bits]
    H, Y, S, n0 = synth_frames(seed, len(snrs), items, T, b, u,
                               {4: "qam16", 6: "qam64", 2: "qpsk"}[bits], list(snrs))
    n0_item = np.repeat(n0, items)
    part = ref.ClusterPartition.uniform(b, c)
    out = dict(H=H, Y=Y, sym=S, n0=n0_item, B=b, C=c, U=u, T=T, bits=bits,
               t_max=t_max if t_max else 0)
    for arch in archs:
        for kind in kinds:
            zs, s2s, nus, decs = [], [], [], []
            for n in range(H.shape[0]):
                h = H[n].astype(np.complex128)
                row = ([], [], [], [])
                for t in range(T):
                    y = Y[n, t].astype(np.complex128)
                    fn = ref_pd if arch == "pd" else ref_fd
                    z, s2, nu = fn(kind, h, y, part, float(n0_item[n]), const, t_max)
                    row[0].append(z)
                    row[1].append(s2)
                    if nu is not None:
                        row[2].append(nu)
                    row[3].append(sym_index(ref.hard_detect(z, const), const))
                zs.append(row[0]); s2s.append(row[1]); nus.append(row[2]); decs.append(row[3])
            key = f"{arch}_{kind}"
            out[f"{key}_z"] = np.array(zs)
            out[f"{key}_sigma2"] = np.array(s2s)
            out[f"{key}_dec"] = np.array(decs).astype(np.uint8)
            if arch == "fd":
                out[f"{key}_nu"] = np.array(nus)
    path = os.path.join(HERE, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


def make_units(seed=2024):
    rng = np.random.default_rng(seed)
    u = {}
    # linear equalizers + unbias on assorted shapes (equalize.py:130-195)
    for i, (b, uu) in enumerate([(8, 2), (10, 5), (24, 6), (32, 16), (64, 16), (48, 8)]):
        h = (rng.standard_normal((b, uu)) + 1j * rng.standard_normal((b, uu))) / np.sqrt(2 * b)
        h = h.astype(np.complex64).astype(np.complex128)
        y = (rng.standard_normal(b) + 1j * rng.standard_normal(b)).astype(np.complex64).astype(np.complex128)
        n0 = float(rng.uniform(0.01, 0.5))
        st = ref.centralized_stats(h, y)
        u[f"lin{i}_h"], u[f"lin{i}_y"], u[f"lin{i}_n0"] = h, y, n0
        u[f"lin{i}_gram"], u[f"lin{i}_ymrc"] = st.gram, st.y_mrc
        for kind in ("mrc", "zf", "lmmse"):
            o = ref.linear_equalize(kind, st, n0)
            u[f"lin{i}_{kind}_z"], u[f"lin{i}_{kind}_sigma2"] = o.z, o.sigma2
            if o.signal_gain is not None:
                u[f"lin{i}_{kind}_gain"] = o.signal_gain
                ub = ref.unbiased_output(o)
                u[f"lin{i}_{kind}_uz"], u[f"lin{i}_{kind}_usigma2"] = ub.z, ub.sigma2
    # LAMA traces (equalize.py:208-259)
    for name in ("qpsk", "qam16", "qam64"):
        const = ref.make_constellation(name)
        cfg = ref.SystemConfig(b=64, u=16, n0=0.05)
        ch = ref.sample_rayleigh_channel(cfg, rng)
        s0 = ref.sample_symbols(const, cfg.u, rng)
        y = ref.transmit(ch, s0, cfg.n0, rng)
        h = ch.h.astype(np.complex64).astype(np.complex128)
        y = y.astype(np.complex64).astype(np.complex128)
        st = ref.centralized_stats(h, y)
        out, tr = ref.lama_equalize(st, const, cfg.n0, cfg.beta, t_max=6)
        u[f"lama_{name}_h"], u[f"lama_{name}_y"] = h, y
        u[f"lama_{name}_z"], u[f"lama_{name}_sigma2"] = out.z, out.sigma2
        u[f"lama_{name}_trace_z"] = np.array([s.z for s in tr])
        u[f"lama_{name}_trace_s"] = np.array([s.s for s in tr])
        u[f"lama_{name}_trace_v"] = np.array([s.v for s in tr])
        u[f"lama_{name}_trace_phi"] = np.array([s.phi for s in tr])
        out2, _ = ref.lama_equalize(st, const, cfg.n0, cfg.beta, t_max=6, damping=0.7)
        u[f"lama_{name}_damped_z"] = out2.z
    # posterior grid (_kernels_py.py:14-28)
    zg = (rng.uniform(-2, 2, 64) + 1j * rng.uniform(-2, 2, 64))
    u["post_z"] = zg
    for name in ("qpsk", "qam16", "qam64"):
        const = ref.make_constellation(name)
        for k, tau in enumerate((1e-3, 0.1, 1.0, 10.0)):
            f, g = ref.kernels.posterior_mean_var(zg, tau, const.symbols)
            u[f"post_{name}_{k}_f"], u[f"post_{name}_{k}_g"] = f, g
    # FD pipeline for C in 1,2,4,8 (fusion.py:127-154)
    const = CONST[4]
    for c in (1, 2, 4, 8):
        cfg = ref.SystemConfig(b=64, u=16, n0=0.1)
        part = ref.ClusterPartition.uniform(cfg.b, c)
        ch = ref.sample_rayleigh_channel(cfg, rng, part)
        s0 = ref.sample_symbols(const, cfg.u, rng)
        y = ref.transmit(ch, s0, cfg.n0, rng).astype(np.complex64).astype(np.complex128)
        h = ch.h.astype(np.complex64).astype(np.complex128)
        u[f"fd{c}_h"], u[f"fd{c}_y"] = h, y
        for kind in ("mrc", "zf", "lmmse", "lama"):
            if kind == "zf" and 64 // c < 16:
                continue
            lp = {"t_max": 5} if kind == "lama" else None
            z, s2, nu = ref_fd(kind, h, y, part, cfg.n0, const, 5)
            u[f"fd{c}_{kind}_z"], u[f"fd{c}_{kind}_sigma2"], u[f"fd{c}_{kind}_nu"] = z, s2, nu
            del lp
    # hard decisions (equalize.py:262-268)
    zh = rng.uniform(-1.5, 1.5, 200) + 1j * rng.uniform(-1.5, 1.5, 200)
    u["hard_z"] = zh
    for name in ("qpsk", "qam16", "qam64"):
        const = ref.make_constellation(name)
        u[f"hard_{name}_idx"] = sym_index(ref.hard_detect(zh, const), const)
    # message volumes (model.py:260-280)
    v = ref.message_volume(16, 1200, 14, 4)
    u["vol_16_1200_14_4"] = np.array([v.pd_bytes, v.fd_bytes, v.cs_bytes])
    path = os.path.join(HERE, "golden_units.npz")
    np.savez_compressed(path, **u)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    make_units()
    for i, (name, spec) in enumerate(CONFIGS.items()):
        make_config(name, spec, seed=1000 + i)
