"""CPU oracle for the decentralized feedforward equalization path.

TEST INFRASTRUCTURE ONLY.  This module is a float64 NumPy restatement of the
reference package's algorithm (``/root/reference/pkg/src/dbp``) for the hot
path: Gram/matched-filter preprocessing, PD fusion, MRC/ZF/L-MMSE, the
Gram-domain LAMA recursion with its discrete-posterior denoiser, FD per-cluster
equalization with SINR-optimal fusion, and nearest-symbol detection.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference`` arm) may import it, and only as the checker or as
the timed CPU baseline.  The product path (``paper_1808_04473_b200``) never
imports it.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (imported
from ``/root/reference/pkg/src`` in the build container) on seeded inputs and
commits the outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this module against those fixtures at 1e-10.

Every function cites the reference file:line it restates.  Shapes follow the
reference's per-vector API; the ``*_batch`` drivers loop the per-vector
functions over ``[n][T]`` exactly as ``montecarlo._equalize`` would.
"""

from __future__ import annotations

import numpy as np

# equalize.py:24 -- variances below -_VAR_TOL signal a numerical fault
VAR_TOL = 1e-9
# fusion.py:23 -- floor applied before inverting variances
VARIANCE_FLOOR = 1e-15

MRC, ZF, LMMSE, LAMA = "mrc", "zf", "lmmse", "lama"


class OracleError(Exception):
    """Raised where the reference raises; ``code`` names the reference type."""

    def __init__(self, code, msg="", iteration=None):
        super().__init__(f"{code}: {msg}")
        self.code = code
        self.iteration = iteration


# --------------------------------------------------------------------------
# constellations (model.py:80-98)
# --------------------------------------------------------------------------
def square_qam(bits_per_symbol):
    """Unit-energy square QAM.  model.py:80-85: per-dimension amplitudes
    -(L-1), ..., L-1 in steps of 2, grid built with meshgrid(indexing='ij') so
    symbol k = i*L + j has real level i and imaginary level j; both the
    points and the levels are divided by the rms of the points."""
    n_levels = {2: 2, 4: 4, 6: 8}[bits_per_symbol]
    amps = np.arange(-(n_levels - 1), n_levels, 2, dtype=float)
    pts = (amps[:, None] + 1j * amps[None, :]).reshape(-1)
    rms = np.sqrt(np.mean(np.abs(pts) ** 2))
    return pts / rms, amps / rms


# --------------------------------------------------------------------------
# preprocessing / PD fusion (equalize.py:85-112)
# --------------------------------------------------------------------------
def gram_mrc(h_c, y_c):
    """equalize.py:85-93: G_c = H_c^H H_c, y_c^mrc = H_c^H y_c."""
    h_c = np.asarray(h_c, dtype=np.complex128)
    y_c = np.asarray(y_c, dtype=np.complex128)
    hh = h_c.conj().T
    return hh @ h_c, hh @ y_c


def fuse_partials(parts):
    """equalize.py:96-107: element-wise sums of the partial statistics."""
    parts = list(parts)
    if not parts:
        raise OracleError("ConfigError", "empty partial list")
    return (np.sum([g for g, _ in parts], axis=0),
            np.sum([m for _, m in parts], axis=0))


def _check_sigma2(s2):
    """equalize.py:115-120."""
    if np.min(s2) < -VAR_TOL:
        raise OracleError("NegativeVarianceError", f"{np.min(s2)}")
    return np.maximum(s2, 0.0)


def _chol_lower(a):
    """equalize.py:123-127 (scipy zpotrf, lower); failure -> SingularGram."""
    try:
        return np.linalg.cholesky(a)
    except np.linalg.LinAlgError:
        raise OracleError("SingularGramError", "not positive definite")


def _tri_solve_lower(l, b):
    """Forward substitution L x = b (b may be a matrix)."""
    n = l.shape[0]
    x = np.array(b, dtype=np.complex128, copy=True)
    for k in range(n):
        x[k] = (x[k] - l[k, :k] @ x[:k]) / l[k, k]
    return x


def _tri_solve_upper(r, b):
    """Back substitution R x = b."""
    n = r.shape[0]
    x = np.array(b, dtype=np.complex128, copy=True)
    for k in range(n - 1, -1, -1):
        x[k] = (x[k] - r[k, k + 1:] @ x[k + 1:]) / r[k, k]
    return x


def linear_equalize(kind, g, y_mrc, n0, es=1.0):
    """equalize.py:130-176.  Returns (z, sigma2, signal_gain|None).

    MRC  (:144-152): d = Re diag G; z = y/d; sigma2 = N0/d + Es*sum_j|G_ij/d_i - delta_ij|^2.
    ZF   (:153-158): L = chol(G); z = cho_solve; sigma2 = N0 * diag(G^-1) from L^-1.
    LMMSE(:159-172): A = (G + rho I)^-1 via Cholesky; z = A y; sigma2 =
         N0*rowsum(AG . conj A) + Es*sum_j|(AG - I)_ij|^2; gain = Re diag(AG).
    """
    g = np.asarray(g, dtype=np.complex128)
    y_mrc = np.asarray(y_mrc, dtype=np.complex128)
    u = y_mrc.shape[0]
    eye = np.eye(u)
    if kind == MRC:
        d = np.real(np.diag(g)).copy()
        if np.any(d <= 0.0):
            raise OracleError("SingularGramError", "MRC diagonal")
        z = y_mrc / d
        s2 = n0 / d + es * np.sum(np.abs(g / d[:, None] - eye) ** 2, axis=1)
        return z, _check_sigma2(s2), None
    if kind == ZF:
        l = _chol_lower(g)
        z = _tri_solve_upper(l.conj().T, _tri_solve_lower(l, y_mrc))
        linv = _tri_solve_lower(l, eye.astype(np.complex128))
        s2 = n0 * np.sum(np.abs(linv) ** 2, axis=0)
        return z, _check_sigma2(s2), None
    if kind == LMMSE:
        if es <= 0:
            raise OracleError("ConfigError", "L-MMSE requires Es > 0")
        rho = n0 / es
        l = _chol_lower(g + rho * eye)
        inv = _tri_solve_upper(l.conj().T, _tri_solve_lower(l, eye.astype(np.complex128)))
        z = inv @ y_mrc
        ag = inv @ g
        noise = n0 * np.real(np.sum(ag * inv.conj(), axis=1))
        interf = es * np.sum(np.abs(ag - eye) ** 2, axis=1)
        gain = np.real(np.diag(ag))
        return z, _check_sigma2(noise + interf), gain
    raise OracleError("ConfigError", f"kind {kind}")


def unbias(z, s2, gain, es=1.0):
    """equalize.py:179-195: z/c with (sigma2 - (1-c)^2 Es)/c^2; pass-through
    when there is no gain."""
    if gain is None:
        return z, s2
    if np.any(gain <= 0):
        raise OracleError("SingularGramError", "nonpositive signal gain")
    s2u = (s2 - (1.0 - gain) ** 2 * es) / gain ** 2
    return z / gain, _check_sigma2(s2u)


# --------------------------------------------------------------------------
# LAMA (equalize.py:208-259) and its denoiser (_kernels_py.py:14-28)
# --------------------------------------------------------------------------
def posterior_mean_var(z, tau, symbols):
    """_kernels_py.py:14-28 / _kernels.pyx:19-50: log-domain weights
    w_k = exp(-(|z-a_k|^2 - min_k |z-a_k|^2)/tau), F = sum w a / sum w,
    G = max(sum w |a|^2 / sum w - |F|^2, 0)."""
    z = np.atleast_1d(np.asarray(z, dtype=np.complex128))
    symbols = np.asarray(symbols, dtype=np.complex128)
    d2 = np.abs(z[:, None] - symbols[None, :]) ** 2
    d2 = d2 - d2.min(axis=1, keepdims=True)
    w = np.exp(-d2 / tau)
    w = w / w.sum(axis=1, keepdims=True)
    f = w @ symbols
    g = np.maximum(w @ (np.abs(symbols) ** 2) - np.abs(f) ** 2, 0.0)
    return f, g


def lama_equalize(g, y_mrc, symbols, es, n0, beta, t_max=10, damping=1.0,
                  want_trace=False):
    """equalize.py:208-259: Gram-domain recursion
        tau^t = N0 + beta phi^t
        z^t = y_mrc + (I - G) s^t + v^t        (divergence check :247-249)
        (F, G) = posterior(z^t, max(tau^t, 1e-300))
        v^{t+1} = beta phi^{t+1} / tau^t (z^t - s^t)
        s^{t+1} = theta F + (1 - theta) s^t
    started at s = mean(symbols), v = 0, phi = Es.  Output z^{t_max} with
    sigma2 = tau^{t_max} broadcast (:257)."""
    if t_max < 1:
        raise OracleError("ConfigError", "t_max must be >= 1")
    if not 0.0 < damping <= 1.0:
        raise OracleError("ConfigError", "damping must lie in (0, 1]")
    g = np.asarray(g, dtype=np.complex128)
    y_mrc = np.asarray(y_mrc, dtype=np.complex128)
    symbols = np.asarray(symbols, dtype=np.complex128)
    u = y_mrc.shape[0]
    a = np.eye(u) - g
    s = np.full(u, symbols.mean(), dtype=np.complex128)
    v = np.zeros(u, dtype=np.complex128)
    phi = float(es)
    trace = []
    z = None
    tau = n0 + beta * phi
    for t in range(1, t_max + 1):
        tau = n0 + beta * phi
        z = y_mrc + a @ s + v
        if not (np.all(np.isfinite(z)) and np.isfinite(tau)
                and np.max(np.abs(z)) < 1e150):
            raise OracleError("DivergenceError", f"t={t}", iteration=t)
        if want_trace:
            trace.append((t, z.copy(), s.copy(), v.copy(), phi))
        f, gv = posterior_mean_var(z, max(tau, 1e-300), symbols)
        phi_next = float(np.mean(gv))
        v = (beta * phi_next) / tau * (z - s)
        s = damping * f + (1.0 - damping) * s
        phi = phi_next
    return z, np.full(u, tau), trace


def lama_receive_domain(y, h, symbols, n0, beta, t_max):
    """The receive-domain message passing the Gram-domain recursion is
    derived from -- the reference's independent check of lama_equalize
    (tests/oracles.py:55-82, used by test_acceptance.py:99-113):
        z^t = s^t + H^H r^t,   eff^t = N0 (1 + tau^t)
        (F, G) = posterior(z^t, eff^t),  tau^{t+1} = beta/N0 mean(G)
        r^{t+1} = y - H F + tau^{t+1} / (1 + tau^t) r^t,  s^{t+1} = F
    from s^1 = E[S], tau^1 = beta Var[S] / N0, r^1 = y - H s^1.  Returns the
    list of (z^t, phi^t = N0 tau^t / beta)."""
    y = np.asarray(y, dtype=np.complex128)
    h = np.asarray(h, dtype=np.complex128)
    symbols = np.asarray(symbols, dtype=np.complex128)
    mean = symbols.mean()
    s = np.full(h.shape[1], mean, dtype=np.complex128)
    tau = beta * float(np.mean(np.abs(symbols - mean) ** 2)) / n0
    r = y - h @ s
    out = []
    for _ in range(t_max):
        z = s + h.conj().T @ r
        out.append((z, n0 * tau / beta))
        f, g = posterior_mean_var(z, n0 * (1.0 + tau), symbols)
        tau_next = beta / n0 * float(np.mean(g))
        r = y - h @ f + (tau_next / (1.0 + tau)) * r
        s, tau = f, tau_next
    return out


def hard_detect_index(z, symbols):
    """equalize.py:262-268: argmin_k |z - a_k|^2, ties to the lowest k
    (np.argmin returns the first minimum).  Returned as indices."""
    z = np.atleast_1d(np.asarray(z, dtype=np.complex128))
    symbols = np.asarray(symbols, dtype=np.complex128)
    return np.argmin(np.abs(z[:, None] - symbols[None, :]) ** 2, axis=1)


# --------------------------------------------------------------------------
# FD (fusion.py:43-154)
# --------------------------------------------------------------------------
def cluster_equalize(kind, h_c, y_c, n0, es=1.0, total_antennas=None,
                     symbols=None, lama_params=None):
    """fusion.py:43-75.  Returns dict(z, sigma2, gain, mrc_gains).
    LAMA runs on the rescaled system G/w_c, y/w_c, N0/w_c with beta_c = U/B_c
    (:60,:66-68); linear kinds run unscaled (:70)."""
    h_c = np.asarray(h_c, dtype=np.complex128)
    b_c, u = h_c.shape
    g, ym = gram_mrc(h_c, y_c)
    w_c = b_c / total_antennas if total_antennas else 1.0
    gain = None
    if kind == LAMA:
        p = dict(lama_params or {})
        z, s2, _ = lama_equalize(g / w_c, ym / w_c, symbols, es, n0 / w_c,
                                 u / b_c, **p)
    else:
        z, s2, gain = linear_equalize(kind, g, ym, n0, es)
    mrc_gains = np.real(np.diag(g)) if kind == MRC else None
    return dict(z=z, sigma2=s2, gain=gain, mrc_gains=mrc_gains)


def optimal_fusion_weights(s2):
    """fusion.py:96-105: nu_{c,u} = (1/max(s2,1e-15)) / sum_c (...);
    ConfigError if any s2 <= 0."""
    s2 = np.asarray(s2, dtype=float)
    if s2.ndim != 2:
        raise OracleError("DimensionMismatchError", "expected C x U")
    if np.any(s2 <= 0):
        raise OracleError("ConfigError", "fusion weights need s2 > 0")
    inv = 1.0 / np.maximum(s2, VARIANCE_FLOOR)
    return inv / inv.sum(axis=0, keepdims=True)


def fuse_estimates(z_stack, s2_stack, nu):
    """fusion.py:108-124: z = sum_c nu z_c; s2 = 1/sum_c 1/max(s2_c, floor)."""
    z = np.sum(nu * z_stack, axis=0)
    s2 = 1.0 / np.sum(1.0 / np.maximum(s2_stack, VARIANCE_FLOOR), axis=0)
    return z, s2


def fd_equalize(kind, h, y, offsets, n0, es=1.0, symbols=None,
                lama_params=None):
    """fusion.py:127-154, additionally returning the weights nu (C x U) and
    the per-cluster raw/unbiased outputs (the reference computes but does not
    return them)."""
    b = h.shape[0]
    outs = []
    for c in range(len(offsets) - 1):
        sl = slice(offsets[c], offsets[c + 1])
        outs.append(cluster_equalize(kind, h[sl], y[sl], n0, es=es,
                                     total_antennas=b, symbols=symbols,
                                     lama_params=lama_params))
    # fusion.py:148 -- fuse in the unbiased domain
    unb = [unbias(o["z"], o["sigma2"], o["gain"], es) for o in outs]
    z_stack = np.stack([zu for zu, _ in unb])
    s2_stack = np.stack([su for _, su in unb])
    if kind == MRC:
        gains = np.stack([o["mrc_gains"] for o in outs])
        nu = gains / gains.sum(axis=0, keepdims=True)  # fusion.py:149-151
    else:
        nu = optimal_fusion_weights(s2_stack)          # fusion.py:153
    z, s2 = fuse_estimates(z_stack, s2_stack, nu)
    return dict(z=z, sigma2=s2, nu=nu, clusters=outs, z_unbiased=z_stack,
                sigma2_unbiased=s2_stack)


def pd_equalize(kind, h, y, offsets, n0, es=1.0, symbols=None,
                lama_params=None):
    """montecarlo.py:131-145 (PD branch): per-cluster preprocess, fuse,
    central equalizer; linear outputs are unbiased before detection, LAMA
    runs with beta = U/B."""
    b, u = h.shape
    parts = [gram_mrc(h[offsets[c]:offsets[c + 1]], y[offsets[c]:offsets[c + 1]])
             for c in range(len(offsets) - 1)]
    g, ym = fuse_partials(parts)
    if kind == LAMA:
        z, s2, _ = lama_equalize(g, ym, symbols, es, n0, u / b,
                                 **dict(lama_params or {}))
        return dict(z=z, sigma2=s2, z_raw=z, gain=None)
    z, s2, gain = linear_equalize(kind, g, ym, n0, es)
    zu, s2u = unbias(z, s2, gain, es)
    return dict(z=zu, sigma2=s2u, z_raw=z, sigma2_raw=s2, gain=gain)


# --------------------------------------------------------------------------
# batched drivers over [n][B][U] channels and [n][T][B] receive vectors
# --------------------------------------------------------------------------
def uniform_offsets(b, c):
    """model.py:158-175 (ClusterPartition.uniform + slices)."""
    if b % c:
        raise OracleError("ConfigError", "B not divisible by C")
    return [i * (b // c) for i in range(c + 1)]


def run_batch(arch, kind, H, Y, offsets, n0, es=1.0, symbols=None,
              lama_params=None, items=None):
    """Apply the per-vector reference path to every (item, t).

    H: [n][B][U], Y: [n][T][B] (complex), n0: scalar or per-item array.
    Returns dict of stacked arrays: z [n][T][U], sigma2 [n][T][U],
    nu [n][T][C][U] (FD), dec [n][T][U] (symbol indices).
    """
    n, t_count = Y.shape[0], Y.shape[1]
    items = range(n) if items is None else items
    n0_arr = np.broadcast_to(np.asarray(n0, dtype=float), (H.shape[0],))
    zs, s2s, nus, decs = [], [], [], []
    for i in items:
        zt, st, nt, dt = [], [], [], []
        for t in range(t_count):
            if arch == "fd":
                r = fd_equalize(kind, H[i], Y[i, t], offsets, n0_arr[i], es,
                                symbols, lama_params)
                nt.append(r["nu"])
            else:
                r = pd_equalize(kind, H[i], Y[i, t], offsets, n0_arr[i], es,
                                symbols, lama_params)
            zt.append(r["z"])
            st.append(r["sigma2"])
            if symbols is not None:
                dt.append(hard_detect_index(r["z"], symbols))
        zs.append(zt)
        s2s.append(st)
        nus.append(nt)
        decs.append(dt)
    out = dict(z=np.array(zs), sigma2=np.array(s2s))
    if arch == "fd":
        out["nu"] = np.array(nus)
    if symbols is not None:
        out["dec"] = np.array(decs)
    return out


# --------------------------------------------------------------------------
# vectorized restatement: the same per-vector algorithm, batched over items
# and symbols with NumPy (the reference recomputes G_c for every receive
# vector; G_c depends only on H, so computing it once per item is the same
# arithmetic).  Used for parity at the BASELINE sizes (>= 1e5 symbols); pinned
# to run_batch by tests/test_oracle_vec.py.  Raises on the first failing item
# like the per-vector path, unless strict=False (then status[n] is returned).
# --------------------------------------------------------------------------
def _linear_vec(kind, g, ym, n0, es):
    """linear_equalize (equalize.py:130-176) for G [n][U][U], y_mrc
    [n][T][U], n0 [n]; returns z [n][T][U], sigma2 [n][U], gain [n][U]|None,
    bad [n] (SingularGram)."""
    n, u = g.shape[0], g.shape[-1]
    eye = np.eye(u)
    bad = np.zeros(n, dtype=bool)
    if kind == MRC:
        d = np.real(np.einsum("nii->ni", g)).copy()
        bad |= np.any(d <= 0.0, axis=1)
        d = np.where(d <= 0.0, 1.0, d)
        z = ym / d[:, None, :]
        s2 = n0[:, None] / d + es * np.sum(np.abs(g / d[:, :, None] - eye) ** 2, axis=2)
        return z, s2, None, bad
    if kind == ZF:
        m = g
    elif kind == LMMSE:
        m = g + (n0 / es)[:, None, None] * eye
    else:
        raise OracleError("ConfigError", f"kind {kind}")
    # Cholesky of each item (zpotrf); failures -> SingularGram
    ok = np.ones(n, dtype=bool)
    try:
        l = np.linalg.cholesky(m)
    except np.linalg.LinAlgError:
        l = np.zeros_like(m)
        for i in range(n):
            try:
                l[i] = np.linalg.cholesky(m[i])
            except np.linalg.LinAlgError:
                ok[i] = False
                l[i] = np.eye(u)
    bad |= ~ok
    inv = np.linalg.inv(l)                        # L^-1
    a = np.conj(np.swapaxes(inv, -1, -2)) @ inv    # M^-1 = L^-H L^-1
    z = np.einsum("nij,ntj->nti", a, ym)
    if kind == ZF:
        s2 = n0[:, None] * np.sum(np.abs(inv) ** 2, axis=1)  # diag(G^-1)
        return z, s2, None, bad
    ag = a @ g
    noise = n0[:, None] * np.real(np.sum(ag * a.conj(), axis=2))
    interf = es * np.sum(np.abs(ag - eye) ** 2, axis=2)
    gain = np.real(np.einsum("nii->ni", ag))
    return z, noise + interf, gain, bad


def _check_sigma2_vec(s2):
    neg = np.any(s2 < -VAR_TOL, axis=tuple(range(1, s2.ndim)))
    return np.maximum(s2, 0.0), neg


def _unbias_vec(z, s2, gain, es):
    if gain is None:
        return z, s2, np.zeros(z.shape[0], dtype=bool)
    badg = np.any(gain <= 0, axis=1)
    g = np.where(gain <= 0, 1.0, gain)
    s2u = (s2 - (1.0 - g) ** 2 * es) / g ** 2
    return z / g[:, None, :], s2u, badg


def _posterior_vec(z, tau, symbols):
    """posterior_mean_var (_kernels_py.py:14-28) for z [...], tau [...]."""
    d2 = np.abs(z[..., None] - symbols) ** 2
    d2 = d2 - d2.min(axis=-1, keepdims=True)
    w = np.exp(-d2 / tau[..., None])
    w = w / w.sum(axis=-1, keepdims=True)
    f = w @ symbols
    g = np.maximum(w @ (np.abs(symbols) ** 2) - np.abs(f) ** 2, 0.0)
    return f, g


def _lama_vec(g, ym, symbols, es, n0, beta, t_max=10, damping=1.0):
    """lama_equalize (equalize.py:208-259) for every (item, symbol):
    G [n][U][U], y_mrc [n][T][U], n0 [n] -> z [n][T][U], tau [n][T],
    diverged-at-iteration [n] (0: none)."""
    n, t_count, u = ym.shape
    a = np.eye(u) - g
    s = np.full((n, t_count, u), symbols.mean(), dtype=np.complex128)
    v = np.zeros((n, t_count, u), dtype=np.complex128)
    phi = np.full((n, t_count), float(es))
    div = np.zeros(n, dtype=int)
    z = None
    tau = n0[:, None] + beta * phi
    for it in range(1, t_max + 1):
        tau = n0[:, None] + beta * phi
        z = ym + np.einsum("nij,ntj->nti", a, s) + v
        bad = ~(np.all(np.isfinite(z), axis=2) & (np.max(np.abs(np.nan_to_num(z, nan=np.inf)), axis=2) < 1e150))
        newly = np.any(bad, axis=1) & (div == 0)
        div[newly] = it
        f, gv = _posterior_vec(np.nan_to_num(z), np.maximum(tau, 1e-300)[:, :, None] * np.ones(u), symbols)
        phi_next = np.mean(gv, axis=2)
        v = (beta * phi_next / tau)[:, :, None] * (z - s)
        s = damping * f + (1.0 - damping) * s
        phi = phi_next
    return z, tau, div


def run_batch_vec(arch, kind, H, Y, offsets, n0, es=1.0, symbols=None, lama_params=None, strict=True):
    """run_batch for whole batches: H [n][B][U], Y [n][T][B], n0 scalar or
    [n].  Returns z [n][T][U], sigma2 [n][T][U], nu [n][C][U] (FD; per
    symbol for LAMA: [n][T][C][U]), dec [n][T][U] and status [n] (0 ok,
    1 singular, 2 negative variance, 3 diverged, 4 bad fusion variance)."""
    H = np.asarray(H, dtype=np.complex128)
    Y = np.asarray(Y, dtype=np.complex128)
    n, b, u = H.shape
    t_count = Y.shape[1]
    n0a = np.broadcast_to(np.asarray(n0, dtype=float), (n,)).astype(float)
    lp = dict(lama_params or {})
    t_max, damping = int(lp.get("t_max", 10)), float(lp.get("damping", 1.0))
    symbols = None if symbols is None else np.asarray(symbols, dtype=np.complex128)
    status = np.zeros(n, dtype=int)

    def flag(mask, code):
        status[(status == 0) & mask] = code

    C = len(offsets) - 1
    if arch == "pd":
        g = np.einsum("nbi,nbj->nij", H.conj(), H)
        ym = np.einsum("nbi,ntb->nti", H.conj(), Y)
        if kind == LAMA:
            z, tau, div = _lama_vec(g, ym, symbols, es, n0a, u / b, t_max, damping)
            flag(div > 0, 3)
            s2 = np.broadcast_to(tau[:, :, None], (n, t_count, u))
        else:
            z, s2, gain, bad = _linear_vec(kind, g, ym, n0a, es)
            flag(bad, 1)
            s2, neg = _check_sigma2_vec(s2)
            flag(neg, 2)
            z, s2, badg = _unbias_vec(z, s2, gain, es)
            flag(badg, 1)
            s2, neg = _check_sigma2_vec(s2)
            flag(neg, 2)
            s2 = np.broadcast_to(s2[:, None, :], (n, t_count, u))
        out = dict(z=z, sigma2=np.array(s2))
    else:
        zc, s2c, wc = [], [], []
        for c in range(C):
            sl = slice(offsets[c], offsets[c + 1])
            hc = H[:, sl]
            b_c = hc.shape[1]
            g = np.einsum("nbi,nbj->nij", hc.conj(), hc)
            ym = np.einsum("nbi,ntb->nti", hc.conj(), Y[:, :, sl])
            if kind == LAMA:
                w_c = b_c / b
                z, tau, div = _lama_vec(g / w_c, ym / w_c, symbols, es, n0a / w_c, u / b_c, t_max, damping)
                flag(div > 0, 3)
                s2 = np.broadcast_to(tau[:, :, None], (n, t_count, u))
            else:
                z, s2, gain, bad = _linear_vec(kind, g, ym, n0a, es)
                flag(bad, 1)
                s2, neg = _check_sigma2_vec(s2)
                flag(neg, 2)
                z, s2, badg = _unbias_vec(z, s2, gain, es)
                flag(badg, 1)
                s2, neg = _check_sigma2_vec(s2)
                flag(neg, 2)
                s2 = np.broadcast_to(s2[:, None, :], (n, t_count, u))
            zc.append(z)
            s2c.append(np.array(s2))
            wc.append(np.real(np.einsum("nii->ni", g)) if kind == MRC else None)
        zs = np.stack(zc, axis=2)      # [n][T][C][U]
        s2s = np.stack(s2c, axis=2)    # [n][T][C][U]
        if kind == MRC:
            gains = np.stack(wc, axis=1)[:, None]          # [n][1][C][U]
            nu = gains / gains.sum(axis=2, keepdims=True)
        else:
            flag(np.any(s2s <= 0, axis=(1, 2, 3)), 4)
            inv = 1.0 / np.maximum(s2s, VARIANCE_FLOOR)
            nu = inv / inv.sum(axis=2, keepdims=True)
        z = np.sum(nu * zs, axis=2)
        s2 = 1.0 / np.sum(1.0 / np.maximum(s2s, VARIANCE_FLOOR), axis=2)
        out = dict(z=z, sigma2=s2, nu=np.broadcast_to(nu, zs.shape).copy())
    if symbols is not None:
        out["dec"] = np.argmin(np.abs(out["z"][..., None] - symbols) ** 2, axis=-1)
    out["status"] = status
    if strict and np.any(status):
        i = int(np.flatnonzero(status)[0])
        names = {1: "SingularGramError", 2: "NegativeVarianceError", 3: "DivergenceError", 4: "ConfigError"}
        raise OracleError(names[int(status[i])], f"item {i}")
    return out


# --------------------------------------------------------------------------
# message volumes (model.py:260-280)
# --------------------------------------------------------------------------
def message_volume(u, n_sc, n_sym, c, bytes_per_entry=8):
    """model.py:274-276: PD moves U^2 N_sc + U N_sc N_sym entries per cluster,
    FD moves U N_sc N_sym, consensus sharing twice FD."""
    pd = (u * u * n_sc + u * n_sc * n_sym) * c * bytes_per_entry
    fd = u * n_sc * n_sym * c * bytes_per_entry
    return pd, fd, 2 * fd


# --------------------------------------------------------------------------
# soft outputs (no reference counterpart -- the
# reference stops at hard decisions, equalize.py:262-268).  Unpinned by
# construction: checked against closed forms in tests/test_llr_oracle.py.
# --------------------------------------------------------------------------
def gray_labels(symbols, levels):
    """Binary-reflected Gray code of the real-level index (high bits) and the
    imaginary-level index (low bits) of symbol k = i*L + j."""
    side = len(levels)
    half = int(np.log2(side))
    k = np.arange(len(symbols))
    i, j = k // side, k % side
    return ((i ^ (i >> 1)) << half) | (j ^ (j >> 1))


def bit_llr(x, s2, symbols, levels, exact=False):
    """Bit LLRs log P(b=0|x)/P(b=1|x) of the decoupled channel x = s + CN(0,
    s2), uniform prior, by brute force over all M symbols; bits MSB first.
    ``x`` and ``s2`` broadcast; output [..., 2 log2 L]."""
    x = np.asarray(x, dtype=np.complex128)
    s2 = np.broadcast_to(np.asarray(s2, dtype=float), x.shape)
    labels = gray_labels(symbols, levels)
    nb = 2 * int(np.log2(len(levels)))
    d = np.abs(x[..., None] - np.asarray(symbols)) ** 2 / s2[..., None]
    out = np.empty(x.shape + (nb,))
    for b in range(nb):
        bit = (labels >> (nb - 1 - b)) & 1
        d0, d1 = d[..., bit == 0], d[..., bit == 1]
        m0, m1 = d0.min(-1), d1.min(-1)
        out[..., b] = m1 - m0
        if exact:
            out[..., b] += (np.log(np.exp(m0[..., None] - d0).sum(-1))
                            - np.log(np.exp(m1[..., None] - d1).sum(-1)))
    return out


# --------------------------------------------------------------------------
# Gauss-Hermite quadratures of the large-system analysis (SURVEY.md 8(f)
# rank 4): _kernels.pyx:74-158 / _kernels_py.py:31-77, nodes and weights of
# kernels.gauss_hermite (kernels.py:34-38, scipy's roots_hermite: numpy's
# hermgauss returns NaN at the default PAM order 2048).  Pinned by tests/golden/golden_quad.npz, made by
# running the reference's own kernels (tests/golden/make_golden_quad.py).
# --------------------------------------------------------------------------
def gauss_hermite(order):
    """kernels.py:34-38: nodes/weights for the weight exp(-x^2)."""
    from scipy.special import roots_hermite

    return roots_hermite(order)


def _post_mean_pam(x, levels, sigma2):
    d2 = (x[..., None] - levels) ** 2
    d2 = d2 - d2.min(axis=-1, keepdims=True)
    w = np.exp(-d2 / sigma2)
    return (w @ levels) / w.sum(axis=-1)


def lama_mse_pam(sigma2, levels, order=2048):
    """_kernels.pyx:99-126: twice the 1-D posterior-mean MSE of the PAM set."""
    nodes, weights = gauss_hermite(order)
    levels = np.asarray(levels, dtype=float)
    x = levels[:, None] + np.sqrt(sigma2) * nodes[None, :]  # [a][j]
    f = _post_mean_pam(x, levels, sigma2)
    total = np.sum(weights[None, :] * (f - levels[:, None]) ** 2)
    return 2.0 * total / (levels.size * np.sqrt(np.pi))


def lama_mse(sigma2, symbols, order=32):
    """_kernels.pyx:74-96: 2-D posterior-mean MSE over the symbol set."""
    nodes, weights = gauss_hermite(order)
    symbols = np.asarray(symbols, dtype=np.complex128)
    noise = np.sqrt(sigma2) * (nodes[:, None] + 1j * nodes[None, :])
    w2 = weights[:, None] * weights[None, :]
    total = 0.0
    for s in symbols:
        f, _ = posterior_mean_var((s + noise).ravel(), sigma2, symbols)
        total += float(np.sum(w2.ravel() * np.abs(f - s) ** 2))
    return total / (symbols.size * np.pi)


def mi_awgn(noise_var, symbols, order=32):
    """_kernels.pyx:129-158: mutual information (bits) of the uniform input
    over complex AWGN, log-sum-exp stabilised."""
    nodes, weights = gauss_hermite(order)
    symbols = np.asarray(symbols, dtype=np.complex128)
    noise = (np.sqrt(noise_var) * (nodes[:, None] + 1j * nodes[None, :])).ravel()
    w2 = (weights[:, None] * weights[None, :]).ravel()
    penalty = 0.0
    for a in symbols:
        e = -(np.abs(a - symbols[None, :] + noise[:, None]) ** 2 - (np.abs(noise) ** 2)[:, None]) / noise_var
        emax = e.max(axis=1)
        lse = emax + np.log(np.sum(np.exp(e - emax[:, None]), axis=1))
        penalty += float(np.sum(w2 * lse)) / np.log(2.0)
    return np.log2(symbols.size) - penalty / (symbols.size * np.pi)
