// Per-unit (item or cluster) epilogues that run on the on-chip Gram G and
// matched filter Z: MRC / ZF / L-MMSE (Cholesky + triangular solves), the
// Gram-domain LAMA recursion, FD fusion accumulation.  All CTA-cooperative on
// shared memory; the caller provides __syncthreads() boundaries between
// units.
#pragma once
#include "dbp_device.cuh"

namespace dbp {

// Shared-memory views of one unit's working set (padded leading dims).
struct Work {
  float2* G;     // [UP][LD]  Gram; after Cholesky: upper = L^H, Ld = diag(L)
  float2* Z;     // [TP][LD]  matched filter y_mrc per OFDM symbol
  float2* X;     // [TP][LD]  per-symbol solution / LAMA z
  float2* W;     // [UP][LD]  L^{-1} unit-vector solves (ZF / L-MMSE variances)
  float2* Sv;    // [TP][LD]  LAMA mean s
  float2* Vv;    // [TP][LD]  LAMA Onsager term v
  float2* Fb;    // [TP][LD]  LAMA posterior mean
  float* gb;     // [TP][LD]  LAMA posterior variance
  float* phi;    // [TP]
  float* coef;   // [TP]
  float* Ld;     // [UP]
  float* s2;     // [UP] linear sigma2 (or [TP] for LAMA)
  float* gn;     // [UP] MRC gain d / L-MMSE signal gain c
  float* dg;     // [UP] original diagonal (pivot tolerance)
  uint16_t* pairs;  // lower-triangle pair table (ii<<8 | kk)
  int* flags;    // [0] status, [1] divergence iteration
  int LD;
};

struct EpiArgs {
  int kind, u, T;
  float n0, es;
  float beta, lama_scale, damping;
  int t_max;
  bool unbias;
};

__device__ __forceinline__ void set_status(int* flags, int st) { atomicCAS(flags, 0, st); }

// ---- Cholesky of the leading u x u block, in place (lower triangle read,
// ---- R = L^H written to the strict upper triangle, diag(L) to Ld).
// One __syncthreads per column; the trailing update of column j is spread over
// all threads via the (ii, kk) pair table.
template <int NT>
__device__ void cholesky(const Work& w, int u) {
  const int tid = threadIdx.x;
  const int LD = w.LD;
  // pivot tolerance: fp32 Schur complements of a rank-deficient Gram come out
  // as rounding noise ~eps*G_jj instead of <= 0 (LAPACK zpotrf's criterion in
  // fp64); treat pivots below 8*u*eps*G_jj as singular.
  const float tolf = 8.f * (float)u * FLT_EPSILON;
  for (int j = 0; j < u; ++j) {
    float pj = w.G[j * LD + j].x;
    const bool bad = !(pj > tolf * w.dg[j]);
    if (bad) {
      if (tid == 0) set_status(w.flags, ST_SINGULAR);
      pj = 1.f;
    }
    const float rinv = rsqrtf(pj);
    const float r2 = rinv * rinv;
    const int n = u - j;
    const int np = n * (n + 1) / 2;
    for (int p = tid; p < np; p += NT) {
      const int pr = w.pairs[p];
      const int ii = pr >> 8, kk = pr & 0xff;
      const int i = j + ii, k = j + kk;
      if (kk == 0) {
        if (ii == 0) {
          w.Ld[j] = sqrtf(pj);
        } else {
          const float2 gij = w.G[i * LD + j];
          w.G[j * LD + i] = make_float2(gij.x * rinv, -gij.y * rinv);  // conj(L_ij) = R_ji
        }
      } else {
        const float2 gij = w.G[i * LD + j];
        const float2 gkj = w.G[k * LD + j];
        float2 acc = w.G[i * LD + k];
        // G_ik -= G_ij conj(G_kj) / p_j
        acc.x -= r2 * (gij.x * gkj.x + gij.y * gkj.y);
        acc.y -= r2 * (gij.y * gkj.x - gij.x * gkj.y);
        w.G[i * LD + k] = acc;
      }
    }
    __syncthreads();
  }
}

// Forward substitution L w = b for one right-hand side held in row `row`
// (length u, stride 1).  b_k is read from `b` (may alias row) or is the unit
// vector e_unit (unit >= 0).  Lanes of a warp run the same (k, m) sequence so
// the R reads are broadcasts.
__device__ __forceinline__ float fwd_solve(const Work& w, float2* row, const float2* b, int unit, int u) {
  const int LD = w.LD;
  float norm2 = 0.f;
  for (int k = 0; k < u; ++k) {
    float2 acc = (unit >= 0) ? make_float2(k == unit ? 1.f : 0.f, 0.f) : b[k];
    const float2* rcol = w.G + k;  // R[m][k] = G[m*LD + k], m < k
#pragma unroll 4
    for (int m = 0; m < k; ++m) c_fms_conj(acc, rcol[m * LD], row[m]);  // L_km = conj(R_mk)
    const float2 v = c_scale(acc, 1.f / w.Ld[k]);
    row[k] = v;
    norm2 += c_abs2(v);
  }
  return norm2;
}

// Back substitution L^H x = w in place.
__device__ __forceinline__ void back_solve(const Work& w, float2* row, int u) {
  const int LD = w.LD;
  for (int k = u - 1; k >= 0; --k) {
    float2 acc = row[k];
    const float2* rrow = w.G + k * LD;
#pragma unroll 4
    for (int m = k + 1; m < u; ++m) c_fms(acc, rrow[m], row[m]);
    row[k] = c_scale(acc, 1.f / w.Ld[k]);
  }
}

// ---- linear equalizers on (G, Z) -> X (per symbol), s2, gn --------------
// equalize.py:130-176 (+ unbiased_output :179-195 when a.unbias).
//  MRC : d = Re G_ii; z = y/d; s2 = N0/d + Es sum_{j!=i}|G_ij|^2/d^2
//  ZF  : G = L L^H; z = L^-H L^-1 y; s2 = N0 ||L^-1 e_i||^2 = N0 [G^-1]_ii
//  LMMSE: G + rho I = L L^H; A_ii = ||L^-1 e_i||^2; s2 = N0 A_ii,
//        c = 1 - rho A_ii (= [AG]_ii); unbiased: z/c, s2 = N0 A_ii / c.
template <int NT>
__device__ void linear_unit(const Work& w, const EpiArgs& a) {
  const int tid = threadIdx.x;
  const int u = a.u, T = a.T, LD = w.LD;
  if (a.kind == EQ_MRC) {
    for (int i = tid; i < u; i += NT) {
      const float d = w.G[i * LD + i].x;
      if (!(d > 0.f)) set_status(w.flags, ST_SINGULAR);
      float off = 0.f;
      for (int j = 0; j < u; ++j)
        if (j != i) off += c_abs2(w.G[i * LD + j]);
      const float rd = 1.f / d;
      w.s2[i] = a.n0 * rd + a.es * off * rd * rd;
      w.gn[i] = d;
    }
    __syncthreads();
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      w.X[t * LD + i] = c_scale(w.Z[t * LD + i], 1.f / w.gn[i]);
    }
    __syncthreads();
    return;
  }
  const float rho = (a.kind == EQ_LMMSE) ? a.n0 / a.es : 0.f;
  for (int i = tid; i < u; i += NT) {
    float d = w.G[i * LD + i].x + rho;
    w.G[i * LD + i].x = d;
    w.dg[i] = d;
  }
  __syncthreads();
  cholesky<NT>(w, u);
  // jobs: warp-aligned groups so the RHS warps and the unit-vector warps run
  // uniform loops (no divergence between the two job kinds).
  const int rhs_threads = ((T + 31) / 32) * 32;
  if (tid < T) {
    float2* row = w.X + tid * LD;
    fwd_solve(w, row, w.Z + tid * LD, -1, u);
    back_solve(w, row, u);
  } else if (tid >= rhs_threads && tid < rhs_threads + u) {
    const int i = tid - rhs_threads;
    const float aii = fwd_solve(w, w.W + i * LD, nullptr, i, u);
    if (a.kind == EQ_ZF) {
      w.s2[i] = a.n0 * aii;
    } else {
      const float c = 1.f - rho * aii;
      w.gn[i] = c;
      if (a.unbias) {
        if (!(c > 0.f)) set_status(w.flags, ST_SINGULAR);
        w.s2[i] = a.n0 * aii / c;
      } else {
        w.s2[i] = a.n0 * aii;
      }
    }
  }
  __syncthreads();
  if (a.kind == EQ_LMMSE && a.unbias) {
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      w.X[t * LD + i] = c_scale(w.X[t * LD + i], 1.f / w.gn[i]);
    }
    __syncthreads();
  }
}

// ---- LAMA (equalize.py:208-259) on (G, Z) scaled by lama_scale ----------
// Per OFDM symbol t an independent recursion; state in shared memory.
// Output: X = z^{t_max}, s2[t] = tau^{t_max}.  The last iteration skips the
// denoiser (its F, G only feed discarded updates).
template <int NT>
__device__ void lama_unit(const Work& w, const EpiArgs& a, const ConstParams& cp, float2* tr_z,
                          float2* tr_s, float2* tr_v, float* tr_phi) {
  const int tid = threadIdx.x;
  const int u = a.u, T = a.T, LD = w.LD;
  const float sc = a.lama_scale;
  const float n0 = a.n0 * sc;
  const float beta = a.beta;
  for (int e = tid; e < u * u; e += NT) {
    const int i = e / u, j = e - i * u;
    w.G[i * LD + j] = c_scale(w.G[i * LD + j], sc);
  }
  for (int e = tid; e < T * u; e += NT) {
    const int t = e / u, i = e - t * u;
    w.Z[t * LD + i] = c_scale(w.Z[t * LD + i], sc);
    w.Sv[t * LD + i] = cp.mean;
    w.Vv[t * LD + i] = make_float2(0.f, 0.f);
  }
  for (int t = tid; t < T; t += NT) w.phi[t] = cp.es;
  __syncthreads();
  for (int it = 1; it <= a.t_max; ++it) {
    const bool last = (it == a.t_max);
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      const float2* srow = w.Sv + t * LD;
      const float2* grow = w.G + i * LD;
      // z = y_mrc + (I - G) s + v
      float2 z = c_add(w.Z[t * LD + i], c_add(srow[i], w.Vv[t * LD + i]));
#pragma unroll 4
      for (int j = 0; j < u; ++j) c_fms(z, grow[j], srow[j]);
      if (!c_finite(z) || !(c_abs2(z) < DIVERGE_ABS2)) atomicMin(w.flags + 1, it);
      w.X[t * LD + i] = z;
      const float phi = w.phi[t];
      if (tr_z) {
        const size_t o = ((size_t)(it - 1) * T + t) * u + i;
        tr_z[o] = z;
        tr_s[o] = srow[i];
        tr_v[o] = w.Vv[t * LD + i];
        if (i == 0) tr_phi[(size_t)(it - 1) * T + t] = phi;
      }
      if (!last) {
        float2 F;
        float g;
        posterior(z, n0 + beta * phi, cp, F, g);
        w.Fb[t * LD + i] = F;
        w.gb[t * LD + i] = g;
      }
    }
    __syncthreads();
    if (last) break;
    for (int t = tid; t < T; t += NT) {
      float sum = 0.f;
      for (int i = 0; i < u; ++i) sum += w.gb[t * LD + i];
      const float phin = sum / (float)u;
      const float tau = n0 + beta * w.phi[t];
      w.coef[t] = beta * phin / tau;
      w.phi[t] = phin;
    }
    __syncthreads();
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      const float2 s = w.Sv[t * LD + i];
      w.Vv[t * LD + i] = c_scale(c_sub(w.X[t * LD + i], s), w.coef[t]);
      w.Sv[t * LD + i] = c_add(c_scale(w.Fb[t * LD + i], a.damping), c_scale(s, 1.f - a.damping));
    }
    __syncthreads();
  }
  for (int t = tid; t < T; t += NT) w.s2[t] = n0 + beta * w.phi[t];
  __syncthreads();
}

}  // namespace dbp
