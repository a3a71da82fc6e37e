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
  float2* W;     // scratch: Gauss-Jordan pivot row/column buffers [4][UP]
  float2* Sv;    // [TP][LD]  LAMA mean s
  float2* Vv;    // [TP][LD]  LAMA Onsager term v
  float2* Fb;    // [TP][LD]  LAMA posterior mean
  float* gb;     // [TP][LD]  LAMA posterior variance
  float* phi;    // [TP]
  float* coef;   // [TP]
  float* s2;     // [UP] linear sigma2 (or [TP] for LAMA)
  float* gn;     // [UP] MRC gain d / L-MMSE signal gain c
  float* dg;     // [UP] original diagonal (pivot tolerance)
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

// ---- linear equalizers on (G, Z) -> X (per symbol), s2, gn --------------
// equalize.py:130-176 (+ unbiased_output :179-195 when a.unbias).
//  MRC  : d = Re G_ii; z = y/d; s2 = N0/d + Es sum_{j!=i}|G_ij|^2/d^2
//  ZF   : A = G^-1;            z = A y; s2 = N0 A_ii
//  LMMSE: A = (G + rho I)^-1;  z = A y; s2 = N0 A_ii, c = 1 - rho A_ii
//         (= [AG]_ii); unbiased: z/c, s2 = N0 A_ii / c.
// (The reference's explicit formulas reduce to these identities exactly,
// e.g. N0 rowsum(AG .* conj A) + Es sum|AG - I|^2 = N0 A_ii for rho = N0/Es.)
// The inverse is an in-place Gauss-Jordan sweep without pivoting (stable for
// Hermitian positive definite matrices, like Cholesky): matrix elements stay
// in registers, each step publishes the old pivot row/column through shared
// memory (double-buffered, one __syncthreads per step).  A pivot below
// 8*u*eps of its original diagonal is SingularGramError: the fp32 counterpart
// of zpotrf's "not positive definite" (a rank-deficient fp32 Gram leaves
// rounding noise ~eps*G_jj instead of an exact zero).
template <int UP, int NT>
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
  constexpr int EPT = (UP * UP + NT - 1) / NT;
  float2 m[EPT];
  float2* rowb = w.W;           // [2][UP] pivot rows (double-buffered)
  float2* colb = w.W + 2 * UP;  // [2][UP] pivot columns
  const float tolf = 8.f * (float)u * FLT_EPSILON;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int e = tid + r * NT;
    const int i = e / UP, j = e % UP;
    float2 v = make_float2(0.f, 0.f);
    if (e < UP * UP && i < u && j < u) {
      v = w.G[i * LD + j];
      if (i == j) {
        v.x += rho;
        v.y = 0.f;
        w.dg[i] = v.x;
      }
    }
    m[r] = v;
  }
  for (int k = 0; k < u; ++k) {
    float2* rk = rowb + (k & 1) * UP;
    float2* ck = colb + (k & 1) * UP;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int e = tid + r * NT;
      const int i = e / UP, j = e % UP;
      if (e < UP * UP) {
        if (i == k) rk[j] = m[r];
        if (j == k) ck[i] = m[r];
      }
    }
    __syncthreads();
    float p = rk[k].x;
    if (!(p > tolf * w.dg[k])) {
      if (tid == 0) set_status(w.flags, ST_SINGULAR);
      p = 1.f;
    }
    const float rp = 1.f / p;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int e = tid + r * NT;
      if (e < UP * UP) {
        const int i = e / UP, j = e % UP;
        if (i == k) {
          m[r] = (j == k) ? make_float2(rp, 0.f) : c_scale(m[r], rp);
        } else if (j == k) {
          m[r] = c_scale(m[r], -rp);
        } else {
          c_fms(m[r], c_scale(ck[i], rp), rk[j]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int e = tid + r * NT;
    const int i = e / UP, j = e % UP;
    if (e < UP * UP && i < u && j < u) w.G[i * LD + j] = m[r];
  }
  __syncthreads();
  // z = A y_mrc per OFDM symbol (+ unbiasing), variances from diag(A)
  const bool unb = (a.kind == EQ_LMMSE) && a.unbias;
  for (int e = tid; e < T * u; e += NT) {
    const int t = e / u, i = e - t * u;
    const float2* arow = w.G + i * LD;
    const float2* zrow = w.Z + t * LD;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int j = 0; j < u; ++j) c_fma(acc, arow[j], zrow[j]);
    if (unb) acc = c_scale(acc, 1.f / (1.f - rho * arow[i].x));
    w.X[t * LD + i] = acc;
  }
  for (int i = tid; i < u; i += NT) {
    const float aii = w.G[i * LD + i].x;
    if (a.kind == EQ_ZF) {
      w.s2[i] = a.n0 * aii;
    } else {
      const float c = 1.f - rho * aii;
      w.gn[i] = c;
      if (a.unbias && !(c > 0.f)) set_status(w.flags, ST_SINGULAR);
      w.s2[i] = a.unbias ? a.n0 * aii / c : a.n0 * aii;
    }
  }
  __syncthreads();
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
