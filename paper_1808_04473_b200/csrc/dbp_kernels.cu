// libdbp_b200: sm_100a kernels for decentralized feedforward equalization
// (arXiv 1808.04473) behind the C ABI of include/dbp_b200.h.
//
// Hot path = one persistent kernel per (arch, U) that streams each item's
// channel block H[n] (B x U) and receive block Y[n] (T x B) through
// shared-memory stages filled by the TMA bulk-copy engine, forms the Gram and
// the matched filter of all T symbols on the tensor cores (tcgen05, 3xTF32,
// TMEM accumulators; dbp_tc.cuh) -- or on FP32 SIMT for U = 64
// (dbp_simt.cuh) -- and runs the equalizer, FD fusion and the QAM slicer on
// chip (dbp_epilogue.cuh).  Only estimates, variances, weights and decisions
// are written back to HBM.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>

#include "../../include/dbp_b200.h"
#include "dbp_device.cuh"
#include "dbp_epilogue.cuh"
#include "dbp_host.h"
#include "dbp_synth.cuh"

namespace dbp {

// FD finalize from summed partials (multi-GPU).
__global__ void fd_finalize_kernel(const float* __restrict__ acc, int64_t n_items, int u, int T, int wdim,
                                   const __grid_constant__ ConstParams cp, float2* xhat, float* sigma2,
                                   uint8_t* dec) {
  const int rec = 2 * T * u + 2 * wdim;
  const int64_t total = n_items * T * u;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / (T * u);
    const int r = (int)(e - n * T * u);
    const int t = r / u, i = r - t * u;
    const float* a = acc + n * rec;
    const float d = a[2 * T * u + ((wdim == u) ? i : t)];
    const float2 x = make_float2(a[2 * r] / d, a[2 * r + 1] / d);
    xhat[e] = x;
    if (dec) dec[e] = (uint8_t)slice_symbol(x, cp);
    if (r < wdim) sigma2[n * wdim + r] = 1.f / a[2 * T * u + wdim + r];
  }
}

__global__ void fd_weights_kernel(const float* __restrict__ wraw, const float* __restrict__ den, int64_t n_items,
                                  int C, int wdim, float* nu) {
  const int64_t total = n_items * C * wdim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / (C * wdim);
    const int k = (int)(e % wdim);
    nu[e] = wraw[e] / den[n * wdim + k];
  }
}

__global__ void posterior_kernel(const float2* __restrict__ z, int64_t n, float tau,
                                 const __grid_constant__ ConstParams cp, float2* f, float* g) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float2 F;
    float G;
    posterior(z[e], tau, cp, F, G);
    f[e] = F;
    g[e] = G;
  }
}

__global__ void hard_detect_kernel(const float2* __restrict__ z, int64_t n, const __grid_constant__ ConstParams cp,
                                   int32_t* idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    idx[e] = slice_symbol(z[e], cp);
}



// Gray-labelled bit LLRs from (x-hat, sigma2) (the
// reference stops at symbol decisions).  Decoupled model x = s + e,
// e ~ CN(0, s2); symbol k = i L + j with label (gray(i) << h) | gray(j),
// h = log2 L, bits MSB first.  Per dimension (the labels factorise):
// LLR_b = log sum_{a: bit 0} exp(-(v-a)^2/s2) - log sum_{a: bit 1} exp(..)
// (exact) or its max-log form (min_{bit 1} - min_{bit 0}) / s2.
//
// One thread per symbol, H = log2 L a template parameter so the level and bit
// loops fully unroll; the CTA's 256 x 2H LLRs are staged in shared memory and
// written back as coalesced float4 rows (a thread's own 2H floats sit at a
// 8-24 B stride, which scalar stores would scatter over 2H sectors per warp
// instruction).  Exact mode shares one exp2 per level (relative to the
// dimension's nearest level) across the H bits and falls back to
// group-relative sums only where the far group's terms would underflow.
constexpr int LLR_THREADS = 256;

template <int H>
__global__ void __launch_bounds__(LLR_THREADS) llr_kernel(const float2* __restrict__ x, const float* __restrict__ s2,
                                                          int64_t n_el, int T, int u, int s2_per_symbol,
                                                          const __grid_constant__ ConstParams cp, int exact,
                                                          float* __restrict__ llr) {
  constexpr int L = 1 << H, NB = 2 * H;
  constexpr float LOG2E = 1.4426950408889634f, LN2 = 0.6931471805599453f;
  __shared__ __align__(16) float tile[LLR_THREADS * NB];
  float lev[L];
#pragma unroll
  for (int l = 0; l < L; ++l) lev[l] = cp.levels[l];
  const uint32_t TU = (uint32_t)(T * u);
  const bool small = n_el <= 0xffffffffll;
  for (int64_t e0 = (int64_t)blockIdx.x * LLR_THREADS; e0 < n_el; e0 += (int64_t)gridDim.x * LLR_THREADS) {
    const int64_t e = e0 + threadIdx.x;
    if (e < n_el) {
      int64_t sidx;
      if (s2_per_symbol) {  // [n][T]: item * T + t = e / u
        sidx = small ? (int64_t)((uint32_t)e / (uint32_t)u) : e / u;
      } else {  // [n][u]: item * u + e % u
        const int64_t item = small ? (int64_t)((uint32_t)e / TU) : e / (int64_t)TU;
        const uint32_t i = small ? (uint32_t)e % (uint32_t)u : (uint32_t)(e % u);
        sidx = item * u + i;
      }
      // distances in log2 units: d_l = (v - a_l)^2 / s2 * log2(e)
      const float inv = LOG2E / fmaxf(__ldg(s2 + sidx), FLT_MIN);
      const float2 z = x[e];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const float v = d ? z.y : z.x;
        float dist[L], dmin = FLT_MAX;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const float q = v - lev[l];
          dist[l] = q * q * inv;
          dmin = fminf(dmin, dist[l]);
        }
        float w[L];
        if (exact) {
#pragma unroll
          for (int l = 0; l < L; ++l) w[l] = exp2f(dmin - dist[l]);
        }
#pragma unroll
        for (int b = 0; b < H; ++b) {  // bit H-1-b of gray(l), MSB first
          const int sh = H - 1 - b;
          float m0 = FLT_MAX, m1 = FLT_MAX, s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int l = 0; l < L; ++l) {
            if (((l ^ (l >> 1)) >> sh) & 1) {
              m1 = fminf(m1, dist[l]);
              if (exact) s1 += w[l];
            } else {
              m0 = fminf(m0, dist[l]);
              if (exact) s0 += w[l];
            }
          }
          float r = m1 - m0;  // max-log, log2 units
          if (exact) {
            // log2 sum_{g} 2^(dmin - d) = (dmin - m_g) + log2 sum_g 2^(m_g - d);
            // the far group's shared sum underflows once m_g - dmin > ~100:
            // recompute it relative to its own minimum there
            if (fmaxf(m0, m1) - dmin > 100.f) {
              const int far = m1 > m0;
              const float mf = far ? m1 : m0;
              float sf = 0.f;
#pragma unroll
              for (int l = 0; l < L; ++l)
                if (((((l ^ (l >> 1)) >> sh) & 1) == far)) sf += exp2f(mf - dist[l]);
              // LLR = log2 s0' - log2 s1' + (m1 - m0) with s_g' group-relative
              const float sn = far ? s0 : s1;  // near group, relative to dmin = its min
              r += far ? (__log2f(sn) - __log2f(sf)) : (__log2f(sf) - __log2f(sn));
            } else {
              r = __log2f(s0) - __log2f(s1);
            }
          }
          tile[threadIdx.x * NB + d * H + b] = r * LN2;
        }
      }
    }
    __syncthreads();
    const int64_t cnt = min((int64_t)LLR_THREADS, n_el - e0) * NB;  // floats in this tile
    float* dst = llr + e0 * NB;
    if (cnt == LLR_THREADS * NB) {
      const float4* src4 = reinterpret_cast<const float4*>(tile);
      float4* dst4 = reinterpret_cast<float4*>(dst);
      for (int q = threadIdx.x; q < LLR_THREADS * NB / 4; q += LLR_THREADS) dst4[q] = src4[q];
    } else {
      for (int q = threadIdx.x; q < cnt; q += LLR_THREADS) dst[q] = tile[q];
    }
    __syncthreads();
  }
}

// Gray bits of hard decisions (the north star's "hard decisions as indices
// plus Gray bits"): symbol index k = i L + j -> label (gray(i) << h) | gray(j),
// h = log2 L, written MSB first as one byte per bit, bits [n][2h].  Indices
// outside [0, L^2) (never produced by the slicers) give all-ones rows.
template <typename IDX>
__global__ void gray_bits_kernel(const IDX* __restrict__ idx, int64_t n, int h, uint8_t* __restrict__ bits) {
  const int L = 1 << h, nb = 2 * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)idx[e];
    const bool ok = k >= 0 && k < L * L;
    const int i = k >> h, j = k & (L - 1);
    const int label = ok ? (((i ^ (i >> 1)) << h) | (j ^ (j >> 1))) : (1 << nb) - 1;
    uint8_t* o = bits + e * nb;
    for (int b = 0; b < nb; ++b) o[b] = (uint8_t)((label >> (nb - 1 - b)) & 1);
  }
}

// Gauss-Hermite quadratures of the large-system analysis (SURVEY.md 8(f)
// rank 4; _kernels.pyx:74-158), fp64 like the reference: one CTA per
// evaluation point, the (symbol, node[, node]) terms strided over its
// threads, a fixed-order tree reduction (deterministic).
//   QK_MSE_PAM: 2/(L sqrt(pi)) sum_a sum_j w_j (F(a + s n_j) - a)^2
//   QK_MSE_2D : 1/(M pi) sum_s sum_jk w_j w_k |F(s + s(n_j + i n_k)) - s|^2
//   QK_MI     : log2 M - 1/(M pi ln 2) sum_a sum_jk w_j w_k lse_b(e_b)
// F = posterior mean of the uniform prior at noise variance x (= sigma^2).
enum { QK_MSE_PAM = 0, QK_MSE_2D = 1, QK_MI = 2 };
struct QuadSet {
  int M;  // symbols (2-D kinds) or levels (PAM)
  double re[MAX_SYMS], im[MAX_SYMS];
};
constexpr int QUAD_THREADS = 256;

// One quadrature sum at x, reduced over the CTA (fixed-order tree:
// deterministic); every thread returns the total.  red: QUAD_THREADS doubles.
__device__ double quad_sum(int kind, double x, const QuadSet& qs, const double* __restrict__ nodes,
                           const double* __restrict__ weights, int q, double* red) {
  const double sigma = sqrt(x);
  const int M = qs.M;
  double acc = 0.0;
  if (kind == QK_MSE_PAM) {
    for (int t = threadIdx.x; t < M * q; t += QUAD_THREADS) {
      const int a = t / q, j = t - a * q;
      const double v = qs.re[a] + sigma * nodes[j];
      double dmin = 1e300;
      for (int k = 0; k < M; ++k) {
        const double d = v - qs.re[k];
        dmin = fmin(dmin, d * d);
      }
      double ws = 0.0, f = 0.0;
      for (int k = 0; k < M; ++k) {
        const double d = v - qs.re[k];
        const double w = exp(-(d * d - dmin) / x);
        ws += w;
        f += w * qs.re[k];
      }
      f /= ws;
      acc += weights[j] * (f - qs.re[a]) * (f - qs.re[a]);
    }
  } else {
    for (int t = threadIdx.x; t < M * q * q; t += QUAD_THREADS) {
      const int a = t / (q * q), r = t - a * q * q, j = r / q, k = r - j * q;
      const double nr = sigma * nodes[j], ni = sigma * nodes[k];
      const double wjk = weights[j] * weights[k];
      if (kind == QK_MSE_2D) {
        const double zr = qs.re[a] + nr, zi = qs.im[a] + ni;
        double dmin = 1e300;
        for (int b = 0; b < M; ++b) {
          const double dr = zr - qs.re[b], di = zi - qs.im[b];
          dmin = fmin(dmin, dr * dr + di * di);
        }
        double ws = 0.0, fr = 0.0, fi = 0.0;
        for (int b = 0; b < M; ++b) {
          const double dr = zr - qs.re[b], di = zi - qs.im[b];
          const double w = exp(-((dr * dr + di * di) - dmin) / x);
          ws += w;
          fr += w * qs.re[b];
          fi += w * qs.im[b];
        }
        const double er = fr / ws - qs.re[a], ei = fi / ws - qs.im[a];
        acc += wjk * (er * er + ei * ei);
      } else {  // QK_MI
        const double n2 = nr * nr + ni * ni;
        double emax = -1e300;
        for (int b = 0; b < M; ++b) {
          const double dr = qs.re[a] - qs.re[b] + nr, di = qs.im[a] - qs.im[b] + ni;
          emax = fmax(emax, -((dr * dr + di * di) - n2) / x);
        }
        double lse = 0.0;
        for (int b = 0; b < M; ++b) {
          const double dr = qs.re[a] - qs.re[b] + nr, di = qs.im[a] - qs.im[b] + ni;
          lse += exp(-((dr * dr + di * di) - n2) / x - emax);
        }
        acc += wjk * (emax + log(lse));
      }
    }
  }
  __syncthreads();  // red may still be read from the previous call
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = QUAD_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double pi = 3.141592653589793, tot = red[0];
  if (kind == QK_MSE_PAM) return 2.0 * tot / (M * sqrt(pi));
  if (kind == QK_MSE_2D) return tot / (M * pi);
  return log2((double)M) - tot / (M * pi * log(2.0));
}

__global__ void __launch_bounds__(QUAD_THREADS) quad_kernel(int kind, const double* __restrict__ xs,
                                                            const __grid_constant__ QuadSet qs,
                                                            const double* __restrict__ nodes,
                                                            const double* __restrict__ weights, int q,
                                                            double* __restrict__ out) {
  __shared__ double red[QUAD_THREADS];
  const double r = quad_sum(kind, xs[blockIdx.x], qs, nodes, weights, q, red);
  if (threadIdx.x == 0) out[blockIdx.x] = r;
}

// Batched state evolution of the message-passing equalizer (the decoupled
// fixed point w sigma2 = N0 + beta Psi(sigma2) of the large-system analysis,
// /root/reference/pkg/src/dbp/asymptotics.py:75-129): one CTA per point
// iterates sigma2 <- (N0 + beta Psi(sigma2)) / w from its start value, the
// MSE Psi by the quadrature above, until |new - old| <= tol * old, entirely
// on the GPU (a whole SNR x beta x cluster grid is one launch).  Started at
// (N0 + beta Es) / w the orbit decreases onto the largest fixed point; from
// just above the noise floor it finds the smallest.  iters[p] = iterations
// taken, negative when max_iter was reached without convergence.
__global__ void __launch_bounds__(QUAD_THREADS) fixed_point_kernel(
    int kind, const double* __restrict__ n0, const double* __restrict__ beta, const double* __restrict__ w,
    const double* __restrict__ start, const __grid_constant__ QuadSet qs, const double* __restrict__ nodes,
    const double* __restrict__ weights, int q, double tol, int max_iter, double* __restrict__ sigma2,
    int* __restrict__ iters) {
  __shared__ double red[QUAD_THREADS];
  const int p = blockIdx.x;
  const double a = n0[p], b = beta[p], c = w[p];
  double s = start[p];
  int it = 1;
  for (;; ++it) {
    const double nxt = (a + b * quad_sum(kind, s, qs, nodes, weights, q, red)) / c;
    const bool done = fabs(nxt - s) <= tol * s;
    s = nxt;
    if (done) break;
    if (it == max_iter) {
      it = -it;
      break;
    }
  }
  if (threadIdx.x == 0) {
    sigma2[p] = s;
    iters[p] = it;
  }
}

// ---- small element-wise kernels behind the per-vector drop-in API --------
// fuse_partials (equalize.py:96-107): out = sum_p parts[p]
__global__ void stats_sum_kernel(const float2* __restrict__ parts, int P, int64_t count, float2* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    float2 s = parts[e];
    for (int q = 1; q < P; ++q) s = c_add(s, parts[(int64_t)q * count + e]);
    out[e] = s;
  }
}

// unbiased_output (equalize.py:179-195): z/c, (s2 - (1-c)^2 Es)/c^2, guard
// c <= 0 (SingularGram) and s2 < -1e-9 (NegativeVariance), clamp at 0.
__global__ void unbias_kernel(const float2* __restrict__ z, const float* __restrict__ s2,
                              const float* __restrict__ gain, int64_t n, int T, int u, float es, float2* z_out,
                              float* s2_out, int32_t* status) {
  const int64_t total = n * T * u;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = e / ((int64_t)T * u);
    const int r = (int)(e - item * T * u);
    const int t = r / u, i = r - t * u;
    const float c = gain[item * u + i];
    if (!(c > 0.f)) atomicCAS(status + item, 0, ST_SINGULAR);
    z_out[e] = c_scale(z[e], 1.f / c);
    if (t == 0) {
      const float d = 1.f - c, a = s2[item * u + i], b = d * d * es;
      const float v = (a - b) / (c * c);
      // _VAR_TOL = 1e-9 (equalize.py:24) plus the fp32 rounding level of the
      // difference, so rounding-level negatives clamp instead of raising
      const float tol = 1e-9f + 4.f * FLT_EPSILON * (fabsf(a) + b) / (c * c);
      if (v < -tol) atomicCAS(status + item, 0, ST_NEGVAR);
      s2_out[item * u + i] = fmaxf(v, 0.f);
    }
  }
}

// optimal_fusion_weights (fusion.py:96-105) over s2 [n][C][u].
__global__ void fusion_weights_kernel(const float* __restrict__ s2, int64_t n, int C, int u, float* nu,
                                      int32_t* status) {
  const int64_t total = n * u;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = e / u;
    const int i = (int)(e - item * u);
    float den = 0.f;
    for (int c = 0; c < C; ++c) {
      const float v = s2[(item * C + c) * u + i];
      if (!(v > 0.f)) atomicCAS(status + item, 0, ST_BADVAR);
      den += 1.f / fmaxf(v, VAR_FLOOR);
    }
    for (int c = 0; c < C; ++c)
      nu[(item * C + c) * u + i] = (1.f / fmaxf(s2[(item * C + c) * u + i], VAR_FLOOR)) / den;
  }
}

// fuse_estimates (fusion.py:108-124) over z/s2/nu [C][rows][u].
__global__ void fuse_estimates_kernel(const float2* __restrict__ z, const float* __restrict__ s2,
                                      const float* __restrict__ nu, int C, int64_t count, float2* z_out,
                                      float* s2_out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    float h = 0.f;
    for (int c = 0; c < C; ++c) {
      const int64_t o = (int64_t)c * count + e;
      acc = c_add(acc, c_scale(z[o], nu[o]));
      h += 1.f / fmaxf(s2[o], VAR_FLOOR);
    }
    z_out[e] = acc;
    s2_out[e] = 1.f / h;
  }
}

}  // namespace dbp

// ============================================================================
// C ABI
// ============================================================================
using namespace dbp;

static thread_local std::string g_err;
thread_local int g_last_kernel = 0;  // dbp_last_kernel()

// Process-wide kernel-selection / staging options (dbp_set_option): explicit
// calls, never the environment, so a stray variable cannot change what the
// library computes.  0 = automatic everywhere.
static std::atomic<int> g_opt[DBP_OPT_COUNT];

namespace dbp {
int opt(int key) { return g_opt[key].load(std::memory_order_relaxed); }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DBP_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return DBP_OK;
}

int sm_count() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// Per-(device, stream) device scratch (FD fold records, U = 64 statistics),
// grown on demand.  Launches on one stream are ordered, so they may share it;
// other streams (and other devices) get their own.  Growth is stream-ordered
// (cudaFreeAsync of the old buffer, cudaMallocAsync of the new one on the same
// stream): no host synchronisation inside a launch, capturable in a CUDA
// graph.  The table is guarded by a mutex (calls are reentrant).
void* stream_scratch(cudaStream_t st, size_t need) {
  struct Entry {
    int dev;
    cudaStream_t st;
    void* ptr;
    size_t bytes;
  };
  static std::mutex mu;
  static Entry tab[64];
  static int used = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  Entry* e = nullptr;
  for (int i = 0; i < used; ++i)
    if (tab[i].st == st && tab[i].dev == dev) e = &tab[i];
  if (!e) {
    if (used == 64) return nullptr;
    e = &tab[used++];
    *e = Entry{dev, st, nullptr, 0};
  }
  if (need > e->bytes) {
    if (e->ptr) cudaFreeAsync(e->ptr, st);  // freed after the work already queued on st
    e->ptr = nullptr;
    e->bytes = 0;
    need = std::max(need, (size_t)1 << 20);
    if (cudaMallocAsync(&e->ptr, need, st) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    e->bytes = need;
  }
  return e->ptr;
}

}  // namespace dbp

static int up_for(int u) { return u <= 8 ? 8 : u <= 16 ? 16 : u <= 32 ? 32 : u <= 64 ? 64 : -1; }

static int fill_const(ConstParams& cp, const float* levels, int L, const float* symbols, int M, float es) {
  memset(&cp, 0, sizeof(cp));
  if (L < 0 || L > MAX_L || M < 0 || M > MAX_SYMS) return fail(DBP_E_ARG, "constellation too large");
  cp.L = L;
  cp.M = M;
  cp.es = es;
  for (int l = 0; l < L; ++l) {
    cp.levels[l] = levels[l];
    cp.lv2[l] = make_float2(levels[l], levels[l]);
    cp.lq2[l] = make_float2(levels[l] * levels[l], levels[l] * levels[l]);
  }
  for (int l = 0; l + 1 < L; ++l) cp.mids[l] = 0.5f * (levels[l] + levels[l + 1]);
  double mr = 0, mi = 0, e2 = 0;
  for (int k = 0; k < M; ++k) {
    cp.syms[k] = make_float2(symbols[2 * k], symbols[2 * k + 1]);
    mr += symbols[2 * k];
    mi += symbols[2 * k + 1];
    e2 += (double)symbols[2 * k] * symbols[2 * k] + (double)symbols[2 * k + 1] * symbols[2 * k + 1];
  }
  if (M > 0) cp.mean = make_float2((float)(mr / M), (float)(mi / M));
  if (M == 0 && L == 0) return fail(DBP_E_ARG, "empty constellation");
  return DBP_OK;
}

// U <= 32 -> tensor-core kernel; U = 64 -> SIMT kernel (2(U+T) > 128).
// DBP_FORCE_SIMT=1 selects the SIMT kernel for every U (A/B measurements).
static int dispatch_stats(EqParams& p, cudaStream_t st);

// FD through per-cluster statistics: {G_c, y_c} on the tensor cores (up = 64:
// wide split-bf16 kernel, 3 parts -- the per-cluster Grams of B_c = U antennas
// are ill-conditioned; up = 32: the 3xTF32 kernel), then per item the cluster
// solves / LAMA recursions and their fusion in stats_kernel.
// In chunks of items: the per-cluster records are as large as the input.
// Returns 1 when the geometry is not covered.
static int fd_wide(EqParams& p, cudaStream_t st, int up = 64) {
  const size_t rec = (size_t)p.u * p.u + (size_t)p.T * p.u;
  const size_t per_item = (size_t)p.C * rec * sizeof(float2);
  int64_t chunk = std::max<int64_t>(1, (int64_t)(((size_t)3 << 30) / per_item));  // ~3 GB of records
  if (opt(DBP_OPT_WIDE_CHUNK) > 0) chunk = opt(DBP_OPT_WIDE_CHUNK);                 // tests
  if (p.n0_dev) chunk = std::max<int64_t>(1, chunk / p.n0_group) * p.n0_group;  // n0 runs stay whole
  chunk = std::min<int64_t>(chunk, p.n_items);
  float2* stats = static_cast<float2*>(stream_scratch(st, (size_t)chunk * per_item));
  if (!stats) return fail(DBP_E_CUDA, "statistics scratch allocation failed");
  const int u = p.u, T = p.T;
  for (int64_t i0 = 0; i0 < p.n_items; i0 += chunk) {
    const int64_t len = std::min<int64_t>(chunk, p.n_items - i0);
    EqParams q = p;
    q.n_items = len;
    q.H = p.H + (size_t)i0 * p.B * p.us;
    q.Y = p.Y + (size_t)i0 * T * p.B;
    q.xhat = p.xhat + (size_t)i0 * T * u;
    if (p.dec) q.dec = p.dec + (size_t)i0 * T * u;
    const int wdim = p.kind == EQ_LAMA ? T : u;  // LAMA: sigma2 [n][T], nu [n][C][T]
    q.sigma2 = p.sigma2 + (size_t)i0 * wdim;
    if (p.nu) q.nu = p.nu + (size_t)i0 * p.C * wdim;
    if (p.gain) q.gain = p.gain + (size_t)i0 * u;
    q.status = p.status + i0;
    if (p.iters) q.iters = p.iters + i0;
    if (p.n0_dev) q.n0_dev = p.n0_dev + i0 / p.n0_group;
    EqParams s = q;
    s.arch = ARCH_STATS;
    s.sum_clusters = 0;
    s.stats_out = stats;
    // up = 32 (FD LAMA): the 3xTF32 kernel -- per-cluster units of 32 antennas
    // are one stage each, where the wide split-bf16 kernel measured slower
    // (cfg4-fd 8.85 -> 10.76 ms)
    int rc = up == 64 ? launch_tcw(s, st, 3) : launch_tc_up(up, s, st);
    g_last_kernel = up == 64 ? DBP_KERNEL_TC_BF16 : DBP_KERNEL_TC_TF32;
    if (rc) return rc;  // 1: geometry not covered (the same for every chunk)
    q.stats_in = stats;
    rc = launch_lama(q, st);  // LAMA (u <= 32): the register-resident recursion kernel
    if (rc == 1) rc = launch_stats_up(up, q, st);
    if (rc) return rc;
  }
  return 0;
}

static int dispatch_stream(EqParams& p, cudaStream_t st) {
  p.g_hermitian = 1;  // the streaming kernels build G themselves (full Hermitian matrix)
  const int pol = opt(DBP_OPT_KERNEL);
  const bool force_simt = pol == DBP_KERNEL_SIMT;
  const int up = up_for(p.u);
  // U <= 16 linear / statistics: the split-bf16 tensor-core kernel
  if ((pol == DBP_KERNEL_AUTO || pol == DBP_KERNEL_TC_BF16) && up <= 16) {
    const int rc = launch_tc2(p, st);
    if (rc == 0) g_last_kernel = DBP_KERNEL_TC_BF16;
    if (rc <= 0) return rc;  // launched (0) or failed (< 0); 1 = not covered
    if (pol == DBP_KERNEL_TC_BF16) return fail(DBP_E_UNSUPPORTED, "geometry not covered by the split-bf16 kernel");
  }
  const bool force_tc = pol == DBP_KERNEL_TC_TF32;
  // the tf32 tensor-core kernel solves one unit per warp: LAMA (10 iterations
  // over T x U state) and FD-MRC (trivial solves, fold-bound) run faster on
  // the CTA-cooperative epilogue of the SIMT kernel (measured, round 1)
  const bool fdk = (p.arch == ARCH_FD || p.arch == ARCH_FD_PARTIAL);
  const bool tc_ok = force_tc || (p.kind != EQ_LAMA && !(fdk && p.kind == EQ_MRC));
  if (!force_simt && up <= 32 && tc_ok) {
    int rc = 1;
    rc = launch_tc_up(up, p, st);
    if (rc == 0) g_last_kernel = DBP_KERNEL_TC_TF32;
    if (rc <= 0) return rc;  // launched (0) or failed (< 0); 1 = use the SIMT kernel
    p.NS = up <= 16 ? 4 : 3;
  }
  // PD LAMA, 16 < u <= 32: the fused statistics on the tensor cores (3xTF32
  // kernel), then the recursions in stats_kernel from them (the SIMT kernel's
  // Gram mainloop was half of the step: cfg4-pd 3.72 -> 3.05 ms).  (FD LAMA
  // the same way, per-cluster records through fd_wide, measured no faster:
  // its step is the recursions.)
  if (!force_simt && up == 32 && p.arch == ARCH_PD && p.kind == EQ_LAMA && !opt(DBP_OPT_NO_WIDE) &&
      !p.tr_z) {
    EqParams q = p;
    q.arch = ARCH_STATS;
    q.sum_clusters = 1;
    const size_t rec = (size_t)p.u * p.u + (size_t)p.T * p.u;
    q.stats_out = static_cast<float2*>(stream_scratch(st, (size_t)p.n_items * rec * sizeof(float2)));
    if (!q.stats_out) return fail(DBP_E_CUDA, "statistics scratch allocation failed");
    // split-bf16 statistics (wide kernel, half of M = 128 used), three parts:
    // cfg4-pd 1.99 -> 1.66 ms against the 3xTF32 kernel (two parts: 1.54 ms,
    // but x-hat 7.7e-6 and decision flips at 8.7e-6 of the symbols, too close
    // to the 1e-5 bar)
    int kid = DBP_KERNEL_TC_BF16;
    int rc = pol != DBP_KERNEL_TC_TF32 ? launch_tcw(q, st, 3) : 1;
    if (rc == 1) {
      kid = DBP_KERNEL_TC_TF32;
      rc = launch_tc_up(32, q, st);
    }
    if (rc < 0) return rc;
    if (rc == 0) {
      g_last_kernel = kid;
      EqParams r = p;
      r.stats_in = q.stats_out;
      r.C = 1;
      const int rl = launch_lama(r, st);
      if (rl <= 0) return rl;
      return launch_stats_up(32, r, st);
    }
  }
  // FD LAMA, 16 < u <= 32: per-cluster statistics on the tensor cores, then
  // the recursions and their fusion in lama_kernel (G in registers)
  if (!force_simt && up == 32 && p.arch == ARCH_FD && p.kind == EQ_LAMA && !opt(DBP_OPT_NO_WIDE) && !p.tr_z &&
      opt(DBP_OPT_LAMA_KERNEL) != 1) {
    const int rc = fd_wide(p, st, 32);  // sets g_last_kernel (the statistics kernel)
    if (rc <= 0) return rc;
  }
  if (!force_simt && up == 64 && p.arch == ARCH_FD && p.kind != EQ_LAMA && !opt(DBP_OPT_NO_WIDE) &&
      pol != DBP_KERNEL_TC_TF32) {
    const int rc = fd_wide(p, st);
    if (rc == 0) g_last_kernel = DBP_KERNEL_TC_BF16;
    if (rc <= 0) return rc;
  }
  // U = 64: statistics {G, y_mrc} on the tensor cores (wide layout); PD
  // linear equalization then runs its solves in stats_kernel on them.  Not
  // FD: its per-cluster Grams (B_c = U = 64 at cfg5) are ill-conditioned, and
  // 3xTF32 (no lo.lo term) left FD-ZF 5e-3 from the float64 reference where
  // the FP32 SIMT Gram stays at 2e-4 (cfg5a, measured), for a 2 % gain.
  const bool wide_ok = !force_simt && up == 64 && !opt(DBP_OPT_NO_WIDE) &&
                       (p.arch == ARCH_STATS || (p.arch == ARCH_PD && p.kind != EQ_LAMA));
  if (wide_ok) {
    if (p.arch == ARCH_STATS) {
      if (pol != DBP_KERNEL_TC_TF32) {  // split-bf16 wide statistics kernel first
        const int rc = launch_tcw(p, st);
        if (rc == 0) g_last_kernel = DBP_KERNEL_TC_BF16;
        if (rc <= 0) return rc;
      }
      const int rc = launch_tc_up(64, p, st);
      if (rc == 0) g_last_kernel = DBP_KERNEL_TC_TF32;
      if (rc <= 0) return rc;
    } else {
      EqParams q = p;
      q.arch = ARCH_STATS;
      q.sum_clusters = 1;
      const size_t rec = (size_t)p.u * p.u + (size_t)p.T * p.u;
      q.stats_out = static_cast<float2*>(stream_scratch(st, (size_t)p.n_items * rec * sizeof(float2)));
      if (!q.stats_out) return fail(DBP_E_CUDA, "statistics scratch allocation failed");
      int kid = DBP_KERNEL_TC_BF16;
      // two bf16 parts for well-conditioned systems (B >= 4 u), else three (see launch_tc2)
      int rc = pol != DBP_KERNEL_TC_TF32 ? launch_tcw(q, st, p.B >= 4 * p.u ? 2 : 3) : 1;
      if (rc == 1) {
        kid = DBP_KERNEL_TC_TF32;
        rc = launch_tc_up(64, q, st);
      }
      if (rc < 0) return rc;
      if (rc == 0) {
        g_last_kernel = kid;
        EqParams r = p;
        r.stats_in = q.stats_out;
        r.C = 1;
        return dispatch_stats(r, st);
      }
    }
    p.NS = 3;
  }
  g_last_kernel = DBP_KERNEL_SIMT;
  return launch_stream_up(up, p, st);
}

static int dispatch_stats(EqParams& p, cudaStream_t st) {
  int rc = launch_t2_stats_solve(p, st);  // u <= 16 ZF / L-MMSE: warp-pair solver
  if (rc <= 0) return rc;
  if (up_for(p.u) == 32) {  // LAMA, 16 < u <= 32: register-resident recursion kernel
    rc = launch_lama(p, st);
    if (rc <= 0) return rc;
  }
  return launch_stats_up(up_for(p.u), p, st);
}

// Build the per-item chunk schedule: clusters in order, <= KC rows each.
static int build_chunks(EqParams& p, int C, const int32_t* offsets) {
  if (C < 1 || C > MAX_C) return fail(DBP_E_ARG, "C must be in [1, 16]");
  if (offsets[0] != 0 || offsets[C] != p.B) return fail(DBP_E_ARG, "cluster offsets must span [0, B]");
  int nc = 0;
  for (int c = 0; c < C; ++c) {
    const int a = offsets[c], b = offsets[c + 1];
    if (b <= a || (a & 1) || (b & 1)) return fail(DBP_E_ARG, "cluster row offsets must be even and increasing");
    for (int r = a; r < b; r += p.KC) {
      if (nc >= MAX_CHUNKS) return fail(DBP_E_UNSUPPORTED, "too many row chunks per item (B too large)");
      ChunkDesc& d = p.chunks[nc++];
      d.row0 = r;
      d.nrows = std::min(p.KC, b - r);
      d.cluster = c;
      d.flags = (r + p.KC >= b) ? CH_CLUSTER_END : 0;
    }
  }
  p.chunks[nc - 1].flags |= CH_ITEM_END;
  p.nchunks = nc;
  p.C = C;
  return DBP_OK;
}

static int common_geometry(EqParams& p, int B, int u, int us, int T) {
  if (u < 1 || up_for(u) < 0) return fail(DBP_E_UNSUPPORTED, "u must be in [1, 64]");
  if (T < 1 || T > MAX_T) return fail(DBP_E_UNSUPPORTED, "T must be in [1, 16]");
  if (us < u || (us & 1) || us > up_for(u)) return fail(DBP_E_ARG, "u_stride must be even, >= u and <= padded u");
  if (B < 2 || (B & 1)) return fail(DBP_E_ARG, "B must be even");
  p.B = B;
  p.u = u;
  p.us = us;
  p.T = T;
  p.TP = align_up(T, 4);
  p.KC = 32;
  p.KCP = p.KC + 2;
  p.NS = up_for(u) <= 16 ? 4 : 3;
  p.stage_f2 = p.KC * us + p.TP * p.KCP;
  return DBP_OK;
}

extern "C" {

int dbp_abi_version(void) { return DBP_ABI_VERSION; }

const char* dbp_last_error(void) { return g_err.c_str(); }

int dbp_last_kernel(void) { return g_last_kernel; }

int dbp_set_option(int key, int value) {
  if (key < 0 || key >= DBP_OPT_COUNT) return fail(DBP_E_ARG, "unknown option");
  return g_opt[key].exchange(value);
}

int dbp_device_query(int* sms, int* major, int* minor, long long* l2) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(DBP_E_CUDA, "no CUDA device");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return fail(DBP_E_CUDA, "cudaGetDeviceProperties failed");
  if (sms) *sms = prop.multiProcessorCount;
  if (major) *major = prop.major;
  if (minor) *minor = prop.minor;
  if (l2) *l2 = prop.l2CacheSize;
  return DBP_OK;
}

int dbp_gram_mrc(const void* H, const void* Y, int64_t n_items, int B, int u, int u_stride, int T, int C,
                 const int32_t* offsets, int sum_clusters, void* stats, void* stream) {
  return dbp_gram_mrc_parts(H, Y, n_items, B, u, u_stride, T, C, offsets, sum_clusters, 0, stats, stream);
}

int dbp_gram_mrc_parts(const void* H, const void* Y, int64_t n_items, int B, int u, int u_stride, int T, int C,
                       const int32_t* offsets, int sum_clusters, int bf16_parts, void* stats, void* stream) {
  if (n_items <= 0) return DBP_OK;
  if (bf16_parts != 0 && bf16_parts != 2 && bf16_parts != 3) return fail(DBP_E_ARG, "bf16_parts must be 0, 2 or 3");
  if (!H || !Y || !stats || !offsets) return fail(DBP_E_ARG, "null pointer");
  EqParams q;
  memset(&q, 0, sizeof(q));
  int rc = common_geometry(q, B, u, u_stride, T);
  if (rc) return rc;
  if ((rc = build_chunks(q, C, offsets))) return rc;
  q.H = static_cast<const float2*>(H);
  q.Y = static_cast<const float2*>(Y);
  q.n_items = n_items;
  q.arch = ARCH_STATS;
  q.kind = EQ_MRC;
  q.sum_clusters = sum_clusters;
  q.nsplit = bf16_parts;
  q.stats_out = static_cast<float2*>(stats);
  return dispatch_stream(q, static_cast<cudaStream_t>(stream));
}

int dbp_equalize_stats(const void* stats, int64_t n_items, int u, int T, int kind, float n0, const float* n0_dev,
                       int64_t n0_group, float es, int unbias, float beta, float lama_scale, int t_max, float damping,
                       const float* levels, int L, const float* symbols, int M, void* xhat, float* sigma2,
                       float* gain, uint8_t* dec, int32_t* status, int32_t* iters, void* tr_z, void* tr_s,
                       void* tr_v, float* tr_phi, void* stream) {
  if (n_items <= 0) return DBP_OK;
  if (!stats || !xhat || !sigma2 || !status) return fail(DBP_E_ARG, "null pointer");
  if (kind < EQ_MRC || kind > EQ_LAMA) return fail(DBP_E_ARG, "unknown equalizer kind");
  if (kind == EQ_LAMA && (t_max < 1 || !(damping > 0.f && damping <= 1.f)))
    return fail(DBP_E_ARG, "LAMA needs t_max >= 1 and damping in (0, 1]");
  if (u < 1 || up_for(u) < 0) return fail(DBP_E_UNSUPPORTED, "u must be in [1, 64]");
  if (T < 1 || T > MAX_T) return fail(DBP_E_UNSUPPORTED, "T must be in [1, 16]");
  EqParams p;
  memset(&p, 0, sizeof(p));
  int rc = fill_const(p.cp, levels, L, symbols, M, es);
  if (rc && (kind == EQ_LAMA || dec)) return rc;
  p.stats_in = static_cast<const float2*>(stats);
  p.n_items = n_items;
  p.u = u;
  p.T = T;
  p.TP = align_up(T, 4);
  p.C = 1;
  p.arch = ARCH_PD;
  p.kind = kind;
  p.unbias = unbias;
  p.n0 = n0;
  p.n0_dev = n0_dev;
  p.n0_group = n0_group > 0 ? n0_group : 1;
  p.es = es;
  p.beta = beta;
  p.lama_scale = lama_scale;
  p.damping = damping;
  p.t_max = t_max;
  p.xhat = static_cast<float2*>(xhat);
  p.sigma2 = sigma2;
  p.gain = gain;
  p.dec = dec;
  p.status = status;
  p.iters = iters;
  p.tr_z = static_cast<float2*>(tr_z);
  p.tr_s = static_cast<float2*>(tr_s);
  p.tr_v = static_cast<float2*>(tr_v);
  p.tr_phi = tr_phi;
  return dispatch_stats(p, static_cast<cudaStream_t>(stream));
}

int dbp_equalize(int arch, int kind, const void* H, const void* Y, int64_t n_items, int B, int u, int u_stride, int T,
                 int C, const int32_t* offsets, const int32_t* real_counts, int B_total, float n0,
                 const float* n0_dev, int64_t n0_group, float es, int unbias, float beta, float lama_scale, int t_max,
                 float damping, const float* levels, int L, const float* symbols, int M, void* xhat, float* sigma2,
                 float* gain, float* nu, uint8_t* dec, int32_t* status, int32_t* iters, float* fd_acc,
                 float* fd_wraw, void* stream) {
  if (n_items <= 0) return DBP_OK;
  if (arch != ARCH_PD && arch != ARCH_FD && arch != ARCH_FD_PARTIAL) return fail(DBP_E_ARG, "unknown architecture");
  if (kind < EQ_MRC || kind > EQ_LAMA) return fail(DBP_E_ARG, "unknown equalizer kind");
  if (!H || !Y || !offsets || !status) return fail(DBP_E_ARG, "null pointer");
  if (arch == ARCH_FD_PARTIAL ? (!fd_acc || !fd_wraw) : (!xhat || !sigma2)) return fail(DBP_E_ARG, "null output");
  if (kind == EQ_LAMA && (t_max < 1 || !(damping > 0.f && damping <= 1.f)))
    return fail(DBP_E_ARG, "LAMA needs t_max >= 1 and damping in (0, 1]");
  EqParams p;
  memset(&p, 0, sizeof(p));
  int rc = common_geometry(p, B, u, u_stride, T);
  if (rc) return rc;
  if ((rc = build_chunks(p, C, offsets))) return rc;
  rc = fill_const(p.cp, levels, L, symbols, M, es);
  if (rc && (kind == EQ_LAMA || dec)) return rc;
  int btot = 0;
  for (int c = 0; c < C; ++c) {
    const int bc = real_counts ? real_counts[c] : offsets[c + 1] - offsets[c];
    if (bc < 1) return fail(DBP_E_ARG, "cluster with no antennas");
    btot += bc;
  }
  if (B_total <= 0) B_total = btot;
  for (int c = 0; c < C; ++c) {
    const int bc = real_counts ? real_counts[c] : offsets[c + 1] - offsets[c];
    p.cl_scale[c] = (float)B_total / (float)bc;  // 1 / w_c (fusion.py:60)
    p.cl_beta[c] = (float)u / (float)bc;         // beta_c = U / B_c (fusion.py:67)
  }
  p.H = static_cast<const float2*>(H);
  p.Y = static_cast<const float2*>(Y);
  p.n_items = n_items;
  p.arch = arch;
  p.kind = kind;
  p.unbias = unbias;
  p.n0 = n0;
  p.n0_dev = n0_dev;
  p.n0_group = n0_group > 0 ? n0_group : 1;
  p.es = es;
  p.beta = beta;
  p.lama_scale = lama_scale;
  p.damping = damping;
  p.t_max = t_max;
  p.xhat = static_cast<float2*>(xhat);
  p.sigma2 = sigma2;
  p.gain = gain;
  p.nu = nu;
  p.dec = dec;
  p.status = status;
  p.iters = iters;
  p.fd_acc = fd_acc;
  p.fd_wraw = fd_wraw;
#ifdef DBP_STUDY
  if (const char* ab = getenv("DBP_ABLATE")) p.ablate = atoi(ab);  // timing studies only (study builds)
#endif
  return dispatch_stream(p, static_cast<cudaStream_t>(stream));
}

int dbp_fd_finalize(const float* fd_acc, int64_t n_items, int u, int T, int wdim, const float* levels, int L,
                    const float* symbols, int M, void* xhat, float* sigma2, uint8_t* dec, void* stream) {
  if (n_items <= 0) return DBP_OK;
  if (!fd_acc || !xhat || !sigma2) return fail(DBP_E_ARG, "null pointer");
  if (wdim != u && wdim != T) return fail(DBP_E_ARG, "wdim must be u or T");
  ConstParams cp;
  int rc = fill_const(cp, levels, L, symbols, M, 1.f);
  if (rc && dec) return rc;
  const int64_t total = n_items * T * u;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8);
  fd_finalize_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(fd_acc, n_items, u, T, wdim, cp,
                                                                          static_cast<float2*>(xhat), sigma2, dec);
  return cuda_check("fd_finalize_kernel");
}

int dbp_fd_weights(const float* wraw, const float* den, int64_t n_items, int C, int wdim, float* nu, void* stream) {
  if (n_items <= 0) return DBP_OK;
  if (!wraw || !den || !nu) return fail(DBP_E_ARG, "null pointer");
  const int64_t total = n_items * C * wdim;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8);
  fd_weights_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(wraw, den, n_items, C, wdim, nu);
  return cuda_check("fd_weights_kernel");
}

int dbp_posterior(const void* z, int64_t n, float tau, const float* symbols, int M, void* f_out, float* g_out,
                  void* stream) {
  if (n <= 0) return DBP_OK;
  if (!z || !f_out || !g_out || !symbols) return fail(DBP_E_ARG, "null pointer");
  if (!(tau > 0.f)) return fail(DBP_E_ARG, "tau must be > 0");
  ConstParams cp;
  int rc = fill_const(cp, nullptr, 0, symbols, M, 1.f);
  if (rc) return rc;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  posterior_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const float2*>(z), n, tau, cp,
                                                                         static_cast<float2*>(f_out), g_out);
  return cuda_check("posterior_kernel");
}

int dbp_hard_detect(const void* z, int64_t n, const float* symbols, int M, int32_t* idx_out, void* stream) {
  if (n <= 0) return DBP_OK;
  if (!z || !idx_out || !symbols) return fail(DBP_E_ARG, "null pointer");
  ConstParams cp;
  int rc = fill_const(cp, nullptr, 0, symbols, M, 1.f);
  if (rc) return rc;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  hard_detect_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const float2*>(z), n, cp,
                                                                          idx_out);
  return cuda_check("hard_detect_kernel");
}


static int grid_for(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8)); }

int dbp_stats_sum(const void* parts, int P, int64_t count, void* out, void* stream) {
  if (count <= 0) return DBP_OK;
  if (!parts || !out || P < 1) return fail(DBP_E_ARG, "bad arguments");
  stats_sum_kernel<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const float2*>(parts), P, count, static_cast<float2*>(out));
  return cuda_check("stats_sum_kernel");
}

int dbp_unbias(const void* z, const float* s2, const float* gain, int64_t n, int T, int u, float es, void* z_out,
               float* s2_out, int32_t* status, void* stream) {
  if (n <= 0) return DBP_OK;
  if (!z || !s2 || !gain || !z_out || !s2_out || !status) return fail(DBP_E_ARG, "null pointer");
  unbias_kernel<<<grid_for(n * T * u), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const float2*>(z), s2, gain, n, T, u, es, static_cast<float2*>(z_out), s2_out, status);
  return cuda_check("unbias_kernel");
}

int dbp_fusion_weights(const float* s2, int64_t n, int C, int u, float* nu, int32_t* status, void* stream) {
  if (n <= 0) return DBP_OK;
  if (!s2 || !nu || !status || C < 1) return fail(DBP_E_ARG, "bad arguments");
  fusion_weights_kernel<<<grid_for(n * u), 256, 0, static_cast<cudaStream_t>(stream)>>>(s2, n, C, u, nu, status);
  return cuda_check("fusion_weights_kernel");
}

int dbp_fuse_estimates(const void* z, const float* s2, const float* nu, int C, int64_t count, void* z_out,
                       float* s2_out, void* stream) {
  if (count <= 0) return DBP_OK;
  if (!z || !s2 || !nu || !z_out || !s2_out || C < 1) return fail(DBP_E_ARG, "bad arguments");
  fuse_estimates_kernel<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const float2*>(z), s2, nu, C, count, static_cast<float2*>(z_out), s2_out);
  return cuda_check("fuse_estimates_kernel");
}

// On-device frame synthesis (dbp_synth.cuh): H, Y (and optionally the symbol
// indices) of items [item0, item0 + n_items).
int dbp_synthesize(uint64_t seed, int64_t n_items, int64_t item0, int B, int u, int T, const float* symbols, int M,
                   float n0, const float* n0_dev, int64_t n0_group, void* H, void* Y, uint8_t* sym, void* stream) {
  if (n_items <= 0) return DBP_OK;
  if (!H || !Y || !symbols) return fail(DBP_E_ARG, "null pointer");
  if (B < 2 || (B & 1) || u < 2 || (u & 1) || u > 64) return fail(DBP_E_UNSUPPORTED, "B and u must be even, u <= 64");
  if (T < 1 || T > MAX_T) return fail(DBP_E_UNSUPPORTED, "T must be in [1, 16]");
  if (M < 1 || M > MAX_SYMS) return fail(DBP_E_ARG, "constellation size out of range");
  ConstParams cp;
  int rc = fill_const(cp, nullptr, 0, symbols, M, 1.f);
  if (rc) return rc;
  const int threads = B >= 256 ? 256 : 128;
  const int64_t grid = std::min<int64_t>(n_items, (int64_t)sm_count() * 8);
  synth_kernel<<<(unsigned)grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, n_items, item0, B, u, T, cp, n0_dev, n0_group > 0 ? n0_group : 1, n0, static_cast<float2*>(H),
      static_cast<float2*>(Y), sym);
  return cuda_check("synth_kernel");
}

// Bit LLRs [n][T][u][2 log2 L] from x-hat [n][T][u] and sigma2 ([n][u], or
// [n][T] when s2_per_symbol) for a square QAM set (PAM levels).
int dbp_llr(const void* xhat, const float* sigma2, int64_t n, int T, int u, int s2_per_symbol, const float* levels,
            int L, int exact, float* llr, void* stream) {
  if (n <= 0) return DBP_OK;
  if (!xhat || !sigma2 || !levels || !llr) return fail(DBP_E_ARG, "null pointer");
  if (L < 2 || L > MAX_L || (L & (L - 1))) return fail(DBP_E_ARG, "LLRs need a square QAM set (L a power of two)");
  ConstParams cp;
  int rc = fill_const(cp, levels, L, nullptr, 0, 1.f);
  if (rc) return rc;
  const int64_t n_el = n * T * u;
  const int64_t grid = std::min<int64_t>((n_el + LLR_THREADS - 1) / LLR_THREADS, (int64_t)sm_count() * 8);
  auto cs = static_cast<cudaStream_t>(stream);
  auto xp = static_cast<const float2*>(xhat);
  if (L == 2) llr_kernel<1><<<(unsigned)grid, LLR_THREADS, 0, cs>>>(xp, sigma2, n_el, T, u, s2_per_symbol, cp, exact, llr);
  else if (L == 4) llr_kernel<2><<<(unsigned)grid, LLR_THREADS, 0, cs>>>(xp, sigma2, n_el, T, u, s2_per_symbol, cp, exact, llr);
  else llr_kernel<3><<<(unsigned)grid, LLR_THREADS, 0, cs>>>(xp, sigma2, n_el, T, u, s2_per_symbol, cp, exact, llr);
  return cuda_check("llr_kernel");
}

// Gray bits [n][2 log2 L] (one byte per bit, MSB first) of symbol indices
// (idx_bytes = 1: uint8 decisions; 4: int32 hard_detect indices).
int dbp_gray_bits(const void* idx, int idx_bytes, int64_t n, int L, uint8_t* bits, void* stream) {
  if (n <= 0) return DBP_OK;
  if (!idx || !bits) return fail(DBP_E_ARG, "null pointer");
  if (L < 2 || L > MAX_L || (L & (L - 1))) return fail(DBP_E_ARG, "Gray bits need a square QAM set (L a power of two)");
  if (idx_bytes != 1 && idx_bytes != 4) return fail(DBP_E_ARG, "index type must be uint8 or int32");
  const int h = 31 - __builtin_clz(L);
  auto cs = static_cast<cudaStream_t>(stream);
  if (idx_bytes == 1)
    gray_bits_kernel<<<grid_for(n), 256, 0, cs>>>(static_cast<const uint8_t*>(idx), n, h, bits);
  else
    gray_bits_kernel<<<grid_for(n), 256, 0, cs>>>(static_cast<const int32_t*>(idx), n, h, bits);
  return cuda_check("gray_bits_kernel");
}

// Gauss-Hermite quadratures at n points x (device,
// fp64): kind 0 = lama_mse_pam (values = M real levels), 1 = lama_mse,
// 2 = mi_awgn (values = M complex symbols, interleaved re/im; host); nodes /
// weights: q-point rule for exp(-x^2) (device).
int dbp_quadrature(int kind, const double* x, int64_t n, const double* values, int M, const double* nodes,
                   const double* weights, int q, double* out, void* stream) {
  if (n <= 0) return DBP_OK;
  if (!x || !values || !nodes || !weights || !out) return fail(DBP_E_ARG, "null pointer");
  if (kind < QK_MSE_PAM || kind > QK_MI) return fail(DBP_E_ARG, "unknown quadrature kind");
  if (M < 1 || M > MAX_SYMS || q < 1) return fail(DBP_E_ARG, "bad set size or order");
  if ((int64_t)M * q * (kind == QK_MSE_PAM ? 1 : q) > (int64_t)1 << 30) return fail(DBP_E_UNSUPPORTED, "order too large");
  if (n > 0x7fffffff) return fail(DBP_E_UNSUPPORTED, "too many points");
  QuadSet qs;
  memset(&qs, 0, sizeof(qs));
  qs.M = M;
  for (int k = 0; k < M; ++k) {
    if (kind == QK_MSE_PAM) {
      qs.re[k] = values[k];
    } else {
      qs.re[k] = values[2 * k];
      qs.im[k] = values[2 * k + 1];
    }
  }
  quad_kernel<<<(unsigned)n, QUAD_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(kind, x, qs, nodes, weights, q,
                                                                                  out);
  return cuda_check("quad_kernel");
}

// Batched fixed points of the state evolution (fixed_point_kernel): P points
// (device arrays n0, beta, w, start), constellation as in dbp_quadrature
// (kind 0: PAM levels, 1: complex symbols).
int dbp_fixed_point(int kind, const double* n0, const double* beta, const double* w, const double* start, int64_t P,
                    const double* values, int M, const double* nodes, const double* weights, int q, double tol,
                    int max_iter, double* sigma2, int32_t* iters, void* stream) {
  if (P <= 0) return DBP_OK;
  if (!n0 || !beta || !w || !start || !values || !nodes || !weights || !sigma2 || !iters)
    return fail(DBP_E_ARG, "null pointer");
  if (kind != QK_MSE_PAM && kind != QK_MSE_2D) return fail(DBP_E_ARG, "fixed points need an MSE quadrature");
  if (M < 1 || M > MAX_SYMS || q < 1 || max_iter < 1) return fail(DBP_E_ARG, "bad set size, order or iteration cap");
  if (P > 0x7fffffff) return fail(DBP_E_UNSUPPORTED, "too many points");
  QuadSet qs;
  memset(&qs, 0, sizeof(qs));
  qs.M = M;
  for (int k = 0; k < M; ++k) {
    if (kind == QK_MSE_PAM) {
      qs.re[k] = values[k];
    } else {
      qs.re[k] = values[2 * k];
      qs.im[k] = values[2 * k + 1];
    }
  }
  fixed_point_kernel<<<(unsigned)P, QUAD_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      kind, n0, beta, w, start, qs, nodes, weights, q, tol, max_iter, sigma2, iters);
  return cuda_check("fixed_point_kernel");
}

}  // extern "C"
