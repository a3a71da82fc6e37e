// dbp::lama_kernel -- the LAMA message-passing recursion (equalize.py:208-259)
// from precomputed statistics records [G (u x u) | y_mrc (T x u)], u <= 32,
// T <= 16: PD (one record per item) and FD (the item's C per-cluster records,
// fused in cluster order as fusion.py:127-154 does, with the LAMA weights
// 1 / tau_c[t] of fusion.py:96-105).
//
// Why a kernel of its own: the recursion is the whole cost of cfg4
// (10 iterations x T symbols x a u x u complex matvec per unit = 573K FMA
// against 11.5 KB of statistics).  The group-owned recursion inside the
// streaming kernels kept G in shared memory and one (symbol, row) per lane:
// every FMA pair needed its own shared-memory operand.  Shared memory delivers
// 4 bytes per lane per wavefront whatever the access width or broadcast
// (measured: a broadcast LDS.128 costs 4 wavefronts), so an FMA-bound matvec
// needs >= 4 FMA per word a lane reads.  Here:
//
//   team = 64 threads (2 warps) per unit; thread (ip, jq), ip = 8 warp +
//   lane / 4 in [0, 16), jq = lane % 4, holds G rows ip and ip + 16, columns
//   8 jq .. 8 jq + 7, in REGISTERS (32) for the whole recursion.  Symbols run
//   in batches of four: every s pair a thread reads (one float4, broadcast
//   over the rows) feeds 16 FFMA (2 rows x 2 columns), 4 FMA per word; a
//   4-lane reduce-scatter (12 shuffles) then leaves thread jq with (G s) of
//   symbol 4b + jq for both rows.  The owned states (y_mrc, s, v of
//   (4b + jq, ip / ip + 16)) sit in per-thread shared-memory slots and the
//   batch loop is not unrolled (the unrolled recursion, 34 KB of code per
//   iteration, stalled on instruction fetch).
//
// Per iteration: matvec, z = y_mrc + s + v - G s (lama_scale applied as in
// the reference's rescaled statistics), the PAM-factorised posterior with the
// two dimensions in packed FP32 pairs, the per-symbol sum of g (shuffles over
// the warp's rows, one partial per warp), and s^{t+1} published to the other
// half of a double-buffered shared array -- ONE CTA barrier per iteration:
// v^{t+1} = beta phi^{t+1} / tau^t (z - s) is stored without its phi factor
// and completed when the next pass reads phi^{t+1}.
#pragma once
#include "dbp_epilogue.cuh"

namespace dbp {

constexpr int LAMA_NT = 64;
// shared s row: 32 columns in four octets, each octet padded by two entries
// so the four jq lanes of a quad read four disjoint bank groups
constexpr int LAMA_SLD = 40;
__device__ __forceinline__ int lama_sidx(int j) { return j + 2 * (j >> 3); }

// packed FP32 pairs (one 64-bit register pair; FFMA2 / FADD2 / FMUL2 on sm_100)
typedef unsigned long long p2_t;
__device__ __forceinline__ p2_t p2(float a, float b) {
  p2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 p2_unpack(p2_t x) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(x));
  return r;
}
__device__ __forceinline__ p2_t p2_fma(p2_t a, p2_t b, p2_t c) {
  p2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ p2_t p2_add(p2_t a, p2_t b) {
  p2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ p2_t p2_sub(p2_t a, p2_t b) {
  p2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ p2_t p2_mul(p2_t a, p2_t b) {
  p2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ p2_t p2_ld(const float2& f) { return *reinterpret_cast<const p2_t*>(&f); }
__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// posterior_t<L> (the PAM-factorised posterior of _kernels.pyx:19-71) with the
// real and imaginary dimensions in one packed pair: weights
// exp(-(d - dmin) / tau) as 2^((dmin - d) tau^-1 log2 e) (one FFMA2 + two
// MUFU.EX2 per level for both dimensions); weights below 2^-126 flush to zero
// (they are below the fp32 resolution of the weight sum, which is >= 1).
template <int L>
__device__ __forceinline__ void lama_post2(float2 z, float tinv, const ConstParams& cp, float2& F, float& gv) {
  const float tl = tinv * 1.44269504088896341f;
  const p2_t zz = p2(z.x, z.y);
  p2_t d[L];
  float mx = FLT_MAX, my = FLT_MAX;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const p2_t e = p2_sub(zz, p2_ld(cp.lv2[l]));
    d[l] = p2_mul(e, e);
    const float2 df = p2_unpack(d[l]);
    mx = fminf(mx, df.x);
    my = fminf(my, df.y);
  }
  const p2_t ntl = p2(-tl, -tl), base = p2(mx * tl, my * tl);
  p2_t ws = p2(0.f, 0.f), s1 = ws, s2 = ws;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const float2 a = p2_unpack(p2_fma(d[l], ntl, base));
    const p2_t w = p2(ex2_ftz(a.x), ex2_ftz(a.y));
    ws = p2_add(ws, w);
    s1 = p2_fma(w, p2_ld(cp.lv2[l]), s1);
    s2 = p2_fma(w, p2_ld(cp.lq2[l]), s2);
  }
  const float2 wsf = p2_unpack(ws);
  const p2_t r = p2(rcp_ftz(wsf.x), rcp_ftz(wsf.y));  // ws in [1, L]
  const float2 mean = p2_unpack(p2_mul(s1, r)), m2 = p2_unpack(p2_mul(s2, r));
  F = mean;
  gv = fmaxf((m2.x - mean.x * mean.x) + (m2.y - mean.y * mean.y), 0.f);
}

#ifndef DBP_LAMA_MINB
#define DBP_LAMA_MINB 8  // CTAs per SM the register budget is cut for (study builds vary it)
#endif
template <int PL>
__global__ void __launch_bounds__(LAMA_NT, DBP_LAMA_MINB) lama_kernel(const __grid_constant__ EqParams p) {
  __shared__ __align__(16) float2 S[2][MAX_T][LAMA_SLD];  // s per (symbol, column), double-buffered
  __shared__ __align__(16) float2 P[2][MAX_T];            // per-warp sums of g per symbol
  __shared__ float2 ZY[4][2][LAMA_NT];                    // per-thread state slots: y_mrc (z at the end),
  __shared__ float2 SS[4][2][LAMA_NT];                    // s,
  __shared__ float2 VV[4][2][LAMA_NT];                    // v / phi' (equalize.py:252)
  __shared__ float2 fnum[4][2][LAMA_NT];                  // FD: per-thread fusion sums
  __shared__ float fden[4][LAMA_NT];
  __shared__ float wb[MAX_C][MAX_T];                      // FD: cluster weights (for nu)
  __shared__ int flags[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ip = warp * 8 + (lane >> 2), jq = lane & 3;
  const int u = p.u, T = p.T;
  const bool fd = p.arch == ARCH_FD;
  const bool herm = p.g_hermitian != 0;
  const int ncl = fd ? p.C : 1;
  const size_t rec = (size_t)u * u + (size_t)T * u;
  const int64_t nrec = p.n_items * ncl;
  const float inv_u = 1.f / (float)u;
  const float damp = p.damping;
  const ConstParams& cp = p.cp;

  // padding rows / columns of s stay zero for the whole launch
  for (int e = tid; e < 2 * MAX_T * LAMA_SLD; e += LAMA_NT) (&S[0][0][0])[e] = make_float2(0.f, 0.f);
  bool valid[4][2];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int r = 0; r < 2; ++r) valid[b][r] = 4 * b + jq < T && ip + 16 * r < u;

  for (int64_t n = blockIdx.x; n < p.n_items; n += gridDim.x) {
    if (tid == 0) {
      flags[0] = 0;
      flags[1] = 0x7fffffff;
    }
    const float n0i = item_n0(p, n);
    for (int c = 0; c < ncl; ++c) {
      const int64_t rr = n * ncl + c;
      const float2* src = p.stats_in + rr * rec;
      {  // the next record into L2 while this one iterates
        const int64_t rn = (c + 1 < ncl) ? rr + 1 : (n + gridDim.x) * ncl;
        if (tid == 0 && rn < nrec) {
          const char* nx = reinterpret_cast<const char*>(p.stats_in + rn * rec);
          const uint32_t bytes = (uint32_t)(rec * sizeof(float2));
          for (uint32_t o = 0; o < bytes; o += 32768) {
            const uint32_t len = min(32768u, bytes - o) & ~15u;
            if (len && !(reinterpret_cast<uintptr_t>(nx + o) & 15))
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx + o), "r"(len) : "memory");
          }
        }
      }
      // G rows ip and ip + 16, columns 8 jq .. 8 jq + 7 (the kernel's own
      // Gram: conj of the columns, as the streaming kernels read it)
      float2 g[2][8];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = ip + 16 * r;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = 8 * jq + k;
          float2 x = make_float2(0.f, 0.f);
          if (i < u && j < u) x = herm ? c_conj(src[(size_t)j * u + i]) : src[(size_t)i * u + j];
          g[r][k] = x;
        }
      }
      const float sc = fd ? p.cl_scale[c] : p.lama_scale;
      const float beta = fd ? p.cl_beta[c] : p.beta;
      const float n0 = n0i * sc;
      __syncthreads();  // the previous unit's last matvec has read S
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int t = 4 * b + jq;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = ip + 16 * r;
          const float2 s0 = valid[b][r] ? cp.mean : make_float2(0.f, 0.f);
          ZY[b][r][tid] = valid[b][r] ? c_scale(src[(size_t)u * u + (size_t)t * u + i], sc) : make_float2(0.f, 0.f);
          SS[b][r][tid] = s0;
          VV[b][r][tid] = make_float2(0.f, 0.f);
          if (valid[b][r]) S[0][t][lama_sidx(i)] = s0;
        }
      }
      __syncthreads();
      int par = 0, dv = 0x7fffffff;  // dv: first divergent iteration of this thread's states
      for (int it = 1;; ++it) {
        const bool last = it == p.t_max;
        // one batch of four symbols per pass (a compact loop body: the fully
        // unrolled recursion missed the instruction cache); the owned states
        // (z, s, v of rows ip, ip + 16) live in per-thread shared-memory slots
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
          const int t = 4 * b + jq;
          // phi^t: the per-symbol mean of g from the previous pass (equalize.py:253)
          const float2 pw = P[par ^ 1][t];
          const float phi = it == 1 ? cp.es : (pw.x + pw.y) * inv_u;
          // ---- (G s)_i for rows ip, ip + 16 and symbols 4b..4b+3 over this
          // thread's eight columns: each s pair read from shared memory feeds
          // 16 FFMA (two rows); rows t >= T of S are zero
          float2 a[2][4];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) a[r][q] = make_float2(0.f, 0.f);
          const float2* sb = &S[par][4 * b][10 * jq];  // lama_sidx(8 jq) = 10 jq
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 sv = *reinterpret_cast<const float4*>(sb + q * LAMA_SLD + 2 * k2);
              const float2 s0 = make_float2(sv.x, sv.y), s1 = make_float2(sv.z, sv.w);
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                c_fma(a[r][q], g[r][2 * k2], s0);
                c_fma(a[r][q], g[r][2 * k2 + 1], s1);
              }
            }
          }
          // reduce-scatter over the quad: lane jq keeps symbol 4b + jq
          const bool h1 = (jq & 2) != 0, h0 = (jq & 1) != 0;
          float2 m[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            float2 k0 = h1 ? a[r][2] : a[r][0], k1 = h1 ? a[r][3] : a[r][1];
            const float2 o0 = h1 ? a[r][0] : a[r][2], o1 = h1 ? a[r][1] : a[r][3];
            k0.x += __shfl_xor_sync(0xffffffffu, o0.x, 2);
            k0.y += __shfl_xor_sync(0xffffffffu, o0.y, 2);
            k1.x += __shfl_xor_sync(0xffffffffu, o1.x, 2);
            k1.y += __shfl_xor_sync(0xffffffffu, o1.y, 2);
            m[r] = h0 ? k1 : k0;
            const float2 om = h0 ? k0 : k1;
            m[r].x += __shfl_xor_sync(0xffffffffu, om.x, 1);
            m[r].y += __shfl_xor_sync(0xffffffffu, om.y, 1);
          }
          const float tau = n0 + beta * phi;
          const float tinv = rcp_ftz(fmaxf(tau, FLT_MIN));  // MUFU.RCP (~1 ulp)
          float gs = 0.f;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = ip + 16 * r;
            const bool ok = 4 * b + jq < T && i < u;
            const float2 sold = SS[b][r][tid];
            // v^t = beta phi^t / tau^{t-1} (z^{t-1} - s^{t-1}): the stored part times phi^t
            const float2 v = it == 1 ? make_float2(0.f, 0.f) : c_scale(VV[b][r][tid], phi);
            // z = y_mrc + (I - G) s + v (equalize.py:243); |z|^2 < 1e36 is
            // false for NaN / inf too (equalize.py:246-249)
            const float2 z = c_sub(c_add(ZY[b][r][tid], c_add(sold, v)), c_scale(m[r], sc));
            dv = (ok && !(c_abs2(z) < DIVERGE_ABS2)) ? min(dv, it) : dv;
            if (last) {  // z^{t_max} parked in the (now unused) y_mrc slot
              ZY[b][r][tid] = z;
              continue;
            }
            // ---- denoiser; s^{t+1} published
            float2 F;
            float gv;
            if constexpr (PL > 0)
              lama_post2<PL>(z, tinv, cp, F, gv);
            else
              posterior_t<0>(z, tau, cp, F, gv);
            gs += ok ? gv : 0.f;
            VV[b][r][tid] = c_scale(c_sub(z, sold), beta * tinv);
            const float2 snew = c_add(c_scale(F, damp), c_scale(sold, 1.f - damp));
            SS[b][r][tid] = snew;
            if (ok) S[par ^ 1][t][lama_sidx(i)] = snew;
          }
          if (!last) {  // this batch's sums of g over the warp's rows -> P
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
            if (lane < 4) (warp ? P[par][t].y : P[par][t].x) = gs;
          }
        }
        if (last) break;
        __syncthreads();
        par ^= 1;
      }
      if (dv < 0x7fffffff) atomicMin(&flags[1], dv);
      // ---- outputs (equalize.py:255-257): z^{t_max}, tau^{t_max}
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int t = 4 * b + jq;
        const float2 pw = P[par ^ 1][t];
        const float phi = p.t_max == 1 ? cp.es : (pw.x + pw.y) * inv_u;
        const float tau = n0 + beta * phi;
        const float wt = 1.f / fmaxf(tau, VAR_FLOOR);  // FD: w = 1 / max(tau, 1e-15) (fusion.py:96-105)
        if (fd && t < T && ip < u && !(tau > 0.f)) set_status(flags, ST_BADVAR);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = ip + 16 * r;
          const float2 z = ZY[b][r][tid];
          if (!fd) {
            if (valid[b][r]) {
              const size_t o = ((size_t)n * T + t) * u + i;
              p.xhat[o] = z;
              if (p.dec) p.dec[o] = (uint8_t)slice_symbol(z, cp);
            }
          } else {  // fold cluster c
            const float2 x = c_scale(z, wt);
            fnum[b][r][tid] = c == 0 ? x : c_add(fnum[b][r][tid], x);
          }
        }
        if (fd) {
          fden[b][tid] = c == 0 ? wt : fden[b][tid] + wt;
          if (ip == 0 && t < T) wb[c][t] = wt;
        } else if (ip == 0 && t < T) {
          p.sigma2[(size_t)n * T + t] = tau;
        }
      }
    }
    if (fd) {  // fuse_estimates (fusion.py:108-124); sigma2 = 1 / sum_c 1 / tau_c
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int t = 4 * b + jq;
        const float den = fden[b][tid];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = ip + 16 * r;
          if (valid[b][r]) {
            const float2 x = c_scale(fnum[b][r][tid], 1.f / den);
            const size_t o = ((size_t)n * T + t) * u + i;
            p.xhat[o] = x;
            if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, cp);
          }
          if (i == 0 && t < T) {
            p.sigma2[(size_t)n * T + t] = 1.f / den;
            if (p.nu)
              for (int cc = 0; cc < ncl; ++cc) p.nu[((size_t)n * ncl + cc) * T + t] = wb[cc][t] / den;
          }
        }
      }
    }
    __syncthreads();  // every status / divergence update of the item is in
    if (tid == 0) {
      int st = flags[0];
      if (flags[1] < 0x7fffffff) st = st ? st : ST_DIVERGED;
      p.status[n] = st;
      if (p.iters) p.iters[n] = (flags[1] < 0x7fffffff) ? flags[1] : 0;
    }
  }
}

}  // namespace dbp
