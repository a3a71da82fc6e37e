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
//   one WARP per unit (4 independent units per CTA, no CTA barrier); lane
//   (ip, jq), ip = lane / 2, jq = lane % 2, holds G rows ip and ip + 16,
//   columns 16 jq .. 16 jq + 15, in REGISTERS (64) as (re, im) pairs for the
//   whole recursion.  Symbols run in pairs: every s pair a lane reads (one
//   float4, broadcast over the 16 lanes of a parity) feeds 8 FFMA2 -- packed
//   FP32 on the G pair with s_r / s_i as the scalar broadcast operand, 16 FMA
//   per 4 words -- and one shuffle exchange leaves lane jq with (G s) of
//   symbol 2b + jq for both rows.  The owned states (y_mrc, v of
//   (2b + jq, ip / ip + 16)) sit in per-lane shared-memory slots, s in the
//   matvec operand array itself, and the batch loop is not unrolled (the
//   unrolled recursion, 34 KB of code per iteration, stalled on instruction
//   fetch).
//
// Per pass over a symbol pair: matvec, z = y_mrc + s + v - G s (lama_scale
// applied as in the reference's rescaled statistics), the PAM-factorised
// posterior with the two dimensions in packed FP32 pairs, phi^{t+1} as a
// shuffle reduction over the 16 lanes of the symbol (the warp holds all u
// rows), v^{t+1} and s^{t+1} written back -- __syncwarp only.
#pragma once
#include "dbp_epilogue.cuh"

namespace dbp {

constexpr int LAMA_WARPS = 4;  // independent units (one per warp) per CTA
constexpr int LAMA_NT = 32 * LAMA_WARPS;
// shared s row: 32 columns in two halves, the second shifted by two entries
// so the two lane parities read disjoint bank groups
constexpr int LAMA_SLD = 36;
__device__ __forceinline__ int lama_sidx(int j) { return j + 2 * (j >> 4); }

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
#define DBP_LAMA_MINB 4  // CTAs per SM the register budget is cut for (study builds vary it)
#endif
// per-warp shared-memory block (one unit / item per warp)
struct __align__(16) LamaWarpSmem {
  float2 S[MAX_T][LAMA_SLD];      // s per (symbol, column): the matvec operand
  float2 ZY[MAX_T / 2][2][32];    // per-lane state slots: y_mrc (z^{t_max} at the end),
  float2 VV[MAX_T / 2][2][32];    // v,
  float PH[MAX_T / 2][2];         // phi per symbol (batch b, lane parity)
  float wb[MAX_C][MAX_T];         // FD: cluster weights (for nu)
  int flags[2];
};

template <int PL>
__global__ void __launch_bounds__(LAMA_NT, DBP_LAMA_MINB) lama_kernel(const __grid_constant__ EqParams p) {
  extern __shared__ __align__(16) char lama_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  LamaWarpSmem& ws = reinterpret_cast<LamaWarpSmem*>(lama_smem)[warp];
  const int ip = lane >> 1, jq = lane & 1;  // rows ip, ip + 16; columns 16 jq .. 16 jq + 15
  const int u = p.u, T = p.T, nb = (T + 1) >> 1;
  const bool fd = p.arch == ARCH_FD;
  const bool herm = p.g_hermitian != 0;
  const int ncl = fd ? p.C : 1;
  const size_t rec = (size_t)u * u + (size_t)T * u;
  const int64_t nrec = p.n_items * ncl;
  const int64_t nwarps = (int64_t)gridDim.x * LAMA_WARPS;
  const float inv_u = 1.f / (float)u;
  const float damp = p.damping;
  const ConstParams& cp = p.cp;

  // padding rows / columns of s stay zero for the whole launch
  for (int e = lane; e < MAX_T * LAMA_SLD; e += 32) (&ws.S[0][0])[e] = make_float2(0.f, 0.f);
  __syncwarp();

  for (int64_t n = (int64_t)blockIdx.x * LAMA_WARPS + warp; n < p.n_items; n += nwarps) {
    const float n0i = item_n0(p, n);
    int dv = 0x7fffffff, st = 0;  // first divergent iteration; status of the item
    for (int c = 0; c < ncl; ++c) {
      const int64_t rr = n * ncl + c;
      const float2* src = p.stats_in + rr * rec;
      {  // the warp's next record into L2 while this one iterates
        const int64_t rn = (c + 1 < ncl) ? rr + 1 : (n + nwarps) * ncl;
        if (lane == 0 && rn < nrec) {
          const char* nx = reinterpret_cast<const char*>(p.stats_in + rn * rec);
          const uint32_t bytes = (uint32_t)(rec * sizeof(float2));
          for (uint32_t o = 0; o < bytes; o += 32768) {
            const uint32_t len = min(32768u, bytes - o) & ~15u;
            if (len && !(reinterpret_cast<uintptr_t>(nx + o) & 15))
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx + o), "r"(len) : "memory");
          }
        }
      }
      // G rows ip and ip + 16, columns 16 jq .. 16 jq + 15, in registers as
      // natural (re, im) pairs; the kernel's own Gram (herm) is read down the
      // columns, G[j][i] = conj G[i][j], the conjugation folded into the
      // recombination below
      p2_t g[2][16];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = ip + 16 * r;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int j = 16 * jq + k;
          g[r][k] = (i < u && j < u) ? *reinterpret_cast<const p2_t*>(src + (herm ? (size_t)j * u + i : (size_t)i * u + j))
                                     : 0ull;
        }
      }
      const float hs = herm ? -1.f : 1.f;
      const float sc = fd ? p.cl_scale[c] : p.lama_scale;
      const float beta = fd ? p.cl_beta[c] : p.beta;
      const float n0 = n0i * sc;
      __syncwarp();  // the previous unit's reads of S / ZY are done
      for (int b = 0; b < nb; ++b) {
        const int t = 2 * b + jq;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = ip + 16 * r;
          const bool ok = t < T && i < u;
          ws.ZY[b][r][lane] = ok ? c_scale(src[(size_t)u * u + (size_t)t * u + i], sc) : make_float2(0.f, 0.f);
          ws.VV[b][r][lane] = make_float2(0.f, 0.f);
          if (ok) ws.S[t][lama_sidx(i)] = cp.mean;
        }
        if (ip == 0) ws.PH[b][jq] = cp.es;
      }
      for (int it = 1;; ++it) {
        const bool last = it == p.t_max;
#pragma unroll 1
        for (int b = 0; b < nb; ++b) {
          __syncwarp();  // S rows 2b, 2b + 1 of the previous pass are published
          const int t = 2 * b + jq;
          // ---- (G s)_i for rows ip, ip + 16 and symbols 2b, 2b + 1 over this
          // lane's 16 columns: FFMA2 on (re, im) pairs of G with s_r / s_i as
          // the broadcast scalar operand, A += g s_r, B += g s_i; each s pair
          // read (one float4, shared by the 16 lanes of a parity) feeds 8 FFMA2
          // = 16 FMA; rows t >= T of S are zero
          p2_t pa[2][2], pb[2][2];  // [row][symbol]
#pragma unroll
          for (int r = 0; r < 2; ++r) pa[r][0] = pa[r][1] = pb[r][0] = pb[r][1] = 0ull;
          const float2* sb = &ws.S[2 * b][lama_sidx(16 * jq)];
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const float4 sv = *reinterpret_cast<const float4*>(sb + q * LAMA_SLD + 2 * k2);
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                pa[r][q] = p2_fma(g[r][2 * k2], p2(sv.x, sv.x), pa[r][q]);
                pb[r][q] = p2_fma(g[r][2 * k2], p2(sv.y, sv.y), pb[r][q]);
                pa[r][q] = p2_fma(g[r][2 * k2 + 1], p2(sv.z, sv.z), pa[r][q]);
                pb[r][q] = p2_fma(g[r][2 * k2 + 1], p2(sv.w, sv.w), pb[r][q]);
              }
            }
          }
          // (G s) = (A.re - B.im, B.re + A.im); conj(G) s = (A.re + B.im, B.re - A.im)
          float2 a[2][2];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const float2 A = p2_unpack(pa[r][q]), B = p2_unpack(pb[r][q]);
              a[r][q] = make_float2(fmaf(-hs, B.y, A.x), fmaf(hs, A.y, B.x));
            }
          // the lane pair exchanges halves: lane jq keeps symbol 2b + jq
          float2 m[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            m[r] = jq ? a[r][1] : a[r][0];
            const float2 o = jq ? a[r][0] : a[r][1];
            m[r].x += __shfl_xor_sync(0xffffffffu, o.x, 1);
            m[r].y += __shfl_xor_sync(0xffffffffu, o.y, 1);
          }
          const float phi = ws.PH[b][jq];
          const float tau = n0 + beta * phi;
          const float tinv = rcp_ftz(fmaxf(tau, FLT_MIN));  // MUFU.RCP (~1 ulp)
          float2 z[2], sold[2], F[2];
          float gs = 0.f;
          __syncwarp();  // every lane has read S rows 2b, 2b + 1
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = ip + 16 * r;
            const bool ok = t < T && i < u;
            sold[r] = ws.S[t][lama_sidx(i)];
            // z = y_mrc + (I - G) s + v (equalize.py:243); |z|^2 < 1e36 is
            // false for NaN / inf too (equalize.py:246-249)
            z[r] = c_sub(c_add(ws.ZY[b][r][lane], c_add(sold[r], ws.VV[b][r][lane])), c_scale(m[r], sc));
            dv = (ok && !(c_abs2(z[r]) < DIVERGE_ABS2)) ? min(dv, it) : dv;
            if (last) {
              ws.ZY[b][r][lane] = z[r];  // z^{t_max} parked in the y_mrc slot
              continue;
            }
            float gv;
            if constexpr (PL > 0)
              lama_post2<PL>(z[r], tinv, cp, F[r], gv);
            else
              posterior_t<0>(z[r], tau, cp, F[r], gv);
            gs += ok ? gv : 0.f;
          }
          if (last) continue;
          // phi^{t+1}: mean of g over the u rows of symbol t (equalize.py:253),
          // the 16 lanes of this parity hold them all
#pragma unroll
          for (int o = 2; o < 32; o <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
          const float phin = gs * inv_u;
          const float coef = beta * phin * tinv;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = ip + 16 * r;
            ws.VV[b][r][lane] = c_scale(c_sub(z[r], sold[r]), coef);
            const float2 snew = c_add(c_scale(F[r], damp), c_scale(sold[r], 1.f - damp));
            if (t < T && i < u) ws.S[t][lama_sidx(i)] = snew;
          }
          __syncwarp();  // every lane has read PH[b] before it is overwritten
          if (ip == 0) ws.PH[b][jq] = phin;
        }
        if (last) break;
      }
      // ---- outputs (equalize.py:255-257): z^{t_max}, tau^{t_max}
      __syncwarp();
      for (int b = 0; b < nb; ++b) {
        const int t = 2 * b + jq;
        const float tau = n0 + beta * ws.PH[b][jq];
        const float wt = 1.f / fmaxf(tau, VAR_FLOOR);  // FD: w = 1 / max(tau, 1e-15) (fusion.py:96-105)
        if (fd && t < T && ip < u && !(tau > 0.f)) st = ST_BADVAR;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = ip + 16 * r;
          const float2 z = ws.ZY[b][r][lane];
          if (!fd) {
            if (t < T && i < u) {
              const size_t o = ((size_t)n * T + t) * u + i;
              p.xhat[o] = z;
              if (p.dec) p.dec[o] = (uint8_t)slice_symbol(z, cp);
            }
          } else if (t < T && i < u) {  // fold cluster c: sum_c w_c z_c, in x-hat itself (L2)
            const size_t o = ((size_t)n * T + t) * u + i;
            const float2 x = c_scale(z, wt);
            p.xhat[o] = c == 0 ? x : c_add(p.xhat[o], x);
          }
        }
        if (fd) {
          if (ip == 0 && t < T) ws.wb[c][t] = wt;
        } else if (ip == 0 && t < T) {
          p.sigma2[(size_t)n * T + t] = tau;
        }
      }
    }
    if (fd) {  // fuse_estimates (fusion.py:108-124); sigma2 = 1 / sum_c 1 / tau_c
      __syncwarp();  // the cluster weights wb are in
      for (int b = 0; b < nb; ++b) {
        const int t = 2 * b + jq;
        float den = 0.f;  // sum_c w_c, in cluster order
        if (t < T)
          for (int cc = 0; cc < ncl; ++cc) den += ws.wb[cc][t];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = ip + 16 * r;
          if (t < T && i < u) {
            const size_t o = ((size_t)n * T + t) * u + i;
            const float2 x = c_scale(p.xhat[o], 1.f / den);
            p.xhat[o] = x;
            if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, cp);
          }
        }
        if (ip == 0 && t < T) {
          p.sigma2[(size_t)n * T + t] = 1.f / den;
          if (p.nu)
            for (int cc = 0; cc < ncl; ++cc) p.nu[((size_t)n * ncl + cc) * T + t] = ws.wb[cc][t] / den;
        }
      }
    }
    // item status: BadVariance first (set during the folds), else divergence
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dv = min(dv, __shfl_xor_sync(0xffffffffu, dv, o));
      st = max(st, __shfl_xor_sync(0xffffffffu, st, o));
    }
    if (lane == 0) {
      if (dv < 0x7fffffff) st = st ? st : ST_DIVERGED;
      p.status[n] = st;
      if (p.iters) p.iters[n] = (dv < 0x7fffffff) ? dv : 0;
    }
  }
}

}  // namespace dbp
