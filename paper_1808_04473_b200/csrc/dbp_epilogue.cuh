// Per-unit epilogues that run on the on-chip Gram G and matched filter Z of
// one unit (a whole item for PD, one cluster for FD): MRC / ZF / L-MMSE
// (Gauss-Jordan inverse), the Gram-domain LAMA recursion, FD fusion, the
// statistics writer and the output stores.  Every function runs on a thread
// Team (the whole CTA, or the epilogue warps of a warp-specialized kernel)
// and only synchronises through Team::sync().
#pragma once
#include "dbp_device.cuh"

namespace dbp {

struct EqParams {
  const float2* H;
  const float2* Y;
  const float2* stats_in;
  int64_t n_items;
  int B, u, us, T, TP;
  int KC, KCP, NS;
  int stage_f2;  // float2 elements per raw stage
  int nchunks;
  int C;
  int arch;
  int kind;
  int unbias;
  int sum_clusters;
  float n0;
  const float* n0_dev;
  int64_t n0_group;
  float es;
  float beta, lama_scale, damping;
  int t_max;
  float cl_scale[MAX_C];
  float cl_beta[MAX_C];
  ChunkDesc chunks[MAX_CHUNKS];
  ConstParams cp;
  // outputs
  float2* xhat;
  float* sigma2;
  float* gain;
  float* nu;
  uint8_t* dec;
  int32_t* status;
  int32_t* iters;
  float2* stats_out;
  float* fd_acc;
  float* fd_wraw;
  float* fd_scratch;  // tensor-core FD: per-(item, cluster) records for the ordered fold
  float2 *tr_z, *tr_s, *tr_v;
  float* tr_phi;
  int pair;        // tensor-core kernel: units per operand tile (1 or 2)
  // tensor-core kernel staging: a stage is `ips` consecutive whole items
  // (spi == 1) or one row block of one item (spi > 1); H part then Y part
  int ips, spi, stage_bytes, stage_hbytes, stage_ystride;
  int tc_simple, tc_bc;  // whole-item stages, full 32-row chunks, clusters of tc_bc rows
  int g_hermitian;       // G is the kernel's own Gram (exactly Hermitian in shared memory)
  int nsplit;            // split-bf16 statistics: bf16 parts per operand (0: the kernel's default)
  int st_row0[MAX_SPI], st_rows[MAX_SPI];
  float* dbg_tile;  // debug: first operand tile of CTA 0 (DBP_TC_DUMP)
  long long* dbg;  // debug: per-role wait-cycle counters [5][4] (DBP_TC_DEBUG)
  int ablate;  // debug: 1 skip solver work, 2 skip MMAs, 4 skip conversion (timing studies only)
};

__device__ __forceinline__ float item_n0(const EqParams& p, int64_t n) {
  return p.n0_dev ? p.n0_dev[n / p.n0_group] : p.n0;
}

// Shared-memory views of one unit's working set (padded leading dims).
struct Work {
  float2* G;     // [UP][LD]  Gram -> inverse after Gauss-Jordan
  float2* Z;     // [TP][LD]  matched filter y_mrc per OFDM symbol
  float2* X;     // [TP][LD]  per-symbol solution / LAMA z
  float2* W;     // [4][UP]   Gauss-Jordan pivot row/column buffers
  float2* Sv;    // [TP][LD]  LAMA mean s
  float2* Vv;    // [TP][LD]  LAMA Onsager term v
  float2* Fb;    // [TP][LD]  LAMA posterior mean
  float* gb;     // [TP][LD]  LAMA posterior variance
  float* phi;    // [TP]
  float* coef;   // [TP]
  float* s2;     // [max(UP,TP)] linear sigma2 (or per-symbol LAMA tau)
  float* gn;     // [UP] MRC gain d / L-MMSE signal gain c
  float* dg;     // [UP] original diagonal (pivot tolerance)
  float2* num;   // FD [TP][LD] sum_c w z
  float* den;    // FD [max(UP,TP)] sum_c w
  float* harm;   // FD [max(UP,TP)] sum_c 1/sigma2
  float* wbuf;   // FD [C][max(UP,TP)] raw weights
  int* flags;    // [0] status, [1] divergence iteration
  int LD;
};

struct EpiArgs {
  int kind, u, T;
  float n0, es;
  float beta, lama_scale, damping;
  int t_max;
  bool unbias;
  int ablate;  // timing studies only (EqParams::ablate)
};

__device__ __forceinline__ void set_status(int* flags, int st) { atomicCAS(flags, 0, st); }

__device__ __forceinline__ float2 shfl2(float2 v, int src) {
  return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// One-warp ZF / L-MMSE solve (the unit epilogue of the tensor-core kernel's
// solver warps).  Lane l owns column j = l % UP of the matrix for rows
// rb + r*RS (rb = l / UP, RS = 32 / UP); the Gauss-Jordan sweep is written
// branch-free as a rank-1 update  m_ij -= c_i r_j  with
//   c_i = m_ik (i != k), c_k = p - 1;   r_j = m_kj / p (j != k), r_k = 1 + 1/p
// (this yields m_kj/p on the pivot row, -m_ik/p on the pivot column and 1/p
// on the pivot), and the pivot row / column reach the lanes by shuffles, so
// a step needs neither shared memory nor a barrier.  Padded rows / columns
// (u < UP) are the identity and stay untouched.
// NU independent units are solved together (NU = 2: their pivot chains
// interleave, hiding the shuffle / reciprocal latency of a lone warp).
template <int UP, int NU>
__device__ void linear_solve_warp_n(const Work* w, const EpiArgs* a, const float* rho, int lane) {
  constexpr int RS = 32 / UP;
  constexpr int EPT = UP * UP / 32;
  const int u = a[0].u, T = a[0].T, LD = w[0].LD;  // units share the geometry
  const int j = lane % UP, rb = lane / UP;
  float2 m[NU][EPT];
  float dgl[NU];  // original diagonal of the (at most one) diagonal element this lane owns
#pragma unroll
  for (int q = 0; q < NU; ++q) {
    dgl[q] = 1.f;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int i = rb + r * RS;
      float2 v;
      if (i < u && j < u) {
        v = w[q].G[i * LD + j];
        if (i == j) {
          v.x += rho[q];
          v.y = 0.f;
          dgl[q] = v.x;
        }
      } else {
        v = make_float2(i == j ? 1.f : 0.f, 0.f);
      }
      m[q][r] = v;
    }
  }
  const float tolf = 8.f * (float)u * FLT_EPSILON;
  bool bad[NU];
#pragma unroll
  for (int q = 0; q < NU; ++q) bad[q] = false;
  // Rotating register order: after every RS pivot steps the row registers
  // rotate by one, so the pivot row is always register 0 (static indices, no
  // selects); UP steps = EPT full rotations restore the order.  Padded steps
  // k >= u act on identity rows/columns and are no-ops.  The loop is unrolled
  // RS-fold only (small instruction footprint).
#pragma unroll 1
  for (int k0 = 0; k0 < UP; k0 += RS) {
#pragma unroll
    for (int kk = 0; kk < RS; ++kk) {
      const int k = k0 + kk;
      const int own = kk * UP + k;  // lane holding (k, k), in register 0
      const bool prow = (rb == kk);  // this lane's register 0 is the pivot row
#pragma unroll
      for (int q = 0; q < NU; ++q) {
        const float2 mk = m[q][0];
        // the pivot owner checks its pivot against the original diagonal and
        // broadcasts 1 for a failed (singular) pivot
        float pv = mk.x;
        if (lane == own && k < u && !(pv > tolf * dgl[q])) {
          bad[q] = true;
          pv = 1.f;
        }
        const float p = __shfl_sync(0xffffffffu, pv, own);
        const float rp = __frcp_rn(p);
        const float2 rkj = shfl2(mk, kk * UP + j);
        const float2 rj = (j == k) ? make_float2(1.f + rp, 0.f) : c_scale(rkj, rp);
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
          float2 ci = shfl2(m[q][r], rb * UP + k);
          if (r == 0 && prow) ci = make_float2(p - 1.f, 0.f);
          c_fms(m[q][r], ci, rj);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NU; ++q) {
      const float2 first = m[q][0];
#pragma unroll
      for (int r = 0; r + 1 < EPT; ++r) m[q][r] = m[q][r + 1];
      m[q][EPT - 1] = first;
    }
  }
#pragma unroll
  for (int q = 0; q < NU; ++q) {
    if (__any_sync(0xffffffffu, bad[q]) && lane == 0) set_status(w[q].flags, ST_SINGULAR);
#pragma unroll
    for (int r = 0; r < EPT; ++r) w[q].G[(rb + r * RS) * LD + j] = m[q][r];
  }
  __syncwarp();
  // z = A y_mrc: lane -> UE i = lane % UP, symbols t = rb, rb + RS, ...
  const int i = j;
  if (i < u) {
#pragma unroll
    for (int q = 0; q < NU; ++q) {
      const bool unb = (a[q].kind == EQ_LMMSE) && a[q].unbias;
      float2 arow[UP];
#pragma unroll
      for (int c = 0; c < UP; c += 2) {
        const float4 v = *reinterpret_cast<const float4*>(w[q].G + i * LD + c);
        arow[c] = make_float2(v.x, v.y);
        arow[c + 1] = make_float2(v.z, v.w);
      }
      const float aii = w[q].G[i * LD + i].x;
      const float cgain = 1.f - rho[q] * aii;
      const float sc = unb ? 1.f / cgain : 1.f;
      for (int t = rb; t < T; t += 2 * RS) {  // two symbols per pass: independent chains
        const int t1 = t + RS;
        const float2* z0 = w[q].Z + t * LD;
        const float2* z1 = w[q].Z + (t1 < T ? t1 : t) * LD;
        float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0, acc2 = acc0, acc3 = acc0;
#pragma unroll
        for (int c = 0; c < UP; c += 2) {
          if (c < u) {
            const float4 v0 = *reinterpret_cast<const float4*>(z0 + c);
            const float4 v1 = *reinterpret_cast<const float4*>(z1 + c);
            c_fma(acc0, arow[c], make_float2(v0.x, v0.y));
            c_fma(acc2, arow[c], make_float2(v1.x, v1.y));
            if (c + 1 < u) {
              c_fma(acc1, arow[c + 1], make_float2(v0.z, v0.w));
              c_fma(acc3, arow[c + 1], make_float2(v1.z, v1.w));
            }
          }
        }
        w[q].X[t * LD + i] = c_scale(c_add(acc0, acc1), sc);
        if (t1 < T) w[q].X[t1 * LD + i] = c_scale(c_add(acc2, acc3), sc);
      }
      if (rb == 0) {
        if (a[q].kind == EQ_ZF) {
          w[q].s2[i] = a[q].n0 * aii;
        } else {
          w[q].gn[i] = cgain;
          if (a[q].unbias && !(cgain > 0.f)) set_status(w[q].flags, ST_SINGULAR);
          w[q].s2[i] = a[q].unbias ? a[q].n0 * aii / cgain : a[q].n0 * aii;
        }
      }
    }
  }
  __syncwarp();
}

template <int UP>
__device__ void linear_solve_warp(const Work& w, const EpiArgs& a, float rho, int lane) {
  linear_solve_warp_n<UP, 1>(&w, &a, &rho, lane);
}

// ---- blocked Gauss-Jordan inverse, U = 64, 256 threads --------------------
// The same in-place sweep as the rank-1 version below (no pivoting, HPD),
// eight pivots per step, so one CTA barrier per eight pivots and a
// register-tiled rank-8 update.  Thread (ti, tj) = (tid / 16, tid % 16) owns
// the 4 x 4 tile rows 4 ti .. 4 ti + 3, cols 4 tj .. 4 tj + 3; warp w owns rows
// 8 w .. 8 w + 7.  For pivot block K = [8 b, 8 b + 8) with P = M[K,K],
// Pinv = P^-1, C = M[:,K], R = M[K,:], one step is
//     M <- M - Ct Rt,   Rt = R except Rt[:,K] = P + I,
//                       Ct = C Pinv except Ct[K,:] = I - Pinv,
// which gives Pinv on M[K,K], Pinv R on the pivot rows, -C Pinv on the pivot
// columns and M - C Pinv R elsewhere (= eight rank-1 Gauss-Jordan steps).
// Warp b owns the pivot rows of block b: right after its update for block
// b - 1 it publishes Rt_b and, with `lookahead`, inverts P_b (eight
// sequential pivots on its lanes, shuffles only) while the other warps reach
// the barrier -- the better choice with two CTAs per SM (stats_kernel);
// without it every warp inverts P_b itself after the barrier (one CTA per SM,
// the streaming kernel: no warp idles).  Every warp then forms Ct for its own
// eight rows, whose C entries it holds itself.  The sequential pivots of P are those of the rank-1 sweep,
// so the singularity test (pivot below 8 u eps of its original diagonal) is
// unchanged.  The scratch (Rt and Pinv, double-buffered by block parity, and
// per-warp C / Ct) lives in the G area, free while the matrix sits in
// registers; A = M^-1 is written back to G at the end.
template <bool lookahead>
__device__ __forceinline__ void gj64_blocked(const Work& w, int u, float rho, int tid) {
  const int LD = w.LD;
  const int ti = tid >> 4, tj = tid & 15, warp = tid >> 5, lane = tid & 31;
  float2 m[4][4];
  // the tile's two 16-byte halves per row, the lanes with (tj / 4) odd taking
  // the second half first: the eight lanes of a quarter-warp then touch eight
  // distinct bank groups (the element-wise loads were 4-way conflicted)
  const bool swp = (tj >> 2) & 1;
  if (u == 64) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = 4 * ti + r;
      const float2* row = w.G + i * LD + 4 * tj;
      const float4 a0 = *reinterpret_cast<const float4*>(row + (swp ? 2 : 0));
      const float4 a1 = *reinterpret_cast<const float4*>(row + (swp ? 0 : 2));
      const float4 lo = swp ? a1 : a0, hi = swp ? a0 : a1;
      m[r][0] = make_float2(lo.x, lo.y);
      m[r][1] = make_float2(lo.z, lo.w);
      m[r][2] = make_float2(hi.x, hi.y);
      m[r][3] = make_float2(hi.z, hi.w);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (4 * ti + r == 4 * tj + c) {
          m[r][c].x += rho;
          m[r][c].y = 0.f;
          w.dg[4 * ti + r] = m[r][c].x;
        }
      }
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * ti + r, j = 4 * tj + c;
        float2 v = make_float2(i == j ? 1.f : 0.f, 0.f);  // padding: identity
        if (i < u && j < u) {
          v = w.G[i * LD + j];
          if (i == j) {
            v.x += rho;
            v.y = 0.f;
            w.dg[i] = v.x;
          }
        }
        m[r][c] = v;
      }
  }
  __syncthreads();  // G is scratch from here on
  // Rt rows are stored column-permuted: columns {4t, 4t+1} at 2t, columns
  // {4t+2, 4t+3} at 32 + 2t, so the eight lanes of a quarter-warp read eight
  // consecutive 16-byte chunks (conflict-free; the natural order put two of
  // them on each bank group: 2x the wavefronts on the update's hottest loads)
  float2* rt = w.G;                                  // [2][8][64]  Rt of the step (block parity)
  auto rtc = [](int j) { return ((j >> 2) << 1) + ((j & 2) << 4) + (j & 1); };
  float2* pinvb = w.G + 2 * 512;                     // [2][8][8]   Pinv of the step (look-ahead)
  float2* cb = w.G + 2 * 512 + 2 * 64 + warp * 192;  // per warp: C [8][8], Ct [8][8], own Pinv [8][8]
  float2* ctb = cb + 64;
  float2* pown = cb + 128;
  const float tolf = 8.f * (float)u * FLT_EPSILON;
  const int nblk = (u + 7) >> 3;
  bool bad = false;
  // warp b: publish Rt_b from its rows
  auto publish = [&](int b) {
    float2* rb = rt + (b & 1) * 512;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int lr = 4 * (ti & 1) + r;
      float2 v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[c] = m[r][c];
        if (4 * tj + c == 8 * b + lr) v[c].x += 1.f;
      }
      *reinterpret_cast<float4*>(rb + lr * 64 + 2 * tj) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
      *reinterpret_cast<float4*>(rb + lr * 64 + 32 + 2 * tj) = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
    }
  };
  // Pinv_b = (Rt_b[:, K] - I)^-1 into pb (one warp)
  auto invert = [&](int b, float2* pb) {
    const float2* rb = rt + (b & 1) * 512;
    // lane l holds P[pr][pc], P[pr + 1][pc] (pr = 2 (l / 8), pc = l % 8)
    const int pc = lane & 7, pr = 2 * (lane >> 3);
    const int pcol = rtc(8 * b + pc);
    float2 q0 = rb[pr * 64 + pcol], q1 = rb[(pr + 1) * 64 + pcol];
    if (pr == pc) q0.x -= 1.f;
    if (pr + 1 == pc) q1.x -= 1.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int src_col = (pr >> 1) * 8 + k;  // lane holding (pr, k), (pr + 1, k)
      const int src_row = (k >> 1) * 8 + pc;  // lane holding (k, pc)
      const int src_piv = (k >> 1) * 8 + k;   // lane holding (k, k)
      const float c0x = __shfl_sync(0xffffffffu, q0.x, src_col), c0y = __shfl_sync(0xffffffffu, q0.y, src_col);
      const float c1x = __shfl_sync(0xffffffffu, q1.x, src_col), c1y = __shfl_sync(0xffffffffu, q1.y, src_col);
      const float rkx = __shfl_sync(0xffffffffu, (k & 1) ? q1.x : q0.x, src_row);
      const float rky = __shfl_sync(0xffffffffu, (k & 1) ? q1.y : q0.y, src_row);
      float p = __shfl_sync(0xffffffffu, (k & 1) ? q1.x : q0.x, src_piv);
      const int kg = 8 * b + k;
      if (kg < u && !(p > tolf * w.dg[kg])) {
        bad = true;
        p = 1.f;
      }
      const float rp = rcp_pivot(p);
      const float2 rj = (pc == k) ? make_float2(1.f + rp, 0.f) : make_float2(rkx * rp, rky * rp);
      const float2 ci0 = (pr == k) ? make_float2(p - 1.f, 0.f) : make_float2(c0x, c0y);
      const float2 ci1 = (pr + 1 == k) ? make_float2(p - 1.f, 0.f) : make_float2(c1x, c1y);
      c_fms(q0, ci0, rj);
      c_fms(q1, ci1, rj);
    }
    pb[pr * 8 + pc] = q0;
    pb[(pr + 1) * 8 + pc] = q1;
  };
  if (warp == 0) {
    publish(0);
    if constexpr (lookahead) {
      __syncwarp();
      invert(0, pinvb);
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int b = 0; b < nblk; ++b) {
    const float2* rb = rt + (b & 1) * 512;
    const float2* pb = pinvb + (b & 1) * 64;
    if constexpr (!lookahead) {  // every warp inverts P_b itself (no warp idles at the barrier)
      invert(b, pown);
      pb = pown;
    }
    // this warp's rows of the pivot columns
    if ((tj >> 1) == b) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int lr = 4 * (ti & 1) + r, c0 = 4 * (tj & 1);
        *reinterpret_cast<float4*>(cb + lr * 8 + c0) = make_float4(m[r][0].x, m[r][0].y, m[r][1].x, m[r][1].y);
        *reinterpret_cast<float4*>(cb + lr * 8 + c0 + 2) = make_float4(m[r][2].x, m[r][2].y, m[r][3].x, m[r][3].y);
      }
    }
    __syncwarp();
    // Ct for the warp's rows: lane -> row lr = lane / 4, columns 2 (lane % 4) + {0, 1}
    {
      const int lr = lane >> 2, c0 = 2 * (lane & 3);
      float2 a0 = make_float2(0.f, 0.f), a1 = a0;
      if (warp == b) {
        const float4 pv = *reinterpret_cast<const float4*>(pb + lr * 8 + c0);
        a0 = make_float2((lr == c0 ? 1.f : 0.f) - pv.x, -pv.y);
        a1 = make_float2((lr == c0 + 1 ? 1.f : 0.f) - pv.z, -pv.w);
      } else {
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const float2 cv = cb[lr * 8 + l];
          const float4 pv = *reinterpret_cast<const float4*>(pb + l * 8 + c0);
          c_fma(a0, cv, make_float2(pv.x, pv.y));
          c_fma(a1, cv, make_float2(pv.z, pv.w));
        }
      }
      *reinterpret_cast<float4*>(ctb + lr * 8 + c0) = make_float4(a0.x, a0.y, a1.x, a1.y);
    }
    __syncwarp();
    // rank-8 update of the tile
#pragma unroll
    for (int l = 0; l < 8; l += 2) {
      float2 cr[4][2], rr[2][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float4 v = *reinterpret_cast<const float4*>(ctb + (4 * (ti & 1) + r) * 8 + l);
        cr[r][0] = make_float2(v.x, v.y);
        cr[r][1] = make_float2(v.z, v.w);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float4 v0 = *reinterpret_cast<const float4*>(rb + (l + e) * 64 + 2 * tj);
        const float4 v1 = *reinterpret_cast<const float4*>(rb + (l + e) * 64 + 32 + 2 * tj);
        rr[e][0] = make_float2(v0.x, v0.y);
        rr[e][1] = make_float2(v0.z, v0.w);
        rr[e][2] = make_float2(v1.x, v1.y);
        rr[e][3] = make_float2(v1.z, v1.w);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          c_fms2(m[r][c], cr[r][0], rr[0][c]);
          c_fms2(m[r][c], cr[r][1], rr[1][c]);
        }
    }
    __syncwarp();  // the warp's Ct / C / Pinv reads are done before the next block rewrites them
    if (warp == b + 1 && b + 1 < nblk) {
      publish(b + 1);
      if constexpr (lookahead) {
        __syncwarp();
        invert(b + 1, pinvb + ((b + 1) & 1) * 64);
      }
    }
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) set_status(w.flags, ST_SINGULAR);
  // (the last barrier of the loop: every scratch read is done)
  if (u == 64) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float2* row = w.G + (4 * ti + r) * LD + 4 * tj;
      const float4 lo = make_float4(m[r][0].x, m[r][0].y, m[r][1].x, m[r][1].y);
      const float4 hi = make_float4(m[r][2].x, m[r][2].y, m[r][3].x, m[r][3].y);
      *reinterpret_cast<float4*>(row + (swp ? 2 : 0)) = swp ? hi : lo;
      *reinterpret_cast<float4*>(row + (swp ? 0 : 2)) = swp ? lo : hi;
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = 4 * ti + r;
    if (i < u) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = 4 * tj + c;
        if (j < u) w.G[i * LD + j] = m[r][c];
      }
    }
  }
}

// The same blocked sweep on a 128-thread team with 8 x 4 tiles: thread
// (ti, tj), ti = tid / 16 in [0, 8), tj = tid % 16, holds rows 8 ti .. 8 ti + 7
// (pivot block ti) x cols 4 tj .. 4 tj + 3; warp w owns pivot blocks 2w, 2w + 1.
// Per pivot column l of the rank-8 update a thread reads its block's 8 Ct
// values (stored transposed: one broadcast float4 run per quarter-warp) and 4
// Rt values: 12 words per 32 complex MACs (5.3 FMA per word; the 4 x 4 tiles
// of gj64_blocked: 4), and four items share an SM.
template <bool lookahead>
__device__ __forceinline__ void gj64_8x4(const Work& w, int u, float rho, int tid) {
  const int LD = w.LD;
  const int ti = tid >> 4, tj = tid & 15, warp = tid >> 5, lane = tid & 31;
  float2 m[8][4];
  const bool swp = (tj >> 2) & 1;  // rotated 16-byte halves: conflict-free quarter-warps
  if (u == 64) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float2* row = w.G + (8 * ti + r) * LD + 4 * tj;
      const float4 a0 = *reinterpret_cast<const float4*>(row + (swp ? 2 : 0));
      const float4 a1 = *reinterpret_cast<const float4*>(row + (swp ? 0 : 2));
      const float4 lo = swp ? a1 : a0, hi = swp ? a0 : a1;
      m[r][0] = make_float2(lo.x, lo.y);
      m[r][1] = make_float2(lo.z, lo.w);
      m[r][2] = make_float2(hi.x, hi.y);
      m[r][3] = make_float2(hi.z, hi.w);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (8 * ti + r == 4 * tj + c) {
          m[r][c].x += rho;
          m[r][c].y = 0.f;
          w.dg[8 * ti + r] = m[r][c].x;
        }
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 8 * ti + r, j = 4 * tj + c;
        float2 v = make_float2(i == j ? 1.f : 0.f, 0.f);  // padding: identity
        if (i < u && j < u) {
          v = w.G[i * LD + j];
          if (i == j) {
            v.x += rho;
            v.y = 0.f;
            w.dg[i] = v.x;
          }
        }
        m[r][c] = v;
      }
  }
  __syncthreads();  // G is scratch from here on
  // Rt rows column-permuted as in gj64_blocked (conflict-free quarter-warps)
  float2* rt = w.G;                                   // [2][8][64]  Rt of the step (block parity)
  auto rtc = [](int j) { return ((j >> 2) << 1) + ((j & 2) << 4) + (j & 1); };
  float2* pinvb = w.G + 2 * 512;                      // [2][8][8]   Pinv of the step (look-ahead)
  float2* cb = w.G + 2 * 512 + 2 * 64 + warp * 320;   // per warp: C [16][8], Ct^T [8][16], own Pinv [8][8]
  float2* ctT = cb + 128;
  float2* pown = cb + 256;
  const float tolf = 8.f * (float)u * FLT_EPSILON;
  const int nblk = (u + 7) >> 3;
  bool bad = false;
  auto publish = [&](int b) {  // the 16 threads of block b's rows
    if (ti != b) return;
    float2* rb = rt + (b & 1) * 512;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float2 v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[c] = m[r][c];
        if (4 * tj + c == 8 * b + r) v[c].x += 1.f;
      }
      *reinterpret_cast<float4*>(rb + r * 64 + 2 * tj) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
      *reinterpret_cast<float4*>(rb + r * 64 + 32 + 2 * tj) = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
    }
  };
  auto invert = [&](int b, float2* pb) {  // Pinv_b = (Rt_b[:, K] - I)^-1 (one warp)
    const float2* rb = rt + (b & 1) * 512;
    const int pc = lane & 7, pr = 2 * (lane >> 3);
    const int pcol = rtc(8 * b + pc);
    float2 q0 = rb[pr * 64 + pcol], q1 = rb[(pr + 1) * 64 + pcol];
    if (pr == pc) q0.x -= 1.f;
    if (pr + 1 == pc) q1.x -= 1.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int src_col = (pr >> 1) * 8 + k;
      const int src_row = (k >> 1) * 8 + pc;
      const int src_piv = (k >> 1) * 8 + k;
      const float c0x = __shfl_sync(0xffffffffu, q0.x, src_col), c0y = __shfl_sync(0xffffffffu, q0.y, src_col);
      const float c1x = __shfl_sync(0xffffffffu, q1.x, src_col), c1y = __shfl_sync(0xffffffffu, q1.y, src_col);
      const float rkx = __shfl_sync(0xffffffffu, (k & 1) ? q1.x : q0.x, src_row);
      const float rky = __shfl_sync(0xffffffffu, (k & 1) ? q1.y : q0.y, src_row);
      float p = __shfl_sync(0xffffffffu, (k & 1) ? q1.x : q0.x, src_piv);
      const int kg = 8 * b + k;
      if (kg < u && !(p > tolf * w.dg[kg])) {
        bad = true;
        p = 1.f;
      }
      const float rp = rcp_pivot(p);
      const float2 rj = (pc == k) ? make_float2(1.f + rp, 0.f) : make_float2(rkx * rp, rky * rp);
      const float2 ci0 = (pr == k) ? make_float2(p - 1.f, 0.f) : make_float2(c0x, c0y);
      const float2 ci1 = (pr + 1 == k) ? make_float2(p - 1.f, 0.f) : make_float2(c1x, c1y);
      c_fms(q0, ci0, rj);
      c_fms(q1, ci1, rj);
    }
    pb[pr * 8 + pc] = q0;
    pb[(pr + 1) * 8 + pc] = q1;
  };
  if (warp == 0) {
    publish(0);
    if constexpr (lookahead) {
      __syncwarp();
      invert(0, pinvb);
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int b = 0; b < nblk; ++b) {
    const float2* rb = rt + (b & 1) * 512;
    const float2* pb = pinvb + (b & 1) * 64;
    if constexpr (!lookahead) {
      invert(b, pown);
      pb = pown;
    }
    // this warp's 16 rows of the pivot columns (threads holding columns 8b..8b+7)
    if ((tj >> 1) == b) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int lr = 8 * (ti & 1) + r, c0 = 4 * (tj & 1);
        *reinterpret_cast<float4*>(cb + lr * 8 + c0) = make_float4(m[r][0].x, m[r][0].y, m[r][1].x, m[r][1].y);
        *reinterpret_cast<float4*>(cb + lr * 8 + c0 + 2) = make_float4(m[r][2].x, m[r][2].y, m[r][3].x, m[r][3].y);
      }
    }
    __syncwarp();
    // Ct^T for the warp's rows: lane -> row lr = lane / 2, columns 4 (lane % 2) + {0..3};
    // the pivot block's own rows take I - Pinv
    {
      const int lr = lane >> 1, c0 = 4 * (lane & 1);
      float2 a[4];
      if ((b >> 1) == warp && (lr >> 3) == (b & 1)) {
        const int rl = lr & 7;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 pv = pb[rl * 8 + c0 + c];
          a[c] = make_float2((rl == c0 + c ? 1.f : 0.f) - pv.x, -pv.y);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = make_float2(0.f, 0.f);
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const float2 cv = cb[lr * 8 + l];
          const float4 p0 = *reinterpret_cast<const float4*>(pb + l * 8 + c0);
          const float4 p1 = *reinterpret_cast<const float4*>(pb + l * 8 + c0 + 2);
          c_fma2(a[0], cv, make_float2(p0.x, p0.y));
          c_fma2(a[1], cv, make_float2(p0.z, p0.w));
          c_fma2(a[2], cv, make_float2(p1.x, p1.y));
          c_fma2(a[3], cv, make_float2(p1.z, p1.w));
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) ctT[(c0 + c) * 16 + lr] = a[c];
    }
    __syncwarp();
    // rank-8 update of the tile
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      float2 cr[8], rr[4];
      const float2* cl = ctT + l * 16 + 8 * (ti & 1);
#pragma unroll
      for (int r = 0; r < 8; r += 2) {
        const float4 v = *reinterpret_cast<const float4*>(cl + r);
        cr[r] = make_float2(v.x, v.y);
        cr[r + 1] = make_float2(v.z, v.w);
      }
      const float4 v0 = *reinterpret_cast<const float4*>(rb + l * 64 + 2 * tj);
      const float4 v1 = *reinterpret_cast<const float4*>(rb + l * 64 + 32 + 2 * tj);
      rr[0] = make_float2(v0.x, v0.y);
      rr[1] = make_float2(v0.z, v0.w);
      rr[2] = make_float2(v1.x, v1.y);
      rr[3] = make_float2(v1.z, v1.w);
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) c_fms2(m[r][c], cr[r], rr[c]);
    }
    __syncwarp();  // the warp's Ct / C / Pinv reads are done before the next block rewrites them
    if (warp == ((b + 1) >> 1) && b + 1 < nblk) {
      publish(b + 1);
      if constexpr (lookahead) {
        __syncwarp();
        invert(b + 1, pinvb + ((b + 1) & 1) * 64);
      }
    }
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) set_status(w.flags, ST_SINGULAR);
  if (u == 64) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float2* row = w.G + (8 * ti + r) * LD + 4 * tj;
      const float4 lo = make_float4(m[r][0].x, m[r][0].y, m[r][1].x, m[r][1].y);
      const float4 hi = make_float4(m[r][2].x, m[r][2].y, m[r][3].x, m[r][3].y);
      *reinterpret_cast<float4*>(row + (swp ? 2 : 0)) = swp ? hi : lo;
      *reinterpret_cast<float4*>(row + (swp ? 0 : 2)) = swp ? lo : hi;
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = 8 * ti + r;
    if (i < u) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = 4 * tj + c;
        if (j < u) w.G[i * LD + j] = m[r][c];
      }
    }
  }
}

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
// memory (double-buffered, one team barrier per step).  A pivot below
// 8*u*eps of its original diagonal is SingularGramError: the fp32 counterpart
// of zpotrf's "not positive definite" (a rank-deficient fp32 Gram leaves
// rounding noise ~eps*G_jj instead of an exact zero).
// LA: the blocked U = 64 solve inverts each pivot block on one warp (look-ahead;
// for kernels with two CTAs per SM), else on every warp
template <int UP, class TM, bool LA = false, bool XZ = false>
__device__ void linear_unit(const Work& w, const EpiArgs& a, const TM& tm) {
  constexpr int NT = TM::N;
  const int tid = tm.t;
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
    tm.sync();
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      w.X[t * LD + i] = c_scale(w.Z[t * LD + i], 1.f / w.gn[i]);
    }
    tm.sync();
    return;
  }
  const float rho = (a.kind == EQ_LMMSE) ? a.n0 / a.es : 0.f;
  if constexpr (NT == 32 && UP <= 32) {
    linear_solve_warp<UP>(w, a, rho, tid);
    return;
  }
  if constexpr (UP == 64 && NT == 256) {
    gj64_blocked<LA>(w, u, rho, tid);  // eight pivots per barrier
  } else if constexpr (UP == 64 && NT == 128) {
    gj64_8x4<LA>(w, u, rho, tid);  // 8 x 4 tiles, 128-thread team
  } else {
    // thread -> elements (i0 + r*RS, j): fixed column, RS-strided rows.  The
    // sweep is the branch-free rank-1 update of linear_solve_warp_n
    //   m_ij -= c_i r_j,  c_i = m_ik (i != k), c_k = p - 1,  r_j = m_kj / p (j != k), r_k = 1 + 1/p,
    // with rotating register order: after every RS steps the row registers
    // rotate by one, so the pivot row is always register 0; the pivot column
    // is published by register slot ([i0][slot], slot = original register).
    constexpr int RS = (NT >= UP) ? NT / UP : 1;
    constexpr int EPT = (UP * UP + NT - 1) / NT;
    static_assert((EPT & (EPT - 1)) == 0, "rows per thread must be a power of two");
    const int j = tid % UP;
    const int i0 = tid / UP;
    const bool live = (i0 < UP);  // threads beyond UP*UP elements (NT > UP*UP) idle
    float2 m[EPT];
    float2* rowb = w.W;           // [2][UP] pivot rows (double-buffered)
    float2* colb = w.W + 2 * UP;  // [2][UP] pivot columns, [i0][slot]
    const float tolf = 8.f * (float)u * FLT_EPSILON;
  #pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int i = i0 + r * RS;
      float2 v = make_float2(i == j ? 1.f : 0.f, 0.f);  // padding: identity
      if (i < u && j < u) {
        v = w.G[i * LD + j];
        if (i == j) {
          v.x += rho;
          v.y = 0.f;
          w.dg[i] = v.x;
        }
      }
      m[r] = v;
    }
    for (int k0 = 0; k0 < UP; k0 += RS) {
      for (int kk = 0; kk < RS && k0 + kk < UP; ++kk) {
        const int k = k0 + kk;
        float2* rk = rowb + (k & 1) * UP;
        float2* ck = colb + (k & 1) * UP;
        if (live) {
          if (i0 == kk) rk[j] = m[0];
          if (j == k) {
            // slot = register index: readers with the same i0 share the writer's
            // rotation state, so register r of every such thread holds the same row
            if constexpr (EPT >= 2) {
  #pragma unroll
              for (int r = 0; r < EPT; r += 2)
                *reinterpret_cast<float4*>(ck + i0 * EPT + r) = make_float4(m[r].x, m[r].y, m[r + 1].x, m[r + 1].y);
            } else {
              ck[i0] = m[0];
            }
          }
        }
        tm.sync();
        float p = rk[k].x;
        if (k < u && !(p > tolf * w.dg[k])) {
          if (tid == 0) set_status(w.flags, ST_SINGULAR);
          p = 1.f;
        }
        if (k >= u) p = 1.f;  // padded step: identity pivot
        const float rp = __frcp_rn(p);  // = 1.f / p (correctly rounded), no division slow path
        if (live) {
          const float2 rj = (j == k) ? make_float2(1.f + rp, 0.f) : c_scale(rk[j], rp);
          if constexpr (EPT >= 2) {
  #pragma unroll
            for (int r = 0; r < EPT; r += 2) {
              const float4 c2 = *reinterpret_cast<const float4*>(ck + i0 * EPT + r);
              float2 ci = make_float2(c2.x, c2.y);
              if (r == 0 && i0 == kk) ci = make_float2(p - 1.f, 0.f);
              c_fms(m[r], ci, rj);
              c_fms(m[r + 1], make_float2(c2.z, c2.w), rj);
            }
          } else {
            const float2 ci = (i0 == kk) ? make_float2(p - 1.f, 0.f) : ck[i0];
            c_fms(m[0], ci, rj);
          }
        }
      }
      if (live) {
        const float2 first = m[0];
  #pragma unroll
        for (int r = 0; r + 1 < EPT; ++r) m[r] = m[r + 1];
        m[EPT - 1] = first;
      }
    }
    if (live) {
  #pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const int i = i0 + r * RS;
        if (i < u && j < u) w.G[i * LD + j] = m[r];
      }
    }
  }
  tm.sync();
  // z = A y_mrc per OFDM symbol (+ unbiasing), two symbols per thread sharing
  // the A row; rows are 16-byte aligned (LD even) -> float4 loads
  const bool unb = (a.kind == EQ_LMMSE) && a.unbias;
  const int th = (T + 1) / 2;
  if (UP == 64 && !(u & 1)) {
    // 2 x 2 register tiles: rows ip, ip + u/2 and symbols t0, t0 + th share
    // each A-row / y load (4 float4 loads per 8 complex MACs instead of 3 per 4;
    // U = 64 only: at UP = 32 the tiles cost stats_kernel<32> its second CTA per SM)
    const int hu = u >> 1;
    auto tile = [&](int e, float2& c00, float2& c01, float2& c10, float2& c11) {
      const int t0 = e / hu, ip = e - t0 * hu;
      const int t1 = t0 + th;
      const float2* ar0 = w.G + ip * LD;
      const float2* ar1 = w.G + (ip + hu) * LD;
      const float2* z0 = w.Z + t0 * LD;
      const float2* z1 = w.Z + (t1 < T ? t1 : t0) * LD;
      c00 = make_float2(0.f, 0.f);  // [row][symbol]
      c01 = c00;
      c10 = c00;
      c11 = c00;
      for (int jj = 0; jj < u; jj += 2) {
        const float4 a0 = *reinterpret_cast<const float4*>(ar0 + jj);
        const float4 a1 = *reinterpret_cast<const float4*>(ar1 + jj);
        const float4 b0 = *reinterpret_cast<const float4*>(z0 + jj);
        const float4 b1 = *reinterpret_cast<const float4*>(z1 + jj);
        c_fma2(c00, make_float2(a0.x, a0.y), make_float2(b0.x, b0.y));
        c_fma2(c01, make_float2(a0.x, a0.y), make_float2(b1.x, b1.y));
        c_fma2(c10, make_float2(a1.x, a1.y), make_float2(b0.x, b0.y));
        c_fma2(c11, make_float2(a1.x, a1.y), make_float2(b1.x, b1.y));
        c_fma2(c00, make_float2(a0.z, a0.w), make_float2(b0.z, b0.w));
        c_fma2(c01, make_float2(a0.z, a0.w), make_float2(b1.z, b1.w));
        c_fma2(c10, make_float2(a1.z, a1.w), make_float2(b0.z, b0.w));
        c_fma2(c11, make_float2(a1.z, a1.w), make_float2(b1.z, b1.w));
      }
      if (unb) {
        const float rc0 = 1.f / (1.f - rho * ar0[ip].x), rc1 = 1.f / (1.f - rho * ar1[ip + hu].x);
        c00 = c_scale(c00, rc0);
        c01 = c_scale(c01, rc0);
        c10 = c_scale(c10, rc1);
        c11 = c_scale(c11, rc1);
      }
    };
    auto put = [&](int e, float2 c00, float2 c01, float2 c10, float2 c11) {
      const int t0 = e / hu, ip = e - t0 * hu;
      const int t1 = t0 + th;
      w.X[t0 * LD + ip] = c00;
      w.X[t0 * LD + ip + hu] = c10;
      if (t1 < T) {
        w.X[t1 * LD + ip] = c01;
        w.X[t1 * LD + ip + hu] = c11;
      }
    };
    if constexpr (XZ) {  // X overwrites y_mrc (make_work_layout x_in_z, T <= 16): tiles held across a barrier
      static_assert(NT == 128, "X in Z: two 2 x 2 tiles per thread of a 128-thread team");
      // both tiles of the thread in one pass (th * hu <= 256 = 2 NT); a missing
      // second tile recomputes the first and is not stored
      const int e0 = tid, e1 = (tid + NT < th * hu) ? tid + NT : tid;
      const int t0a = e0 / hu, ipa = e0 - t0a * hu, t0b = e1 / hu, ipb = e1 - t0b * hu;
      const float2* ra0 = w.G + ipa * LD;
      const float2* ra1 = w.G + (ipa + hu) * LD;
      const float2* rb0 = w.G + ipb * LD;
      const float2* rb1 = w.G + (ipb + hu) * LD;
      const float2* za0 = w.Z + t0a * LD;
      const float2* za1 = w.Z + (t0a + th < T ? t0a + th : t0a) * LD;
      const float2* zb0 = w.Z + t0b * LD;
      const float2* zb1 = w.Z + (t0b + th < T ? t0b + th : t0b) * LD;
      float2 ha[4], hb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) ha[q] = hb[q] = make_float2(0.f, 0.f);
      const bool live0 = e0 < th * hu;
      for (int jj = 0; jj < u; jj += 2) {
        const float4 a0 = *reinterpret_cast<const float4*>(ra0 + jj);
        const float4 a1 = *reinterpret_cast<const float4*>(ra1 + jj);
        const float4 b0 = *reinterpret_cast<const float4*>(za0 + jj);
        const float4 b1 = *reinterpret_cast<const float4*>(za1 + jj);
        const float4 c0 = *reinterpret_cast<const float4*>(rb0 + jj);
        const float4 c1 = *reinterpret_cast<const float4*>(rb1 + jj);
        const float4 d0 = *reinterpret_cast<const float4*>(zb0 + jj);
        const float4 d1 = *reinterpret_cast<const float4*>(zb1 + jj);
        c_fma2(ha[0], make_float2(a0.x, a0.y), make_float2(b0.x, b0.y));
        c_fma2(ha[1], make_float2(a0.x, a0.y), make_float2(b1.x, b1.y));
        c_fma2(ha[2], make_float2(a1.x, a1.y), make_float2(b0.x, b0.y));
        c_fma2(ha[3], make_float2(a1.x, a1.y), make_float2(b1.x, b1.y));
        c_fma2(ha[0], make_float2(a0.z, a0.w), make_float2(b0.z, b0.w));
        c_fma2(ha[1], make_float2(a0.z, a0.w), make_float2(b1.z, b1.w));
        c_fma2(ha[2], make_float2(a1.z, a1.w), make_float2(b0.z, b0.w));
        c_fma2(ha[3], make_float2(a1.z, a1.w), make_float2(b1.z, b1.w));
        c_fma2(hb[0], make_float2(c0.x, c0.y), make_float2(d0.x, d0.y));
        c_fma2(hb[1], make_float2(c0.x, c0.y), make_float2(d1.x, d1.y));
        c_fma2(hb[2], make_float2(c1.x, c1.y), make_float2(d0.x, d0.y));
        c_fma2(hb[3], make_float2(c1.x, c1.y), make_float2(d1.x, d1.y));
        c_fma2(hb[0], make_float2(c0.z, c0.w), make_float2(d0.z, d0.w));
        c_fma2(hb[1], make_float2(c0.z, c0.w), make_float2(d1.z, d1.w));
        c_fma2(hb[2], make_float2(c1.z, c1.w), make_float2(d0.z, d0.w));
        c_fma2(hb[3], make_float2(c1.z, c1.w), make_float2(d1.z, d1.w));
      }
      if (unb) {
        const float sa0 = 1.f / (1.f - rho * ra0[ipa].x), sa1 = 1.f / (1.f - rho * ra1[ipa + hu].x);
        const float sb0 = 1.f / (1.f - rho * rb0[ipb].x), sb1 = 1.f / (1.f - rho * rb1[ipb + hu].x);
        ha[0] = c_scale(ha[0], sa0);
        ha[1] = c_scale(ha[1], sa0);
        ha[2] = c_scale(ha[2], sa1);
        ha[3] = c_scale(ha[3], sa1);
        hb[0] = c_scale(hb[0], sb0);
        hb[1] = c_scale(hb[1], sb0);
        hb[2] = c_scale(hb[2], sb1);
        hb[3] = c_scale(hb[3], sb1);
      }
      tm.sync();
      if (live0) put(e0, ha[0], ha[1], ha[2], ha[3]);
      if (e1 != e0) put(e1, hb[0], hb[1], hb[2], hb[3]);
    } else {
      for (int e = tid; e < th * hu; e += NT) {
        float2 c00, c01, c10, c11;
        tile(e, c00, c01, c10, c11);
        put(e, c00, c01, c10, c11);
      }
    }
  } else
  for (int e = tid; e < th * u; e += NT) {
    const int t0 = e / u, i = e - t0 * u;
    const int t1 = t0 + th;
    const float2* arow = w.G + i * LD;
    const float2* z0 = w.Z + t0 * LD;
    const float2* z1 = w.Z + (t1 < T ? t1 : t0) * LD;
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
    for (int jj = 0; jj < u; jj += 2) {
      const float4 av = *reinterpret_cast<const float4*>(arow + jj);
      const float4 b0 = *reinterpret_cast<const float4*>(z0 + jj);
      const float4 b1 = *reinterpret_cast<const float4*>(z1 + jj);
      c_fma2(acc0, make_float2(av.x, av.y), make_float2(b0.x, b0.y));
      c_fma2(acc1, make_float2(av.x, av.y), make_float2(b1.x, b1.y));
      if (jj + 1 < u) {
        c_fma2(acc0, make_float2(av.z, av.w), make_float2(b0.z, b0.w));
        c_fma2(acc1, make_float2(av.z, av.w), make_float2(b1.z, b1.w));
      }
    }
    if (unb) {
      const float rc = 1.f / (1.f - rho * arow[i].x);
      acc0 = c_scale(acc0, rc);
      acc1 = c_scale(acc1, rc);
    }
    w.X[t0 * LD + i] = acc0;
    if (t1 < T) w.X[t1 * LD + i] = acc1;
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
  tm.sync();
}

// ---- LAMA, group-owned symbols (u <= 32) -----------------------------------
// The T recursions of lama_equalize are independent per OFDM symbol and only
// share G (read-only), so each group of GS lanes (GS = u rounded up to a power
// of two, within one warp) owns whole symbols: lane i keeps z, s, v of UE i in
// registers, the s rows are published through shared memory for the matvec
// (broadcast reads), and the per-symbol mean of g is a shuffle reduction --
// no team barrier inside the t_max iterations.  A group can run K symbols'
// recursions interleaved (independent dependency chains, one G load feeding
// all); K = 1 measured best (K = 2 costs the second CTA per SM).  lama_scale
// is applied to the matvec result and to y_mrc
// instead of rescaling G in place.
template <int GS, int PL, class TM>
__device__ void lama_unit_groups(const Work& w, const EpiArgs& a, const ConstParams& cp, float2* tr_z, float2* tr_s,
                                 float2* tr_v, float* tr_phi, const TM& tm, bool herm) {
  constexpr int NT = TM::N;
  constexpr int NG = NT / GS;  // groups in the team
  constexpr int K = 1;         // symbols per group and round (2: 169 regs, one CTA per SM, slower)
  const int tid = tm.t;
  const int i = tid & (GS - 1), g = tid / GS;
  const int u = a.u, T = a.T, LD = w.LD;
  const int ic = i < u ? i : 0;
  const float sc = a.lama_scale;
  const float n0 = a.n0 * sc;
  const float beta = a.beta, damp = a.damping;
  const float inv_u = 1.f / (float)u;
  // warp-uniform trip count: slots without a symbol in the last round run a
  // clamped symbol and write nothing (the shuffles need every lane)
  const int rounds = (T + K * NG - 1) / (K * NG);
  for (int r = 0; r < rounds; ++r) {
    int t[K];
    bool act[K], live[K];
    const float2* srow[K];
    float2 zy[K], s[K], v[K], z[K];
    float phi[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int tq = g + (r * K + k) * NG;
      live[k] = tq < T;
      t[k] = live[k] ? tq : T - 1;
      act[k] = live[k] && i < u;
      srow[k] = w.Sv + t[k] * LD;
      zy[k] = c_scale(w.Z[t[k] * LD + ic], sc);
      s[k] = cp.mean;
      v[k] = make_float2(0.f, 0.f);
      phi[k] = cp.es;
      if (act[k]) w.Sv[t[k] * LD + i] = s[k];
    }
    __syncwarp();
    for (int it = 1;; ++it) {
      // z = y_mrc + (I - G) s + v
      float2 m[K];
#pragma unroll
      for (int k = 0; k < K; ++k) m[k] = make_float2(0.f, 0.f);
      int j = 0;
      if (herm) {
#pragma unroll 2
        for (; j + 1 < u; j += 2) {
          const float2 g0 = w.G[j * LD + ic], g1 = w.G[(j + 1) * LD + ic];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float4 sj = *reinterpret_cast<const float4*>(srow[k] + j);
            c_fma_conj(m[k], g0, make_float2(sj.x, sj.y));
            c_fma_conj(m[k], g1, make_float2(sj.z, sj.w));
          }
        }
        if (j < u) {
          const float2 g0 = w.G[j * LD + ic];
#pragma unroll
          for (int k = 0; k < K; ++k) c_fma_conj(m[k], g0, srow[k][j]);
        }
      } else {
        const float2* grow = w.G + ic * LD;
#pragma unroll 2
        for (; j + 1 < u; j += 2) {
          const float4 gj = *reinterpret_cast<const float4*>(grow + j);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float4 sj = *reinterpret_cast<const float4*>(srow[k] + j);
            c_fma(m[k], make_float2(gj.x, gj.y), make_float2(sj.x, sj.y));
            c_fma(m[k], make_float2(gj.z, gj.w), make_float2(sj.z, sj.w));
          }
        }
        if (j < u) {
#pragma unroll
          for (int k = 0; k < K; ++k) c_fma(m[k], grow[j], srow[k][j]);
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        z[k] = c_sub(c_add(zy[k], c_add(s[k], v[k])), c_scale(m[k], sc));
        if (act[k] && (!c_finite(z[k]) || !(c_abs2(z[k]) < DIVERGE_ABS2))) atomicMin(w.flags + 1, it);
        if (tr_z && act[k]) {
          const size_t o = ((size_t)(it - 1) * T + t[k]) * u + i;
          tr_z[o] = z[k];
          tr_s[o] = s[k];
          tr_v[o] = v[k];
          if (i == 0) tr_phi[(size_t)(it - 1) * T + t[k]] = phi[k];
        }
      }
      if (it == a.t_max) break;
      float2 F[K];
      float gv[K], tau[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        tau[k] = n0 + beta * phi[k];
        posterior_t<PL>(z[k], tau[k], cp, F[k], gv[k]);
        gv[k] = act[k] ? gv[k] : 0.f;
      }
#pragma unroll
      for (int o = GS / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) gv[k] += __shfl_xor_sync(0xffffffffu, gv[k], o);
      }
      __syncwarp();  // every lane has read the old rows
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float phin = gv[k] * inv_u;
        const float coef = beta * phin / tau[k];
        phi[k] = phin;
        v[k] = c_scale(c_sub(z[k], s[k]), coef);
        s[k] = c_add(c_scale(F[k], damp), c_scale(s[k], 1.f - damp));
        if (act[k]) w.Sv[t[k] * LD + i] = s[k];
      }
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (act[k]) w.X[t[k] * LD + i] = z[k];
      if (live[k] && i == 0) w.s2[t[k]] = n0 + beta * phi[k];
    }
  }
  tm.sync();
}

// ---- LAMA (equalize.py:208-259) on (G, Z) scaled by lama_scale ----------
// Per OFDM symbol t an independent recursion; state in shared memory.
// Output: X = z^{t_max}, s2[t] = tau^{t_max}.  The last iteration skips the
// denoiser (its F, G only feed discarded updates).
template <int UP = 0, class TM>
__device__ void lama_unit(const Work& w, const EpiArgs& a, const ConstParams& cp, float2* tr_z, float2* tr_s,
                          float2* tr_v, float* tr_phi, const TM& tm, bool herm = false) {
  constexpr int NT = TM::N;
  // group-owned schedule with GS = UP lanes per symbol (one instantiation per
  // kernel keeps the register budget of the kernel's other phases);
  // ablate bit 64 selects the team-wide schedule below (timing studies)
  if constexpr (UP > 0 && UP <= 32 && NT % 32 == 0) {
    if (!(a.ablate & 64) && a.u <= UP) {  // PL: PAM levels per dimension (0: generic set)
      if (cp.L == 4) return lama_unit_groups<UP, 4>(w, a, cp, tr_z, tr_s, tr_v, tr_phi, tm, herm);
      if (cp.L == 8) return lama_unit_groups<UP, 8>(w, a, cp, tr_z, tr_s, tr_v, tr_phi, tm, herm);
      if (cp.L == 2) return lama_unit_groups<UP, 2>(w, a, cp, tr_z, tr_s, tr_v, tr_phi, tm, herm);
      return lama_unit_groups<UP, 0>(w, a, cp, tr_z, tr_s, tr_v, tr_phi, tm, herm);
    }
  }
  const int tid = tm.t;
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
  tm.sync();
  for (int it = 1; it <= a.t_max; ++it) {
    const bool last = (it == a.t_max);
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      const float2* srow = w.Sv + t * LD;
      const float2* grow = w.G + i * LD;
      // z = y_mrc + (I - G) s + v
      float2 z = c_add(w.Z[t * LD + i], c_add(srow[i], w.Vv[t * LD + i]));
      if (herm) {
        // G Hermitian (the kernel's own Gram): (G s)_i = sum_j conj(G_ji) s_j;
        // lanes with consecutive i then read consecutive words of row j
        // (no bank conflicts) and s_j is a broadcast
#pragma unroll 4
        for (int j = 0; j < u; ++j) c_fms_conj(z, w.G[j * LD + i], srow[j]);
      } else {
#pragma unroll 4
        for (int j = 0; j < u; ++j) c_fms(z, grow[j], srow[j]);
      }
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
    tm.sync();
    if (last) break;
    for (int t = tid; t < T; t += NT) {
      float sum = 0.f;
      for (int i = 0; i < u; ++i) sum += w.gb[t * LD + i];
      const float phin = sum / (float)u;
      const float tau = n0 + beta * w.phi[t];
      w.coef[t] = beta * phin / tau;
      w.phi[t] = phin;
    }
    tm.sync();
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      const float2 s = w.Sv[t * LD + i];
      w.Vv[t * LD + i] = c_scale(c_sub(w.X[t * LD + i], s), w.coef[t]);
      w.Sv[t * LD + i] = c_add(c_scale(w.Fb[t * LD + i], a.damping), c_scale(s, 1.f - a.damping));
    }
    tm.sync();
  }
  for (int t = tid; t < T; t += NT) w.s2[t] = n0 + beta * w.phi[t];
  tm.sync();
}

template <class TM>
__device__ __forceinline__ void reset_flags(const Work& w, const TM& tm) {
  if (tm.t == 0) {
    w.flags[0] = 0;
    w.flags[1] = 0x7fffffff;
  }
}

template <class TM>
__device__ __forceinline__ void write_status(const Work& w, const EqParams& p, int64_t n, const TM& tm) {
  if (tm.t == 0) {
    int st = w.flags[0];
    if (w.flags[1] < 0x7fffffff) st = st ? st : ST_DIVERGED;
    p.status[n] = st;
    if (p.iters) p.iters[n] = (w.flags[1] < 0x7fffffff) ? w.flags[1] : 0;
  }
}

// The unit epilogue after G and Z of one unit are in shared memory (and the
// team is synchronised).  PD: equalize + outputs; FD: equalize one cluster +
// fold into the fusion sums, finalize on the item's last cluster; STATS:
// write {G, y_mrc}.  Ends with a team barrier.
// CLS: equalizer class known at compile time (0 stats only, 1 linear, 2 LAMA)
// so a kernel instantiated for one class carries no code of the others; -1
// decides at run time (SIMT kernels).
template <int UP, class TM, int CLS = -1, bool LA = false, bool XZ = false>
__device__ void unit_epilogue(const Work& w, const EqParams& p, int64_t n, int cluster, bool item_end,
                              int& cl_first, const TM& tm, long long* dbg_solve = nullptr,
                              float n0_pre = -1.f) {
  constexpr int NT = TM::N;
  const int tid = tm.t;
  const int u = p.u, T = p.T, LD = w.LD;
  if (CLS == 0 || (CLS < 0 && p.arch == ARCH_STATS)) {
    const int ncl = p.sum_clusters ? 1 : p.C;
    const int cl = p.sum_clusters ? 0 : cluster;
    float2* dst = p.stats_out + ((size_t)n * ncl + cl) * (size_t)(u * u + T * u);
    if (u == UP && !(reinterpret_cast<uintptr_t>(p.stats_out) & 15)) {
      // rows of UP complex as float4 pairs, shifts instead of divisions (a
      // lone writer warp moves 40 KB per unit at U = 64)
      constexpr int SH = (UP == 8) ? 2 : (UP == 16) ? 3 : (UP == 32) ? 4 : 5;  // log2(UP / 2)
      float4* d4 = reinterpret_cast<float4*>(dst);  // record length even: 16-byte aligned
      for (int e = tid; e < (UP * UP + T * UP) / 2; e += NT) {
        const int r = e >> SH, c = 2 * (e & (UP / 2 - 1));
        const float2* src = (r < UP) ? w.G + r * LD + c : w.Z + (r - UP) * LD + c;
        d4[e] = *reinterpret_cast<const float4*>(src);
      }
    } else {
      for (int e = tid; e < u * u; e += NT) dst[e] = w.G[(e / u) * LD + (e % u)];
      for (int e = tid; e < T * u; e += NT) dst[u * u + e] = w.Z[(e / u) * LD + (e % u)];
    }
    tm.sync();
    return;
  }
  const float n0 = (n0_pre >= 0.f) ? n0_pre : item_n0(p, n);
  const bool lama = CLS == 2 || (CLS < 0 && p.kind == EQ_LAMA);
  EpiArgs a;
  a.kind = p.kind;
  a.u = u;
  a.T = T;
  a.n0 = n0;
  a.es = p.es;
  a.damping = p.damping;
  a.t_max = p.t_max;
  a.ablate = p.ablate;
  if (p.arch == ARCH_PD) {
    a.beta = p.beta;
    a.lama_scale = p.lama_scale;
    a.unbias = p.unbias != 0;
    if (lama) {
      float2 *tz = nullptr, *ts = nullptr, *tv = nullptr;
      float* tp = nullptr;
      if (p.tr_z) {
        const size_t o = (size_t)n * p.t_max * T * u;
        tz = p.tr_z + o;
        ts = p.tr_s + o;
        tv = p.tr_v + o;
        tp = p.tr_phi + (size_t)n * p.t_max * T;
      }
      lama_unit<UP>(w, a, p.cp, tz, ts, tv, tp, tm, p.g_hermitian != 0);
    } else {
      const long long t0 = dbg_solve ? clock64() : 0;
      linear_unit<UP, TM, LA, XZ>(w, a, tm);
      if (dbg_solve) *dbg_solve += clock64() - t0;
    }
    if (u == UP) {  // shifts instead of divisions
      for (int e = tid; e < T * UP; e += NT) {
        const int t = e / UP, i = e % UP;
        const float2 x = w.X[t * LD + i];
        const size_t o = (size_t)n * T * UP + e;
        p.xhat[o] = x;
        if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
      }
    } else {
      for (int e = tid; e < T * u; e += NT) {
        const int t = e / u, i = e - t * u;
        const float2 x = w.X[t * LD + i];
        const size_t o = ((size_t)n * T + t) * u + i;
        p.xhat[o] = x;
        if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
      }
    }
    if (lama) {
      for (int t = tid; t < T; t += NT) p.sigma2[(size_t)n * T + t] = w.s2[t];
    } else {
      for (int i = tid; i < u; i += NT) {
        p.sigma2[(size_t)n * u + i] = w.s2[i];
        if (p.gain && (p.kind == EQ_LMMSE || p.kind == EQ_MRC)) p.gain[(size_t)n * u + i] = w.gn[i];
      }
    }
    write_status(w, p, n, tm);
    tm.sync();
    reset_flags(w, tm);
    return;  // the next unit's writes to G/Z follow a barrier in the caller
  }
  // ---- FD: equalize this cluster (fusion.py:141-148), fold into the sums ----
  a.beta = p.cl_beta[cluster];
  a.lama_scale = p.cl_scale[cluster];
  a.unbias = true;  // fusion.py:148 -- fuse in the unbiased domain
  if (lama)
    lama_unit<UP>(w, a, p.cp, nullptr, nullptr, nullptr, nullptr, tm, p.g_hermitian != 0);
  else
    linear_unit<UP, TM, LA, XZ>(w, a, tm);
  // weights: MRC -> Gram diagonal (fusion.py:149-151), otherwise
  // 1/max(sigma2, 1e-15) (fusion.py:96-105); sigma2 <= 0 is a ConfigError
  const int wdim = lama ? T : u;
  const bool first = cl_first != 0;
  for (int e = tid; e < wdim; e += NT) {
    const float s2 = w.s2[e];
    if (p.kind != EQ_MRC && !(s2 > 0.f)) set_status(w.flags, ST_BADVAR);
    const float inv = 1.f / fmaxf(s2, VAR_FLOOR);
    const float wt = (p.kind == EQ_MRC) ? w.gn[e] : inv;
    w.wbuf[cluster * wdim + e] = wt;
    w.den[e] = first ? wt : w.den[e] + wt;
    w.harm[e] = first ? inv : w.harm[e] + inv;
  }
  tm.sync();
  for (int e = tid; e < T * u; e += NT) {
    const int t = e / u, i = e - t * u;
    const float wt = w.wbuf[cluster * wdim + (lama ? t : i)];
    const float2 x = c_scale(w.X[t * LD + i], wt);
    w.num[t * LD + i] = first ? x : c_add(w.num[t * LD + i], x);
  }
  tm.sync();
  cl_first = 0;
  if (!item_end) return;
  if (p.arch == ARCH_FD) {
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      const float2 x = c_scale(w.num[t * LD + i], 1.f / w.den[lama ? t : i]);
      const size_t o = ((size_t)n * T + t) * u + i;
      p.xhat[o] = x;
      if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
    }
    for (int e = tid; e < wdim; e += NT) p.sigma2[(size_t)n * wdim + e] = 1.f / w.harm[e];
    if (p.nu)
      for (int e = tid; e < p.C * wdim; e += NT) p.nu[(size_t)n * p.C * wdim + e] = w.wbuf[e] / w.den[e % wdim];
  } else {  // FD_PARTIAL: raw sums for a cross-GPU reduction
    const int rec = 2 * T * u + 2 * wdim;
    float* dst = p.fd_acc + (size_t)n * rec;
    for (int e = tid; e < T * u; e += NT) {
      const int t = e / u, i = e - t * u;
      const float2 v = w.num[t * LD + i];
      dst[2 * e] = v.x;
      dst[2 * e + 1] = v.y;
    }
    for (int e = tid; e < wdim; e += NT) {
      dst[2 * T * u + e] = w.den[e];
      dst[2 * T * u + wdim + e] = w.harm[e];
    }
    for (int e = tid; e < p.C * wdim; e += NT) p.fd_wraw[(size_t)n * p.C * wdim + e] = w.wbuf[e];
  }
  write_status(w, p, n, tm);
  tm.sync();
  reset_flags(w, tm);
  cl_first = 1;
}

}  // namespace dbp
