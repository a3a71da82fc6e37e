// Split-bf16 tensor-core streaming kernel for U <= 16 (the headline path:
// cfg1-cfg3 linear PD/FD and the statistics of U <= 16).
//
// Per unit (an item for PD / summed statistics, one cluster of an item for
// FD / per-cluster statistics) the Gram and the matched filter of all T
// symbols are one real GEMM over the unit's K antennas:
//     P = Xh^T [Xh | Xy],  Xh = [Re/Im H features] (K x 2U),
//                          Xy = [Re/Im Y features] (K x 2T)
//     G[u][v] = P[(u,re)][(v,re)] + P[(u,im)][(v,im)] + i (P[(u,re)][(v,im)] - P[(u,im)][(v,re)])
//     y_t[u]  = P[(u,re)][(t,re)] + P[(u,im)][(t,im)] + i (P[(u,re)][(t,im)] - P[(u,im)][(t,re)])
// Four units share one tcgen05.mma (kind::f16, M = 128 = 4 x 32 H features,
// N = 256 = [4 x 32 H features | 4 x 32 Y features], K = 16 antennas per
// instruction); the accumulator lane quarter q holds unit q's rows, so the
// solver warp of quarter q reads its unit's G and y_mrc straight from TMEM.
//
// Precision: every operand x is split into bf16 parts, x = h + m (+ l), and
// P is accumulated in fp32 from the products h.h + h.m + m.h (NSPLIT = 2:
// ~2^-17 relative per Gram entry, x-hat within ~1e-5 at cfg2) or additionally
// m.m + h.l + l.h (NSPLIT = 3: ~3xTF32 accuracy, for ill-conditioned FD-ZF).
// Plain TF32 would miss the 1e-4 tolerance.
//
// Stage = 4 units (cluster c of 4 consecutive items) x 32 antennas: the TMA
// (tensor maps, zero fill past the unit's antennas / the last item) lands H
// as [item][32 antennas][2U floats] and Y as [item][T][68 floats] (4 floats
// of row padding so the converter's column reads spread over all banks).  The converter warps load
// the whole stage into registers, meet at a named barrier, and write the bf16
// splits IN PLACE as MN-major, 128-byte-swizzled operand tiles
// ([split][4 MN blocks of 64 features][32 K rows of 128 B], 16-byte chunk j of
// K row k at position j ^ (k % 8); LBO = 4096, SBO = 1024, verified by
// tools/umma_bf16_test.cu).  Every converter load and store is bank-conflict
// free for U = 16.
//
// Roles (one persistent CTA per SM, contiguous range of 4-unit groups):
//   warp 0          TMA producer
//   warp 1          MMA issuer (one thread): NSPLIT-products x 2 K-steps per
//                   stage into accumulator (group & 1) (2 x 256 TMEM columns)
//   warps 2..       converters (T2_NCONV warps)
//   then            8 solvers in 2 sets; set s owns accumulator s (groups
//                   s, s + 2, ...); per pass warp (s, q) reads unit q of
//                   groups g and g + 2 -- 32 lanes x 64 columns each --
//                   releasing the accumulator right after each read,
//                   recombines G / y_mrc into its two shared-memory work areas
//                   and solves the two units on its two half-warps
//                   (t2_solve_pair), writing the outputs (PD) or the FD fold
//                   records directly.
//   (An L2 prefetch of the stages NS ahead, cp.async.bulk.prefetch.tensor,
//   measured 3.5 % slower on cfg2 and 6 % on the U = 64 statistics: the
//   stage ring alone keeps enough loads in flight.)
#pragma once
#include <cuda.h>

// timing-study ablations (study builds only: make study): 1 solvers skip the
// epilogue, 2 no MMAs, 4 converters skip the conversion
#if defined(DBP_STUDY) && !defined(T2X_NOABL)
#define T2_ABLATE(bit) (p.ablate & (bit))
#else
#define T2_ABLATE(bit) false
#endif
#if defined(DBP_STUDY) && !defined(T2X_NOCLK)
// per-warp wait-cycle counters (DBP_TC_DEBUG): [warp][total, wait1, wait2, -]
#define T2_WAIT(bar, par, slot)           \
  do {                                    \
    const long long t0_ = clock64();      \
    mbar_wait(bar, par);                  \
    dbgc[slot] += clock64() - t0_;        \
  } while (0)
#elif defined(T2X_CLKMASK)
#define T2_WAIT(bar, par, slot) T2_WAITR(bar, par, slot, 15)
#else
#define T2_WAIT(bar, par, slot) mbar_wait(bar, par)
#endif
#if defined(T2X_CLKMASK)
#define T2_WAITR(bar, par, slot, role)                 \
  do {                                                 \
    if (T2X_CLKMASK & (role)) {                        \
      const long long t0_ = clock64();                 \
      mbar_wait(bar, par);                             \
      dbgc[slot] += clock64() - t0_;                   \
    } else {                                           \
      mbar_wait(bar, par);                             \
    }                                                  \
  } while (0)
#else
#define T2_WAITR(bar, par, slot, role) T2_WAIT(bar, par, slot)
#endif

#include "dbp_tc.cuh"

namespace dbp {

#ifndef DBP_T2_NCONV
#define DBP_T2_NCONV 4
#endif
constexpr int T2_NCONV = DBP_T2_NCONV;               // converter warps
constexpr int T2_FIRST_CONV = 2;
constexpr int T2_FIRST_SOLV = T2_FIRST_CONV + T2_NCONV;
constexpr int T2_NSOLV = 8;                          // solver warps: 2 sets x 4 TMEM lane quarters
constexpr int T2_NWORK = 2 * T2_NSOLV;               // work areas: two units in flight per solver warp
constexpr int T2_THREADS = 32 * (T2_FIRST_SOLV + T2_NSOLV);
constexpr int T2_CT = 32 * T2_NCONV;                 // converter threads
constexpr int T2_YROW = 68;                          // floats per staged Y row (64 + 4 pad)
constexpr int T2_SPLIT_BYTES = 16384;                // one bf16 split of a stage tile
constexpr int T2_FD_CNT = 64;

// one kernel per epilogue class, so each binary carries only its own solver
// code (instruction-cache footprint)
enum { T2_STATS = 0, T2_PD = 1, T2_FD = 2 };

// Geometry of one launch (host-computed).
struct Tc2Geom {
  int K;        // antennas per unit
  int nchunk;   // stages per group = ceil(K / 32)
  int upi;      // units per item (1: PD / summed statistics; C: per cluster) = groups per item block
  int us;       // complex entries per H row (u_stride, even, <= 16)
  int T;
  int NS;       // stage ring depth
  int stage_bytes;
  int hbytes;   // bytes of the H box (4 units x 32 x 2us floats)
  int ybox;     // bytes of the Y box (4 items x T rows x 68 floats)
  int lean;     // compact solver work areas (G, y_mrc, pivot columns, flags)
  int quad;     // u <= 8: four units per solver warp pass (t2_solve_quad)
  int64_t n_items;
  int64_t G_tot;  // groups in the launch = ceil(n_items / 4) * upi
};

struct Tc2Layout {
  int bars, tmem_slot, stg, work, work_stride, fdacc, fdacc_stride, total;
  WorkLayout w;
};

// FD fusion sums of one solver warp (T2FdAcc): num [2][T][16] float2, den /
// harm [2][16], wb [C][16], status
__host__ __device__ inline int t2_fdacc_bytes(int T, int C) {
  return align_up(2 * T * 16 * 8 + 2 * 2 * 16 * 4 + C * 16 * 4 + 16, 128);
}

__host__ __device__ inline Tc2Layout make_tc2_layout(const Tc2Geom& g, int TP, int C, bool fd) {
  Tc2Layout L;
  int o = 0;
  L.bars = o;
  o += (3 * g.NS + 4) * 8;
  L.tmem_slot = o;
  o += 16;
  o = align_up(o, 1024);
  L.stg = o;
  o += g.NS * g.stage_bytes;
  L.work = o;
  L.w = make_work_layout(0, 16, TP, C, false, false);
  const int UPW = g.quad ? 8 : 16;  // unit width of a work area
  {  // compact work area: G, y_mrc, status flags
    const int LD = UPW + 2;
    int q = 0;
    L.w.G = q;
    q += UPW * LD * 8;
    L.w.Z = q;
    q += TP * LD * 8;
    L.w.W = q;
    L.w.flags = q;
    L.w.X = L.w.Sv = L.w.Vv = L.w.Fb = L.w.gb = L.w.num = L.w.Z;
    L.w.phi = L.w.coef = L.w.s2 = L.w.gn = L.w.dg = L.w.den = L.w.harm = L.w.wbuf = L.w.Z;
    L.w.total = align_up(q + 16, 128);
  }
  // +16 bytes: neighbouring work areas start 4 banks apart
  L.work_stride = L.w.total + 16;
  o += (g.quad ? 2 : 1) * T2_NWORK * L.work_stride;
  L.fdacc = o;
  L.fdacc_stride = (fd && !g.quad) ? t2_fdacc_bytes(g.T, C) : 0;
  o += T2_NSOLV * L.fdacc_stride;
  L.total = align_up(o, 128);
  return L;
}

// Stream order of a CTA's groups: item blocks go in pairs (2 bp, 2 bp + 1)
// whose groups alternate, (block 2bp, cluster 0), (2bp + 1, 0), (2bp, 1), ...,
// so consecutive groups alternate the two accumulators and both solver sets
// (set s reads the blocks of parity s) stay busy; an unpaired last block runs
// its clusters in order.
__device__ __forceinline__ void t2_group(int gl, int upi, int nblocks, int& lb, int& c) {
  const int bp = gl / (2 * upi), r = gl - bp * 2 * upi;
  if (2 * bp + 1 < nblocks) {
    lb = 2 * bp + (r & 1);
    c = r >> 1;
  } else {
    lb = 2 * bp;
    c = r;
  }
}

// ---- PTX wrappers ------------------------------------------------------------
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// Shared-memory matrix descriptor, MN-major bf16, 128-byte swizzle (layout
// type 2): LBO = stride between 64-element MN blocks, SBO = stride between
// 8-row K groups.
__device__ __forceinline__ uint64_t umma_desc_mn16(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::f16 with bf16 A/B, fp32 accumulate, MN-major A and B
__host__ __device__ constexpr uint32_t umma_idesc_bf16_mn(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns (no wait)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns (no wait)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// bf16 splits of a float pair (x0 at the lower address): h = rn(x), m =
// rn(x - h) (, l = rn(x - h - m)); returns packed bf16x2 words.  The residual
// of the pair is one packed FP32 subtraction (FADD2, sm_100).
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint32_t bf2_rn(uint64_t x) {  // {lo float, hi float} -> bf16x2
  uint32_t h;
  asm("{\n\t.reg .f32 a, b;\n\tmov.b64 {a, b}, %1;\n\tcvt.rn.bf16x2.f32 %0, b, a;\n\t}" : "=r"(h) : "l"(x));
  return h;
}
__device__ __forceinline__ uint64_t bf2_unpack(uint32_t h) {  // bf16x2 -> {lo float, hi float}
  return f2_pack(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u));
}
template <int NSPLIT>
__device__ __forceinline__ void split2(float x0, float x1, uint32_t (&w)[NSPLIT]) {
  const uint64_t x = f2_pack(x0, x1);
  const uint32_t h = bf2_rn(x);
  w[0] = h;
  const uint64_t r = f2_sub(x, bf2_unpack(h));
  const uint32_t m = bf2_rn(r);
  w[1] = m;
  if constexpr (NSPLIT == 3) w[2] = bf2_rn(f2_sub(r, bf2_unpack(m)));
}

// byte offset of MN element e (multiple of 8 / 4) of MN block b, K row k
__device__ __forceinline__ int t2_off(int b, int k, int e) {
  return b * 4096 + k * 128 + ((((e >> 3) ^ (k & 7))) << 4) + (e & 7) * 2;
}

// ---- solver of the split-bf16 kernel --------------------------------------
// Nearest symbol (equalize.py:262-268): per-dimension PAM slicer for square
// QAM (ties to the lower level), generic set otherwise; a short runtime loop
// (compact code: the solver shares the instruction cache with the other roles)
__device__ __forceinline__ int t2_slice(float2 z, const ConstParams& cp) {
  if (cp.L == 0) return slice_symbol(z, cp);
  int i = 0, j = 0;
#pragma unroll 1
  for (int l = 0; l < cp.L - 1; ++l) {
    const float mid = cp.mids[l];
    i += (z.x > mid) ? 1 : 0;
    j += (z.y > mid) ? 1 : 0;
  }
  return i * cp.L + j;
}

// FD fusion sums of one warp's item (fusion.py:108-124), accumulated in
// shared memory per half-warp in cluster order; combined at the item's end.
struct T2FdAcc {
  float2* num;  // [2][TP][16]  sum_c w_c z_c
  float* den;   // [2][16]      sum_c w_c
  float* harm;  // [2][16]      sum_c 1 / max(sigma2_c, floor)
  float* wb;    // [C][16]      w_c (for nu)
  int* st;      // status of the item (first failing cluster's code)
};


// In-place Gauss-Jordan inverse of a 16 x 16 HPD unit on one half-warp, in
// 4 x 4 blocks: lane (bi, bj) = ((lane / 4) % 4, lane % 4) of the half owns
// rows 4 bi .., cols 4 bj .. .  The branch-free rank-1 step of t2_solve_pair,
//   m_ij -= c_i r_j,  c_i = M_ik (i != k), c_k = p - 1;  r_j = M_kj / p (j != k), r_k = 1 + 1/p,
// needs per lane only the pivot row's 4 entries of its columns and the pivot
// column's 4 entries of its rows (shuffles from the two owning lanes): 18
// shuffles per step for 16 complex updates, half the traffic of a column per
// lane (a shared-memory exchange instead measured 4 % slower on cfg3-zf).  A pivot below 8 u eps of its original diagonal is singular (replaced
// by 1 and flagged).  Padded rows / columns (>= u) are the identity and their
// steps no-ops.  Reads G (+ rho on the diagonal) from, and writes A to, the
// unit's work area (rows / cols < u).
// FR: pivot reciprocals by rcp_pivot (MUFU + one Newton step) instead of
// __frcp_rn -- measured 1.3 % faster on cfg3-zf (FD) but 1.2 % slower on cfg2
// (PD), so only the FD instantiation uses it
template <bool FR>
__device__ __forceinline__ void t2_gj2d(float2* Gw, int LD, int u, float rho, bool act, int lane, bool& bad) {
  const int h16 = lane & 16, bi = (lane >> 2) & 3, bj = lane & 3;
  float2 m[4][4];
  float dgl[4];
  // full units: the block's rows as two 16-byte halves, lanes with bi odd
  // taking the second half first, so a quarter-warp's eight lanes hit eight
  // distinct bank groups (element-wise loads / stores were 4-way conflicted)
  const bool full = act && u == 16, swp = bi & 1;
  if (full) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float2* row = Gw + (4 * bi + r) * LD + 4 * bj;
      const float4 a0 = *reinterpret_cast<const float4*>(row + (swp ? 2 : 0));
      const float4 a1 = *reinterpret_cast<const float4*>(row + (swp ? 0 : 2));
      const float4 lo = swp ? a1 : a0, hi = swp ? a0 : a1;
      m[r][0] = make_float2(lo.x, lo.y);
      m[r][1] = make_float2(lo.z, lo.w);
      m[r][2] = make_float2(hi.x, hi.y);
      m[r][3] = make_float2(hi.z, hi.w);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (bi == bj && r == c) {
          m[r][c].x += rho;
          m[r][c].y = 0.f;
        }
      dgl[r] = m[r][r].x;  // the original diagonal (meaningful on the diagonal lanes bi == bj)
    }
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * bi + r, jj = 4 * bj + c;
        float2 v = make_float2(i == jj ? 1.f : 0.f, 0.f);
        if (act && i < u && jj < u) {
          v = Gw[i * LD + jj];
          if (i == jj) {
            v.x += rho;
            v.y = 0.f;
          }
        }
        m[r][c] = v;
      }
      dgl[r] = m[r][r].x;  // the original diagonal (meaningful on the diagonal lanes bi == bj)
    }
  }
  const float tolf = 8.f * (float)u * FLT_EPSILON;
  const int nkb = (u + 3) >> 2;
#pragma unroll 1
  for (int kb = 0; kb < nkb; ++kb) {
    const int srow = h16 | (kb << 2) | bj;  // owner of (row block kb, my column block)
    const int scol = h16 | (bi << 2) | kb;  // owner of (my row block, column block kb)
    const int spiv = h16 | (kb << 2) | kb;  // owner of the pivot block
#pragma unroll
    for (int kr = 0; kr < 4; ++kr) {
      float2 R[4], C[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) R[c] = shfl2(m[kr][c], srow);
#pragma unroll
      for (int r = 0; r < 4; ++r) C[r] = shfl2(m[r][kr], scol);
      float pv = __shfl_sync(0xffffffffu, m[kr][kr].x, spiv);
      const float dgk = __shfl_sync(0xffffffffu, dgl[kr], spiv);
      if (act && 4 * kb + kr < u && !(pv > tolf * dgk)) {
        if (lane == spiv) bad = true;
        pv = 1.f;
      }
      const float rp = FR ? rcp_pivot(pv) : __frcp_rn(pv);
      float2 rr[4], cr[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) rr[c] = (bj == kb && c == kr) ? make_float2(1.f + rp, 0.f) : c_scale(R[c], rp);
#pragma unroll
      for (int r = 0; r < 4; ++r) cr[r] = (bi == kb && r == kr) ? make_float2(pv - 1.f, 0.f) : C[r];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) c_fms2(m[r][c], cr[r], rr[c]);
    }
  }
  if (full) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float2* row = Gw + (4 * bi + r) * LD + 4 * bj;
      const float4 lo = make_float4(m[r][0].x, m[r][0].y, m[r][1].x, m[r][1].y);
      const float4 hi = make_float4(m[r][2].x, m[r][2].y, m[r][3].x, m[r][3].y);
      *reinterpret_cast<float4*>(row + (swp ? 2 : 0)) = swp ? hi : lo;
      *reinterpret_cast<float4*>(row + (swp ? 0 : 2)) = swp ? lo : hi;
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 4 * bi + r, jj = 4 * bj + c;
      if (act && i < u && jj < u) Gw[i * LD + jj] = m[r][c];
    }
}

// Two units per warp, one per half-warp: MRC / ZF / L-MMSE (equalize.py:130-
// 195).  ZF / L-MMSE: A = (G + rho I)^-1 in place by t2_gj2d (4 x 4 blocks
// per lane; measured 3.4 % faster on cfg3-zf than a column per lane with the
// pivot column shuffled in whole); then lane (h = lane / 16, j = lane % 16)
// loads column j of A (all 16 rows).  A is Hermitian, so lane j also holds
// row j of A (conjugated): x_t[j] = sum_i conj(A_ij) y_t[i], sigma2 = N0 A_jj,
// c = 1 - rho A_jj, unbiased z / c and N0 A_jj / c.  MRC: d = G_jj, z = y / d,
// sigma2 = N0/d + Es sum_{v != j} |G_jv|^2 / d^2.  A pivot below 8 u eps of
// its original diagonal is SingularGramError (the fp32 counterpart of
// zpotrf's "not positive definite").  PD writes x-hat / decisions / sigma2 /
// gain / status; FD adds w z, w, 1/sigma2 (w = 1/max(sigma2, 1e-15), MRC: the
// Gram diagonal, fusion.py:96-105,149-151) to the half-warp's sums in `acc`.
// F2: FFMA2 complex MACs in the A y products (measured: cfg2 -2 %, cfg3-zf
// -1.5 %; off in the FD two-part instantiation, which only MRC runs and whose
// MRC path measured 5 % slower with the FFMA2 variant compiled in)
template <bool FD, bool F2 = true>
__device__ void t2_solve_pair(const Work* w, const EqParams& p, const int64_t* n, const int* c, const float* n0,
                              const bool* valid, int lane, const T2FdAcc* acc = nullptr) {
  const int h = lane >> 4, j = lane & 15;
  const int u = p.u, T = p.T, LD = w[0].LD;
  const bool lmmse = p.kind == EQ_LMMSE, mrc = p.kind == EQ_MRC;
  const bool act = h ? valid[1] : valid[0];
  const int64_t nh = h ? n[1] : n[0];
  const int ch = h ? c[1] : c[0];
  const float n0h = h ? n0[1] : n0[0];
  float2* G = h ? w[1].G : w[0].G;
  const float2* Z = h ? w[1].Z : w[0].Z;
  const float rho = lmmse ? n0h / p.es : 0.f;
  bool bad = false;
  if (!mrc) {  // ZF / L-MMSE: A = (G + rho I)^-1 in place (4 x 4 blocks per lane)
    t2_gj2d<FD>(G, LD, u, rho, act, lane, bad);
    __syncwarp();
  }
  // lane j: column j of A (or of G for MRC), all 16 rows
  float2 m[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float2 v = make_float2(i == j ? 1.f : 0.f, 0.f);  // padding (u < 16, idle half): identity
    if (act && i < u && j < u) v = G[i * LD + j];
    m[i] = v;
  }
  // per-lane scalars: A_jj (ZF / L-MMSE) or d = G_jj and the off-diagonal
  // row energy (MRC; row j = conj(column j))
  float ajj = 0.f, off = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i == j) ajj = m[i].x;
    else if (mrc && i < u) off += c_abs2(m[i]);
  }
  if (mrc && act && j < u && !(ajj > 0.f)) bad = true;  // MRC: Gram diagonal <= 0
  const bool unb = lmmse && (FD || p.unbias);
  const float cgain = 1.f - rho * ajj;
  const float sc = mrc ? __frcp_rn(ajj) : unb ? __frcp_rn(cgain) : 1.f;
  const bool badc = act && j < u && unb && !(cgain > 0.f);
  const unsigned bm = __ballot_sync(0xffffffffu, bad || badc);
  int st = ((bm >> (16 * h)) & 0xffffu) ? ST_SINGULAR : ST_OK;
  float s2 = 0.f;
  if (mrc) {
    const float rd = __frcp_rn(ajj);
    s2 = n0h * rd + p.es * off * rd * rd;
  } else {
    const float nv = n0h * ajj;
    s2 = (p.kind == EQ_ZF) ? nv : (unb ? nv / cgain : nv);
  }
  // FD weight of this cluster for UE j (fusion.py:96-105,149-151)
  const float inv = 1.f / fmaxf(s2, VAR_FLOOR);
  const float wgt = mrc ? ajj : inv;
  if (FD && !mrc && act && j < u && !(s2 > 0.f)) st = ST_BADVAR;  // optimal_fusion_weights rejects sigma2 <= 0
  const int hb = FD ? h * 16 : 0;
  if (act && j < u) {
    for (int t = 0; t < T; t += 2) {  // symbols t, t + 1: four independent chains
      const int t1 = (t + 1 < T) ? t + 1 : t;
      const float2* z0 = Z + t * LD;
      const float2* z1 = Z + t1 * LD;
      float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
      if (mrc) {
        a0 = z0[j];
        b0 = z1[j];
      } else {
#pragma unroll
        for (int i0 = 0; i0 < 16; i0 += 8) {  // half a row of loads in flight at a time
          if (i0 >= u) break;
          float4 y0[4], y1[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = i0 + 2 * e;
            y0[e] = (i < u) ? *reinterpret_cast<const float4*>(z0 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            y1[e] = (i < u) ? *reinterpret_cast<const float4*>(z1 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = i0 + 2 * e;
            // y_t[i] beyond u is zero (the recombination zeroes it; its A column is zero)
            if constexpr (F2) {
              c_fma2_conj(a0, m[i], make_float2(y0[e].x, y0[e].y));
              c_fma2_conj(b0, m[i], make_float2(y1[e].x, y1[e].y));
              c_fma2_conj(a1, m[i + 1], make_float2(y0[e].z, y0[e].w));
              c_fma2_conj(b1, m[i + 1], make_float2(y1[e].z, y1[e].w));
            } else {
              c_fma_conj(a0, m[i], make_float2(y0[e].x, y0[e].y));
              c_fma_conj(b0, m[i], make_float2(y1[e].x, y1[e].y));
              c_fma_conj(a1, m[i + 1], make_float2(y0[e].z, y0[e].w));
              c_fma_conj(b1, m[i + 1], make_float2(y1[e].z, y1[e].w));
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (e == 1 && t + 1 >= T) break;
        const int te = t + e;
        const float2 x = c_scale(e ? c_add(b0, b1) : c_add(a0, a1), sc);
        if constexpr (FD) {
          float2& sum = acc->num[(h * T + te) * 16 + j];
          sum = c_add(sum, c_scale(x, wgt));
        } else {
          const size_t o = ((size_t)nh * T + te) * u + j;
          p.xhat[o] = x;
          if (p.dec) p.dec[o] = (uint8_t)t2_slice(x, p.cp);
        }
      }
    }
    if constexpr (FD) {
      acc->den[hb + j] += wgt;
      acc->harm[hb + j] += inv;
      acc->wb[ch * 16 + j] = wgt;
    } else {
      p.sigma2[(size_t)nh * u + j] = s2;
      if (p.gain && (lmmse || mrc)) p.gain[(size_t)nh * u + j] = mrc ? ajj : cgain;
    }
  }
  if constexpr (FD) {
    // the first failing cluster's code (half 0 holds the earlier cluster)
    const unsigned bv = __ballot_sync(0xffffffffu, act && j < u && st == ST_BADVAR);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int code = ((bm >> (16 * hh)) & 0xffffu) ? ST_SINGULAR : ((bv >> (16 * hh)) & 0xffffu) ? ST_BADVAR : 0;
      if (lane == 0 && code) atomicCAS(acc->st, 0, code);
    }
  } else if (act && j == 0) {
    p.status[nh] = st;
    if (p.iters) p.iters[nh] = 0;
  }
}

// Four units per warp, one per quarter-warp, for u <= 8: the same solves as
// t2_solve_pair on 8 x 8 matrices (lane (qq, j) = (lane / 8, lane % 8) owns
// column j of unit qq, eight rows in registers; pivot columns by shuffles
// within the quarter).  PD writes every item's outputs; FD (units of one item
// in consecutive quarters, upi = 1, 2 or 4 clusters) fuses the item's
// clusters with xor-shuffles across its quarters (fusion.py:96-124) and its
// first quarter writes x-hat / decisions / sigma2, every quarter its nu.
template <bool FD>
__device__ void t2_solve_quad(const Work* w, const EqParams& p, const int64_t* n, const int* c, const float* n0,
                              const bool* valid, int lane, int upi) {
  const int qq = lane >> 3, j = lane & 7;
  const int u = p.u, T = p.T, LD = w[0].LD;
  const bool lmmse = p.kind == EQ_LMMSE, mrc = p.kind == EQ_MRC;
  bool act = valid[0];
  int64_t nq = n[0];
  int cq = c[0];
  float n0q = n0[0];
  const float2* G = w[0].G;
  const float2* Z = w[0].Z;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (qq == k) {
      act = valid[k];
      nq = n[k];
      cq = c[k];
      n0q = n0[k];
      G = w[k].G;
      Z = w[k].Z;
    }
  const float rho = lmmse ? n0q / p.es : 0.f;
  float2 m[8];
  float dg = 1.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 v = make_float2(i == j ? 1.f : 0.f, 0.f);  // padding (u < 8, idle quarter): identity
    if (act && i < u && j < u) {
      v = G[i * LD + j];
      if (i == j) {
        v.x += rho;
        v.y = 0.f;
        dg = v.x;
      }
    }
    m[i] = v;
  }
  bool bad = false;
  if (!mrc) {
    const float tolf = 8.f * (float)u * FLT_EPSILON;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= u) break;  // padded steps are identity pivots (u is warp-uniform)
      const int src = (lane & 24) | k;
      float2 cc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) cc[i] = shfl2(m[i], src);
      const float dgk = __shfl_sync(0xffffffffu, dg, src);
      if (act && !(cc[k].x > tolf * dgk)) {
        if (j == k) bad = true;
        cc[k] = make_float2(1.f, 0.f);
      }
      const float pv = cc[k].x;
      const float rp = rcp_pivot(pv);
      const float2 r = (j == k) ? make_float2(1.f + rp, 0.f) : c_scale(m[k], rp);
      cc[k] = make_float2(pv - 1.f, 0.f);
#pragma unroll
      for (int i = 0; i < 8; ++i) c_fms2(m[i], cc[i], r);
    }
  }
  float ajj = 0.f, off = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i == j) ajj = m[i].x;
    else if (mrc && i < u) off += c_abs2(m[i]);
  }
  const bool live = act && j < u;
  if (mrc && live && !(ajj > 0.f)) bad = true;  // MRC: Gram diagonal <= 0
  const bool unb = lmmse && (FD || p.unbias);
  const float cgain = 1.f - rho * ajj;
  const float sc = mrc ? __frcp_rn(ajj) : unb ? __frcp_rn(cgain) : 1.f;
  const bool badc = live && unb && !(cgain > 0.f);
  const unsigned bm = __ballot_sync(0xffffffffu, bad || badc);
  float s2;
  if (mrc) {
    const float rd = __frcp_rn(ajj);
    s2 = n0q * rd + p.es * off * rd * rd;
  } else {
    const float nv = n0q * ajj;
    s2 = (p.kind == EQ_ZF) ? nv : (unb ? nv / cgain : nv);
  }
  const float inv = live ? 1.f / fmaxf(s2, VAR_FLOOR) : 0.f;
  const float wgt = live ? (mrc ? ajj : inv) : 0.f;
  const unsigned bv = __ballot_sync(0xffffffffu, FD && !mrc && live && !(s2 > 0.f));
  // FD: sums over the item's quarters (consecutive, upi of them)
  auto fuse = [&](float v) {
    if (FD && upi >= 2) v += __shfl_xor_sync(0xffffffffu, v, 8);
    if (FD && upi == 4) v += __shfl_xor_sync(0xffffffffu, v, 16);
    return v;
  };
  const float den = fuse(wgt), harm = fuse(inv);
  const bool lead = !FD || cq == 0;  // the quarter that writes the item's outputs
  for (int t = 0; t < T; ++t) {
    const float2* z = Z + t * LD;
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
    if (live) {
      if (mrc) {
        a0 = z[j];
      } else {
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          if (i >= u) break;
          const float4 y = *reinterpret_cast<const float4*>(z + i);  // y_t[i] beyond u is zero
          c_fma2_conj(a0, m[i], make_float2(y.x, y.y));
          c_fma2_conj(a1, m[i + 1], make_float2(y.z, y.w));
        }
      }
    }
    float2 x = c_scale(c_add(a0, a1), sc);
    if constexpr (FD) {
      const float2 xw = c_scale(x, wgt);
      x = c_scale(make_float2(fuse(xw.x), fuse(xw.y)), 1.f / den);
    }
    if (live && lead) {
      const size_t o = ((size_t)nq * T + t) * u + j;
      p.xhat[o] = x;
      if (p.dec) p.dec[o] = (uint8_t)t2_slice(x, p.cp);
    }
  }
  if (live) {
    if constexpr (FD) {
      if (lead) p.sigma2[(size_t)nq * u + j] = 1.f / harm;
      if (p.nu) p.nu[((size_t)nq * p.C + cq) * u + j] = wgt / den;
    } else {
      p.sigma2[(size_t)nq * u + j] = s2;
      if (p.gain && (lmmse || mrc)) p.gain[(size_t)nq * u + j] = mrc ? ajj : cgain;
    }
  }
  if (act && lead && j == 0) {
    int code = 0;  // FD: the first failing cluster's code (clusters in quarter order)
    for (int e = 0; e < (FD ? upi : 1); ++e) {
      const int qe = qq + e;
      const int ce = ((bm >> (8 * qe)) & 0xffu) ? ST_SINGULAR : ((bv >> (8 * qe)) & 0xffu) ? ST_BADVAR : 0;
      if (!code) code = ce;
    }
    p.status[nq] = code;
    if (p.iters) p.iters[nq] = 0;
  }
}

// The item's FD fusion (fusion.py:108-124, 141-154) from the two half-warps'
// sums: x = sum_c w_c z_c / sum_c w_c, sigma2 = 1 / sum_c 1/max(sigma2_c,
// 1e-15), nu_c = w_c / sum w; or the raw sums for a cross-GPU reduction
// (ARCH_FD_PARTIAL: fd_acc [n][2Tu + 2u], fd_wraw [n][C][u]).
__device__ inline void t2_fd_finish(const T2FdAcc& acc, const EqParams& p, int64_t n, int lane) {
  const int u = p.u, T = p.T, C = p.C;
  const int h = lane >> 4, j = lane & 15;
  const int st = *acc.st;
  if (j < u) {
    const float den = acc.den[j] + acc.den[16 + j], harm = acc.harm[j] + acc.harm[16 + j];
    if (p.arch == ARCH_FD) {
      const float rden = 1.f / den;
      for (int t = h; t < T; t += 2) {
        const float2 x = c_scale(c_add(acc.num[t * 16 + j], acc.num[(T + t) * 16 + j]), rden);
        const size_t o = ((size_t)n * T + t) * u + j;
        p.xhat[o] = x;
        if (p.dec) p.dec[o] = (uint8_t)t2_slice(x, p.cp);
      }
      if (h == 0) p.sigma2[(size_t)n * u + j] = 1.f / harm;
      if (p.nu)
        for (int c = h; c < C; c += 2) p.nu[((size_t)n * C + c) * u + j] = acc.wb[c * 16 + j] * rden;
    } else {
      float* dst = p.fd_acc + (size_t)n * (2 * T * u + 2 * u);
      for (int t = h; t < T; t += 2) {
        const float2 v = c_add(acc.num[t * 16 + j], acc.num[(T + t) * 16 + j]);
        dst[2 * (t * u + j)] = v.x;
        dst[2 * (t * u + j) + 1] = v.y;
      }
      if (h == 0) {
        dst[2 * T * u + j] = den;
        dst[2 * T * u + u + j] = harm;
      }
      for (int c = h; c < C; c += 2) p.fd_wraw[((size_t)n * C + c) * u + j] = acc.wb[c * 16 + j];
    }
  }
  if (lane == 0) {
    p.status[n] = st;
    if (p.iters) p.iters[n] = 0;
  }
}

// Central solve from fused statistics {G, y_mrc} (linear_equalize +
// unbiased_output on FusedStats, equalize.py:130-195; the central node of the
// multi-GPU PD path after dbp_pd_reduce_scatter) for u <= 16, ZF / L-MMSE:
// each warp stages two items' statistics into its two work areas (G
// Hermitian from its lower triangle, as the reference's Cholesky reads it;
// y_mrc zero past u) and runs t2_solve_pair.
constexpr int T2S_WARPS = 4;
template <int UP = 16>  // (a template so that the header can be included by several units)
__global__ void __launch_bounds__(32 * T2S_WARPS) t2_stats_solve_kernel(const __grid_constant__ EqParams p,
                                                                        int work_stride) {
  extern __shared__ __align__(16) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = p.u, T = p.T, LD = 16 + 2;
  const int rec = u * u + T * u;
  Work w[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    char* base = smem + (2 * warp + k) * work_stride;
    w[k].G = reinterpret_cast<float2*>(base);
    w[k].Z = reinterpret_cast<float2*>(base + 16 * LD * 8);
    w[k].W = reinterpret_cast<float2*>(base + (16 + p.TP) * LD * 8);  // layout of launch_t2_stats_solve
    w[k].flags = reinterpret_cast<int*>(base + (16 + p.TP) * LD * 8 + 32 * 8);
    w[k].X = w[k].Z;
    w[k].LD = LD;
  }
  const int64_t pairs = (p.n_items + 1) / 2;
  for (int64_t pr = (int64_t)blockIdx.x * T2S_WARPS + warp; pr < pairs; pr += (int64_t)gridDim.x * T2S_WARPS) {
    int64_t n[2];
    int c[2] = {0, 0};
    float n0[2];
    bool valid[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      n[k] = 2 * pr + k;
      valid[k] = n[k] < p.n_items;
      n0[k] = valid[k] ? item_n0(p, n[k]) : 0.f;
      if (!valid[k]) continue;
      const float2* src = p.stats_in + (size_t)n[k] * rec;
      if (!(u & 1) && !(reinterpret_cast<uintptr_t>(src) & 15)) {
        // coalesced: the record's rows as float4 pairs, then the upper
        // triangle mirrored from the lower one in shared memory
        const int hu = u >> 1;
        const float4* s4 = reinterpret_cast<const float4*>(src);
        for (int e = lane; e < (u + T) * hu; e += 32) {
          const int r = e / hu, cc = 2 * (e - r * hu);
          float2* dst = (r < u) ? w[k].G + r * LD + cc : w[k].Z + (r - u) * LD + cc;
          *reinterpret_cast<float4*>(dst) = s4[e];
        }
        for (int e = lane; e < T * (16 - u); e += 32) {  // zero y past u (read by t2_solve_pair)
          const int t = e / (16 - u), i = u + e - t * (16 - u);
          w[k].Z[t * LD + i] = make_float2(0.f, 0.f);
        }
        __syncwarp();
        for (int e = lane; e < u * u; e += 32) {
          const int i = e / u, j = e - i * u;
          if (i < j) w[k].G[i * LD + j] = c_conj(w[k].G[j * LD + i]);
        }
      } else {
        for (int e = lane; e < u * u; e += 32) {
          const int i = e / u, j = e - i * u;
          const float2 v = (i >= j) ? src[e] : c_conj(src[j * u + i]);
          w[k].G[i * LD + j] = v;
        }
        for (int e = lane; e < T * 16; e += 32) {
          const int t = e >> 4, i = e & 15;
          w[k].Z[t * LD + i] = (i < u) ? src[u * u + t * u + i] : make_float2(0.f, 0.f);
        }
      }
    }
    __syncwarp();
    t2_solve_pair<false>(w, p, n, c, n0, valid, lane);
    __syncwarp();
  }
}

template <int MODE, int NSPLIT, int QUAD = 0>
// register cap: a warp lives on one of the 4 SM sub-partitions (16K registers
// each), which hold ceil(warps / 4) warps
__global__ void __maxnreg__(16384 / (32 * ((T2_THREADS / 32 + 3) / 4)) / 8 * 8)
    tc2_kernel(const __grid_constant__ EqParams p, const __grid_constant__ CUtensorMap hmap,
               const __grid_constant__ CUtensorMap ymap, const __grid_constant__ Tc2Geom g) {
  extern __shared__ __align__(1024) char smem[];
  constexpr bool fd = (MODE == T2_FD);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int NS = g.NS;
  const Tc2Layout L = make_tc2_layout(g, p.TP, p.C, fd);
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* conv_full = raw_full + NS;
  uint64_t* stage_empty = conv_full + NS;
  uint64_t* acc_full = stage_empty + NS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&conv_full[s], T2_NCONV);
      mbar_init(&stage_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#if defined(DBP_STUDY) || defined(T2X_CLKMASK)
  long long dbgc[4] = {0, 0, 0, 0};
  const long long t_start = clock64();
#endif

  // Groups are item-major: group g = (item block b = g / upi, cluster
  // c = g % upi) holds cluster c of items 4b .. 4b + 3 (unit q = item 4b + q),
  // so a solver warp's lane quarter sees every cluster of one item and can
  // fuse them (FD) without leaving the warp.  A CTA owns whole item blocks.
  const int64_t nblk = g.G_tot / g.upi;
  const int64_t per_cta = nblk / gridDim.x, extra = nblk % gridDim.x;
  const int64_t b_first = blockIdx.x * per_cta + min((int64_t)blockIdx.x, extra);
  const int nblocks = (int)(per_cta + (blockIdx.x < extra ? 1 : 0));
  const int ngroups = nblocks * g.upi;
  const int nch = g.nchunk;
  const uint32_t stg0 = smem_u32(smem + L.stg);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ----
    if (lane == 0) {
      prefetch_tmap(&hmap);
      prefetch_tmap(&ymap);
      const uint64_t policy = l2_evict_first_policy();
      const int total = ngroups * nch;
      // stage sequence number -> (group, chunk) coordinates
      auto coords = [&](int sq, int& j, int& item0, int& c0) {
        const int gl = sq / nch;
        j = sq - gl * nch;
        int lb;
        t2_group(gl, g.upi, nblocks, lb, c0);
        item0 = (int)((b_first + lb) * 4);
      };
      int s = 0;
      uint32_t ph = 0;
      for (int sq = 0; sq < total; ++sq) {
        if (sq >= NS) T2_WAITR(&stage_empty[s], ph ^ 1u, 1, 1);
        int j, item0, c0;
        coords(sq, j, item0, c0);
        const uint32_t bar = smem_u32(&raw_full[s]);
        mbar_arrive_expect_tx(&raw_full[s], (uint32_t)(g.hbytes + g.ybox));
        const uint32_t dst = stg0 + (uint32_t)(s * g.stage_bytes);
        tma_load_4d(dst, &hmap, 0, 32 * j, c0, item0, bar, policy);
        tma_load_4d(dst + g.hbytes, &ymap, 64 * j, c0, 0, item0, bar, policy);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer ----
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16_mn(128, 256);
      // products (a split, b split): h.h, h.m, m.h [, m.m, h.l, l.h]
      constexpr int NP = NSPLIT == 2 ? 3 : 6;
      constexpr int PA[6] = {0, 0, 1, 1, 0, 2};
      constexpr int PB[6] = {0, 1, 0, 1, 2, 0};
      int s = 0;
      uint32_t ph = 0;
      int uses[2] = {0, 0};  // groups written into each accumulator so far
      for (int gl = 0; gl < ngroups; ++gl) {
        int lb, cg;
        t2_group(gl, g.upi, nblocks, lb, cg);
        const int a = lb & 1;  // item blocks alternate accumulators
        if (uses[a] >= 1) T2_WAITR(&acc_empty[a], (uint32_t)((uses[a] - 1) & 1), 2, 2);
        ++uses[a];
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(256 * a);
        for (int j = 0; j < nch; ++j) {
          T2_WAITR(&conv_full[s], ph, 1, 2);
          tc_fence_after();
          const uint32_t base = stg0 + (uint32_t)(s * g.stage_bytes);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
            for (int pr = 0; pr < NP; ++pr) {
              const uint64_t da = umma_desc_mn16(base + PA[pr] * T2_SPLIT_BYTES + ks * 2048);
              const uint64_t db = umma_desc_mn16(base + PB[pr] * T2_SPLIT_BYTES + ks * 2048);
              if (!T2_ABLATE(2)) umma_bf16(d, da, db, idesc, (j | ks | pr) ? 1u : 0u);
            }
          }
          umma_commit(&stage_empty[s]);
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
        }
        umma_commit(&acc_full[a]);
      }
    }
    __syncwarp();
  } else if (warp < T2_FIRST_SOLV) {
    // -------------------------------------------------------- converters ----
    const int ct = tid - 32 * T2_FIRST_CONV;
    const int us = g.us, T = g.T;
    const int qpr = us >> 1;           // float4 (2 UEs) per H row
    const int nh = 4 * 32 * qpr;       // H tasks per stage
    constexpr int HT = 4 * 32 * 8 / T2_CT;  // H tasks per thread at us = 16
    constexpr int YT = 4 * 16 * 4 / T2_CT;  // Y tasks per thread (T <= 16)
    static_assert(HT * T2_CT == 1024 && YT * T2_CT == 256, "converter task split");
    // per-thread task tables, the same for every stage (float index of the
    // load in the stage, byte offset of the store in a split tile)
    // H task e: quad jq of antenna row k (+4 r) of unit q; 16-lane phases =
    // 8 quads x rows {k, k + 4} (conflict-free loads and 8-byte stores)
    int hld[HT], hst[HT];
#pragma unroll
    for (int i = 0; i < HT; ++i) {
      const int e = ct + i * T2_CT;
      const int jq = e % qpr, e2 = e / qpr;
      const int r = e2 & 1, kk = (e2 >> 1) & 15, q = e2 >> 5;
      const int k = (kk & 3) + 8 * (kk >> 2) + 4 * r;
      hld[i] = (q * 32 + k) * 2 * us + 4 * jq;
      hst[i] = (e < nh) ? t2_off(q >> 1, k, 32 * (q & 1) + 4 * jq) : -1;
    }
    // Y task e: antenna pair kp, symbol block tb (t = 4 tb .. 4 tb + 3) of
    // unit q; 8-lane phases = 4 antenna pairs x 2 symbol blocks.  The store
    // for antenna 2kp + 1 sits at the next 128-byte K row, its chunk position
    // the XOR with (k % 8) flipped in bit 0.
    int yld[YT], yst0[YT], yst1[YT], yt0[YT];
#pragma unroll
    for (int i = 0; i < YT; ++i) {
      const int e = ct + i * T2_CT;
      const int kp = (e & 3) + 4 * ((e >> 3) & 3);
      const int tb = ((e >> 2) & 1) + 2 * ((e >> 5) & 1);
      const int q = e >> 6;
      yt0[i] = 4 * tb;
      yld[i] = (g.hbytes >> 2) + (q * T + 4 * tb) * T2_YROW + 4 * kp;
      yst0[i] = t2_off(2 + (q >> 1), 2 * kp, 32 * (q & 1) + 8 * tb);
      yst1[i] = yst0[i] + 128 + (((yst0[i] >> 4) & 1) ? -16 : 16);
    }
    int s = 0;
    uint32_t ph = 0;
    for (int gl = 0; gl < ngroups; ++gl) {
      for (int j = 0; j < nch; ++j) {
        T2_WAITR(&raw_full[s], ph, 1, 4);
        char* st = smem + L.stg + s * g.stage_bytes;
        if (T2_ABLATE(4)) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv_full[s]);
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
          continue;
        }
        const float* sf = reinterpret_cast<const float*>(st);
        float4 hv[HT];
#pragma unroll
        for (int i = 0; i < HT; ++i)
          hv[i] = (hst[i] >= 0) ? *reinterpret_cast<const float4*>(sf + hld[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 yv[YT][4];
#pragma unroll
        for (int i = 0; i < YT; ++i)
#pragma unroll
          for (int x = 0; x < 4; ++x)
            yv[i][x] = (yt0[i] + x < T) ? *reinterpret_cast<const float4*>(sf + yld[i] + x * T2_YROW)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        named_bar(1, T2_CT);  // every load of the stage done: convert in place
#pragma unroll
        for (int i = 0; i < HT; ++i) {
          if (hst[i] < 0) continue;
          uint32_t w0[NSPLIT], w1[NSPLIT];
          split2<NSPLIT>(hv[i].x, hv[i].y, w0);
          split2<NSPLIT>(hv[i].z, hv[i].w, w1);
#pragma unroll
          for (int sp = 0; sp < NSPLIT; ++sp)
            *reinterpret_cast<uint2*>(st + sp * T2_SPLIT_BYTES + hst[i]) = make_uint2(w0[sp], w1[sp]);
        }
#pragma unroll
        for (int i = 0; i < YT; ++i) {
          // antenna 2kp: (y_t.x, y_t.y) of the 4 symbols; antenna 2kp + 1: (.z, .w)
          uint32_t a0[NSPLIT], a1[NSPLIT], a2[NSPLIT], a3[NSPLIT];
          uint32_t b0[NSPLIT], b1[NSPLIT], b2[NSPLIT], b3[NSPLIT];
          split2<NSPLIT>(yv[i][0].x, yv[i][0].y, a0);
          split2<NSPLIT>(yv[i][1].x, yv[i][1].y, a1);
          split2<NSPLIT>(yv[i][2].x, yv[i][2].y, a2);
          split2<NSPLIT>(yv[i][3].x, yv[i][3].y, a3);
          split2<NSPLIT>(yv[i][0].z, yv[i][0].w, b0);
          split2<NSPLIT>(yv[i][1].z, yv[i][1].w, b1);
          split2<NSPLIT>(yv[i][2].z, yv[i][2].w, b2);
          split2<NSPLIT>(yv[i][3].z, yv[i][3].w, b3);
#pragma unroll
          for (int sp = 0; sp < NSPLIT; ++sp) {
            *reinterpret_cast<uint4*>(st + sp * T2_SPLIT_BYTES + yst0[i]) = make_uint4(a0[sp], a1[sp], a2[sp], a3[sp]);
            *reinterpret_cast<uint4*>(st + sp * T2_SPLIT_BYTES + yst1[i]) = make_uint4(b0[sp], b1[sp], b2[sp], b3[sp]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_full[s]);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // ----------------------------------------------------------- solvers ----
    // set s = 0, 1 owns accumulator s, i.e. the item blocks of parity s; warp
    // (s, q) handles item 4b + q of each of its blocks, reading the units of
    // its lane quarter in order, two per pass (one per half-warp)
    const int sv = warp - T2_FIRST_SOLV;
    const int sset = sv >> 2;  // = the accumulator this warp reads
    const int q = warp & 3;    // TMEM lane quarter this warp may access
    const Team<32, -1> tm{lane};
    if constexpr (QUAD) {
      // u <= 8: four units per pass (consecutive in the warp's unit sequence;
      // FD items, upi | 4 units, never straddle a pass), one per quarter-warp
      Work w4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        WorkLayout wl = L.w;
        const int base = L.work + (4 * sv + k) * L.work_stride;
        wl.G += base; wl.Z += base; wl.X += base; wl.W += base; wl.Sv += base; wl.Vv += base; wl.Fb += base;
        wl.gb += base; wl.num += base; wl.phi += base; wl.coef += base; wl.s2 += base; wl.gn += base;
        wl.dg += base; wl.den += base; wl.harm += base; wl.wbuf += base; wl.flags += base;
        w4[k] = make_work(smem, wl, 8);
      }
      const int u = p.u, T = p.T, LD = w4[0].LD, upi = g.upi;
      const int uh = lane >> 1, s_im = lane & 1;
      const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
      const int units = ((nblocks - sset + 1) / 2) * upi;
      int use = 0;
      for (int k0 = 0; k0 < units; k0 += 4) {
        int64_t n[4];
        int c[4];
        float n0[4];
        bool valid[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          valid[k] = false;
          n[k] = 0;
          c[k] = 0;
          n0[k] = 0.f;
          const int uix = k0 + k;
          if (uix >= units) continue;
          const int lb = sset + 2 * (uix / upi);
          c[k] = uix - (uix / upi) * upi;
          n[k] = (b_first + lb) * 4 + q;
          valid[k] = n[k] < g.n_items;
          if (valid[k]) n0[k] = item_n0(p, n[k]);
          T2_WAITR(&acc_full[sset], (uint32_t)(use & 1), 1, 8);
          ++use;
          tc_fence_after();
          uint32_t gr[16], yr[32];
          tmem_ld16_nw(tq + (uint32_t)(256 * sset + 32 * q), gr);
          tmem_ld32_nw(tq + (uint32_t)(256 * sset + 128 + 32 * q), yr);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[sset]);
          if (!valid[k]) continue;
          float* Gf = reinterpret_cast<float*>(w4[k].G);
          float* Zf = reinterpret_cast<float*>(w4[k].Z);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const float mine = __uint_as_float(gr[2 * v]);
            const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(gr[2 * v + 1]), 1);
            const float val = s_im ? (po - mine) : (mine + po);
            if (uh < u && v < u) Gf[(v * LD + uh) * 2 + s_im] = s_im ? -val : val;  // G[v][uh] = conj(G[uh][v])
          }
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const float mine = __uint_as_float(yr[2 * t]);
            const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(yr[2 * t + 1]), 1);
            const float val = s_im ? (po - mine) : (mine + po);
            if (t < T && uh < 8) Zf[(t * LD + uh) * 2 + s_im] = (uh < u) ? val : 0.f;
          }
        }
        __syncwarp();
        t2_solve_quad<MODE == T2_FD>(w4, p, n, c, n0, valid, lane, upi);
        __syncwarp();
      }
    } else {
    Work w[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      WorkLayout wl = L.w;
      const int base = L.work + (2 * sv + k) * L.work_stride;
      wl.G += base; wl.Z += base; wl.X += base; wl.W += base; wl.Sv += base; wl.Vv += base; wl.Fb += base;
      wl.gb += base; wl.num += base; wl.phi += base; wl.coef += base; wl.s2 += base; wl.gn += base;
      wl.dg += base; wl.den += base; wl.harm += base; wl.wbuf += base; wl.flags += base;
      w[k] = make_work(smem, wl, 16);
    }
    const int u = p.u, T = p.T, LD = w[0].LD, upi = g.upi;
    const int uh = lane >> 1, s_im = lane & 1;  // this lane's H feature: UE uh, re/im
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    int cl_first = 1;
    T2FdAcc acc;
    if constexpr (fd) {
      char* ab = smem + L.fdacc + sv * L.fdacc_stride;
      acc.num = reinterpret_cast<float2*>(ab);
      acc.den = reinterpret_cast<float*>(ab + 2 * T * 16 * 8);
      acc.harm = acc.den + 32;
      acc.wb = acc.harm + 32;
      acc.st = reinterpret_cast<int*>(acc.wb + upi * 16);
    }
    // this warp's unit sequence: (block lb, cluster c), lb = sset, sset + 2, ...
    const int units = ((nblocks - sset + 1) / 2) * upi;
    int use = 0;  // reads of accumulator sset so far (mbarrier phase)
    for (int k0 = 0; k0 < units; k0 += 2) {
      int64_t n[2];
      int c[2];
      float n0[2];
      bool valid[2];
      int lbk[2];
      int cnt = 0;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        valid[k] = false;
        n[k] = 0;
        c[k] = 0;
        n0[k] = 0.f;
        lbk[k] = -1;
        const int uix = k0 + k;
        if (uix >= units) continue;
        const int lb = sset + 2 * (uix / upi);
        const int cc = uix - (uix / upi) * upi;
        if (fd && k == 1 && cc == 0) continue;  // FD pairs stay inside one item block
        ++cnt;
        lbk[k] = lb;
        c[k] = cc;
        n[k] = (b_first + lb) * 4 + q;
        valid[k] = n[k] < g.n_items;
        if (valid[k] && MODE != T2_STATS) n0[k] = item_n0(p, n[k]);  // global load before the wait
        T2_WAITR(&acc_full[sset], (uint32_t)(use & 1), 1, 8);
        ++use;
        tc_fence_after();
        uint32_t gr[32], yr[32];
        tmem_ld32_nw(tq + (uint32_t)(256 * sset + 32 * q), gr);
        tmem_ld32_nw(tq + (uint32_t)(256 * sset + 128 + 32 * q), yr);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[sset]);
        if (T2_ABLATE(1)) valid[k] = false;
        if (!valid[k]) continue;
        // re/im recombination (one shuffle per column pair): even lanes form
        // the real parts, odd lanes the imaginary parts
        float* Gf = reinterpret_cast<float*>(w[k].G);
        float* Zf = reinterpret_cast<float*>(w[k].Z);
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float mine = __uint_as_float(gr[2 * v]);
          const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(gr[2 * v + 1]), 1);
          const float val = s_im ? (po - mine) : (mine + po);
          // stored as G[v][uh] = conj(G[uh][v]) (G is Hermitian): lanes hit 32 banks
          if (uh < u && v < u) Gf[(v * LD + uh) * 2 + s_im] = s_im ? -val : val;
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const float mine = __uint_as_float(yr[2 * t]);
          const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(yr[2 * t + 1]), 1);
          const float val = s_im ? (po - mine) : (mine + po);
          if (t < T) Zf[(t * LD + uh) * 2 + s_im] = (uh < u) ? val : 0.f;  // zero past u: read by t2_solve_pair
        }
        reset_flags(w[k], tm);
      }
      k0 -= 2 - cnt;  // a unit not taken (FD block boundary) is read in the next pass
      __syncwarp();
      if constexpr (MODE == T2_STATS) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (valid[k]) unit_epilogue<16, Team<32, -1>, 0>(w[k], p, n[k], c[k], true, cl_first, tm, nullptr, 0.f);
        continue;
      } else if constexpr (MODE == T2_PD) {
        t2_solve_pair<false>(w, p, n, c, n0, valid, lane);
      } else {
        const bool item_ok = lbk[0] >= 0 && (b_first + lbk[0]) * 4 + q < g.n_items;
        if (c[0] == 0 && lbk[0] >= 0) {  // a new item: clear its fusion sums
          for (int e = lane; e < 2 * T * 16; e += 32) acc.num[e] = make_float2(0.f, 0.f);
          acc.den[lane] = 0.f;
          acc.harm[lane] = 0.f;
          if (lane == 0) *acc.st = 0;
          __syncwarp();
        }
        t2_solve_pair<true, NSPLIT != 2>(w, p, n, c, n0, valid, lane, &acc);
        __syncwarp();
        const int clast = (lbk[1] >= 0) ? c[1] : c[0];
        if (item_ok && clast == upi - 1) t2_fd_finish(acc, p, n[0], lane);
      }
      __syncwarp();
    }
    }  // !QUAD
  }
#ifdef DBP_STUDY
  if (p.dbg && lane == 0) {
    dbgc[0] = clock64() - t_start;
    for (int k = 0; k < 4; ++k)
      atomicAdd(reinterpret_cast<unsigned long long*>(p.dbg + warp * 4 + k), (unsigned long long)dbgc[k]);
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace dbp
