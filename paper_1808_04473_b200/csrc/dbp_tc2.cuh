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
// Stage = 4 units x 32 antennas: the TMA (tensor maps, zero fill past the
// unit's antennas / the last unit) lands H as [unit][32 antennas][2U floats]
// and Y as [cluster][item][T][68 floats] (4 floats of row padding so the
// converter's column reads spread over all banks).  The converter warps load
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
//   then            solvers: T2_NSET sets of 4 warps; set s takes groups
//                   s, s + NSET, ...; warp (s, q) reads unit q's 32 lanes x
//                   64 columns, releases the accumulator, recombines G / y_mrc
//                   into its shared-memory work area and runs the unit
//                   epilogue (dbp_epilogue.cuh).
#pragma once
#include <cuda.h>

#include "dbp_tc.cuh"

namespace dbp {

#ifndef DBP_T2_NCONV
#define DBP_T2_NCONV 4
#endif
#ifndef DBP_T2_NSET
#define DBP_T2_NSET 2
#endif
constexpr int T2_NCONV = DBP_T2_NCONV;               // converter warps
constexpr int T2_NSET = DBP_T2_NSET;                 // solver sets (4 warps each)
constexpr int T2_FIRST_CONV = 2;
constexpr int T2_FIRST_SOLV = T2_FIRST_CONV + T2_NCONV;
constexpr int T2_NSOLV = 4 * T2_NSET;
constexpr int T2_THREADS = 32 * (T2_FIRST_SOLV + T2_NSOLV);
constexpr int T2_CT = 32 * T2_NCONV;                 // converter threads
constexpr int T2_YROW = 68;                          // floats per staged Y row (64 + 4 pad)
constexpr int T2_SPLIT_BYTES = 16384;                // one bf16 split of a stage tile
constexpr int T2_FD_CNT = 64;

enum { T2_STATS = 0, T2_PD = 1, T2_FD = 2 };

// Geometry of one launch (host-computed).
struct Tc2Geom {
  int K;        // antennas per unit
  int nchunk;   // stages per group = ceil(K / 32)
  int upi;      // units per item (1: PD / summed statistics; C: per cluster)
  int gc, gn;   // a group = gn items x gc clusters (gc * gn = 4)
  int us;       // complex entries per H row (u_stride, even, <= 16)
  int T;
  int NS;       // stage ring depth
  int stage_bytes;
  int hbytes;   // bytes of the H box (4 units x 32 x 2us floats)
  int ybox;     // bytes of one Y box (gn items x T rows x 68 floats)
  int ystride;  // shared-memory stride between the Y boxes (128-byte aligned)
  int64_t U_tot;  // units in the launch
  int64_t G_tot;  // groups in the launch
};

struct Tc2Layout {
  int bars, tmem_slot, fdc, stg, work, work_stride, total;
  WorkLayout w;
};

__host__ __device__ inline Tc2Layout make_tc2_layout(const Tc2Geom& g, int TP, int C, bool fd) {
  Tc2Layout L;
  int o = 0;
  L.bars = o;
  o += (3 * g.NS + 4) * 8;
  L.tmem_slot = o;
  o += 16;
  L.fdc = o;
  o += fd ? T2_FD_CNT * 4 : 0;
  o = align_up(o, 1024);
  L.stg = o;
  o += g.NS * g.stage_bytes;
  L.work = o;
  L.w = make_work_layout(0, 16, TP, C, false, fd);
  L.work_stride = L.w.total;
  o += T2_NSOLV * L.work_stride;
  L.total = align_up(o, 128);
  return L;
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
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// bf16 splits of a float pair (x0 at the lower address): h = rn(x), m =
// rn(x - h) (, l = rn(x - h - m)); returns packed bf16x2 words
template <int NSPLIT>
__device__ __forceinline__ void split2(float x0, float x1, uint32_t (&w)[NSPLIT]) {
  uint32_t h;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
  w[0] = h;
  float r0 = x0 - __uint_as_float(h << 16), r1 = x1 - __uint_as_float(h & 0xffff0000u);
  uint32_t m;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(m) : "f"(r1), "f"(r0));
  w[1] = m;
  if constexpr (NSPLIT == 3) {
    r0 -= __uint_as_float(m << 16);
    r1 -= __uint_as_float(m & 0xffff0000u);
    uint32_t l;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(r1), "f"(r0));
    w[2] = l;
  }
}

// byte offset of MN element e (multiple of 8 / 4) of MN block b, K row k
__device__ __forceinline__ int t2_off(int b, int k, int e) {
  return b * 4096 + k * 128 + ((((e >> 3) ^ (k & 7))) << 4) + (e & 7) * 2;
}

template <int MODE, int NSPLIT>
__global__ void __launch_bounds__(T2_THREADS, 1)
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
  int* fd_count = reinterpret_cast<int*>(smem + L.fdc);
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
  if (fd)
    for (int k = tid; k < T2_FD_CNT; k += blockDim.x) fd_count[k] = 0;
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // contiguous range of whole items per CTA: blocks of gpi = max(1, upi / 4)
  // groups (groups never straddle items: upi | 4 or 4 | upi), so all clusters
  // of an item meet at one CTA's FD arrival counter
  const int gpi = g.upi > 4 ? g.upi / 4 : 1;
  const int64_t nblk = g.G_tot / gpi;
  const int64_t per_cta = nblk / gridDim.x, extra = nblk % gridDim.x;
  const int64_t g_first = (blockIdx.x * per_cta + min((int64_t)blockIdx.x, extra)) * gpi;
  const int ngroups = (int)(per_cta + (blockIdx.x < extra ? 1 : 0)) * gpi;
  const int nch = g.nchunk;
  const uint32_t stg0 = smem_u32(smem + L.stg);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ----
    if (lane == 0) {
      prefetch_tmap(&hmap);
      prefetch_tmap(&ymap);
      const uint64_t policy = l2_evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      int sq = 0;
      for (int gl = 0; gl < ngroups; ++gl) {
        const int64_t u0 = (g_first + gl) * 4;
        const int n0 = (int)(u0 / g.upi), c0 = (int)(u0 % g.upi);
        for (int j = 0; j < nch; ++j, ++sq) {
          if (sq >= NS) mbar_wait(&stage_empty[s], ph ^ 1u);
          const uint32_t bar = smem_u32(&raw_full[s]);
          mbar_arrive_expect_tx(&raw_full[s], (uint32_t)(g.hbytes + g.gc * g.ybox));
          const uint32_t dst = stg0 + (uint32_t)(s * g.stage_bytes);
          tma_load_3d(dst, &hmap, 0, 32 * j, (int)u0, bar, policy);
          for (int cl = 0; cl < g.gc; ++cl)
            tma_load_4d(dst + g.hbytes + cl * g.ystride, &ymap, 64 * j, c0 + cl, 0, n0, bar, policy);
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
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
      for (int gl = 0; gl < ngroups; ++gl) {
        const int a = gl & 1;
        if (gl >= 2) mbar_wait(&acc_empty[a], (uint32_t)(((gl >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(256 * a);
        for (int j = 0; j < nch; ++j) {
          mbar_wait(&conv_full[s], ph);
          tc_fence_after();
          const uint32_t base = stg0 + (uint32_t)(s * g.stage_bytes);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
            for (int pr = 0; pr < NP; ++pr) {
              const uint64_t da = umma_desc_mn16(base + PA[pr] * T2_SPLIT_BYTES + ks * 2048);
              const uint64_t db = umma_desc_mn16(base + PB[pr] * T2_SPLIT_BYTES + ks * 2048);
              umma_bf16(d, da, db, idesc, (j | ks | pr) ? 1u : 0u);
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
    int s = 0;
    uint32_t ph = 0;
    for (int gl = 0; gl < ngroups; ++gl) {
      for (int j = 0; j < nch; ++j) {
        mbar_wait(&raw_full[s], ph);
        char* st = smem + L.stg + s * g.stage_bytes;
        const float* hraw = reinterpret_cast<const float*>(st);
        const float* yraw = reinterpret_cast<const float*>(st + g.hbytes);
        // H task e: quad jq of antenna row k (+4 r) of unit q; 16-lane phases
        // = 8 quads x rows {k, k + 4} (conflict-free loads and 8-byte stores)
        float4 hv[HT];
        int hoff[HT];
#pragma unroll
        for (int i = 0; i < HT; ++i) {
          const int e = ct + i * T2_CT;
          int jq, r, kk, q;
          if (qpr == 8) {
            jq = e & 7;
            r = (e >> 3) & 1;
            kk = (e >> 4) & 15;
            q = e >> 8;
          } else {
            jq = e % qpr;
            const int e2 = e / qpr;
            r = e2 & 1;
            kk = (e2 >> 1) & 15;
            q = e2 >> 5;
          }
          const int k = (kk & 3) + 8 * (kk >> 2) + 4 * r;
          hoff[i] = -1;
          hv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (e < nh) {
            hv[i] = *reinterpret_cast<const float4*>(hraw + (q * 32 + k) * 2 * us + 4 * jq);
            hoff[i] = t2_off(q >> 1, k, 32 * (q & 1) + 4 * jq);
          }
        }
        // Y task e: antenna pair kp, symbol block tb (t = 4 tb .. 4 tb + 3) of
        // unit q; 8-lane phases = 4 antenna pairs x 2 symbol blocks
        float4 yv[YT][4];
        int yoff[YT];
#pragma unroll
        for (int i = 0; i < YT; ++i) {
          const int e = ct + i * T2_CT;
          const int kp = (e & 3) + 4 * ((e >> 3) & 3);
          const int tb = ((e >> 2) & 1) + 2 * ((e >> 5) & 1);
          const int q = e >> 6;
          const int nl = q / g.gc, cl = q - nl * g.gc;
          const float* yq = yraw + cl * (g.ystride >> 2) + nl * T * T2_YROW;
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int t = 4 * tb + x;
            yv[i][x] = (t < T) ? *reinterpret_cast<const float4*>(yq + t * T2_YROW + 4 * kp)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          yoff[i] = t2_off(2 + (q >> 1), 2 * kp, 32 * (q & 1) + 8 * tb);
        }
        named_bar(1, T2_CT);  // every load of the stage done: convert in place
#pragma unroll
        for (int i = 0; i < HT; ++i) {
          if (hoff[i] < 0) continue;
          uint32_t w0[NSPLIT], w1[NSPLIT];
          split2<NSPLIT>(hv[i].x, hv[i].y, w0);
          split2<NSPLIT>(hv[i].z, hv[i].w, w1);
#pragma unroll
          for (int sp = 0; sp < NSPLIT; ++sp)
            *reinterpret_cast<uint2*>(st + sp * T2_SPLIT_BYTES + hoff[i]) = make_uint2(w0[sp], w1[sp]);
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
          // row 2kp + 1 sits at the next 128-byte K row; its chunk position is
          // the XOR with (k % 8) flipped in bit 0
          const int o0 = yoff[i];
          const int o1 = o0 + 128 + (((o0 >> 4) & 1) ? -16 : 16);
#pragma unroll
          for (int sp = 0; sp < NSPLIT; ++sp) {
            *reinterpret_cast<uint4*>(st + sp * T2_SPLIT_BYTES + o0) = make_uint4(a0[sp], a1[sp], a2[sp], a3[sp]);
            *reinterpret_cast<uint4*>(st + sp * T2_SPLIT_BYTES + o1) = make_uint4(b0[sp], b1[sp], b2[sp], b3[sp]);
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
    const int sv = warp - T2_FIRST_SOLV;
    const int sset = sv >> 2;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const Team<32, -1> tm{lane};
    Work w;
    {
      WorkLayout wl = L.w;
      const int base = L.work + sv * L.work_stride;
      wl.G += base; wl.Z += base; wl.X += base; wl.W += base; wl.Sv += base; wl.Vv += base; wl.Fb += base;
      wl.gb += base; wl.num += base; wl.phi += base; wl.coef += base; wl.s2 += base; wl.gn += base;
      wl.dg += base; wl.den += base; wl.harm += base; wl.wbuf += base; wl.flags += base;
      w = make_work(smem, wl, 16);
    }
    const int u = p.u, T = p.T, LD = w.LD;
    const int uh = lane >> 1, s_im = lane & 1;  // this lane's H feature: UE uh, re/im
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    int cl_first = 1;
    for (int gl = sset; gl < ngroups; gl += T2_NSET) {
      const int a = gl & 1;
      const int64_t uid = (g_first + gl) * 4 + q;
      const bool valid = uid < g.U_tot;
      const int64_t n = uid / g.upi;
      const int c = (int)(uid - n * g.upi);
      const float n0 = (valid && MODE != T2_STATS) ? item_n0(p, n) : 0.f;  // global load before the wait
      mbar_wait(&acc_full[a], (uint32_t)((gl >> 1) & 1));
      tc_fence_after();
      uint32_t gr[32], yr[32];
      tmem_ld32_nw(tq + (uint32_t)(256 * a + 32 * q), gr);
      tmem_ld32_nw(tq + (uint32_t)(256 * a + 128 + 32 * q), yr);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
      if (!valid) continue;
      // re/im recombination (one shuffle per column pair): even lanes form
      // the real parts, odd lanes the imaginary parts
      float* Gf = reinterpret_cast<float*>(w.G);
      float* Zf = reinterpret_cast<float*>(w.Z);
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const float mine = __uint_as_float(gr[2 * v]), po = __shfl_xor_sync(0xffffffffu, __uint_as_float(gr[2 * v + 1]), 1);
        const float val = s_im ? (po - mine) : (mine + po);
        if (uh < u && v < u) Gf[(uh * LD + v) * 2 + s_im] = val;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float mine = __uint_as_float(yr[2 * t]), po = __shfl_xor_sync(0xffffffffu, __uint_as_float(yr[2 * t + 1]), 1);
        const float val = s_im ? (po - mine) : (mine + po);
        if (uh < u && t < T) Zf[(t * LD + uh) * 2 + s_im] = val;
      }
      reset_flags(w, tm);
      tm.sync();
      if constexpr (MODE == T2_STATS) {
        unit_epilogue<16, Team<32, -1>, 0>(w, p, n, c, true, cl_first, tm, nullptr, n0);
      } else if constexpr (MODE == T2_PD) {
        unit_epilogue<16, Team<32, -1>, 1>(w, p, n, 0, true, cl_first, tm, nullptr, n0);
      } else {
        EpiArgs ea;
        ea.kind = p.kind;
        ea.u = u;
        ea.T = T;
        ea.n0 = n0;
        ea.es = p.es;
        ea.damping = p.damping;
        ea.t_max = p.t_max;
        ea.beta = p.cl_beta[c];
        ea.lama_scale = p.cl_scale[c];
        ea.unbias = true;  // fusion.py:148 -- fuse in the unbiased domain
        ea.ablate = 0;
        linear_unit<16>(w, ea, tm);
        // stash this cluster's estimate, count the arrival; the last of the
        // item's C clusters folds the records in cluster order
        fd_stash(w, p, n, c, tm);
        __threadfence_block();
        tm.sync();
        int last = 0;
        if (lane == 0) last = (atomicAdd(&fd_count[n & (T2_FD_CNT - 1)], 1) == p.C - 1);
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          if (lane == 0) fd_count[n & (T2_FD_CNT - 1)] = 0;
          __threadfence_block();
          fd_finish(reinterpret_cast<float*>(w.X), p, n, tm);
        }
      }
      tm.sync();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace dbp
