// Wide statistics kernel (U = 64): per-unit Gram and matched filter
//   G = H^H H,  y_mrc[t] = H^H y_t        (equalize.py:85-93, 96-107)
// for 32 < u <= 64 on the tcgen05 tensor cores, with the operands split into
// bf16 parts (x = h + m (+ l)) like the U <= 16 kernel (dbp_tc2.cuh).
//
// Here one unit fills the MMA: its 2u <= 128 real H features are M, and
// N = 128 H features + 32 Y features (2T <= 32), so one
// tcgen05.mma.kind::f16 (M = 128, N = 160, K = 16) per bf16 product and
// 16 antennas computes P = Xh^T [Xh | Xy] with no idle rows; accumulator
// lane 2v + s / column 2w + s' hold the re/im cross products that recombine
// into G[v][w] and y_mrc[t][v].
//
// A unit is one item (PD: every antenna, sum_clusters) or one cluster of an
// item (per-cluster statistics); its K antennas (a multiple of 32) stream in
// stages of 32.  Per stage two TMA loads (H box 32 antennas x 128 floats, Y
// box T rows x 64 floats) land in a stage slot; the converter warps load the
// whole slot, meet at a named barrier and write the bf16 parts in place as
// MN-major 128-byte-swizzled tiles ([part][3 MN blocks of 64][32 K rows of
// 128 B]; block 2 holds the Y features); the MMA warp issues 2 K-steps x
// (3 or 6) products into one of two TMEM accumulators (256 columns each);
// four epilogue warps (one per TMEM lane quarter = 16 UEs) read the
// accumulator, release it, recombine re/im with one shuffle per column pair
// and store the statistics record [G (u x u) | y_mrc (T x u)] -- G written
// conjugate-transposed (G is Hermitian), so every warp store is 128
// contiguous bytes.
//
// Roles: warp 0 TMA producer, warp 1 MMA issuer, TW_NCONV converter warps,
// four epilogue warps.  Persistent: one CTA per SM, contiguous unit ranges.
#pragma once
#include "dbp_tc2.cuh"

namespace dbp {

#ifndef DBP_TW_NCONV
#define DBP_TW_NCONV 8
#endif
constexpr int TW_NCONV = DBP_TW_NCONV;  // converter warps (4 or 8)
constexpr int TW_FIRST_CONV = 2;
constexpr int TW_FIRST_EPI = TW_FIRST_CONV + TW_NCONV;
constexpr int TW_NEPI = 4;
constexpr int TW_THREADS = 32 * (TW_FIRST_EPI + TW_NEPI);
constexpr int TW_CT = 32 * TW_NCONV;
constexpr int TW_SPLIT = 3 * 4096;  // one bf16 part: MN blocks [H 0..63][H 64..127][Y 0..31]
constexpr int TW_YROW = 64;         // floats per raw Y row (32 antennas, re/im)
constexpr int TW_HBYTES = 32 * 128 * 4;

struct TcwGeom {
  int K;       // antennas per unit (multiple of 32)
  int nchunk;  // K / 32
  int upi;     // units per item (1: summed over clusters, C: per cluster)
  int T;
  int NS, stage_bytes;
  int64_t n_units;
};

__host__ __device__ inline int tcw_bars_bytes(int NS) { return align_up((3 * NS + 4) * 8 + 16, 1024); }

template <int NSPLIT>
__global__ void __launch_bounds__(TW_THREADS, 1)
    tcw_stats_kernel(const __grid_constant__ EqParams p, const __grid_constant__ CUtensorMap hmap,
                     const __grid_constant__ CUtensorMap ymap, const __grid_constant__ TcwGeom g) {
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int NS = g.NS;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* conv_full = raw_full + NS;
  uint64_t* stage_empty = conv_full + NS;
  uint64_t* acc_full = stage_empty + NS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  char* stages = smem + tcw_bars_bytes(NS);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&conv_full[s], TW_NCONV);
      mbar_init(&stage_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], TW_NEPI);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t per = g.n_units / gridDim.x, extra = g.n_units % gridDim.x;
  const int64_t u_first = blockIdx.x * per + min((int64_t)blockIdx.x, extra);
  const int nunits = (int)(per + (blockIdx.x < extra ? 1 : 0));
  const int nch = g.nchunk;
  const uint32_t stg0 = smem_u32(stages);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ----
    if (lane == 0) {
      prefetch_tmap(&hmap);
      prefetch_tmap(&ymap);
      const uint64_t policy = l2_evict_first_policy();
      const int total = nunits * nch;
      auto coords = [&](int sq, int& a0, int& item) {
        const int ul = sq / nch, j = sq - ul * nch;
        const int64_t un = u_first + ul;
        item = (int)(un / g.upi);
        const int c = (int)(un - (int64_t)item * g.upi);
        a0 = c * g.K + 32 * j;  // first antenna of the stage
      };
      int s = 0;
      uint32_t ph = 0;
      for (int sq = 0; sq < total; ++sq) {
        if (sq >= NS) mbar_wait(&stage_empty[s], ph ^ 1u);
        int a0, item;
        coords(sq, a0, item);
        const uint32_t bar = smem_u32(&raw_full[s]);
        mbar_arrive_expect_tx(&raw_full[s], (uint32_t)(TW_HBYTES + g.T * TW_YROW * 4));
        const uint32_t dst = stg0 + (uint32_t)(s * g.stage_bytes);
        tma_load_3d(dst, &hmap, 0, a0, item, bar, policy);
        tma_load_3d(dst + TW_HBYTES, &ymap, 2 * a0, 0, item, bar, policy);
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
      constexpr uint32_t idesc = umma_idesc_bf16_mn(128, 160);
      constexpr int NP = NSPLIT == 2 ? 3 : 6;
      constexpr int PA[6] = {0, 0, 1, 1, 0, 2};
      constexpr int PB[6] = {0, 1, 0, 1, 2, 0};
      int s = 0;
      uint32_t ph = 0;
      int uses[2] = {0, 0};
      for (int ul = 0; ul < nunits; ++ul) {
        const int a = ul & 1;
        if (uses[a] >= 1) mbar_wait(&acc_empty[a], (uint32_t)((uses[a] - 1) & 1));
        ++uses[a];
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
              const uint64_t da = umma_desc_mn16(base + PA[pr] * TW_SPLIT + ks * 2048);
              const uint64_t db = umma_desc_mn16(base + PB[pr] * TW_SPLIT + ks * 2048);
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
  } else if (warp < TW_FIRST_EPI) {
    // -------------------------------------------------------- converters ----
    const int ct = tid - 32 * TW_FIRST_CONV;
    const int T = g.T;
    constexpr int RSTEP = TW_CT / 32;   // antenna rows (H) / symbol pairs (Y) per task round
    constexpr int HT = 32 / RSTEP;      // H tasks per thread
    constexpr int YT = 8 / RSTEP;       // Y tasks per thread (T <= 16: 8 symbol pairs)
    static_assert(HT >= 1 && YT >= 1, "converter task split");
    // H task i: quad jq (features 4 jq .. 4 jq + 3) of antenna row k0 + RSTEP i;
    // Y task i: symbol pair tp = k0 + RSTEP i (symbols 2 tp, 2 tp + 1) of antenna jq
    const int jq = ct & 31, k0 = ct >> 5;
    int s = 0;
    uint32_t ph = 0;
    const int total = nunits * nch;
    for (int sq = 0; sq < total; ++sq) {
      mbar_wait(&raw_full[s], ph);
      char* st = stages + s * g.stage_bytes;
      const float* sf = reinterpret_cast<const float*>(st);
      const float* yf = sf + TW_HBYTES / 4;
      float4 hv[HT];
#pragma unroll
      for (int i = 0; i < HT; ++i) hv[i] = *reinterpret_cast<const float4*>(sf + (k0 + RSTEP * i) * 128 + 4 * jq);
      float2 ya[YT], yb[YT];
#pragma unroll
      for (int i = 0; i < YT; ++i) {
        const int tp = k0 + RSTEP * i;
        ya[i] = (2 * tp < T) ? *reinterpret_cast<const float2*>(yf + (2 * tp) * TW_YROW + 2 * jq) : make_float2(0.f, 0.f);
        yb[i] = (2 * tp + 1 < T) ? *reinterpret_cast<const float2*>(yf + (2 * tp + 1) * TW_YROW + 2 * jq)
                                 : make_float2(0.f, 0.f);
      }
      named_bar(1, TW_CT);  // the whole slot is in registers: overwrite it in place
      if (T2_ABLATE(4)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_full[s]);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < HT; ++i) {
        uint32_t w0[NSPLIT], w1[NSPLIT];
        split2<NSPLIT>(hv[i].x, hv[i].y, w0);
        split2<NSPLIT>(hv[i].z, hv[i].w, w1);
        const int off = t2_off(jq >> 4, k0 + RSTEP * i, 4 * (jq & 15));
#pragma unroll
        for (int sp = 0; sp < NSPLIT; ++sp)
          *reinterpret_cast<uint2*>(st + sp * TW_SPLIT + off) = make_uint2(w0[sp], w1[sp]);
      }
#pragma unroll
      for (int i = 0; i < YT; ++i) {
        const int tp = k0 + RSTEP * i;
        uint32_t w0[NSPLIT], w1[NSPLIT];
        split2<NSPLIT>(ya[i].x, ya[i].y, w0);
        split2<NSPLIT>(yb[i].x, yb[i].y, w1);
        const int off = t2_off(2, jq, 4 * tp);
#pragma unroll
        for (int sp = 0; sp < NSPLIT; ++sp)
          *reinterpret_cast<uint2*>(st + sp * TW_SPLIT + off) = make_uint2(w0[sp], w1[sp]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv_full[s]);
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue ----
    const int q = warp & 3;  // TMEM lane quarter: H features 32 q .. 32 q + 31 = UEs 16 q .. 16 q + 15
    const int u = p.u, T = p.T;
    const int s_im = lane & 1, ue = 16 * q + (lane >> 1);
    const size_t rec = (size_t)u * u + (size_t)T * u;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    int use[2] = {0, 0};
    for (int ul = 0; ul < nunits; ++ul) {
      const int a = ul & 1;
      mbar_wait(&acc_full[a], (uint32_t)(use[a] & 1));
      ++use[a];
      tc_fence_after();
      const int64_t un = u_first + ul;
      const int64_t item = un / g.upi;
      const int cl = (int)(un - item * g.upi);
      float* dst = reinterpret_cast<float*>(p.stats_out + (size_t)(item * g.upi + cl) * rec);
      uint32_t r[32];
#pragma unroll 1
      for (int cc = 0; cc < 5; ++cc) {
        tmem_ld32_nw(tq + (uint32_t)(256 * a + 32 * cc), r);
        tmem_ld_wait();
        if (cc == 4) {  // every column read: the accumulator is free
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[a]);
        }
        if (T2_ABLATE(1)) continue;
        // lane (ue, s_im) forms component s_im of G[ue][w] (or y_mrc[t][ue]):
        // re = P[2ue][2w] + P[2ue+1][2w+1], im = P[2ue][2w+1] - P[2ue+1][2w];
        // G goes out conjugate-transposed, G[w][ue] = re - i im: one FFMA each
        const float sg = s_im ? -1.f : 1.f;
        if (u == 64) {  // full tiles: fixed strides, no bounds
          float* gcol = dst + ue * 2 + s_im;  // G[w][ue] at gcol[w * 128]
          if (cc < 4) {
#pragma unroll
            for (int v = 0; v < 16; ++v) {
              const float mine = __uint_as_float(r[2 * v]);
              const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(r[2 * v + 1]), 1);
              gcol[(16 * cc + v) * 128] = fmaf(sg, po, mine);
            }
          } else {
            float* ycol = gcol + 64 * 64 * 2;  // y_mrc[t][ue] at ycol[t * 128]
#pragma unroll
            for (int v = 0; v < 16; ++v) {
              const float mine = __uint_as_float(r[2 * v]);
              const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(r[2 * v + 1]), 1);
              if (v < T) ycol[v * 128] = fmaf(sg, mine, po);
            }
          }
          continue;
        }
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float mine = __uint_as_float(r[2 * v]);
          const float po = __shfl_xor_sync(0xffffffffu, __uint_as_float(r[2 * v + 1]), 1);
          if (ue < u) {
            if (cc < 4) {  // G[ue][w] stored as G[w][ue] = conj(G[ue][w])
              const int wc = 16 * cc + v;
              if (wc < u) dst[((size_t)wc * u + ue) * 2 + s_im] = fmaf(sg, po, mine);
            } else if (v < T) {  // y_mrc[t = v][ue]
              dst[((size_t)u * u + (size_t)v * u + ue) * 2 + s_im] = fmaf(sg, mine, po);
            }
          }
        }
      }
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
