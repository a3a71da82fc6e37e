// libdbp_b200: sm_100a kernels for decentralized feedforward equalization
// (arXiv 1808.04473) behind the C ABI of include/dbp_b200.h.
//
// Hot path = one persistent kernel per (arch, u) that streams each item's
// channel block H[n] (B x u) and receive block Y[n] (T x B) through a ring of
// shared-memory stages filled by the TMA bulk-copy engine (cp.async.bulk +
// mbarrier), accumulates the Gram and the matched filter of all T symbols in
// registers (register-tiled complex outer products, K split over thread
// groups), and runs the equalizer, FD fusion and the QAM slicer on chip.  Only
// estimates, variances, weights and decisions are written back to HBM.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "../../include/dbp_b200.h"
#include "dbp_device.cuh"
#include "dbp_epilogue.cuh"

namespace dbp {

struct EqParams {
  const float2* H;
  const float2* Y;
  const float2* stats_in;
  int64_t n_items;
  int B, u, us, T, TP;
  int KC, KCP, NS;
  int stage_f2;  // float2 elements per stage
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
  float2 *tr_z, *tr_s, *tr_v;
  float* tr_phi;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

// Shared-memory carve-up (byte offsets), identical on host and device.
struct Layout {
  int bars, stages, red, G, Z, X, W, Sv, Vv, Fb, gb, num, phi, coef, s2, gn, dg, den, harm, wbuf,
      flags, total;
};

__host__ __device__ inline Layout make_layout(int UP, int NT, int TP, int stage_bytes, int NS,
                                              int C, int red_f2, bool lama, bool fd) {
  Layout L;
  const int LD = UP + 1;
  int o = 0;
  L.bars = o;
  o += align_up(NS * 8, 16);
  o = align_up(o, 128);
  L.stages = o;
  o += NS * stage_bytes;
  o = align_up(o, 16);
  L.red = o;
  o += red_f2 * 8;
  L.G = o;
  o += UP * LD * 8;
  L.Z = o;
  o += TP * LD * 8;
  L.X = o;
  o += TP * LD * 8;
  L.W = o;
  o += lama ? 0 : 4 * UP * 8;
  L.Sv = o;
  o += lama ? TP * LD * 8 : 0;
  L.Vv = o;
  o += lama ? TP * LD * 8 : 0;
  L.Fb = o;
  o += lama ? TP * LD * 8 : 0;
  L.gb = o;
  o += lama ? TP * LD * 4 : 0;
  L.num = o;
  o += fd ? TP * LD * 8 : 0;
  const int V = (UP > TP ? UP : TP);
  L.phi = o;
  o += TP * 4;
  L.coef = o;
  o += TP * 4;
  L.s2 = o;
  o += V * 4;
  L.gn = o;
  o += UP * 4;
  L.dg = o;
  o += UP * 4;
  L.den = o;
  o += fd ? V * 4 : 0;
  L.harm = o;
  o += fd ? V * 4 : 0;
  L.wbuf = o;
  o += fd ? C * V * 4 : 0;
  L.flags = o;
  o += 16;
  L.total = align_up(o, 128);
  (void)NT;
  return L;
}

__device__ __forceinline__ Work make_work(char* smem, const Layout& L, int UP) {
  Work w;
  w.G = reinterpret_cast<float2*>(smem + L.G);
  w.Z = reinterpret_cast<float2*>(smem + L.Z);
  w.X = reinterpret_cast<float2*>(smem + L.X);
  w.W = reinterpret_cast<float2*>(smem + L.W);
  w.Sv = reinterpret_cast<float2*>(smem + L.Sv);
  w.Vv = reinterpret_cast<float2*>(smem + L.Vv);
  w.Fb = reinterpret_cast<float2*>(smem + L.Fb);
  w.gb = reinterpret_cast<float*>(smem + L.gb);
  w.phi = reinterpret_cast<float*>(smem + L.phi);
  w.coef = reinterpret_cast<float*>(smem + L.coef);
  w.s2 = reinterpret_cast<float*>(smem + L.s2);
  w.gn = reinterpret_cast<float*>(smem + L.gn);
  w.dg = reinterpret_cast<float*>(smem + L.dg);
  w.flags = reinterpret_cast<int*>(smem + L.flags);
  w.LD = UP + 1;
  return w;
}

__device__ __forceinline__ float item_n0(const EqParams& p, int64_t n) {
  return p.n0_dev ? p.n0_dev[n / p.n0_group] : p.n0;
}

// Register tile owned by one thread: a 4x4 block of the output
// O = H^H [H | Y^T]; G tiles (ib <= jb) cover the upper Hermitian half of the
// Gram, Z tiles cover y_mrc for 4 OFDM symbols.  `g` is the thread's K group.
struct TileInfo {
  int ib, jb, isz, g, S, active;
};

template <int UP>
__device__ __forceinline__ TileInfo decode_tile(int tid, int TB, int NT) {
  constexpr int UB = UP / 4;
  constexpr int NG = UB * (UB + 1) / 2;
  const int ntiles = NG + UB * TB;
  TileInfo ti;
  ti.S = NT / ntiles;
  const int tile = tid % ntiles;
  ti.g = tid / ntiles;
  ti.active = ti.g < ti.S;
  if (tile < NG) {
    int r = tile, ib = 0;
    while (r >= UB - ib) {
      r -= UB - ib;
      ++ib;
    }
    ti.ib = ib;
    ti.jb = ib + r;
    ti.isz = 0;
  } else {
    const int z = tile - NG;
    ti.ib = z % UB;
    ti.jb = z / UB;
    ti.isz = 1;
  }
  return ti;
}

// Accumulate one chunk (nrows antenna rows) into the 4x4 tile.
__device__ __forceinline__ void accumulate_chunk(float2 (&acc)[4][4], const float2* __restrict__ Hs,
                                                 const float2* __restrict__ Ys, int nrows, int us, int KCP,
                                                 const TileInfo& ti) {
  const float2* ap = Hs + 4 * ti.ib + ti.g * us;
  const float2* xp;
  int xstep, cs;
  if (ti.isz) {
    xp = Ys + 4 * ti.jb * KCP + ti.g;
    xstep = ti.S;
    cs = KCP;
  } else {
    xp = Hs + 4 * ti.jb + ti.g * us;
    xstep = ti.S * us;
    cs = 1;
  }
  const int astep = ti.S * us;
#pragma unroll 2
  for (int k = ti.g; k < nrows; k += ti.S) {
    const float4 a01 = *reinterpret_cast<const float4*>(ap);
    const float4 a23 = *reinterpret_cast<const float4*>(ap + 2);
    const float2 a[4] = {make_float2(a01.x, a01.y), make_float2(a01.z, a01.w), make_float2(a23.x, a23.y),
                         make_float2(a23.z, a23.w)};
    const float2 x[4] = {xp[0], xp[cs], xp[2 * cs], xp[3 * cs]};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) c_fma_conj(acc[r][c], a[r], x[c]);
    ap += astep;
    xp += xstep;
  }
}

// Reduce the K groups' tiles into G / Z (shared), then zero the accumulators.
// Groups g >= 1 park their partial tiles in `red`; the g == 0 owner of each
// tile adds them and writes the tile (and its Hermitian mirror).
template <int UP, int NT>
__device__ __forceinline__ void reduce_tiles(float2 (&acc)[4][4], const TileInfo& ti, float2* red, const Work& w,
                                             int T, int ntiles) {
  const int tid = threadIdx.x;
  const int LD = w.LD;
  if (ti.S > 1) {
    const int tile = tid % ntiles;
    if (ti.active && ti.g > 0) {
#pragma unroll
      for (int e = 0; e < 16; ++e) red[((ti.g - 1) * 16 + e) * ntiles + tile] = acc[e >> 2][e & 3];
    }
    __syncthreads();
    if (ti.g == 0) {
      for (int g = 1; g < ti.S; ++g)
#pragma unroll
        for (int e = 0; e < 16; ++e)
          acc[e >> 2][e & 3] = c_add(acc[e >> 2][e & 3], red[((g - 1) * 16 + e) * ntiles + tile]);
    }
  }
  if (ti.active && ti.g == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * ti.ib + r;
        if (ti.isz) {
          const int t = 4 * ti.jb + c;
          if (t < T) w.Z[t * LD + i] = acc[r][c];
        } else {
          const int j = 4 * ti.jb + c;
          w.G[i * LD + j] = acc[r][c];
          if (ti.ib != ti.jb) w.G[j * LD + i] = c_conj(acc[r][c]);
        }
      }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
  __syncthreads();
}

// Write X (per-symbol estimates) + decisions of one item.
template <int NT>
__device__ __forceinline__ void store_estimates(const Work& w, const EqParams& p, int64_t n, bool divide_gain) {
  const int u = p.u, T = p.T, LD = w.LD;
  for (int e = threadIdx.x; e < T * u; e += NT) {
    const int t = e / u, i = e - t * u;
    float2 x = w.X[t * LD + i];
    if (divide_gain) x = c_scale(x, 1.f / w.gn[i]);
    const size_t o = ((size_t)n * T + t) * u + i;
    p.xhat[o] = x;
    if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
  }
}

// The unit epilogue for PD / single-cluster calls: equalize, write outputs.
template <int UP, int NT>
__device__ void pd_epilogue(const Work& w, const EqParams& p, int64_t n, float n0) {
  EpiArgs a;
  a.kind = p.kind;
  a.u = p.u;
  a.T = p.T;
  a.n0 = n0;
  a.es = p.es;
  a.beta = p.beta;
  a.lama_scale = p.lama_scale;
  a.damping = p.damping;
  a.t_max = p.t_max;
  a.unbias = p.unbias != 0;
  const int tid = threadIdx.x;
  if (p.kind == EQ_LAMA) {
    float2* tz = nullptr;
    float2* ts = nullptr;
    float2* tv = nullptr;
    float* tp = nullptr;
    if (p.tr_z) {
      const size_t o = (size_t)n * p.t_max * p.T * p.u;
      tz = p.tr_z + o;
      ts = p.tr_s + o;
      tv = p.tr_v + o;
      tp = p.tr_phi + (size_t)n * p.t_max * p.T;
    }
    lama_unit<NT>(w, a, p.cp, tz, ts, tv, tp);
    store_estimates<NT>(w, p, n, false);
    for (int t = tid; t < p.T; t += NT) p.sigma2[(size_t)n * p.T + t] = w.s2[t];
  } else {
    linear_unit<UP, NT>(w, a);
    store_estimates<NT>(w, p, n, false);
    for (int i = tid; i < p.u; i += NT) {
      p.sigma2[(size_t)n * p.u + i] = w.s2[i];
      if (p.gain && (p.kind == EQ_LMMSE || p.kind == EQ_MRC)) p.gain[(size_t)n * p.u + i] = w.gn[i];
    }
  }
  if (tid == 0) {
    int st = w.flags[0];
    if (w.flags[1] < 0x7fffffff) st = st ? st : ST_DIVERGED;
    p.status[n] = st;
    if (p.iters) p.iters[n] = (w.flags[1] < 0x7fffffff) ? w.flags[1] : 0;
  }
}

// FD: fold one cluster's equalized output into the fusion sums
// (fusion.py:141-153 -- unbiased estimates; MRC weights = Gram diagonal,
// otherwise 1/max(sigma2, 1e-15); sigma2 <= 0 is a ConfigError).
template <int NT>
__device__ void fd_accumulate(const Work& w, float2* num, float* den, float* harm, float* wbuf, const EqParams& p,
                              int c, bool first) {
  const int u = p.u, T = p.T, LD = w.LD;
  const bool lama = p.kind == EQ_LAMA;
  const int wdim = lama ? T : u;
  for (int e = threadIdx.x; e < wdim; e += NT) {
    const float s2 = w.s2[e];
    if (p.kind != EQ_MRC && !(s2 > 0.f)) set_status(w.flags, ST_BADVAR);
    const float inv = 1.f / fmaxf(s2, VAR_FLOOR);
    const float wt = (p.kind == EQ_MRC) ? w.gn[e] : inv;
    wbuf[c * wdim + e] = wt;
    den[e] = first ? wt : den[e] + wt;
    harm[e] = first ? inv : harm[e] + inv;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < T * u; e += NT) {
    const int t = e / u, i = e - t * u;
    const float wt = wbuf[c * wdim + (lama ? t : i)];
    const float2 x = c_scale(w.X[t * LD + i], wt);
    num[t * LD + i] = first ? x : c_add(num[t * LD + i], x);
  }
  // caller syncs before the next unit reuses X
}

// ============================================================================
// Persistent streaming kernel: (H, Y) -> stats | PD outputs | FD outputs.
// ============================================================================
template <int UP, int NT>
__global__ void __launch_bounds__(NT) stream_kernel(const __grid_constant__ EqParams p) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x;
  const bool lama = p.kind == EQ_LAMA;
  const bool fd = (p.arch == ARCH_FD || p.arch == ARCH_FD_PARTIAL);
  const int TB = p.TP / 4;
  constexpr int UB = UP / 4;
  constexpr int NG = UB * (UB + 1) / 2;
  const int ntiles = NG + UB * TB;
  const TileInfo ti = decode_tile<UP>(tid, TB, NT);
  const int red_f2 = (ti.S > 1) ? (ti.S - 1) * ntiles * 16 : 0;
  const Layout L = make_layout(UP, NT, p.TP, p.stage_f2 * 8, p.NS, p.C, red_f2, lama, fd);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  float2* red = reinterpret_cast<float2*>(smem + L.red);
  Work w = make_work(smem, L, UP);
  float2* num = reinterpret_cast<float2*>(smem + L.num);
  float* den = reinterpret_cast<float*>(smem + L.den);
  float* harm = reinterpret_cast<float*>(smem + L.harm);
  float* wbuf = reinterpret_cast<float*>(smem + L.wbuf);

  if (tid == 0) {
    for (int s = 0; s < p.NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    w.flags[0] = 0;
    w.flags[1] = 0x7fffffff;
  }
  __syncthreads();

  const int64_t my_items = (p.n_items > blockIdx.x) ? (p.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_items * p.nchunks;
  const uint64_t policy = l2_evict_first_policy();
  const int stage_bytes = p.stage_f2 * 8;

  auto issue = [&](int64_t q) {
    if (q >= total) return;
    const int qi = (int)q;
    const int il = qi / p.nchunks;
    const int j = qi - il * p.nchunks;
    const int64_t n = blockIdx.x + (int64_t)il * gridDim.x;
    const ChunkDesc cd = p.chunks[j];
    const int s = qi % p.NS;
    char* st = smem + L.stages + s * stage_bytes;
    const uint32_t hbytes = (uint32_t)cd.nrows * p.us * 8;
    const uint32_t ybytes = (uint32_t)cd.nrows * 8;
    mbar_arrive_expect_tx(&bars[s], hbytes + ybytes * p.T);
    bulk_g2s(st, p.H + ((size_t)n * p.B + cd.row0) * p.us, hbytes, &bars[s], policy);
    float2* ys = reinterpret_cast<float2*>(st) + p.KC * p.us;
    const float2* ysrc = p.Y + (size_t)n * p.T * p.B + cd.row0;
    for (int t = 0; t < p.T; ++t) bulk_g2s(ys + t * p.KCP, ysrc + (size_t)t * p.B, ybytes, &bars[s], policy);
  };
  if (tid == 0)
    for (int q = 0; q < p.NS; ++q) issue(q);

  float2 acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);

  int cl_first = 1;  // FD: first cluster of the current item
  int jn = 0, sn = 0;  // chunk-in-item and stage of the next chunk
  uint32_t phase = 0;
  int64_t nn = blockIdx.x;
  for (int64_t q = 0; q < total; ++q) {
    const ChunkDesc cd = p.chunks[jn];
    const int s = sn;
    const int64_t n = nn;
    mbar_wait(&bars[s], phase);
    if (++sn == p.NS) {
      sn = 0;
      phase ^= 1u;
    }
    if (++jn == p.nchunks) {
      jn = 0;
      nn += gridDim.x;
    }
    const float2* Hs = reinterpret_cast<const float2*>(smem + L.stages + s * stage_bytes);
    const float2* Ys = Hs + p.KC * p.us;
    if (ti.active) accumulate_chunk(acc, Hs, Ys, cd.nrows, p.us, p.KCP, ti);
    __syncthreads();  // stage s consumed
    if (tid == 0) issue(q + p.NS);

    const bool item_end = (cd.flags & CH_ITEM_END) != 0;
    const bool per_cluster = fd || (p.arch == ARCH_STATS && !p.sum_clusters);
    const bool unit_end = item_end || (per_cluster && (cd.flags & CH_CLUSTER_END));
    if (!unit_end) continue;

    reduce_tiles<UP, NT>(acc, ti, red, w, p.T, ntiles);
    const float n0 = item_n0(p, n);

    if (p.arch == ARCH_STATS) {
      const int ncl = p.sum_clusters ? 1 : p.C;
      const int cl = p.sum_clusters ? 0 : cd.cluster;
      const int u = p.u;
      float2* dst = p.stats_out + ((size_t)n * ncl + cl) * (size_t)(u * u + p.T * u);
      for (int e = tid; e < u * u; e += NT) dst[e] = w.G[(e / u) * w.LD + (e % u)];
      for (int e = tid; e < p.T * u; e += NT) dst[u * u + e] = w.Z[(e / u) * w.LD + (e % u)];
      __syncthreads();
      continue;
    }
    if (p.arch == ARCH_PD) {
      pd_epilogue<UP, NT>(w, p, n, n0);
      __syncthreads();
      if (tid == 0) {
        w.flags[0] = 0;
        w.flags[1] = 0x7fffffff;
      }
      __syncthreads();
      continue;
    }
    // ---- FD: equalize this cluster, fold into the fusion sums ----
    {
      const int c = cd.cluster;
      EpiArgs a;
      a.kind = p.kind;
      a.u = p.u;
      a.T = p.T;
      a.n0 = n0;
      a.es = p.es;
      a.beta = p.cl_beta[c];
      a.lama_scale = p.cl_scale[c];
      a.damping = p.damping;
      a.t_max = p.t_max;
      a.unbias = true;  // fusion.py:148 -- fuse in the unbiased domain
      if (lama)
        lama_unit<NT>(w, a, p.cp, nullptr, nullptr, nullptr, nullptr);
      else
        linear_unit<UP, NT>(w, a);
      fd_accumulate<NT>(w, num, den, harm, wbuf, p, c, cl_first != 0);
      __syncthreads();
      cl_first = 0;
    }
    if (!item_end) continue;
    {
      const int u = p.u, T = p.T, LD = w.LD;
      const int wdim = lama ? T : u;
      if (p.arch == ARCH_FD) {
        for (int e = tid; e < T * u; e += NT) {
          const int t = e / u, i = e - t * u;
          const float2 x = c_scale(num[t * LD + i], 1.f / den[lama ? t : i]);
          const size_t o = ((size_t)n * T + t) * u + i;
          p.xhat[o] = x;
          if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
        }
        for (int e = tid; e < wdim; e += NT) p.sigma2[(size_t)n * wdim + e] = 1.f / harm[e];
        if (p.nu)
          for (int e = tid; e < p.C * wdim; e += NT) {
            const int k = e % wdim;
            p.nu[(size_t)n * p.C * wdim + e] = wbuf[e] / den[k];
          }
      } else {  // FD_PARTIAL: raw sums for a cross-GPU reduction
        const int rec = 2 * T * u + 2 * wdim;
        float* dst = p.fd_acc + (size_t)n * rec;
        for (int e = tid; e < T * u; e += NT) {
          const int t = e / u, i = e - t * u;
          const float2 v = num[t * LD + i];
          dst[2 * e] = v.x;
          dst[2 * e + 1] = v.y;
        }
        for (int e = tid; e < wdim; e += NT) {
          dst[2 * T * u + e] = den[e];
          dst[2 * T * u + wdim + e] = harm[e];
        }
        for (int e = tid; e < p.C * wdim; e += NT) p.fd_wraw[(size_t)n * p.C * wdim + e] = wbuf[e];
      }
      if (tid == 0) {
        int st = w.flags[0];
        if (w.flags[1] < 0x7fffffff) st = st ? st : ST_DIVERGED;
        p.status[n] = st;
        if (p.iters) p.iters[n] = (w.flags[1] < 0x7fffffff) ? w.flags[1] : 0;
      }
      __syncthreads();
      if (tid == 0) {
        w.flags[0] = 0;
        w.flags[1] = 0x7fffffff;
      }
      cl_first = 1;
      __syncthreads();
    }
  }
}

// ============================================================================
// Equalization from precomputed statistics (PD central node after the
// reduce-scatter; linear_equalize / lama_equalize API).
// ============================================================================
template <int UP, int NT>
__global__ void __launch_bounds__(NT) stats_kernel(const __grid_constant__ EqParams p) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x;
  const bool lama = p.kind == EQ_LAMA;
  const Layout L = make_layout(UP, NT, p.TP, 0, 0, 1, 0, lama, false);
  Work w = make_work(smem, L, UP);
  const int u = p.u, T = p.T;
  const size_t rec = (size_t)u * u + (size_t)T * u;
  for (int64_t n = blockIdx.x; n < p.n_items; n += gridDim.x) {
    if (tid == 0) {
      w.flags[0] = 0;
      w.flags[1] = 0x7fffffff;
    }
    const float2* src = p.stats_in + n * rec;
    for (int e = tid; e < u * u; e += NT) w.G[(e / u) * w.LD + (e % u)] = src[e];
    for (int e = tid; e < T * u; e += NT) w.Z[(e / u) * w.LD + (e % u)] = src[u * u + e];
    __syncthreads();
    pd_epilogue<UP, NT>(w, p, n, item_n0(p, n));
    __syncthreads();
  }
}

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
      const float d = 1.f - c;
      const float v = (s2[item * u + i] - d * d * es) / (c * c);
      if (v < -1e-9f) atomicCAS(status + item, 0, ST_NEGVAR);
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

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static int cuda_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DBP_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return DBP_OK;
}

static int sm_count() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

static int up_for(int u) { return u <= 8 ? 8 : u <= 16 ? 16 : u <= 32 ? 32 : u <= 64 ? 64 : -1; }

static int fill_const(ConstParams& cp, const float* levels, int L, const float* symbols, int M, float es) {
  memset(&cp, 0, sizeof(cp));
  if (L < 0 || L > MAX_L || M < 0 || M > MAX_SYMS) return fail(DBP_E_ARG, "constellation too large");
  cp.L = L;
  cp.M = M;
  cp.es = es;
  for (int l = 0; l < L; ++l) cp.levels[l] = levels[l];
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

template <int UP, int NT>
static int launch_stream(EqParams& p, cudaStream_t st) {
  const bool lama = p.kind == EQ_LAMA;
  const bool fd = (p.arch == ARCH_FD || p.arch == ARCH_FD_PARTIAL);
  const int TB = p.TP / 4;
  constexpr int UB = UP / 4;
  const int ntiles = UB * (UB + 1) / 2 + UB * TB;
  const int S = NT / ntiles;
  if (S < 1) return fail(DBP_E_UNSUPPORTED, "too many output tiles for the CTA (u, T too large)");
  const int red_f2 = S > 1 ? (S - 1) * ntiles * 16 : 0;
  const Layout L = make_layout(UP, NT, p.TP, p.stage_f2 * 8, p.NS, p.C, red_f2, lama, fd);
  auto kern = stream_kernel<UP, NT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return fail(DBP_E_CUDA, "shared memory request too large");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, L.total);
  if (per_sm < 1) return fail(DBP_E_UNSUPPORTED, "kernel does not fit on an SM");
  const int64_t grid = std::min<int64_t>(p.n_items, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, NT, L.total, st>>>(p);
  return cuda_check("stream_kernel");
}

template <int UP, int NT>
static int launch_stats(EqParams& p, cudaStream_t st) {
  const bool lama = p.kind == EQ_LAMA;
  const Layout L = make_layout(UP, NT, p.TP, 0, 0, 1, 0, lama, false);
  auto kern = stats_kernel<UP, NT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return fail(DBP_E_CUDA, "shared memory request too large");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, L.total);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>(p.n_items, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, NT, L.total, st>>>(p);
  return cuda_check("stats_kernel");
}

static int dispatch_stream(EqParams& p, cudaStream_t st) {
  switch (up_for(p.u)) {
    case 8: return launch_stream<8, 128>(p, st);
    case 16: return launch_stream<16, 128>(p, st);
    case 32: return launch_stream<32, 256>(p, st);
    case 64: return launch_stream<64, 256>(p, st);
  }
  return fail(DBP_E_UNSUPPORTED, "u must be <= 64");
}

static int dispatch_stats(EqParams& p, cudaStream_t st) {
  switch (up_for(p.u)) {
    case 8: return launch_stats<8, 128>(p, st);
    case 16: return launch_stats<16, 128>(p, st);
    case 32: return launch_stats<32, 256>(p, st);
    case 64: return launch_stats<64, 256>(p, st);
  }
  return fail(DBP_E_UNSUPPORTED, "u must be <= 64");
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
  if (n_items <= 0) return DBP_OK;
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

}  // extern "C"
