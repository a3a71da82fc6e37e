// CTA-synchronous streaming kernel with an FP32 SIMT Gram/matched-filter
// mainloop (register-tiled complex outer products).  Used for U = 64, where the
// real-embedded operand (2(U+T) = 156 rows) exceeds one tcgen05 M=128 tile;
// U <= 32 runs on the tensor-core kernel in dbp_tc.cuh.  Also the
// statistics-input kernel (central node of the multi-GPU PD path).
#pragma once
#include "dbp_epilogue.cuh"

namespace dbp {

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

// Shared-memory carve-up of the unit working set (byte offsets from `base`).
struct WorkLayout {
  int G, Z, X, W, Sv, Vv, Fb, gb, num, phi, coef, s2, gn, dg, den, harm, wbuf, flags, total;
};

// x_in_z: the solution X overwrites y_mrc in Z (linear solves of the FD U = 64
// statistics kernel: 8.4 KB less, four 128-thread teams per SM; the A y pass
// then holds its tiles in registers across a barrier, see linear_unit)
__host__ __device__ inline WorkLayout make_work_layout(int base, int UP, int TP, int C, bool lama, bool fd,
                                                       bool x_in_z = false) {
  WorkLayout L;
  const int LD = UP + 2;  // even: 16-byte aligned rows for float4 access
  const int V = (UP > TP ? UP : TP);
  int o = align_up(base, 16);
  L.G = o;
  o += UP * LD * 8;
  L.Z = o;
  o += TP * LD * 8;
  L.X = x_in_z ? L.Z : o;
  o += x_in_z ? 0 : TP * LD * 8;
  L.W = o;
  o += 4 * UP * 8;
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
  return L;
}

__device__ __forceinline__ Work make_work(char* smem, const WorkLayout& L, int UP) {
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
  w.num = reinterpret_cast<float2*>(smem + L.num);
  w.den = reinterpret_cast<float*>(smem + L.den);
  w.harm = reinterpret_cast<float*>(smem + L.harm);
  w.wbuf = reinterpret_cast<float*>(smem + L.wbuf);
  w.flags = reinterpret_cast<int*>(smem + L.flags);
  w.LD = UP + 2;
  return w;
}

// SIMT kernel smem: [bars][stages][red][work]
struct SimtLayout {
  int bars, stages, red, work;
  WorkLayout w;
  int total;
};

__host__ __device__ inline SimtLayout make_simt_layout(int UP, int TP, int stage_bytes, int NS, int C, int red_f2,
                                                       bool lama, bool fd) {
  SimtLayout L;
  int o = 0;
  L.bars = o;
  o += align_up(NS * 8, 16);
  o = align_up(o, 128);
  L.stages = o;
  o += NS * stage_bytes;
  o = align_up(o, 16);
  L.red = o;
  o += red_f2 * 8;
  L.work = o;
  L.w = make_work_layout(o, UP, TP, C, lama, fd);
  L.total = L.w.total;
  return L;
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
  __syncthreads();
}

// Persistent streaming kernel: (H, Y) -> stats | PD outputs | FD outputs.
// CLS: epilogue class (0 stats, 1 linear, 2 LAMA), one instantiation each so
// a kernel carries (and allocates registers for) only its own epilogue.
template <int UP, int NT, int CLS>
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
  const SimtLayout L = make_simt_layout(UP, p.TP, p.stage_f2 * 8, p.NS, p.C, red_f2, lama, fd);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  float2* red = reinterpret_cast<float2*>(smem + L.red);
  const Work w = make_work(smem, L.w, UP);
  const Team<NT, 0> tm{tid};

  if (tid == 0) {
    for (int s = 0; s < p.NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  reset_flags(w, tm);
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

  int cl_first = 1;
  int jn = 0, sn = 0;
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
    if (ti.active && !(p.ablate & 2)) accumulate_chunk(acc, Hs, Ys, cd.nrows, p.us, p.KCP, ti);
    __syncthreads();  // stage s consumed
    if (tid == 0) issue(q + p.NS);

    const bool item_end = (cd.flags & CH_ITEM_END) != 0;
    const bool per_cluster = fd || (p.arch == ARCH_STATS && !p.sum_clusters);
    const bool unit_end = item_end || (per_cluster && (cd.flags & CH_CLUSTER_END));
    if (!unit_end) continue;
    reduce_tiles<UP, NT>(acc, ti, red, w, p.T, ntiles);
    if (!(p.ablate & 1)) unit_epilogue<UP, Team<NT, 0>, CLS>(w, p, n, cd.cluster, item_end, cl_first, tm);
    // the accumulators restart after the epilogue (not before it: zeroed
    // registers kept live across the epilogue made the LAMA instantiation spill)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
    __syncthreads();
  }
}

// Equalization from precomputed statistics (PD central node after the
// reduce-scatter; linear_equalize / lama_equalize API; and FD at U = 64, where
// the records are the per-cluster statistics [n][C] of the wide tensor-core
// kernel and each item's clusters are solved and fused in order).
// U = 64: three CTAs per SM (80 registers, a few spills): the blocked
// Gauss-Jordan waits on its pivot-block chain at the barriers and a third
// item per SM fills them (cfg5-pd512 13.3 -> 12.7 ms, fd512 75.6 -> 71.6 ms)
#ifndef DBP_STATS_LA
#define DBP_STATS_LA true  // U = 64 solve: look-ahead pivot-block inversion on one warp
#endif
#ifndef DBP_STATS64_MINB
#define DBP_STATS64_MINB 3  // U = 64, 256-thread team (4 x 4 tiles); the 128-thread team (8 x 4) runs four per SM
#endif
// FD linear solves at U = 64 run on the 128-thread team with X in Z
// (make_work_layout x_in_z: four teams per SM; cfg5-fd512 64.2 -> 61.6 ms)
inline bool stats_x_in_z(const EqParams& p) {
  return p.arch == ARCH_FD && p.kind != EQ_LAMA && !(p.u & 1) && p.T <= 16;
}
template <int UP, int NT, bool XZ = false>
__global__ void __launch_bounds__(NT, (UP == 64 ? (NT == 128 ? 4 : DBP_STATS64_MINB) : 512 / NT)) stats_kernel(const __grid_constant__ EqParams p) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x;
  const bool lama = p.kind == EQ_LAMA;
  const bool fd = p.arch == ARCH_FD;
  const int ncl = fd ? p.C : 1;
  const WorkLayout L = make_work_layout(0, UP, p.TP, ncl, lama, fd, XZ);
  const Work w = make_work(smem, L, UP);
  const Team<NT, 0> tm{tid};
  const int u = p.u, T = p.T;
  const size_t rec = (size_t)u * u + (size_t)T * u;
  const int64_t nrec = p.n_items * ncl;
  int cl_first = 1;
  for (int64_t n = blockIdx.x; n < p.n_items; n += gridDim.x) {
    reset_flags(w, tm);
    for (int c = 0; c < ncl; ++c) {
      const int64_t r = n * ncl + c;
      const float2* src = p.stats_in + r * rec;
      const int64_t rn = (c + 1 < ncl) ? r + 1 : (n + gridDim.x) * ncl;  // the record after this one
      if (tid == 0 && rn < nrec) {  // into L2 while this one solves
        const char* nx = reinterpret_cast<const char*>(p.stats_in + rn * rec);
        const uint32_t bytes = (uint32_t)(rec * sizeof(float2));
        for (uint32_t o = 0; o < bytes; o += 32768) {
          const uint32_t len = min(32768u, bytes - o) & ~15u;
          if (len && !(reinterpret_cast<uintptr_t>(nx + o) & 15))
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx + o), "r"(len) : "memory");
        }
      }
      if (u == UP && !(reinterpret_cast<uintptr_t>(p.stats_in) & 15)) {  // float4 pairs, shifts instead of divisions
        constexpr int SH = (UP == 8) ? 2 : (UP == 16) ? 3 : (UP == 32) ? 4 : 5;  // log2(UP / 2)
        const float4* s4 = reinterpret_cast<const float4*>(src);  // rec is even: 16-byte aligned
        // global -> shared without a register round trip (cp.async, 16 B each):
        // every copy of the thread in flight at once, no registers held
        for (int e = tid; e < (UP * UP + T * UP) / 2; e += NT) {
          const int rr = e >> SH, cc = 2 * (e & (UP / 2 - 1));
          float2* dst = (rr < UP) ? w.G + rr * w.LD + cc : w.Z + (rr - UP) * w.LD + cc;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(s4 + e) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
      } else {
        for (int e = tid; e < u * u; e += NT) w.G[(e / u) * w.LD + (e % u)] = src[e];
        for (int e = tid; e < T * u; e += NT) w.Z[(e / u) * w.LD + (e % u)] = src[u * u + e];
      }
      __syncthreads();
      // two CTAs per SM: look-ahead solve
      unit_epilogue<UP, Team<NT, 0>, -1, DBP_STATS_LA, XZ>(w, p, n, c, c + 1 == ncl, cl_first, tm);
      __syncthreads();
    }
  }
}

}  // namespace dbp
