// Warp-specialized tensor-core streaming kernel (U <= 32).
//
// The Gram and the matched filter of one unit are one real GEMM:
//     P = Xr^T Hr,   Xr = [Re H | Im H | Re Y^T | Im Y^T]  (K = antennas),
//                    Hr = [Re H | Im H]      (columns interleaved re/im)
// M = 2(U+T) <= 128 rows, N = 2U, K = B.  G and y_mrc follow from P:
//     G[u][v]   = P[(u,re)][(v,re)] + P[(u,im)][(v,im)]
//               + i (P[(u,re)][(v,im)] - P[(u,im)][(v,re)])
//     y_t[v]    = P[(t,re)][(v,re)] + P[(t,im)][(v,im)]
//               + i (P[(t,im)][(v,re)] - P[(t,re)][(v,im)])
// It runs on tcgen05 (kind::tf32, M=128, accumulator in TMEM) with a 3xTF32
// split (x = hi + lo, P = hi.hi + hi.lo + lo.hi) so the result keeps fp32
// accuracy (plain TF32 would miss the 1e-4 tolerance: SURVEY.md 8(c)).
//
// Roles (one persistent CTA per SM):
//   warp 0       TMA producer: bulk copies of each chunk (<= 32 antenna rows
//                of one cluster) of H and Y into a ring of raw stages
//   warp 1       MMA issuer (one thread): 3 x ceil(rows/8) tcgen05.mma per
//                chunk into one of two TMEM accumulator slots
//   warps 2-5    converters: raw stage -> hi/lo operand tiles in the canonical
//                K-major core-matrix layout (8 rows x 16 B per core matrix)
//   warps 6-9    assemblers: tcgen05.ld of the accumulator (warp w owns TMEM
//                lanes 32(w%4)..+31), G / y_mrc written into a solver's slot
//   warps 10..   solvers: one warp per unit (round robin), the whole unit
//                epilogue (solve, outputs) with __syncwarp only; FD units of
//                one item are folded into an item ring in cluster order
// Everything is pipelined through mbarriers: loads, conversions and MMAs of
// later units overlap the solves of earlier ones, and several units are
// solved concurrently.
#pragma once
#include "dbp_simt.cuh"

namespace dbp {

constexpr int TC_CONV_W = 4;  // converter warps (2..5)
constexpr int TC_ASM_W = 4;   // assembler warps (6..9)
constexpr int TC_FIRST_SOLVER = 2 + TC_CONV_W + TC_ASM_W;
constexpr int TC_MAX_SOLV = 6;
constexpr int TC_NOP = 4;  // operand tile ring depth (converter -> MMA)
constexpr int TC_CONV = 32 * TC_CONV_W;
constexpr int TC_ASM = 32 * TC_ASM_W;
constexpr int TC_MAX_THREADS = 32 * (TC_FIRST_SOLVER + TC_MAX_SOLV);

// byte offset of (feature f, antenna quad qd) in a K=32 operand tile,
// K-major with the 128-byte swizzle (see umma_desc_sw128)
__device__ __forceinline__ int sw128_off(int f, int qd) {
  return (f >> 3) * 1024 + (f & 7) * 128 + ((qd ^ (f & 7)) << 4);
}

// FD item ring slot: the fusion sums of one item, folded cluster by cluster.
struct ItemSlotLayout {
  int num, den, harm, wbuf, flags, total;
};

__host__ __device__ inline ItemSlotLayout make_item_slot(int UP, int TP, int C) {
  ItemSlotLayout S;
  const int LD = UP + 2, V = (UP > TP ? UP : TP);
  int o = 0;
  S.num = o;
  o += TP * LD * 8;
  S.den = o;
  o += V * 4;
  S.harm = o;
  o += V * 4;
  S.wbuf = o;
  o += C * V * 4;
  S.flags = o;
  o += 16;  // [0] status, [1] divergence iteration, [2] turn counter
  S.total = align_up(o, 128);
  return S;
}

struct TcLayout {
  int bars, tmem_slot, hst, hbytes, yst, ybytes, ops, opb, slack, work, work_stride, items, item_stride, nir, total;
  WorkLayout w;  // offsets relative to a solver's work base
};

// Raw staging: a ring of NS H chunks (KC antenna rows each, one bulk copy)
// and a ring of NY whole-item Y blocks (T x B, one bulk copy per item -- the
// per-symbol rows of a chunk are only 8*KC bytes and would cost T tiny copies).
__host__ __device__ inline TcLayout make_tc_layout(int UP, int TP, int T, int B, int us, int KC, int NS, int NY,
                                                   int C, bool lama, bool fd, int nsolv) {
  TcLayout L;
  const int MB = (2 * UP + 2 * T + 7) / 8;  // 8-row core-matrix blocks used
  int o = 0;
  L.bars = o;
  o += (2 * NS + 2 * NY + 2 * TC_NOP + 4 + 2 * TC_MAX_SOLV) * 8;
  L.tmem_slot = o;
  o += 16;
  o = align_up(o, 128);
  L.hbytes = align_up(KC * us * 8, 128);
  L.hst = o;
  o += NS * L.hbytes;
  L.ybytes = align_up(T * B * 8, 128);
  L.yst = o;
  o += NY * L.ybytes;
  o = align_up(o, 1024);
  L.ops = o;
  L.opb = MB * 1024;  // one K=32 tile: MB blocks x 8 k-quads x 128 B
  o += 2 * TC_NOP * L.opb;  // [hi0][lo0][hi1][lo1]...
  L.work = o;
  L.w = make_work_layout(0, UP, TP, C, lama, false);
  L.work_stride = L.w.total;
  o += nsolv * L.work_stride;
  L.items = o;
  const ItemSlotLayout S = make_item_slot(UP, TP, C);
  L.item_stride = S.total;
  L.nir = fd ? (nsolv + C - 1) / C + 2 : 0;
  o += L.nir * L.item_stride;
  // the M=128 MMA reads 16 blocks (16 KB) from each tile base; rows past
  // MB*8 are never written and only produce ignored accumulator rows, but
  // they must stay inside the CTA's shared memory
  const int after_last = o - (L.work - L.opb);
  L.slack = (after_last < 16 * 1024) ? 16 * 1024 - after_last : 0;
  o += L.slack;
  L.total = align_up(o, 128);
  return L;
}

__device__ __forceinline__ Work work_at(char* smem, const TcLayout& L, int sv, int UP) {
  WorkLayout wl = L.w;
  const int base = L.work + sv * L.work_stride;
  wl.G += base;
  wl.Z += base;
  wl.X += base;
  wl.W += base;
  wl.Sv += base;
  wl.Vv += base;
  wl.Fb += base;
  wl.gb += base;
  wl.num += base;
  wl.phi += base;
  wl.coef += base;
  wl.s2 += base;
  wl.gn += base;
  wl.dg += base;
  wl.den += base;
  wl.harm += base;
  wl.wbuf += base;
  wl.flags += base;
  return make_work(smem, wl, UP);
}

// FD: fold one solved cluster into its item's ring slot, strictly in cluster
// order (deterministic sums; a solver waits for its turn), and finalize the
// item on its last cluster (fusion.py:141-154).  Runs on one warp.
template <int UP, class TM>
__device__ void fd_fold(const Work& w, char* slot, const ItemSlotLayout& S, const EqParams& p, int64_t n, int il,
                        int c, int nir, const TM& tm) {
  const int u = p.u, T = p.T, LD = w.LD, C = p.C;
  const bool lama = p.kind == EQ_LAMA;
  const int wdim = lama ? T : u;
  float2* num = reinterpret_cast<float2*>(slot + S.num);
  float* den = reinterpret_cast<float*>(slot + S.den);
  float* harm = reinterpret_cast<float*>(slot + S.harm);
  float* wbuf = reinterpret_cast<float*>(slot + S.wbuf);
  int* flags = reinterpret_cast<int*>(slot + S.flags);
  volatile int* turn = flags + 2;
  const int key = il * C + c;
  if (tm.t == 0) {
    while (*turn != key) __nanosleep(32);
  }
  tm.sync();
  __threadfence_block();
  const bool first = (c == 0);
  for (int e = tm.t; e < wdim; e += TM::N) {
    const float s2 = w.s2[e];
    if (p.kind != EQ_MRC && !(s2 > 0.f)) set_status(w.flags, ST_BADVAR);
    const float inv = 1.f / fmaxf(s2, VAR_FLOOR);
    const float wt = (p.kind == EQ_MRC) ? w.gn[e] : inv;
    wbuf[c * wdim + e] = wt;
    den[e] = first ? wt : den[e] + wt;
    harm[e] = first ? inv : harm[e] + inv;
  }
  for (int e = tm.t; e < T * u; e += TM::N) {
    const int t = e / u, i = e - t * u;
    const int k = lama ? t : i;
    const float s2 = w.s2[k];
    const float wt = (p.kind == EQ_MRC) ? w.gn[k] : 1.f / fmaxf(s2, VAR_FLOOR);
    const float2 x = c_scale(w.X[t * LD + i], wt);
    num[t * LD + i] = first ? x : c_add(num[t * LD + i], x);
  }
  tm.sync();
  if (tm.t == 0) {
    if (first) {
      flags[0] = 0;
      flags[1] = 0x7fffffff;
    }
    if (w.flags[0] && flags[0] == 0) flags[0] = w.flags[0];
    if (w.flags[1] < flags[1]) flags[1] = w.flags[1];
  }
  if (c == C - 1) {
    tm.sync();
    __threadfence_block();
    if (p.arch == ARCH_FD) {
      for (int e = tm.t; e < T * u; e += TM::N) {
        const int t = e / u, i = e - t * u;
        const float2 x = c_scale(num[t * LD + i], 1.f / den[lama ? t : i]);
        const size_t o = ((size_t)n * T + t) * u + i;
        p.xhat[o] = x;
        if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
      }
      for (int e = tm.t; e < wdim; e += TM::N) p.sigma2[(size_t)n * wdim + e] = 1.f / harm[e];
      if (p.nu)
        for (int e = tm.t; e < C * wdim; e += TM::N) p.nu[(size_t)n * C * wdim + e] = wbuf[e] / den[e % wdim];
    } else {  // FD_PARTIAL: raw sums for a cross-GPU reduction
      const int rec = 2 * T * u + 2 * wdim;
      float* dst = p.fd_acc + (size_t)n * rec;
      for (int e = tm.t; e < T * u; e += TM::N) {
        const int t = e / u, i = e - t * u;
        const float2 v = num[t * LD + i];
        dst[2 * e] = v.x;
        dst[2 * e + 1] = v.y;
      }
      for (int e = tm.t; e < wdim; e += TM::N) {
        dst[2 * T * u + e] = den[e];
        dst[2 * T * u + wdim + e] = harm[e];
      }
      for (int e = tm.t; e < C * wdim; e += TM::N) p.fd_wraw[(size_t)n * C * wdim + e] = wbuf[e];
    }
    if (tm.t == 0) {
      int st = flags[0];
      if (flags[1] < 0x7fffffff) st = st ? st : ST_DIVERGED;
      p.status[n] = st;
      if (p.iters) p.iters[n] = (flags[1] < 0x7fffffff) ? flags[1] : 0;
    }
  }
  tm.sync();
  __threadfence_block();
  if (tm.t == 0) *turn = (c == C - 1) ? (il + nir) * C : key + 1;
}

// Debug instrumentation (p.dbg != nullptr, set by DBP_TC_DEBUG): per-CTA
// cycle counters of each role's waits, for pipeline studies.
struct WaitClock {
  long long* acc;  // nullptr when disabled
  __device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity, int slot) {
    if (!acc) {
      mbar_wait(bar, parity);
      return;
    }
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc[slot] += clock64() - t0;
  }
};

template <int UP>
__global__ void __launch_bounds__(TC_MAX_THREADS, 1) tc_kernel(const __grid_constant__ EqParams p, int nsolv,
                                                                int ny) {
  extern __shared__ __align__(1024) char smem[];
  constexpr int N = 2 * UP;
  // independent accumulator chains per unit: hi.hi / hi.lo / lo.hi products
  // (x2 by k-step parity for U <= 16) accumulate into separate TMEM column
  // blocks, so consecutive tcgen05.mma do not serialise on one accumulator;
  // the assembler sums the chains
  constexpr int NCH = 1;
  constexpr int SW = NCH * N;  // TMEM columns per accumulator slot
  constexpr uint32_t TMEM_COLS = (2 * SW <= 32) ? 32 : (2 * SW <= 64) ? 64 : (2 * SW <= 128) ? 128
                                 : (2 * SW <= 256) ? 256 : 512;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool lama = p.kind == EQ_LAMA;
  const bool fd = (p.arch == ARCH_FD || p.arch == ARCH_FD_PARTIAL);
  const int NS = p.NS;
  const int NY = ny;
  const int MU = 2 * UP + 2 * p.T;
  const int MB = (MU + 7) / 8;
  const TcLayout L = make_tc_layout(UP, p.TP, p.T, p.B, p.us, p.KC, NS, NY, p.C, lama, fd, nsolv);
  const ItemSlotLayout IS = make_item_slot(UP, p.TP, p.C);
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + L.bars);  // H chunk ring
  uint64_t* raw_empty = raw_full + NS;
  uint64_t* y_full = raw_empty + NS;  // Y item ring
  uint64_t* y_empty = y_full + NY;
  uint64_t* op_full = y_empty + NY;
  uint64_t* op_empty = op_full + TC_NOP;
  uint64_t* acc_full = op_empty + TC_NOP;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* slot_full = acc_empty + 2;
  uint64_t* slot_empty = slot_full + TC_MAX_SOLV;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], TC_CONV);
    }
    for (int y = 0; y < NY; ++y) {
      mbar_init(&y_full[y], 1);
      mbar_init(&y_empty[y], TC_CONV);
    }
    for (int b = 0; b < TC_NOP; ++b) {
      mbar_init(&op_full[b], TC_CONV);
      mbar_init(&op_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], TC_ASM);
    }
    for (int v = 0; v < nsolv; ++v) {
      mbar_init(&slot_full[v], TC_ASM);
      mbar_init(&slot_empty[v], 1);
    }
    fence_mbar_init();
  }
  for (int k = tid; k < L.nir; k += blockDim.x) {
    int* f = reinterpret_cast<int*>(smem + L.items + k * L.item_stride + IS.flags);
    f[0] = 0;
    f[1] = 0x7fffffff;
    f[2] = k * p.C;  // turn: first cluster of CTA-local item k
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t my_items = (p.n_items > blockIdx.x) ? (p.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int total = (int)(my_items * p.nchunks);
  const bool per_cluster = fd || (p.arch == ARCH_STATS && !p.sum_clusters);
  // role id for the debug counters: 0 producer, 1 mma, 2 converter, 3 assembler, 4 solver
  const int role = warp == 0 ? 0 : warp == 1 ? 1 : warp < 2 + TC_CONV_W ? 2 : warp < TC_FIRST_SOLVER ? 3 : 4;
  const bool rec = p.dbg && lane == 0 && (warp < 3 || warp == 2 + TC_CONV_W || warp == TC_FIRST_SOLVER);
  long long cnt[4] = {0, 0, 0, 0};
  WaitClock wc{rec ? cnt : nullptr};
  const long long t_start = clock64();

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ----
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      int j = 0, s = 0, il = 0;
      uint32_t ph = 0;
      int64_t n = blockIdx.x;
      for (int q = 0; q < total; ++q) {
        if (j == 0) {  // whole-item Y block
          const int y = il % NY;
          if (il >= NY) wc.wait(&y_empty[y], (uint32_t)(((il / NY) - 1) & 1), 1);
          const uint32_t yb = (uint32_t)p.T * p.B * 8;
          mbar_arrive_expect_tx(&y_full[y], yb);
          bulk_g2s(smem + L.yst + y * L.ybytes, p.Y + (size_t)n * p.T * p.B, yb, &y_full[y], policy);
        }
        if (q >= NS) wc.wait(&raw_empty[s], ph ^ 1u, 2);
        const ChunkDesc cd = p.chunks[j];
        const uint32_t hb = (uint32_t)cd.nrows * p.us * 8;
        mbar_arrive_expect_tx(&raw_full[s], hb);
        bulk_g2s(smem + L.hst + s * L.hbytes, p.H + ((size_t)n * p.B + cd.row0) * p.us, hb, &raw_full[s], policy);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
        if (++j == p.nchunks) {
          j = 0;
          n += gridDim.x;
          ++il;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer ----
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(128, N);
      const uint32_t ops = smem_u32(smem + L.ops);
      int j = 0, unit = 0;
      bool first = true;
      bool written[2] = {false, false};  // chain groups (k-step parity) touched in this unit
      for (int q = 0; q < total; ++q) {
        const int b = q % TC_NOP;
        wc.wait(&op_full[b], (uint32_t)((q / TC_NOP) & 1), 1);
        const ChunkDesc cd = p.chunks[j];
        const int a = unit & 1;
        if (first) {
          if (unit >= 2) wc.wait(&acc_empty[a], (uint32_t)(((unit >> 1) - 1) & 1), 2);
          written[0] = written[1] = false;
        }
        tc_fence_after();
        const uint32_t dslot = tmem + (uint32_t)(a * SW);
        const uint32_t hi = ops + (uint32_t)(2 * b * L.opb);
        const uint32_t lo = hi + (uint32_t)L.opb;
        const int nk8 = (cd.nrows + 7) >> 3;
        for (int ks = 0; ks < ((p.ablate & 2) ? 0 : nk8); ++ks) {
          const int grp = (NCH == 6) ? (ks & 1) : 0;
          const uint32_t acc = written[grp] ? 1u : 0u;
          written[grp] = true;
          const uint32_t d = dslot + (uint32_t)(3 * grp * N);
          const uint64_t ah = umma_desc_sw128(hi + ks * 32, 1024);
          const uint64_t al = umma_desc_sw128(lo + ks * 32, 1024);
          umma_tf32(d, ah, ah, idesc, acc);
          umma_tf32(NCH >= 3 ? d + N : d, ah, al, idesc, NCH >= 3 ? acc : 1u);
          umma_tf32(NCH >= 3 ? d + 2 * N : d, al, ah, idesc, NCH >= 3 ? acc : 1u);
        }
        umma_commit(&op_empty[b]);
        const bool unit_end = (cd.flags & CH_ITEM_END) || (per_cluster && (cd.flags & CH_CLUSTER_END));
        if (unit_end) {
          umma_commit(&acc_full[a]);
          ++unit;
        }
        first = unit_end;
        if (++j == p.nchunks) j = 0;
      }
    }
    __syncwarp();
  } else if (warp < 2 + TC_CONV_W) {
    // -------------------------------------------------------- converters ----
    // hi = x with the low 13 mantissa bits cleared (exact TF32), lo = x - hi.
    // Tile layout (K-major, 128-byte swizzle): feature f, antenna k ->
    // (f/8)*1024 + (f%8)*128 + ((k/4) ^ (f%8))*16 + (k%4)*4 bytes.  H tasks move a 4-feature x 4-antenna block (4x4
    // transpose in registers), Y tasks one symbol's (re, im) rows x 4 antennas.
    const int ct = tid - 64;
    const int us2 = 2 * p.us;
    constexpr int HG = UP / 2;  // 4-feature groups of the H part
    // rows between 2(U+T) and MB*8, and H columns past the stored row width
    // (odd U), are zero forever
    for (int e = ct; e < 2 * TC_NOP * MB * 8 * 8; e += TC_CONV) {
      const int buf = e / (MB * 64), r = e % (MB * 64);
      const int f = r / 8, qd = r % 8;
      if (f >= MU || (f < 2 * UP && f >= us2))
        *reinterpret_cast<float4*>(smem + L.ops + buf * L.opb + sw128_off(f, qd)) =
            make_float4(0.f, 0.f, 0.f, 0.f);
    }
    auto split = [](float x, float& h, float& l) {
      h = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
      l = x - h;
    };
    // static task list of this thread for a full KC=32-row chunk:
    // task = (group g, antenna quad qd); g < HG: H features 4g..4g+3,
    // else symbol t = g - HG (re, im rows)
    const int ng = HG + p.T;
    constexpr int MAXT = 2;  // (UP/2 + T) * 8 <= 2 * TC_CONV for UP <= 32, T <= 16
    int t_ld[MAXT], t_st[MAXT], t_kind[MAXT];
    int nt_mine = 0;
#pragma unroll
    for (int r = 0; r < MAXT; ++r) {
      const int task = ct + r * TC_CONV;
      t_kind[r] = -1;
      t_ld[r] = t_st[r] = 0;
      if (task < ng * 8) {
        const int qd = task / ng, g = task - qd * ng;
        if (g < HG) {
          if (4 * g < us2) {
            t_kind[r] = 0;
            t_ld[r] = 4 * qd * us2 + 4 * g;
            t_st[r] = (4 * g) * 16 + qd;  // packed: feature base, quad
          }
        } else {
          const int t = g - HG;
          t_kind[r] = 1;
          t_ld[r] = (t * p.B + 4 * qd) * 2;
          t_st[r] = (2 * UP + 2 * t) * 16 + qd;
        }
        nt_mine = r + 1;
      }
    }
    int j = 0, s = 0, il = 0;
    uint32_t ph = 0;
    for (int q = 0; q < total; ++q) {
      const int b = q % TC_NOP;
      const int y = il % NY;
      wc.wait(&raw_full[s], ph, 1);
      wc.wait(&y_full[y], (uint32_t)((il / NY) & 1), 2);
      if (q >= TC_NOP) wc.wait(&op_empty[b], (uint32_t)(((q / TC_NOP) - 1) & 1), 3);
      const ChunkDesc cd = p.chunks[j];
      const float* Hf = reinterpret_cast<const float*>(smem + L.hst + s * L.hbytes);
      const float* Yf = reinterpret_cast<const float*>(smem + L.yst + y * L.ybytes) + 2 * cd.row0;
      char* hi = smem + L.ops + 2 * b * L.opb;
      char* lo = hi + L.opb;
      if (cd.nrows == 32 && !(p.ablate & 4)) {
#pragma unroll
        for (int r = 0; r < MAXT; ++r) {
          if (r >= nt_mine || t_kind[r] < 0) continue;
          const int fb = t_st[r] >> 4, qd = t_st[r] & 15;
          if (t_kind[r] == 0) {
            const float* src = Hf + t_ld[r];
            const float4 r0 = *reinterpret_cast<const float4*>(src);
            const float4 r1 = *reinterpret_cast<const float4*>(src + us2);
            const float4 r2 = *reinterpret_cast<const float4*>(src + 2 * us2);
            const float4 r3 = *reinterpret_cast<const float4*>(src + 3 * us2);
            const float cols[4][4] = {{r0.x, r1.x, r2.x, r3.x}, {r0.y, r1.y, r2.y, r3.y},
                                      {r0.z, r1.z, r2.z, r3.z}, {r0.w, r1.w, r2.w, r3.w}};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              float4 h, l;
              split(cols[c][0], h.x, l.x);
              split(cols[c][1], h.y, l.y);
              split(cols[c][2], h.z, l.z);
              split(cols[c][3], h.w, l.w);
              const int off = sw128_off(fb + c, qd);
              *reinterpret_cast<float4*>(hi + off) = h;
              *reinterpret_cast<float4*>(lo + off) = l;
            }
          } else {
            const float* yr = Yf + t_ld[r];
            const float4 a0 = *reinterpret_cast<const float4*>(yr);
            const float4 a1 = *reinterpret_cast<const float4*>(yr + 4);
            float4 h, l;
            split(a0.x, h.x, l.x);
            split(a0.z, h.y, l.y);
            split(a1.x, h.z, l.z);
            split(a1.z, h.w, l.w);
            int off = sw128_off(fb, qd);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
            split(a0.y, h.x, l.x);
            split(a0.w, h.y, l.y);
            split(a1.y, h.z, l.z);
            split(a1.w, h.w, l.w);
            off = sw128_off(fb + 1, qd);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
          }
        }
      } else {
        const int nr = cd.nrows;
        const int nq = 2 * ((nr + 7) >> 3);  // k-quads incl. zero padding to K % 8
        const bool full = (nr & 7) == 0;
        const int ntask = (p.ablate & 4) ? 0 : ng * nq;
        for (int task = ct; task < ntask; task += TC_CONV) {
          const int qd = task / ng;
          const int g = task - qd * ng;
          const int k0 = 4 * qd;
          if (g < HG) {
            const int f0 = 4 * g;
            float4 r[4];
  #pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int k = k0 + i;
              r[i] = (f0 < us2 && (full || k < nr)) ? *reinterpret_cast<const float4*>(Hf + k * us2 + f0)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const float c0[4] = {r[0].x, r[1].x, r[2].x, r[3].x};
            const float c1[4] = {r[0].y, r[1].y, r[2].y, r[3].y};
            const float c2[4] = {r[0].z, r[1].z, r[2].z, r[3].z};
            const float c3[4] = {r[0].w, r[1].w, r[2].w, r[3].w};
            const float* cols[4] = {c0, c1, c2, c3};
  #pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int f = f0 + c;
              float4 h, l;
              split(cols[c][0], h.x, l.x);
              split(cols[c][1], h.y, l.y);
              split(cols[c][2], h.z, l.z);
              split(cols[c][3], h.w, l.w);
              const int off = sw128_off(f, qd);
              *reinterpret_cast<float4*>(hi + off) = h;
              *reinterpret_cast<float4*>(lo + off) = l;
            }
          } else {
            const int t = g - HG;
            const float* yr = Yf + (t * p.B + k0) * 2;  // 4 complex = 2 float4
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
            if (full || k0 + 3 < nr) {
              a0 = *reinterpret_cast<const float4*>(yr);
              a1 = *reinterpret_cast<const float4*>(yr + 4);
            } else {
              if (k0 < nr) {
                a0.x = yr[0];
                a0.y = yr[1];
              }
              if (k0 + 1 < nr) {
                a0.z = yr[2];
                a0.w = yr[3];
              }
              if (k0 + 2 < nr) {
                a1.x = yr[4];
                a1.y = yr[5];
              }
            }
            const int fr = 2 * UP + 2 * t;
            float4 h, l;
            split(a0.x, h.x, l.x);
            split(a0.z, h.y, l.y);
            split(a1.x, h.z, l.z);
            split(a1.z, h.w, l.w);
            int off = sw128_off(fr, qd);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
            split(a0.y, h.x, l.x);
            split(a0.w, h.y, l.y);
            split(a1.y, h.z, l.z);
            split(a1.w, h.w, l.w);
            off = sw128_off(fr + 1, qd);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
          }
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&op_full[b]);
      mbar_arrive(&raw_empty[s]);
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
      if (++j == p.nchunks) {
        mbar_arrive(&y_empty[y]);  // item's last chunk converted
        j = 0;
        ++il;
      }
    }
  } else if (warp < TC_FIRST_SOLVER) {
    // -------------------------------------------------------- assemblers ----
    const int wq = warp & 3;       // TMEM lane quarter this warp may access
    const int m = 32 * wq + lane;  // accumulator row owned by this thread
    const bool odd = (m & 1) != 0;
    const bool has_rows = 32 * wq < MU;
    int j = 0, unit = 0, uks = 0;
    for (int q = 0; q < total; ++q) {
      const ChunkDesc cd = p.chunks[j];
      if (++j == p.nchunks) j = 0;
      uks += (cd.nrows + 7) >> 3;
      const bool unit_end = (cd.flags & CH_ITEM_END) || (per_cluster && (cd.flags & CH_CLUSTER_END));
      if (!unit_end) continue;
      const int nch = (NCH == 6 && uks < 2) ? 3 : NCH;  // chain group 1 untouched
      uks = 0;
      const int sv = unit % nsolv;
      if (unit >= nsolv) wc.wait(&slot_empty[sv], (uint32_t)(((unit / nsolv) - 1) & 1), 1);
      const int a = unit & 1;
      wc.wait(&acc_full[a], (uint32_t)((unit >> 1) & 1), 2);
      tc_fence_after();
      if (has_rows) {
        const Work w = work_at(smem, L, sv, UP);
        float* Gf = reinterpret_cast<float*>(w.G);
        float* Zf = reinterpret_cast<float*>(w.Z);
        const int LD = w.LD;
        const uint32_t taddr = tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)(a * SW);
        // 16 accumulator columns = 8 UE columns (re, im) per tcgen05.ld; the
        // partner row (m ^ 1) holds the other component of the same complex row
#pragma unroll
        for (int h = 0; h < N / 16; ++h) {
          float v[16];
          tmem_ld16(taddr + 16 * h, v);
          for (int ch = 1; ch < nch; ++ch) {
            float t16[16];
            tmem_ld16(taddr + ch * N + 16 * h, t16);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += t16[i];
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float po = __shfl_xor_sync(0xffffffffu, v[2 * c + 1], 1);
            const int col = 8 * h + c;
            if (m < 2 * UP) {
              const float val = odd ? (po - v[2 * c]) : (v[2 * c] + po);
              Gf[((m >> 1) * LD + col) * 2 + (odd ? 1 : 0)] = val;
            } else if (m < MU) {
              const float val = odd ? (v[2 * c] - po) : (v[2 * c] + po);
              Zf[(((m - 2 * UP) >> 1) * LD + col) * 2 + (odd ? 1 : 0)] = val;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[a]);
      mbar_arrive(&slot_full[sv]);
      ++unit;
    }
  } else {
    // ----------------------------------------------------------- solvers ----
    const int sv = warp - TC_FIRST_SOLVER;
    const Team<32, -1> tm{lane};
    const Work w = work_at(smem, L, sv, UP);
    int j = 0, unit = 0, il = 0, cl_first = 1;
    int64_t n = blockIdx.x;
    for (int q = 0; q < total; ++q) {
      const ChunkDesc cd = p.chunks[j];
      const int64_t n_cur = n;
      const int il_cur = il;
      if (++j == p.nchunks) {
        j = 0;
        n += gridDim.x;
        ++il;
      }
      const bool item_end = (cd.flags & CH_ITEM_END) != 0;
      const bool unit_end = item_end || (per_cluster && (cd.flags & CH_CLUSTER_END));
      if (!unit_end) continue;
      const int my = (unit % nsolv == sv);
      const int round = unit / nsolv;
      ++unit;
      if (!my) continue;
      wc.wait(&slot_full[sv], (uint32_t)(round & 1), 1);
      reset_flags(w, tm);
      tm.sync();
      if (p.ablate & 1) {
      } else if (!fd) {
        unit_epilogue<UP>(w, p, n_cur, cd.cluster, item_end, cl_first, tm);
      } else {
        const int c = cd.cluster;
        EpiArgs a;
        a.kind = p.kind;
        a.u = p.u;
        a.T = p.T;
        a.n0 = item_n0(p, n_cur);
        a.es = p.es;
        a.damping = p.damping;
        a.t_max = p.t_max;
        a.beta = p.cl_beta[c];
        a.lama_scale = p.cl_scale[c];
        a.unbias = true;  // fusion.py:148 -- fuse in the unbiased domain
        if (lama)
          lama_unit(w, a, p.cp, nullptr, nullptr, nullptr, nullptr, tm);
        else
          linear_unit<UP>(w, a, tm);
        char* slot = smem + L.items + (il_cur % L.nir) * L.item_stride;
        fd_fold<UP>(w, slot, IS, p, n_cur, il_cur, c, L.nir, tm);
      }
      tm.sync();
      if (lane == 0) mbar_arrive(&slot_empty[sv]);
    }
  }
  if (rec) {
    cnt[0] = clock64() - t_start;
    for (int k = 0; k < 4; ++k) atomicAdd(reinterpret_cast<unsigned long long*>(p.dbg + role * 4 + k),
                                          (unsigned long long)cnt[k]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace dbp
