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
// Operand tiles are MN-major with the 128-byte swizzle: one 1 KB atom holds 32
// features (M or N index, 128 B) of 8 antennas (K).  H is stored [antenna]
// [features] in HBM, i.e. already MN-major, so its conversion is a row-wise
// streaming pass; only Y ([symbol][antenna]) is transposed, as (symbol pair,
// antenna) float4 blocks.  Every converter load and store is conflict-free.
// M rows of a tile: [H features of the pair's units][Y block of unit 0]
// [Y block of unit 1], Y blocks 32-row aligned (feature 2t + re/im); the
// B operand (N) is the H part of the same tile.
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
//
// DBP_ABLATE (timing studies only; results are wrong when set): 1 no solver
// work, 2 no MMAs, 4 no conversion, 32 no TMEM read-back, 64 LAMA team
// schedule, 128 no operand ring / MMA / assembly / solve (stream + convert),
// 256 no proxy fence, 512 H copies only, 1024 one stage wait + release per
// pair (with 128: stream only).  tools/gpu_ablate.sh, tools/gpu_skel.sh.
#pragma once
#include "dbp_simt.cuh"

namespace dbp {

constexpr int TC_CONV_SETS = 1;              // converter warp sets, alternating pair-chunks
constexpr int TC_CONV_W = 4 * TC_CONV_SETS;  // converter warps (2..)
constexpr int TC_MMA_W = 1;   // MMA issuer warps (2 = alternate chunks, one partial accumulator each; measured slower overall: fewer solver registers)
constexpr int TC_ASM_W = 4;   // assembler warps
constexpr int TC_FIRST_CONV = 1 + TC_MMA_W;
constexpr int TC_FIRST_ASM = TC_FIRST_CONV + TC_CONV_W;
constexpr int TC_FIRST_SOLVER = TC_FIRST_ASM + TC_ASM_W;
constexpr int TC_MAX_SOLV = 6;
#ifndef DBP_TC_NOP
#define DBP_TC_NOP 2
#endif
constexpr int TC_NOP = DBP_TC_NOP;  // operand tile ring depth (converter -> MMA)
constexpr int TC_CONV = 128;  // threads of one converter set (barrier arrival count)
constexpr int TC_ASM = 32 * TC_ASM_W;
constexpr int TC_MAX_THREADS = 32 * (TC_FIRST_SOLVER + TC_MAX_SOLV);
constexpr int FD_CNT = 64;  // FD arrival counters per CTA (items in flight in the solver stage)

// byte offset of (M row f, antenna kr) in an operand tile: MN-major tf32
// (128-byte rows, 32-byte granules swizzled by kr % 4; umma_desc_mn_sw128),
// M blocks of 32 rows `lbo` bytes apart, antenna rows 128 B apart; f is
// 4-aligned (one 16-byte chunk = 4 consecutive M rows of one antenna)
__device__ __forceinline__ int mn_off(int f, int kr, int lbo) {
  return (f >> 5) * lbo + kr * 128 + ((((f & 31) >> 3) ^ (kr & 3)) << 5) + (f & 4) * 4;
}
// first M row of the Y blocks
__host__ __device__ constexpr int tc_yrow0(int UP, int pair) { return ((pair * 2 * UP + 31) / 32) * 32; }

struct TcLayout {
  int bars, tmem_slot, chunks, stg, sbytes, ops, opb, lbo, work, work_stride, items, total;
  WorkLayout w;  // offsets relative to a solver's work base
};

// Raw staging: a ring of NS stages, each `sbytes` of H rows then Y rows of
// `ips` consecutive items (or one row block of an item), filled by 2 bulk
// copies (whole items) or 1 + T copies (row block); then the operand tiles.
__host__ __device__ inline TcLayout make_tc_layout(int UP, int TP, int sbytes, int KC, int NS, int C, bool lama,
                                                   bool fd, int nsolv) {
  TcLayout L;
  int o = 0;
  L.bars = o;
  o += (2 * NS + 2 * TC_NOP + 4 + 2 * TC_MAX_SOLV) * 8;
  L.tmem_slot = o;
  o += 16;
  L.chunks = o;  // copy of the chunk table (+ stage rows): dynamic param loads are slow
  o += (MAX_CHUNKS + 2 * MAX_SPI) * 16;
  o = align_up(o, 128);
  L.sbytes = align_up(sbytes, 128);
  L.stg = o;
  o += NS * L.sbytes;
  o = align_up(o, 1024);
  L.ops = o;
  L.lbo = (KC / 8) * 1024;  // one 32-row M block of a K=KC tile
  // 4 M blocks = the 128 rows one MMA reads; wide (U = 64): 5 blocks, the
  // 128 H features (A) and the Y block after them (B = all 160 rows)
  L.opb = (UP > 32 ? 5 : 4) * L.lbo;
  o += 2 * TC_NOP * L.opb;  // [hi0][lo0][hi1][lo1]...
  L.work = o;
  L.w = make_work_layout(0, UP, TP, C, lama, false);
  L.work_stride = L.w.total;
  o += nsolv * L.work_stride;
  L.items = o;  // FD: per-item arrival counters (ring of FD_CNT)
  o += fd ? FD_CNT * 4 : 0;
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

// FD fusion without waiting (fusion.py:141-154).  Every solved cluster is
// stashed as a record {unbiased z_c [T][u], sigma2_c [wdim], MRC gain [u],
// status, divergence iteration} in an L2-resident scratch array; the solver
// that brings the item's arrival count to C then folds the C records in
// cluster order (the reference's summation order: deterministic results) and
// writes the outputs.  No solver ever waits for another one.
__host__ __device__ inline int fd_record_floats(int u, int T, int wdim) {
  return align_up(2 * T * u + wdim + u + 2, 4);
}

template <class TM>
__device__ void fd_stash(const Work& w, const EqParams& p, int64_t n, int c, const TM& tm) {
  const int u = p.u, T = p.T, LD = w.LD, C = p.C;
  const int wdim = (p.kind == EQ_LAMA) ? T : u;
  float* rec = p.fd_scratch + ((size_t)n * C + c) * fd_record_floats(u, T, wdim);
  float2* z = reinterpret_cast<float2*>(rec);
  for (int e = tm.t; e < T * u; e += TM::N) {
    const int t = e / u, i = e - t * u;
    z[e] = w.X[t * LD + i];
  }
  for (int e = tm.t; e < wdim; e += TM::N) rec[2 * T * u + e] = w.s2[e];
  if (p.kind == EQ_MRC)
    for (int e = tm.t; e < u; e += TM::N) rec[2 * T * u + wdim + e] = w.gn[e];
  if (tm.t == 0) {
    int* f = reinterpret_cast<int*>(rec + 2 * T * u + wdim + u);
    f[0] = w.flags[0];
    f[1] = w.flags[1];
  }
}

// Ordered fold of the item's C records by one warp.  scratch: >= (C + 1) *
// wdim floats of the solver's shared memory.
template <class TM>
__device__ void fd_finish(float* scratch, const EqParams& p, int64_t n, const TM& tm) {
  const int u = p.u, T = p.T, C = p.C;
  const bool lama = p.kind == EQ_LAMA, mrc = p.kind == EQ_MRC;
  const int wdim = lama ? T : u;
  const int rf = fd_record_floats(u, T, wdim);
  const float* recs = p.fd_scratch + (size_t)n * C * rf;
  float* den = scratch;         // [wdim]
  float* wts = scratch + wdim;  // [C][wdim]
  int st = 0, it = 0x7fffffff;
  for (int e = tm.t; e < wdim; e += TM::N) {
    float dsum = 0.f, hsum = 0.f;
#pragma unroll 8  // batch the L2 loads of the records
    for (int c = 0; c < C; ++c) {
      const float* rec = recs + (size_t)c * rf;
      const float s2 = __ldcg(rec + 2 * T * u + e);
      if (!mrc && !(s2 > 0.f)) st = ST_BADVAR;  // optimal_fusion_weights rejects sigma2 <= 0
      const float inv = 1.f / fmaxf(s2, VAR_FLOOR);
      const float wt = mrc ? __ldcg(rec + 2 * T * u + wdim + e) : inv;
      wts[c * wdim + e] = wt;
      dsum += wt;
      hsum += inv;
    }
    den[e] = dsum;
    if (p.arch == ARCH_FD) {
      p.sigma2[(size_t)n * wdim + e] = 1.f / hsum;
    } else {
      float* dst = p.fd_acc + (size_t)n * (2 * T * u + 2 * wdim);
      dst[2 * T * u + e] = dsum;
      dst[2 * T * u + wdim + e] = hsum;
    }
  }
  tm.sync();
  if (p.arch == ARCH_FD) {
    if (p.nu)
      for (int e = tm.t; e < C * wdim; e += TM::N) p.nu[(size_t)n * C * wdim + e] = wts[e] / den[e % wdim];
  } else {
    for (int e = tm.t; e < C * wdim; e += TM::N) p.fd_wraw[(size_t)n * C * wdim + e] = wts[e];
  }
  for (int e = tm.t; e < T * u; e += TM::N) {
    const int t = e / u, i = e - t * u;
    const int k = lama ? t : i;
    float2 num = make_float2(0.f, 0.f);
#pragma unroll 8  // batch the L2 loads of the records
    for (int c = 0; c < C; ++c) {
      const float2 zc = __ldcg(reinterpret_cast<const float2*>(recs + (size_t)c * rf) + e);
      num = c_add(num, c_scale(zc, wts[c * wdim + k]));
    }
    if (p.arch == ARCH_FD) {
      const float2 x = c_scale(num, 1.f / den[k]);
      const size_t o = (size_t)n * T * u + e;
      p.xhat[o] = x;
      if (p.dec) p.dec[o] = (uint8_t)slice_symbol(x, p.cp);
    } else {
      float* dst = p.fd_acc + (size_t)n * (2 * T * u + 2 * wdim);
      dst[2 * e] = num.x;
      dst[2 * e + 1] = num.y;
    }
  }
  // status: first failing cluster's code, else divergence (earliest iteration)
  for (int c = 0; c < C; ++c) {
    const int* f = reinterpret_cast<const int*>(recs + (size_t)c * rf + 2 * T * u + wdim + u);
    const int fs = __ldcg(f), fi = __ldcg(f + 1);
    if (st == 0 && fs) st = fs;
    if (fi < it) it = fi;
  }
  // combine the lanes' variance checks
  for (int o = 16; o > 0; o >>= 1) {
    const int so = __shfl_xor_sync(0xffffffffu, st, o);
    if (st == 0) st = so;
  }
  if (tm.t == 0) {
    if (it < 0x7fffffff && st == 0) st = ST_DIVERGED;
    p.status[n] = st;
    if (p.iters) p.iters[n] = (it < 0x7fffffff) ? it : 0;
  }
  tm.sync();
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

// Stream order.  A CTA owns U_tot units (items for PD / STATS-summed, clusters
// for FD / STATS-per-cluster), unit u = (CTA-local item u / upi, cluster
// u % upi).  With pair == 2 two units share every operand tile (rows
// [h*2UP, (h+1)*2UP) = H features of half h, rows 2*2UP + h*2T.. = its Y
// features) and every tcgen05.mma (N = 2 * 2UP): the fixed ~46-cycle cost of
// one small tf32 MMA is paid once for two units.  Stream position q walks
// pairs v, then chunk j < cpu of a unit, then half h < pair.
struct Stream {
  int pair, cpu, upi, U_tot;
  int v, j, h;  // current position
  __device__ __forceinline__ void advance() {
    if (++h == pair) {
      h = 0;
      if (++j == cpu) {
        j = 0;
        ++v;
      }
    }
  }
  __device__ __forceinline__ int unit() const { return v * pair + h; }
  __device__ __forceinline__ bool null() const { return unit() >= U_tot; }
  __device__ __forceinline__ int item() const { return unit() / upi; }
  __device__ __forceinline__ int cluster() const { return unit() % upi; }
  __device__ __forceinline__ int chunk_index() const { return cluster() * cpu + j; }
};

// MODE: what the unit epilogue does, fixed per instantiation so that each
// kernel carries only its own epilogue code (instruction-cache footprint)
enum { TC_STATS = 0, TC_PD_LIN = 1, TC_PD_LAMA = 2, TC_FD_LIN = 3, TC_FD_LAMA = 4 };

template <int UP, int MODE>
__global__ void __launch_bounds__(TC_MAX_THREADS, 1) tc_kernel(const __grid_constant__ EqParams p, int nsolv) {
  extern __shared__ __align__(1024) char smem[];
  // wide (U = 64, statistics only): the 2U = 128 H features fill M, so the Y
  // block moves to N: A = tile rows [0, 128) (H), B = rows [0, 160) ([H | Y])
  // of the same operand tile; accumulator lane = H feature, columns = [H | Y]
  constexpr bool WIDE = UP > 32;
  static_assert(!WIDE || MODE == 0, "the wide layout only produces statistics");
  const int pair = WIDE ? 1 : p.pair;
  const int N = WIDE ? 2 * UP + 32 : pair * 2 * UP;  // MMA N
  constexpr int SW = WIDE ? 2 * UP + 32 : 2 * 2 * UP;  // TMEM columns per accumulator slot (room for pair == 2)
  // accumulators: 2 buffers (pairs v, v+1) x TC_MMA_W partial sums (one per
  // MMA issuer warp), column (2 a + m) * SW
  constexpr int TCOLS = 2 * TC_MMA_W * SW;
  constexpr uint32_t TMEM_COLS = (TCOLS <= 32) ? 32 : (TCOLS <= 64) ? 64 : (TCOLS <= 128) ? 128
                                 : (TCOLS <= 256) ? 256 : 512;
  // warp index broadcast from lane 0: the compiler then treats the role
  // branches as warp-uniform, so shuffles inside them compile to plain SHFL
  // instead of divergence-safe COLLECTIVE sequences
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  constexpr bool lama = (MODE == TC_PD_LAMA || MODE == TC_FD_LAMA);
  constexpr bool fd = (MODE == TC_FD_LIN || MODE == TC_FD_LAMA);
  constexpr int CLS = (MODE == TC_STATS) ? 0 : lama ? 2 : 1;
  const int NS = p.NS;
  const int T = p.T;
  const int HR = pair * 2 * UP;          // H rows of the tile (= MMA N)
  const int YB = tc_yrow0(UP, pair);     // first Y row (32-aligned)
  const int MU = YB + pair * 32;         // rows in use
  const TcLayout L = make_tc_layout(UP, p.TP, p.stage_bytes, p.KC, NS, p.C, lama, fd, nsolv);
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + L.bars);  // stage ring
  uint64_t* raw_empty = raw_full + NS;
  uint64_t* op_full = raw_empty + NS;
  uint64_t* op_empty = op_full + TC_NOP;
  uint64_t* acc_full = op_empty + TC_NOP;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* slot_full = acc_empty + 2;
  uint64_t* slot_empty = slot_full + TC_MAX_SOLV;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
  // chunks per unit, and how many MMA warps contribute to each pair's accumulator
  const int cpu_ = p.nchunks / ((fd || (p.arch == ARCH_STATS && !p.sum_clusters)) ? p.C : 1);
  const int cpu_mma = cpu_ < TC_MMA_W ? cpu_ : TC_MMA_W;
  ChunkDesc* chunks = reinterpret_cast<ChunkDesc*>(smem + L.chunks);
  int* st_row0 = reinterpret_cast<int*>(chunks + MAX_CHUNKS);
  int* st_rows = st_row0 + MAX_SPI;
  for (int e = threadIdx.x; e < p.nchunks; e += blockDim.x) chunks[e] = p.chunks[e];
  for (int e = threadIdx.x; e < MAX_SPI; e += blockDim.x) {
    st_row0[e] = p.st_row0[e];
    st_rows[e] = p.st_rows[e];
  }

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], TC_CONV);
    }
    for (int b = 0; b < TC_NOP; ++b) {
      mbar_init(&op_full[b], TC_CONV);
      mbar_init(&op_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], cpu_mma);
      mbar_init(&acc_empty[b], TC_ASM);
    }
    for (int v = 0; v < nsolv; ++v) {
      mbar_init(&slot_full[v], TC_ASM);
      mbar_init(&slot_empty[v], 1);
    }
    fence_mbar_init();
  }
  int* fd_count = reinterpret_cast<int*>(smem + L.items);
  if (fd)
    for (int k = tid; k < FD_CNT; k += blockDim.x) fd_count[k] = 0;
  // operand tiles start zeroed: pad features (odd U, T < 16) and unused M
  // blocks are never written afterwards
  for (int e = tid; e < 2 * TC_NOP * L.opb / 16; e += blockDim.x)
    reinterpret_cast<float4*>(smem + L.ops)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);  // allocated / freed by MMA warp 0
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // a contiguous range of items per CTA (so a stage can hold consecutive items)
  const int64_t per_cta = p.n_items / gridDim.x, extra = p.n_items % gridDim.x;
  const int64_t first = blockIdx.x * per_cta + min((int64_t)blockIdx.x, extra);
  const int64_t my_items = per_cta + (blockIdx.x < extra ? 1 : 0);
  const bool per_cluster = fd || (p.arch == ARCH_STATS && !p.sum_clusters);
  const int upi = per_cluster ? p.C : 1;
  const int cpu = p.nchunks / upi;
  const int U_tot = (int)my_items * upi;
  const int n_pairs = (U_tot + pair - 1) / pair;
  const int S_tot = n_pairs * pair * cpu;  // stream length
  const Stream s0{pair, cpu, upi, U_tot, 0, 0, 0};
  const bool rec = p.dbg && lane == 0;
  long long cnt[4] = {0, 0, 0, 0};
  WaitClock wc{rec ? cnt : nullptr};
  const long long t_start = clock64();

  const int ips = p.ips, spi = p.spi;
  const int n_groups = (int)((my_items + ips - 1) / ips);
  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ----
    // stage (group g, row block k): lane 0 arms the barrier, then the copies
    // are issued from several lanes (one bulk copy costs the issuing thread
    // a few hundred cycles; a stage is at most 2 + T copies)
    const uint64_t policy = l2_evict_first_policy();
    int s = 0;
    uint32_t ph = 0;
    int seq = 0;
    for (int g = 0; g < n_groups; ++g) {
      const int64_t n0 = first + (int64_t)g * ips;
      const int cnt = (int)min((int64_t)ips, my_items - (int64_t)g * ips);
      for (int k = 0; k < spi; ++k, ++seq) {
        const int r0 = st_row0[k], R = st_rows[k];
        const uint32_t hb = (uint32_t)cnt * R * p.us * 8, yb = (uint32_t)cnt * T * R * 8;  // bytes landing
        const bool no_y = (p.ablate & 512) != 0;  // timing study only: H copies alone
        if (lane == 0) {
          if (seq >= NS) wc.wait(&raw_empty[s], ph ^ 1u, 2);
          mbar_arrive_expect_tx(&raw_full[s], no_y ? hb : hb + yb);
        }
        __syncwarp();
        char* dst = smem + L.stg + s * L.sbytes;
        // H rows of the `cnt` items: one copy when whole items are staged
        // (consecutive items are contiguous), else one per item; Y: one copy
        // per (item, symbol) row into the padded row layout, spread over lanes
        if (spi == 1) {
          if (lane == 0) bulk_g2s(dst, p.H + (size_t)n0 * p.B * p.us, hb, &raw_full[s], policy);
        } else if (lane == 0) {
          bulk_g2s(dst, p.H + ((size_t)n0 * p.B + r0) * p.us, hb, &raw_full[s], policy);
        }
        for (int r = lane; r < (no_y ? 0 : cnt * T); r += 32)
          bulk_g2s(dst + p.stage_hbytes + r * p.stage_ystride, p.Y + ((size_t)n0 * T + r) * p.B + r0, R * 8,
                   &raw_full[s], policy);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp < TC_FIRST_CONV) {
    // ------------------------------------------------------- MMA issuers ----
    // Warp 1 + mw issues the MMAs of pair-chunks pq = mw (mod 2), i.e. always
    // tile mw (TC_NOP = 2), into its own partial accumulator of the pair; the
    // assembler adds the partials.  Two issuing threads overlap one another's
    // wait / fence / commit latency.
    const int mw = warp - 1;
    if (lane == 0 && !(p.ablate & 128)) {  // ablate 128: stream-only skeleton
      const uint32_t idesc = umma_idesc_tf32_mn(128, N);
      const uint32_t lbo = (uint32_t)L.lbo;
      const uint32_t ops = smem_u32(smem + L.ops);
      for (int v = 0; v < n_pairs; ++v) {
        const int a = v & 1;
        bool first = true;
        for (int j = 0; j < cpu; ++j) {
          const int pq = v * cpu + j;
          if (pq % TC_MMA_W != mw) continue;
          const int b = pq % TC_NOP;
          const uint32_t bph = (uint32_t)((pq / TC_NOP) & 1);
          wc.wait(&op_full[b], bph, 1);
          const ChunkDesc cd = chunks[j];  // units share the chunk structure
          if (first && v >= 2) wc.wait(&acc_empty[a], (uint32_t)(((v >> 1) - 1) & 1), 2);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)((TC_MMA_W * a + mw) * SW);
          const uint32_t hi = ops + (uint32_t)(2 * b * L.opb);
          const uint32_t lo = hi + (uint32_t)L.opb;
          const int nk8 = (p.ablate & 2) ? 0 : (cd.nrows + 7) >> 3;
          const long long t_mma = rec ? clock64() : 0;
          for (int ks = 0; ks < nk8; ++ks) {
            const uint32_t acc = (first && ks == 0) ? 0u : 1u;
            const uint64_t ah = umma_desc_mn_sw128(hi + ks * 1024, lbo, 512);
            const uint64_t al = umma_desc_mn_sw128(lo + ks * 1024, lbo, 512);
            umma_tf32(d, ah, ah, idesc, acc);
            umma_tf32(d, ah, al, idesc, 1u);
            umma_tf32(d, al, ah, idesc, 1u);
            // U = 64 (B up to 1024 antennas, 64 x 64 solves): the lo.lo term
            // too (4-term split, ~2^-20 per product instead of ~2^-18), so the
            // decision-mismatch rate stays below 1e-5 at cfg5 (VERDICT r1 task 5)
            if constexpr (WIDE) umma_tf32(d, al, al, idesc, 1u);
          }
          if (rec) cnt[3] += clock64() - t_mma;
          first = false;
          const bool last_mine = (j + TC_MMA_W >= cpu);  // no later chunk of this pair for this warp
          umma_commit(&op_empty[b]);
          if (last_mine) umma_commit(&acc_full[a]);
        }
      }
    }
    __syncwarp();
  } else if (warp < TC_FIRST_ASM) {
    // -------------------------------------------------------- converters ----
    // hi = x with the low 13 mantissa bits cleared (exact TF32), lo = x - hi.
    // H rows: one float4 (2 UEs) per task, written to the same antenna row of
    // the tile (4 rows x 8 chunks per warp: one wavefront per row).  Y: task
    // (symbol pair tp, antenna pair k) reads Y[2tp][k..k+1], Y[2tp+1][k..k+1]
    // and writes chunk tp of antenna rows k and k+1; a warp takes 4 symbol
    // pairs x 8 antenna pairs, so its loads are 4 whole 128-byte row segments
    // and its stores hit every chunk position of the swizzle 4 times (4
    // wavefronts, the minimum).  Pad rows/features of the tiles were zeroed at
    // kernel start and are never written.  Full chunks (KC rows) use per-thread
    // task offsets computed once; one iteration converts a whole pair-chunk.
    // two sets of 4 warps convert alternating pair-chunks, so one set's
    // load / barrier latency overlaps the other's work
    const int cset = (warp - TC_FIRST_CONV) >> 2;
    const int ct = ((warp - TC_FIRST_CONV) & 3) * 32 + lane;  // thread index within the set
    const int us2 = 2 * p.us;
    const int hq = p.us / 2;             // float4 per stored H row
    constexpr int HQ = UP / 2;           // float4 slots per H row of the tile
    constexpr int HT = 32 * HQ / TC_CONV;  // H tasks per thread in a full chunk
    static_assert(HT * TC_CONV == 32 * HQ, "full-chunk H tasks must divide evenly");
    const int lbo = L.lbo;
    const int tpairs = (T + 1) / 2;
    auto split = [](float x, float& h, float& l) {
      h = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
      l = x - h;
    };
    auto put = [&](char* hi, char* lo, int off, float4 v) {
      float4 hh, ll;
      split(v.x, hh.x, ll.x);
      split(v.y, hh.y, ll.y);
      split(v.z, hh.z, ll.z);
      split(v.w, hh.w, ll.w);
      *reinterpret_cast<float4*>(hi + off) = hh;
      *reinterpret_cast<float4*>(lo + off) = ll;
    };
    // per-thread task tables of a full chunk (half h adds its own store offsets)
    int h_ld[HT], h_st[2][HT];
    bool h_ok[HT];
#pragma unroll
    for (int r = 0; r < HT; ++r) {
      const int e = ct + r * TC_CONV;
      const int kr = e / HQ, c4 = e % HQ;
      h_ok[r] = c4 < hq;
      h_ld[r] = kr * us2 + 4 * c4;
      h_st[0][r] = mn_off(4 * c4, kr, lbo);
      h_st[1][r] = mn_off(2 * UP + 4 * c4, kr, lbo);
    }
    // Y task of a full chunk: 8 symbol pairs x 16 antenna pairs over the 128
    // converter threads; a quarter-warp takes 4 symbol pairs x 2 antenna
    // pairs, so its 16-byte loads (padded staged rows) and its stores (the
    // operand swizzle) each hit 8 distinct bank groups
    const int ytp = (ct & 3) + 4 * ((ct >> 5) & 1);
    const int yk = 2 * (((ct >> 2) & 1) + 2 * ((ct >> 3) & 3) + 8 * (ct >> 6));
    const bool y_ok = ytp < tpairs;
    const bool y_ok1 = 2 * ytp + 1 < T;
    // Y loads: symbol rows 2tp, 2tp+1 of the staged block (row stride yrow)
    int y_st[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      y_st[h][0] = mn_off(YB + 32 * h + 4 * ytp, yk, lbo);
      y_st[h][1] = mn_off(YB + 32 * h + 4 * ytp, yk + 1, lbo);
    }
    int b = 0;
    uint32_t bph = 0;
    // unit cursor: (item, cluster) of the next unit, its slot in the stage
    // group and the ring position / phase of the group's first stage (no
    // divisions in the loop: a lone warp pays ~100 cycles per division)
    int cu_il = 0, cu_c = 0, cu_sl = 0, cu_gpos = 0;
    uint32_t cu_gph = 0;
    for (int v = 0; v < n_pairs; ++v) {
      int il[2], cl[2], sl[2], gpos[2];
      uint32_t gph[2];
      bool real[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        il[h] = cu_il;
        cl[h] = cu_c;
        sl[h] = cu_sl;
        gpos[h] = cu_gpos;
        gph[h] = cu_gph;
        real[h] = (h < pair) && (v * pair + h < U_tot);
        if (h < pair && ++cu_c == upi) {
          cu_c = 0;
          ++cu_il;
          if (++cu_sl == ips) {
            cu_sl = 0;
            cu_gpos += spi;
            while (cu_gpos >= NS) {
              cu_gpos -= NS;
              cu_gph ^= 1u;
            }
          }
        }
      }
      if (p.ablate & 1024) {  // timing study only: one wait + release per stage, no chunk loop
        if (spi == 1) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (h < pair && real[h]) wc.wait(&raw_full[gpos[h]], gph[h], 1);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (h < pair && real[h] && cl[h] == upi - 1 && (sl[h] == ips - 1 || il[h] == my_items - 1))
              mbar_arrive(&raw_empty[gpos[h]]);
        }
        continue;
      }
      for (int j = 0; j < cpu; ++j) {
        const int pq = v * cpu + j;
        if ((pq % TC_CONV_SETS) != cset) continue;
        b = pq % TC_NOP;
        bph = (uint32_t)((pq / TC_NOP) & 1);
        if (p.tc_simple && !(p.ablate & 4)) {
          // simple geometry: every address is arithmetic (no table lookups:
          // a lone warp pays ~30 cycles per dependent shared-memory load)
          // one stage holds every chunk of the pair's items (spi == 1): wait
          // for it once, at the first chunk (a completed-phase wait per chunk
          // costs the converter hundreds of cycles: stream-only study)
          if (j == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (h < pair && real[h]) wc.wait(&raw_full[gpos[h]], gph[h], 1);
          }
          if (pq >= TC_NOP && !(p.ablate & 128)) wc.wait(&op_empty[b], bph ^ 1u, 1);
          const long long t_body = rec ? clock64() : 0;
          char* hi = smem + L.ops + 2 * b * L.opb;
          char* lo = hi + L.opb;
          float4 hv[2][HT], ya[2], yb[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            ya[h] = make_float4(0.f, 0.f, 0.f, 0.f);
            yb[h] = ya[h];
            if (h >= pair || !real[h]) continue;
            const int row = cl[h] * p.tc_bc + 32 * j;  // first antenna row of the chunk in its item
            const char* sb = smem + L.stg + gpos[h] * L.sbytes;
            const float* Hq = reinterpret_cast<const float*>(sb) + (size_t)(sl[h] * p.B + row) * us2;
            const float* Yq = reinterpret_cast<const float*>(sb + p.stage_hbytes +
                                                              (size_t)sl[h] * T * p.stage_ystride) + 2 * row;
            const int yq = p.stage_ystride / 4;
#pragma unroll
            for (int r = 0; r < HT; ++r)
              if (h_ok[r]) hv[h][r] = *reinterpret_cast<const float4*>(Hq + h_ld[r]);
            if (y_ok) {
              ya[h] = *reinterpret_cast<const float4*>(Yq + 2 * ytp * yq + 2 * yk);
              if (y_ok1) yb[h] = *reinterpret_cast<const float4*>(Yq + (2 * ytp + 1) * yq + 2 * yk);
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h >= pair || !real[h]) continue;
#pragma unroll
            for (int r = 0; r < HT; ++r)
              if (h_ok[r]) put(hi, lo, h_st[h][r], hv[h][r]);
            if (y_ok) {
              put(hi, lo, y_st[h][0], make_float4(ya[h].x, ya[h].y, yb[h].x, yb[h].y));
              put(hi, lo, y_st[h][1], make_float4(ya[h].z, ya[h].w, yb[h].z, yb[h].w));
            }
          }
          if (rec) cnt[2] += clock64() - t_body;
          if (!(p.ablate & 256)) fence_proxy_async_smem();  // ablate 256: timing study only
          if (!(p.ablate & 128)) mbar_arrive(&op_full[b]);
          // an item's stage is free after its last chunk (multi-item stages:
          // after the group's last item)
          if (j == cpu - 1) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (h < pair && real[h] && cl[h] == upi - 1 && (sl[h] == ips - 1 || il[h] == my_items - 1))
                mbar_arrive(&raw_empty[gpos[h]]);
          }
          continue;
        }
        // wait for the stages of both halves, then for the operand tile
        int sslot[2], sflags[2];
        #pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= pair) continue;
          if (!real[h]) continue;
          sflags[h] = chunks[cl[h] * cpu + j].flags;
          int pos = gpos[h] + ((sflags[h] >> CH_STAGE_SHIFT) & 0xff);
          uint32_t sp = gph[h];
          while (pos >= NS) {
            pos -= NS;
            sp ^= 1u;
          }
          sslot[h] = pos;
          wc.wait(&raw_full[pos], sp, 1);
        }
        if (pq >= TC_NOP && !(p.ablate & 128)) wc.wait(&op_empty[b], bph ^ 1u, 1);
        const long long t_body = rec ? clock64() : 0;
        char* hi = smem + L.ops + 2 * b * L.opb;
        char* lo = hi + L.opb;
        #pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= pair) continue;
          if (!real[h] || (p.ablate & 4)) continue;  // null half: rows/columns never read
          const ChunkDesc cd = chunks[cl[h] * cpu + j];
          const int nr = cd.nrows;
          const int k = (cd.flags >> CH_STAGE_SHIFT) & 0xff;
          const int R = st_rows[k], dr = cd.row0 - st_row0[k], slot = sl[h];
          const char* sb = smem + L.stg + sslot[h] * L.sbytes;
          const float* Hf = reinterpret_cast<const float*>(sb) + (size_t)(slot * R + dr) * us2;
          const float* Yf =
              reinterpret_cast<const float*>(sb + p.stage_hbytes + (size_t)slot * T * p.stage_ystride) + 2 * dr;
          const int yrow = p.stage_ystride / 4;  // floats per staged Y symbol row
          if (nr == 32) {
            float4 hv[HT], ya = make_float4(0.f, 0.f, 0.f, 0.f), yb = ya;
#pragma unroll
            for (int r = 0; r < HT; ++r)
              if (h_ok[r]) hv[r] = *reinterpret_cast<const float4*>(Hf + h_ld[r]);
            if (y_ok) {
              ya = *reinterpret_cast<const float4*>(Yf + 2 * ytp * yrow + 2 * yk);
              if (y_ok1) yb = *reinterpret_cast<const float4*>(Yf + (2 * ytp + 1) * yrow + 2 * yk);
            }
#pragma unroll
            for (int r = 0; r < HT; ++r)
              if (h_ok[r]) put(hi, lo, h_st[h][r], hv[r]);
            if (y_ok) {
              put(hi, lo, y_st[h][0], make_float4(ya.x, ya.y, yb.x, yb.y));
              put(hi, lo, y_st[h][1], make_float4(ya.z, ya.w, yb.z, yb.w));
            }
            continue;
          }
          // partial chunk (ragged cluster): generic loops, K rows zero-padded to 8
          const int nr8 = (nr + 7) & ~7;
          const int fh = h * 2 * UP;
          const int fy = YB + 32 * h;
          for (int e = ct; e < nr8 * HQ; e += TC_CONV) {
            const int kr = e / HQ, c4 = e % HQ;
            if (c4 >= hq) continue;
            const float4 v4 = (kr < nr) ? *reinterpret_cast<const float4*>(Hf + kr * us2 + 4 * c4)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            put(hi, lo, mn_off(fh + 4 * c4, kr, lbo), v4);
          }
          const int kb8 = (nr8 / 2 + 7) / 8;
          const int ntask = 32 * kb8 * ((tpairs + 3) / 4);
          for (int e = ct; e < ntask; e += TC_CONV) {
            const int blk = e >> 5;
            const int tp = 4 * (blk / kb8) + ((e >> 3) & 3);
            const int k = 2 * ((e & 7) + 8 * (blk % kb8));
            if (tp >= tpairs || k >= nr8) continue;
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
            if (k < nr) {
              a0 = *reinterpret_cast<const float4*>(Yf + 2 * tp * yrow + 2 * k);
              if (2 * tp + 1 < T) a1 = *reinterpret_cast<const float4*>(Yf + (2 * tp + 1) * yrow + 2 * k);
            }
            const int f = fy + 4 * tp;
            put(hi, lo, mn_off(f, k, lbo), make_float4(a0.x, a0.y, a1.x, a1.y));
            put(hi, lo, mn_off(f, k + 1, lbo), make_float4(a0.z, a0.w, a1.z, a1.w));
          }
        }
        const long long t_fence = rec ? clock64() : 0;
        if (rec) cnt[2] += t_fence - t_body;
        if (!(p.ablate & 256)) fence_proxy_async_smem();  // ablate 256: timing study only
        if (!(p.ablate & 128)) mbar_arrive(&op_full[b]);
        if (rec) cnt[3] += clock64() - t_fence;
        // release a stage after the last chunk that reads it (host-computed
        // per item; a multi-item stage after its last item)
        #pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= pair) continue;
          if (!real[h] || !(sflags[h] & CH_STAGE_REL)) continue;
          if (spi == 1 && sl[h] != ips - 1 && il[h] != my_items - 1) continue;
          mbar_arrive(&raw_empty[sslot[h]]);
        }
      }
    }
  } else if (warp < TC_FIRST_SOLVER) {
    // -------------------------------------------------------- assemblers ----
    const int wq = warp & 3;       // TMEM lane quarter this warp may access
    const int m = 32 * wq + lane;  // accumulator row owned by this thread
    const bool odd = (m & 1) != 0;
    // which half / part this row belongs to
    const bool is_h = m < HR;
    const int hh = is_h ? m / (2 * UP) : (m - YB) / 32;
    const bool has_row = is_h || (m >= YB && m < MU && ((m - YB) & 31) < 2 * T);
    const bool warp_rows = 32 * wq < MU;
    int ssl = 0;  // solver slot of unit v * pair (round robin, no divisions)
    uint32_t sph = 0;
    for (int v = 0; v < ((p.ablate & 128) ? 0 : n_pairs); ++v) {
      const int a = v & 1;
      int slot[2];
      uint32_t sphase[2];
      #pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h >= pair) continue;
        slot[h] = ssl;
        sphase[h] = sph;
        if (++ssl == nsolv) {
          ssl = 0;
          sph ^= 1u;
        }
      }
      // both halves' solver slots must be free before writing either
      #pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h >= pair) continue;
        const int u = v * pair + h;
        if (u < U_tot && u >= nsolv) wc.wait(&slot_empty[slot[h]], sphase[h] ^ 1u, 1);
      }
      wc.wait(&acc_full[a], (uint32_t)((v >> 1) & 1), 2);
      tc_fence_after();
      const int u_mine = v * pair + hh;
      if (warp_rows && !(p.ablate & 32)) {  // ablate 32: timing study without the TMEM read-back
        const bool write = has_row && u_mine < U_tot;
        const Work w = work_at(smem, L, hh ? slot[1] : slot[0], UP);
        float* Gf = reinterpret_cast<float*>(w.G);
        float* Zf = reinterpret_cast<float*>(w.Z);
        const int LD = w.LD;
        // tcgen05.ld takes one warp-uniform address, and a warp may hold rows of
        // both halves (e.g. rows 64..95 = Y of half 0 and of half 1): read all
        // pair * 2UP columns and let each thread keep its half's columns
        // [hh * 2UP, (hh + 1) * 2UP)
        // partial accumulators of the pair: one per contributing MMA warp
        // (with one chunk per unit only warp (v mod 2) contributes)
        const uint32_t taddr = tmem + ((uint32_t)(32 * wq) << 16) +
                               (uint32_t)((TC_MMA_W * a + (cpu_mma == 1 ? (v * cpu) % TC_MMA_W : 0)) * SW);
        const int rloc = is_h ? (m - hh * 2 * UP) : ((m - YB) & 31);  // row within the half
        for (int c16 = 0; c16 < (WIDE ? SW : pair * 2 * UP) / 16; ++c16) {
          float vv[16];
          tmem_ld16(taddr + 16 * c16, vv);
          for (int mm = 1; mm < cpu_mma; ++mm) {
            float v2[16];
            tmem_ld16(taddr + mm * SW + 16 * c16, v2);
#pragma unroll
            for (int c = 0; c < 16; ++c) vv[c] += v2[c];
          }
          const int colbase = 8 * c16 - hh * UP;  // UE column of vv[0] within this row's half
          const bool mine = write && colbase >= 0 && colbase < UP;
          if (WIDE && colbase >= UP) {
            // Y columns (symbol t = colbase - UP + c): y_t[u] for this lane's
            // UE u, same re/im recombination as G (rows are H features here)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float po = __shfl_xor_sync(0xffffffffu, vv[2 * c + 1], 1);
              const int t = colbase - UP + c;
              if (write && t < T) {
                const float val = odd ? (po - vv[2 * c]) : (vv[2 * c] + po);
                Zf[(t * LD + (rloc >> 1)) * 2 + (odd ? 1 : 0)] = val;
              }
            }
            continue;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float po = __shfl_xor_sync(0xffffffffu, vv[2 * c + 1], 1);
            const int col = colbase + c;
            if (mine) {
              if (is_h) {
                const float val = odd ? (po - vv[2 * c]) : (vv[2 * c] + po);
                Gf[((rloc >> 1) * LD + col) * 2 + (odd ? 1 : 0)] = val;
              } else {
                const float val = odd ? (vv[2 * c] - po) : (vv[2 * c] + po);
                Zf[((rloc >> 1) * LD + col) * 2 + (odd ? 1 : 0)] = val;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[a]);
      #pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h >= pair) continue;
        const int u = v * pair + h;
        if (u < U_tot) mbar_arrive(&slot_full[slot[h]]);
      }
    }
  } else {
    // ----------------------------------------------------------- solvers ----
    const int sv = warp - TC_FIRST_SOLVER;
    const Team<32, -1> tm{lane};
    const Work w = work_at(smem, L, sv, UP);
    int cl_first = 1;
    int il = 0, c = sv;  // (item, cluster) of unit u, advanced without divisions
    while (c >= upi) {
      c -= upi;
      ++il;
    }
    uint32_t ph = 0;
    for (int u = sv; u < ((p.ablate & 128) ? 0 : U_tot); u += nsolv, ph ^= 1u) {
      const int64_t n = first + il;
      const bool item_end = (c == upi - 1);
      const float n0 = item_n0(p, n);  // global load issued before the wait
      wc.wait(&slot_full[sv], ph, 1);
      reset_flags(w, tm);
      tm.sync();
      if (p.ablate & 1) {
      } else if (!fd) {
        const long long t0 = rec ? clock64() : 0;
        unit_epilogue<UP, Team<32, -1>, CLS>(w, p, n, c, item_end, cl_first, tm, rec ? cnt + 2 : nullptr, n0);
        if (rec) cnt[3] += clock64() - t0;
      } else {
        EpiArgs a;
        a.kind = p.kind;
        a.u = p.u;
        a.T = T;
        a.n0 = n0;
        a.es = p.es;
        a.damping = p.damping;
        a.t_max = p.t_max;
        a.beta = p.cl_beta[c];
        a.lama_scale = p.cl_scale[c];
        a.unbias = true;  // fusion.py:148 -- fuse in the unbiased domain
        a.ablate = p.ablate;
        const long long t0 = rec ? clock64() : 0;
        if constexpr (lama)
          lama_unit<UP>(w, a, p.cp, nullptr, nullptr, nullptr, nullptr, tm, true);
        else
          linear_unit<UP>(w, a, tm);
        // stash this cluster's estimate, count the arrival; the last of the
        // item's C clusters folds them in cluster order
        fd_stash(w, p, n, c, tm);
        __threadfence_block();
        tm.sync();
        if (rec) cnt[2] += clock64() - t0;  // FD: solve + stash (c2), fold (c3)
        int last = 0;
        if (lane == 0) last = (atomicAdd(&fd_count[il & (FD_CNT - 1)], 1) == p.C - 1);
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          if (lane == 0) fd_count[il & (FD_CNT - 1)] = 0;
          __threadfence_block();
          const long long t1 = rec ? clock64() : 0;
          fd_finish(reinterpret_cast<float*>(w.X), p, n, tm);
          if (rec) cnt[3] += clock64() - t1;
        }
      }
      tm.sync();
      if (lane == 0) mbar_arrive(&slot_empty[sv]);
      c += nsolv;
      while (c >= upi) {
        c -= upi;
        ++il;
      }
    }
  }
  if (rec) {
    cnt[0] = clock64() - t_start;
    for (int k = 0; k < 4; ++k) atomicAdd(reinterpret_cast<unsigned long long*>(p.dbg + warp * 4 + k),
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
