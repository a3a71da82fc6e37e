// Host launcher of the 3xTF32 tensor-core streaming kernel (dbp_tc.cuh).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "../../include/dbp_b200.h"
#include "dbp_host.h"

namespace dbp {

template <int UP>
static int launch_tc(EqParams& p, cudaStream_t st) {
  const bool lama = p.kind == EQ_LAMA;
  const bool fd = (p.arch == ARCH_FD || p.arch == ARCH_FD_PARTIAL);
  // U = 64 ("wide": A = the 128 H features, B = [H | Y], N = 160) computes
  // statistics only; its solves run in stats_kernel (dispatch_stream)
  constexpr bool WIDE = UP > 32;
  if (WIDE && p.arch != ARCH_STATS) return 1;
  if (!WIDE && 2 * UP + 32 > 128) return fail(DBP_E_UNSUPPORTED, "2U + 32 > 128 rows on the tensor-core path");
  int dev = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // two units per operand tile / MMA when both fit in M = 128 rows and every
  // unit has the same chunk structure (uniform clusters for per-cluster units)
  const bool per_cluster = fd || (p.arch == ARCH_STATS && !p.sum_clusters);
  bool uniform = true;
  const int upi = per_cluster ? p.C : 1;
  if (p.nchunks % upi) uniform = false;
  const int cpu = uniform ? p.nchunks / upi : 0;
  for (int c = 1; uniform && c < upi; ++c)
    for (int j = 0; j < cpu; ++j)
      if (p.chunks[c * cpu + j].nrows != p.chunks[j].nrows || p.chunks[c * cpu + j].cluster != c) uniform = false;
  if (!uniform) return 1;  // ragged clusters: SIMT kernel
  // pair two units per tile when M allows; per-cluster units pair within an
  // item (even cluster count), items pair within a stage
  p.pair = (tc_yrow0(UP, 2) + 2 * 32 <= 128) ? 2 : 1;
  if (upi > 1 && (upi & 1)) p.pair = 1;
  if (opt(DBP_OPT_TC_PAIR)) p.pair = std::max(1, std::min(2, opt(DBP_OPT_TC_PAIR)));
  if (WIDE) p.pair = 1;
  // staging plan: whole items (several per stage when small) or row blocks
  const int hrow = p.us * 8, yrow = p.T * 8;  // bytes per antenna row of H / Y
  const int item_bytes = p.B * (hrow + yrow);
  int smax = 64 * 1024;
  if (opt(DBP_OPT_TC_SMAX_KB)) smax = opt(DBP_OPT_TC_SMAX_KB) * 1024;
  int nsolv = TC_MAX_SOLV;
  for (int attempt = 0;; ++attempt) {  // shrink the stages until the layout fits
  // (paired items may sit in different stages: the converter waits for both,
  // and the ring keeps at least 2 stages, all filled in order)
  if (item_bytes <= smax) {
    p.spi = 1;
    p.ips = std::max(1, smax / item_bytes);
    p.st_row0[0] = 0;
    p.st_rows[0] = p.B;
  } else {
    // row blocks at chunk boundaries (cluster-pair boundaries when units pair
    // inside an item), each at most smax bytes
    p.ips = 1;
    p.spi = 0;
    const int unit_step = (p.pair == 2 && upi > 1) ? 2 : 1;
    int r0 = 0, rows = 0;
    for (int j = 0; j < p.nchunks; ++j) {
      const ChunkDesc& cd = p.chunks[j];
      const bool boundary = (cd.row0 == p.chunks[(cd.cluster / unit_step) * unit_step * cpu].row0) || !per_cluster;
      if (rows > 0 && boundary && (rows + cd.nrows) * (hrow + yrow) + 16 * p.T > smax) {
        if (p.spi == MAX_SPI) return 1;
        p.st_row0[p.spi] = r0;
        p.st_rows[p.spi++] = rows;
        r0 = cd.row0;
        rows = 0;
      }
      rows += cd.nrows;
    }
    if (p.spi == MAX_SPI) return 1;
    p.st_row0[p.spi] = r0;
    p.st_rows[p.spi++] = rows;
  }
  int rmax = 0;
  for (int k = 0; k < p.spi; ++k) rmax = std::max(rmax, p.st_rows[k]);
  // Y symbol rows are staged with a 16-byte pad (row stride = 65 16-byte
  // chunks for 128 antennas) so that the converter's transposing loads of
  // symbols 2tp, 2tp+1 spread over all banks
  p.stage_hbytes = p.ips * rmax * hrow;
  p.stage_ystride = rmax * 8 + 16;
  p.stage_bytes = p.stage_hbytes + p.ips * p.T * p.stage_ystride;
  // chunk -> stage, and the last chunk of the item's visit order touching
  // each stage (units of an item in order; paired clusters interleave)
  for (int j = 0; j < p.nchunks; ++j) {
    int k = 0;
    while (k + 1 < p.spi && p.chunks[j].row0 >= p.st_row0[k + 1]) ++k;
    p.chunks[j].flags = (p.chunks[j].flags & 0xff) | (k << CH_STAGE_SHIFT);
  }
  {
    int last[MAX_SPI];
    for (int k = 0; k < MAX_SPI; ++k) last[k] = -1;
    const int ps = (p.pair == 2 && upi > 1) ? 2 : 1;  // units of an item sharing a tile
    for (int c0 = 0; c0 < upi; c0 += ps)
      for (int j = 0; j < cpu; ++j)
        for (int h = 0; h < ps; ++h) {
          const int idx = (c0 + h) * cpu + j;
          last[(p.chunks[idx].flags >> CH_STAGE_SHIFT) & 0xff] = idx;
        }
    for (int k = 0; k < p.spi; ++k)
      if (last[k] >= 0) p.chunks[last[k]].flags |= CH_STAGE_REL;
  }
  // simple geometry: the converter derives every address arithmetically
  // (chunk j of cluster c starts at row c * B/upi + 32 j) instead of through
  // the chunk table
  p.tc_bc = p.B / upi;
  p.tc_simple = (p.spi == 1) && (p.B % upi == 0);
  for (int c = 0; p.tc_simple && c < upi; ++c)
    for (int j = 0; j < cpu; ++j) {
      const ChunkDesc& cd = p.chunks[c * cpu + j];
      if (cd.nrows != 32 || cd.row0 != c * p.tc_bc + 32 * j) p.tc_simple = 0;
    }
  auto fits = [&](int ns, int nsv) {
    return make_tc_layout(UP, p.TP, p.stage_bytes, p.KC, ns, p.C, lama, fd, nsv).total <= smem_max;
  };
  // ring depth: ~96 KB of stages when they fit (>= 2), then solver warps
  p.NS = std::max(2, std::min(8, (96 * 1024 + p.stage_bytes - 1) / p.stage_bytes));
  nsolv = TC_MAX_SOLV;
  // tuning overrides (timing studies only)
  if (opt(DBP_OPT_TC_NS)) p.NS = opt(DBP_OPT_TC_NS);
  if (opt(DBP_OPT_TC_NSOLV)) nsolv = std::max(2, std::min(TC_MAX_SOLV, opt(DBP_OPT_TC_NSOLV)));
  while (nsolv > 4 && !fits(p.NS, nsolv)) --nsolv;
  while (p.NS > 2 && !fits(p.NS, nsolv)) --p.NS;
  while (nsolv > (WIDE ? 1 : 2) && !fits(p.NS, nsolv)) --nsolv;  // wide: one statistics writer suffices
  if (fits(p.NS, nsolv)) break;
  if (attempt == 6 || smax < 8 * 1024) return 1;  // does not fit: caller falls back to the SIMT kernel
  smax = smax * 3 / 4;
  }
  const TcLayout L = make_tc_layout(UP, p.TP, p.stage_bytes, p.KC, p.NS, p.C, lama, fd, nsolv);
  if (fd) {  // per-(item, cluster) fold records: L2-resident scratch, one per stream, grown on demand
    const size_t need = (size_t)p.n_items * p.C * fd_record_floats(p.u, p.T, lama ? p.T : p.u) * sizeof(float);
    p.fd_scratch = static_cast<float*>(stream_scratch(st, need));
    if (!p.fd_scratch) return fail(DBP_E_CUDA, "FD scratch allocation failed");
  }
  const bool fdm = (p.arch == ARCH_FD || p.arch == ARCH_FD_PARTIAL);
  void (*kern)(EqParams, int) = tc_kernel<UP, TC_STATS>;
  if constexpr (!WIDE)
    kern = (p.arch == ARCH_STATS) ? tc_kernel<UP, TC_STATS>
           : fdm ? (lama ? tc_kernel<UP, TC_FD_LAMA> : tc_kernel<UP, TC_FD_LIN>)
                 : (lama ? tc_kernel<UP, TC_PD_LAMA> : tc_kernel<UP, TC_PD_LIN>);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return fail(DBP_E_CUDA, "shared memory request too large");
  const int threads = 32 * (TC_FIRST_SOLVER + nsolv);
  const int64_t grid = std::min<int64_t>(p.n_items, (int64_t)sm_count());
#ifdef DBP_STUDY
  static float* dtile = nullptr;
  if (getenv("DBP_TC_DUMP")) {
    if (!dtile) cudaMalloc(&dtile, 128 * 1024);
    p.dbg_tile = dtile;
  }
  static long long* dbg = nullptr;
  const bool debug = getenv("DBP_TC_DEBUG") != nullptr;
  if (debug) {
    if (!dbg) cudaMalloc(&dbg, 128 * sizeof(long long));
    cudaMemsetAsync(dbg, 0, 128 * sizeof(long long), st);
    p.dbg = dbg;
  }
#endif
  kern<<<(unsigned)grid, threads, L.total, st>>>(p, nsolv);
#ifdef DBP_STUDY
  if (p.dbg_tile) {
    static float ht[32768];
    cudaMemcpy(ht, dtile, L.opb, cudaMemcpyDeviceToHost);
    FILE* f = fopen("gpurun_out/tile_dump.bin", "wb");
    if (f) {
      fwrite(ht, 1, L.opb, f);
      fclose(f);
    }
  }
  if (debug) {
    long long h[128];
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[dbp tc debug] NS=%d stage=%d B ips=%d spi=%d pair=%d nsolv=%d (cycles summed over CTAs)\n",
            p.NS, p.stage_bytes, p.ips, p.spi, p.pair, nsolv);
    for (int w = 0; w < threads / 32; ++w) {
      const char* name = w == 0 ? "producer" : w < TC_FIRST_CONV ? "mma" : w < TC_FIRST_ASM ? "converter"
                         : w < TC_FIRST_SOLVER ? "assembler" : "solver";
      fprintf(stderr, "  w%-2d %-9s total %.3e  c1 %.3e  c2 %.3e  c3 %.3e\n", w, name, (double)h[w * 4],
              (double)h[w * 4 + 1], (double)h[w * 4 + 2], (double)h[w * 4 + 3]);
    }
  }
#endif
  return cuda_check("tc_kernel");
}

int launch_tc_up(int up, EqParams& p, cudaStream_t st) {
  switch (up) {
    case 8: return launch_tc<8>(p, st);
    case 16: return launch_tc<16>(p, st);
    case 32: return launch_tc<32>(p, st);
    case 64: return launch_tc<64>(p, st);
  }
  return 1;
}

}  // namespace dbp
