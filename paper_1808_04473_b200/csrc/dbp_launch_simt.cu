// Host launchers of the FP32-SIMT streaming kernel and the statistics-input
// kernel (dbp_simt.cuh), one translation unit so the library builds in
// parallel.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "../../include/dbp_b200.h"
#include "dbp_host.h"

namespace dbp {

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
  auto kern = p.arch == ARCH_STATS ? stream_kernel<UP, NT, 0>
              : p.kind == EQ_LAMA   ? stream_kernel<UP, NT, 2>
                                    : stream_kernel<UP, NT, -1>;
  // ring depth: the deepest ring (<= p.NS, >= 2) that still lets a second CTA
  // share the SM, so one CTA's Gram overlaps the other's epilogue (U = 64:
  // 3 stages = one CTA per SM; 2 stages = two, cfg5 57 -> 46 ms)
  int per_sm = 0, ns = p.NS;
  if (opt(DBP_OPT_SIMT_NS)) ns = std::max(2, opt(DBP_OPT_SIMT_NS));  // tuning studies
  SimtLayout L = make_simt_layout(UP, p.TP, p.stage_f2 * 8, ns, p.C, red_f2, lama, fd);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return fail(DBP_E_CUDA, "shared memory request too large");
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, L.total);
  for (int k = ns - 1; k >= 2 && per_sm < 2 && !opt(DBP_OPT_SIMT_NS); --k) {
    const SimtLayout L2 = make_simt_layout(UP, p.TP, p.stage_f2 * 8, k, p.C, red_f2, lama, fd);
    int per2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, kern, NT, L2.total);
    if (per2 > per_sm) {
      ns = k;
      L = L2;
      per_sm = per2;
    }
  }
  p.NS = ns;
  if (per_sm < 1) return fail(DBP_E_UNSUPPORTED, "kernel does not fit on an SM");
  const int64_t grid = std::min<int64_t>(p.n_items, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, NT, L.total, st>>>(p);
  return cuda_check("stream_kernel");
}

template <int UP, int NT, bool XZ = false>
static int launch_stats(EqParams& p, cudaStream_t st) {
  const bool lama = p.kind == EQ_LAMA;
  const bool fd = p.arch == ARCH_FD;
  const WorkLayout L = make_work_layout(0, UP, p.TP, fd ? p.C : 1, lama, fd, XZ);
  auto kern = stats_kernel<UP, NT, XZ>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return fail(DBP_E_CUDA, "shared memory request too large");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, L.total);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>(p.n_items, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, NT, L.total, st>>>(p);
  return cuda_check("stats_kernel");
}

int launch_stream_up(int up, EqParams& p, cudaStream_t st) {
  switch (up) {
    case 8: return launch_stream<8, 128>(p, st);
    case 16: return launch_stream<16, 128>(p, st);
    case 32: return launch_stream<32, 256>(p, st);
    case 64: return launch_stream<64, 256>(p, st);
  }
  return fail(DBP_E_UNSUPPORTED, "u must be <= 64");
}

int launch_stats_up(int up, EqParams& p, cudaStream_t st) {
  switch (up) {
    case 8: return launch_stats<8, 128>(p, st);
    case 16: return launch_stats<16, 128>(p, st);
    case 32: return launch_stats<32, 256>(p, st);
    // U = 64 solves: 128-thread teams with 8 x 4 tiles, four per SM (PD:
    // cfg5-pd512 11.9 -> 11.6 ms); FD linear solves fit four per SM with X in Z
    // (FD LAMA / odd u keep the 256-thread team)
    case 64:
      if (p.arch != ARCH_FD) return launch_stats<64, 128>(p, st);
      return stats_x_in_z(p) ? launch_stats<64, 128, true>(p, st) : launch_stats<64, 256>(p, st);
  }
  return fail(DBP_E_UNSUPPORTED, "u must be <= 64");
}

}  // namespace dbp
