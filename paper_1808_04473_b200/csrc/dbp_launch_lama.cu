// Host launcher of the LAMA recursion kernel (dbp_lama.cuh), its own
// translation unit so the library builds in parallel.
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/dbp_b200.h"
#include "dbp_host.h"
#include "dbp_lama.cuh"

namespace dbp {

// 0 launched, < 0 error, 1 not covered (u > 32, traces, the multi-GPU
// partial-sum architecture: the caller keeps the streaming-kernel recursion)
int launch_lama(EqParams& p, cudaStream_t st) {
  if (p.kind != EQ_LAMA || p.u > 32 || p.T > MAX_T || p.tr_z || (p.arch != ARCH_PD && p.arch != ARCH_FD) ||
      opt(DBP_OPT_LAMA_KERNEL) == 1)
    return 1;
  auto kern = p.cp.L == 4 ? lama_kernel<4> : p.cp.L == 8 ? lama_kernel<8> : p.cp.L == 2 ? lama_kernel<2>
                                                                                        : lama_kernel<0>;
  const size_t smem = sizeof(LamaWarpSmem) * LAMA_WARPS;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(DBP_E_CUDA, "shared memory request too large");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LAMA_NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>((p.n_items + LAMA_WARPS - 1) / LAMA_WARPS, (int64_t)sm_count() * per_sm);
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, LAMA_NT, smem, st>>>(p);
  return cuda_check("lama_kernel");
}

}  // namespace dbp
