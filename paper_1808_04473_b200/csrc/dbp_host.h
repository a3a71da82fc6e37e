// Host-side internals shared by the translation units of libdbp_b200.so
// (dbp_kernels.cu: C ABI and dispatch; dbp_launch_*.cu: kernel launchers).
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "dbp_simt.cuh"
#include "dbp_tc.cuh"
#include "dbp_tc2.cuh"

extern thread_local int g_last_kernel;

namespace dbp {
int opt(int key);                                   // dbp_set_option value
int fail(int code, const std::string& msg);         // sets dbp_last_error
int cuda_check(const char* where);
int sm_count();
void* stream_scratch(cudaStream_t st, size_t need);  // per-(device, stream) scratch
// launchers: 0 launched, < 0 error, 1 geometry not covered (caller falls back)
int launch_tc2(EqParams& p, cudaStream_t st);
int launch_t2_stats_solve(EqParams& p, cudaStream_t st);
// U = 64 statistics on the split-bf16 tensor cores; bf16 parts: 3 for the
// statistics API (~3xTF32 accuracy), 2 inside PD equalization (x-hat ~2e-5)
int launch_tcw(EqParams& p, cudaStream_t st, int nsplit_default = 3);
int launch_tc_up(int up, EqParams& p, cudaStream_t st);
int launch_stream_up(int up, EqParams& p, cudaStream_t st);
int launch_stats_up(int up, EqParams& p, cudaStream_t st);
// LAMA recursions from statistics records (u <= 32, PD / FD): 1 = not covered
int launch_lama(EqParams& p, cudaStream_t st);
}  // namespace dbp
