// Micro-benchmark: issue rate of tcgen05.mma kind::tf32 (cta_group::1) for
// the shapes the equalizer uses, one CTA per SM, operands in shared memory
// (K-major, 128-byte swizzle), accumulator in TMEM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_bench tools/umma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1808_04473_b200/csrc/dbp_device.cuh"

using namespace dbp;

__device__ __forceinline__ void umma_tf32_ts(uint32_t dtmem, uint32_t atmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int M, int N, bool F16>
__global__ void bench2(int iters, long long* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = F16 ? ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                               : umma_idesc_tf32(M, N);
    const uint32_t a = smem_u32(smem);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t da = umma_desc_sw128(a + ks * 32, 1024);
        if constexpr (F16)
          umma_f16(tmem, da, da, idesc, (it | ks) ? 1u : 0u);
        else
          umma_tf32(tmem, da, da, idesc, (it | ks) ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int M, int N, bool F16>
void run2(int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int iters = 256;
  cudaFuncSetAttribute(bench2<M, N, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  bench2<M, N, F16><<<sms, 128, 64 * 1024>>>(iters, d);
  bench2<M, N, F16><<<sms, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[200];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("%s M=%3d N=%3d: %7.1f cycles/mma (%s)\n", F16 ? "f16 " : "tf32", M, N, avg / (iters * 4),
         cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int CHAINS, bool ATMEM = false>
__global__ void bench(int iters, long long* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_tf32(128, N);
    const uint32_t a = smem_u32(smem);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t da = umma_desc_sw128(a + ks * 32, 1024);
        const uint32_t d = tmem + (uint32_t)((ks % CHAINS) * N);
        if constexpr (ATMEM)
          umma_tf32_ts(d, tmem + 256 + ks * 8, da, idesc, (it | ks) ? 1u : 0u);
        else
          umma_tf32(d, da, da, idesc, (it | ks) ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, int CHAINS, bool ATMEM = false>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int iters = 256;
  cudaFuncSetAttribute(bench<N, CHAINS, ATMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  bench<N, CHAINS, ATMEM><<<sms, 128, 64 * 1024>>>(iters, d);
  bench<N, CHAINS, ATMEM><<<sms, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[200];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("tf32 M=128 N=%3d chains=%d A=%s: %7.1f cycles/mma (%s)\n", N, CHAINS, ATMEM ? "tmem" : "smem",
         avg / (iters * 4), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16, 1>(sms);
  run<32, 1>(sms);
  run<32, 4>(sms);
  run<64, 1>(sms);
  run<128, 1>(sms);
  run<256, 1>(sms);
  run2<64, 32, false>(sms);
  run2<64, 64, false>(sms);
  run2<128, 32, true>(sms);
  run2<128, 64, true>(sms);
  run2<64, 32, true>(sms);
  run2<64, 64, true>(sms);
  run2<128, 128, true>(sms);
  run2<128, 256, true>(sms);
  return 0;
}
