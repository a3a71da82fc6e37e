// Issue rate of the kernel's MMA pattern: per k-step three tcgen05.mma
// kind::tf32 (hi.hi, hi.lo, lo.hi), M = 128, operands MN-major (SW128 with
// 32-byte atoms) vs K-major (SW128), A from shared memory or from TMEM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_rate tools/umma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1808_04473_b200/csrc/dbp_device.cuh"
using namespace dbp;

template <int N, int MODE>  // MODE 0: MN-major SS, 1: K-major SS, 2: A in TMEM + B MN-major
__global__ void bench(int iters, long long* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 13);
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
    const uint32_t hi = smem_u32(smem), lo = hi + 16384;
    const uint32_t idesc = MODE == 0 ? umma_idesc_tf32_mn(128, N) : MODE == 1 ? umma_idesc_tf32(128, N)
                                                                  : umma_idesc_tf32_tmem_a(128, N);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (it | ks) ? 1u : 0u;
        const uint32_t d = tmem + (it & 1) * 128;
        if (MODE == 0) {
          const uint64_t ah = umma_desc_mn_sw128(hi + ks * 1024, 4096, 512);
          const uint64_t al = umma_desc_mn_sw128(lo + ks * 1024, 4096, 512);
          umma_tf32(d, ah, ah, idesc, acc);
          umma_tf32(d, ah, al, idesc, 1u);
          umma_tf32(d, al, ah, idesc, 1u);
        } else if (MODE == 1) {
          const uint64_t ah = umma_desc_sw128(hi + ks * 32, 1024);
          const uint64_t al = umma_desc_sw128(lo + ks * 32, 1024);
          umma_tf32(d, ah, ah, idesc, acc);
          umma_tf32(d, ah, al, idesc, 1u);
          umma_tf32(d, al, ah, idesc, 1u);
        } else {
          const uint64_t bh = umma_desc_mn_sw128(hi + ks * 1024, 4096, 512);
          const uint64_t bl = umma_desc_mn_sw128(lo + ks * 1024, 4096, 512);
          const uint32_t at = tmem + 256 + ks * 8;
          umma_tf32_ts(d, at, bh, idesc, acc);
          umma_tf32_ts(d, at, bl, idesc, 1u);
          umma_tf32_ts(d, at + 32, bh, idesc, 1u);
        }
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

template <int N, int MODE>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int iters = 200;
  cudaFuncSetAttribute(bench<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  bench<N, MODE><<<sms, 128, 65536>>>(iters, d);
  bench<N, MODE><<<sms, 128, 65536>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[200];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const char* nm[3] = {"MN-major SS", "K-major SS ", "A-TMEM, B MN"};
  printf("%s N=%3d: %6.1f cycles per MMA (%s)\n", nm[MODE], N, avg / (iters * 12), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<32, 0>(sms); run<64, 0>(sms); run<128, 0>(sms);
  run<32, 1>(sms); run<64, 1>(sms); run<128, 1>(sms);
  run<32, 2>(sms); run<64, 2>(sms); run<128, 2>(sms);
  return 0;
}
