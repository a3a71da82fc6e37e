// Correctness probe for tcgen05.mma kind::tf32 with MN-major, 128-byte
// swizzled operands (the layout dbp_tc.cuh uses), plus the TF32 operand
// rounding mode (truncation vs round-to-nearest) of the tensor core.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_mn_test tools/umma_mn_test.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1808_04473_b200/csrc/dbp_device.cuh"
using namespace dbp;

constexpr int M = 128, N = 64, K = 16;
constexpr int LBO = 4096;  // M-block stride
constexpr int SBO = 512;   // 4-row K-group stride

__host__ __device__ inline int off(int m, int k) {
  return (m >> 5) * LBO + k * 128 + ((((m & 31) >> 3) ^ (k & 3)) << 5) + (m & 7) * 4;
}

__global__ void kern(const float* A, float* D, int lbo_f, int sbo_f, int mode) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<float*>(smem + off(m, k)) = A[i];
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 64);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_tf32_mn(M, N);
    const uint32_t a = smem_u32(smem);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint32_t st = a + ks * 1024;
      const uint64_t da = umma_desc_mn_sw128(st, lbo_f, sbo_f);
      umma_tf32(tmem, da, da, idesc, ks ? 1u : 0u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  float v[16];
  for (int c = 0; c < N / 16; ++c) {
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16 * c, v);
    for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * N + 16 * c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

static float trunc_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  memcpy(&x, &u, 4);
  return x;
}
static float round_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x1000u;
  u &= 0xffffe000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  static float A[M * K], D[M * N];
  float *dA, *dD;
  cudaMalloc(&dA, sizeof(A));
  cudaMalloc(&dD, sizeof(D));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  // 1) layout: small integers (exact in tf32)
  srand(1);
  for (int i = 0; i < M * K; ++i) A[i] = (float)(rand() % 7 - 3);
  cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice);
  const int var[2][2] = {{LBO, SBO}, {SBO, LBO}};
  for (int vi = 0; vi < 2; ++vi) {
    cudaMemset(dD, 0, sizeof(D));
    kern<<<1, 128, 16384>>>(dA, dD, var[vi][0], var[vi][1], 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * A[n * K + k];
        err = fmax(err, fabs(r - D[m * N + n]));
        mx = fmax(mx, fabs(D[m * N + n]));
      }
    printf("layout lbo_field=%d sbo_field=%d: max err %.3g (max |D| %.3g) %s\n", var[vi][0], var[vi][1], err, mx,
           cudaGetErrorString(e));
  }
  // 2) rounding: random fp32 operands
  for (int i = 0; i < M * K; ++i) A[i] = 1.0f + (float)rand() / RAND_MAX;
  cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice);
  kern<<<1, 128, 16384>>>(dA, dD, LBO, SBO, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
  double et = 0, er = 0, ef = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double rt = 0, rr = 0, rf = 0;
      for (int k = 0; k < K; ++k) {
        rt += (double)trunc_tf32(A[m * K + k]) * trunc_tf32(A[n * K + k]);
        rr += (double)round_tf32(A[m * K + k]) * round_tf32(A[n * K + k]);
        rf += (double)A[m * K + k] * A[n * K + k];
      }
      et = fmax(et, fabs(rt - D[m * N + n]));
      er = fmax(er, fabs(rr - D[m * N + n]));
      ef = fmax(ef, fabs(rf - D[m * N + n]));
    }
  printf("rounding: max err vs truncated %.3g, vs rounded %.3g, vs fp32 %.3g\n", et, er, ef);
  return 0;
}
