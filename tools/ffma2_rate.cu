// FP32 FMA issue study: scalar FFMA (3-register form) vs packed FFMA2
// (fma.rn.f32x2) throughput per SM, independent chains, full occupancy.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ffma2_rate tools/ffma2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;      // independent accumulator chains per thread
constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float acc[CH];
  float x = a + threadIdx.x * 1e-7f, y = b - threadIdx.x * 1e-7f;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = c * 0.5f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      acc[c] = fmaf(x, acc[c], y);
      acc[c] = fmaf(y, acc[c], x);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long acc[CH / 2];
  float2 xf = make_float2(a + threadIdx.x * 1e-7f, a), yf = make_float2(b - threadIdx.x * 1e-7f, b);
  unsigned long long x = *reinterpret_cast<unsigned long long*>(&xf), y = *reinterpret_cast<unsigned long long*>(&yf);
#pragma unroll
  for (int c = 0; c < CH / 2; ++c) {
    float2 f = make_float2(c * 0.5f, c * 0.25f);
    acc[c] = *reinterpret_cast<unsigned long long*>(&f);
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) {
      acc[c] = ffma2(x, acc[c], y);
      acc[c] = ffma2(y, acc[c], x);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH / 2; ++c) {
    float2 f = *reinterpret_cast<float2*>(&acc[c]);
    s += f.x + f.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = (double)blocks * threads * ITERS * CH * 2;
    printf("FFMA : %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM @1.9GHz\n", ms, fma / ms / 1e9, fma / (ms * 1e-3) / sms / 1.9e9);
    cudaEventRecord(e0);
    k_ffma2<<<blocks, threads>>>(out, 1.0001f, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM @1.9GHz\n", ms, fma / ms / 1e9, fma / (ms * 1e-3) / sms / 1.9e9);
  }
  return 0;
}
