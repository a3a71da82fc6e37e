// Micro-benchmark of the one-warp ZF / L-MMSE unit solve (linear_solve_warp)
// with G, y_mrc in shared memory: cycles per unit for 1..8 concurrent warps.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/solver_bench tools/solver_bench.cu
#include <cstdio>
#include "../paper_1808_04473_b200/csrc/dbp_tc.cuh"
using namespace dbp;

template <int UP, int NU>
__global__ void bench(int iters, int T, long long* out, float* sink) {
  extern __shared__ __align__(1024) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WorkLayout wl = make_work_layout(0, UP, 16, 1, false, false);
  Work ws[NU];
  for (int q = 0; q < NU; ++q) ws[q] = make_work(smem + (warp * NU + q) * wl.total, wl, UP);
  Work& w = ws[0];
  for (int q = 0; q < NU; ++q) {
    for (int e = lane; e < UP * w.LD; e += 32) {
      const int i = e / w.LD, j = e % w.LD;
      ws[q].G[e] = make_float2(i == j ? 4.f : 0.1f / (1 + i + j), (i == j) ? 0.f : 0.01f * (i - j));
    }
    for (int e = lane; e < 16 * w.LD; e += 32) ws[q].Z[e] = make_float2(0.3f, -0.2f);
    if (lane == 0) {
      ws[q].flags[0] = 0;
      ws[q].flags[1] = 0x7fffffff;
    }
  }
  __syncwarp();
  EpiArgs a;
  a.kind = EQ_LMMSE;
  a.u = UP;
  a.T = T;
  a.n0 = 0.1f;
  a.es = 1.f;
  a.unbias = true;
  const long long t0 = clock64();
  EpiArgs as[NU];
  float rh[NU];
  for (int q = 0; q < NU; ++q) {
    as[q] = a;
    rh[q] = 0.1f;
  }
  for (int it = 0; it < iters; ++it) linear_solve_warp_n<UP, NU>(ws, as, rh, lane);
  const long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (w.X[0].x == 12345.f) sink[0] = 1.f;
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 32 * sizeof(long long));
  cudaMalloc(&sink, 4);
  const int iters = 50;
  for (int NU : {1, 2})
  for (int T : {0, 14})
  for (int nw : {1, 4, 8}) {
    const int smem = nw * NU * make_work_layout(0, 16, 16, 1, false, false).total;
    auto k = NU == 1 ? bench<16, 1> : bench<16, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 32 * nw, smem>>>(iters, T, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148 * 32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int wv = 0; wv < nw; ++wv) avg += h[wv];
    avg /= nw;
    printf("U=16 NU=%d T=%2d warps/CTA %d: %8.0f cycles per unit (per warp, latency)  SM throughput %6.0f cyc/unit (%s)\n",
           NU, T, nw, avg / iters / NU, avg / iters / NU / nw, cudaGetErrorString(e));
  }
  return 0;
}
