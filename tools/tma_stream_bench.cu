// Micro-benchmark: how fast can one persistent CTA per SM stream items
// (H block + Y block per item) from HBM into a shared-memory ring with
// cp.async.bulk?  Varies the copy granularity (split = copies per item),
// the number of issuing lanes, the ring depth and the item order
// (strided over CTAs or contiguous per CTA).  Consumers only wait and release.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream_bench tools/tma_stream_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1808_04473_b200/csrc/dbp_device.cuh"
#ifndef EXTRA_WARPS
#define EXTRA_WARPS 0  // idle warps parked at the final barrier (the kernel has 16 warps)
#endif
#ifndef EXTRA_SMEM
#define EXTRA_SMEM 0  // extra dynamic shared memory (the kernel uses ~230 KB)
#endif
#ifndef CONSUMER_WARPS
#define CONSUMER_WARPS 1  // warps that wait on every stage and release it (the kernel has 4 converters)
#endif
using namespace dbp;

struct Cfg {
  const char* src;
  long long n_items;
  int item_bytes;   // bytes per item (H + Y)
  int split;        // copies per item
  int stages;       // ring depth (items)
  int lanes;        // issuing lanes
  int contiguous;   // items contiguous per CTA
  int rows;         // > 0: tensor-core kernel pattern: one copy of the first (item_bytes - rows * rowb)
  int rowb;         //      bytes, then `rows` copies of rowb bytes to 16-byte padded slots
  const char* src2; // non-null: the row copies read a second array (H and Y as separate tensors)
};

__global__ void __launch_bounds__(32 * (CONSUMER_WARPS + 1 + EXTRA_WARPS), 1) stream(Cfg c, long long* sink) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < c.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32 * CONSUMER_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long per = (c.n_items + gridDim.x - 1) / gridDim.x;
  const long long my = c.contiguous ? max(0LL, min(per, c.n_items - blockIdx.x * per))
                                    : (c.n_items > blockIdx.x ? (c.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  const int cb = c.item_bytes / c.split;
  const uint64_t pol = l2_evict_first_policy();
  if (warp == 0) {
    for (long long k = 0; k < my; ++k) {
      const int s = (int)(k % c.stages);
      const long long n = c.contiguous ? blockIdx.x * per + k : blockIdx.x + k * gridDim.x;
      if (lane == 0 && k >= c.stages) mbar_wait(&empty[s], (uint32_t)(((k / c.stages) - 1) & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)c.item_bytes);
      __syncwarp();
      if (c.rows > 0) {
        const int hb = c.item_bytes - c.rows * c.rowb;
        char* dst = smem + s * (c.item_bytes + 16 * c.rows);
        const char* src = c.src2 ? c.src + n * hb : c.src + n * c.item_bytes;
        const char* ysrc = c.src2 ? c.src2 + n * (c.item_bytes - hb) : src + hb;
        if (lane == 0) bulk_g2s(dst, src, hb, &full[s], pol);
        for (int r = lane; r < c.rows; r += 32)
          bulk_g2s(dst + hb + r * (c.rowb + 16), ysrc + r * c.rowb, c.rowb, &full[s], pol);
      } else {
        for (int q = lane; q < c.split; q += c.lanes)
          if (lane < c.lanes)
            bulk_g2s(smem + s * c.item_bytes + q * cb, c.src + n * c.item_bytes + q * cb, cb, &full[s], pol);
      }
    }
  } else if (warp <= CONSUMER_WARPS) {
    long long acc = 0;
    for (long long k = 0; k < my; ++k) {
      const int s = (int)(k % c.stages);
      mbar_wait(&full[s], (uint32_t)((k / c.stages) & 1));
      acc += reinterpret_cast<const int*>(smem + s * (c.item_bytes + 16 * c.rows))[lane];
      mbar_arrive(&empty[s]);
    }
    if (acc == 12345) sink[0] = acc;
  }
  __syncthreads();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long total = 1LL << 30;  // 1 GiB of input
  char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct V { int item, split, stages, lanes, contig, rows = 0, rowb = 0, sep = 0; };
  const V vs[] = {
      {61440, 2, 2, 2, 1}, {61440, 2, 3, 2, 1}, {30720, 2, 2, 2, 1}, {30720, 2, 3, 2, 1}, {30720, 2, 4, 2, 1},
      {30720, 2, 6, 2, 1}, {45056, 2, 2, 2, 1}, {45056, 2, 4, 2, 1}, {92160, 2, 2, 2, 1}, {15360, 2, 8, 2, 1},
      // cfg2 stage geometry: 2 items (H 2 x 16 KB) + 28 Y rows of 1 KB = 30 copies of ~2 KB
      {61440, 30, 2, 32, 1}, {61440, 60, 2, 32, 1}, {61440, 15, 2, 32, 1}, {30720, 15, 3, 32, 1},
      // the cfg2 tensor-core producer: 2 items per stage = one 32 KB H copy + 28 Y rows of 1 KB
      {61440, 1, 2, 32, 1, 28, 1024}, {61440, 1, 3, 32, 1, 28, 1024}, {61440, 1, 2, 32, 1, 14, 2048},
      // ... with H and Y in separate arrays, as the detector's inputs are
      {61440, 1, 2, 32, 1, 28, 1024, 1}, {61440, 1, 3, 32, 1, 28, 1024, 1},
  };
  for (const V& v : vs) {
    Cfg c{src, total / v.item, v.item, v.split, v.stages, v.lanes, v.contig, v.rows, v.rowb,
          v.sep ? src + (total / v.item) * (long long)(v.item - v.rows * v.rowb) : nullptr};
    const int sb = (v.item + 16 * v.rows) * v.stages;
    if (sb + EXTRA_SMEM > 226 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) stream<<<sms, 32 * (CONSUMER_WARPS + 1 + EXTRA_WARPS), sb + EXTRA_SMEM>>>(c, sink);
    cudaEventRecord(a);
    const int R = 5;
    for (int rep = 0; rep < R; ++rep) stream<<<sms, 32 * (CONSUMER_WARPS + 1 + EXTRA_WARPS), sb + EXTRA_SMEM>>>(c, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("item %6d B split %2d (copy %6d B) rows %2d x %4d B stages %2d lanes %2d %s: %7.1f GB/s  %s\n", v.item,
           v.split, v.item / v.split, v.rows, v.rowb, v.stages, v.lanes, v.contig ? "contig " : "strided",
           (double)total * R / (ms * 1e6), cudaGetErrorString(e));
  }
  return 0;
}
