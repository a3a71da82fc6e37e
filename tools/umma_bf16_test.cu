// Probe for the building blocks of the bf16x2 split-Gram kernel (dbp_tc2.cuh):
//  1) tcgen05.mma kind::f16 (bf16 operands, fp32 accumulate) with MN-major,
//     128-byte swizzled operands: 4 MN blocks of 64 elements, 32 K rows of
//     128 B each, 16-byte chunk j of K row k at position j ^ (k % 8);
//     M = 128 (blocks 0-1), N = 256 (blocks 0-3), two K16 steps.  Tries the
//     two (LBO, SBO) assignments.
//  2) TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver
//     entry point) for the H box [4 units][32 antennas][2U floats] and the
//     padded Y box [units][T][68 floats] (4 floats of the next antennas as row
//     padding).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_bf16_test tools/umma_bf16_test.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_1808_04473_b200/csrc/dbp_device.cuh"
using namespace dbp;

constexpr int MNT = 256, KT = 32, M = 128, N = 256;

__host__ __device__ inline int mn_off16(int mn, int k) {  // byte offset of element (mn, k)
  const int b = mn >> 6, e = mn & 63;
  return b * 4096 + k * 128 + ((((e >> 3) ^ (k & 7))) << 4) + (e & 7) * 2;
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void mma_kern(const float* X, float* D, int lbo, int sbo) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < MNT * KT; i += blockDim.x) {
    const int mn = i / KT, k = i % KT;
    *reinterpret_cast<__nv_bfloat16*>(smem + mn_off16(mn, k)) = __float2bfloat16(X[i]);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a = smem_u32(smem);
    for (int ks = 0; ks < KT / 16; ++ks) {
      const uint64_t da = desc_sw128(a + ks * 2048, lbo, sbo);
      umma_bf16(tmem, da, da, idesc, ks ? 1u : 0u);
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
    tmem_dealloc(tmem, 256);
  }
}

// ---- TMA tensor map probe -------------------------------------------------
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__global__ void tma_kern(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap ymap,
                         int hbytes, int ybytes, int c_h1, int c_h2, int c_y0, int c_y1, int c_y3, float* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, hbytes + ybytes);
    tma_load_3d(smem, &hmap, 0, c_h1, c_h2, &bar);
    tma_load_4d(smem + hbytes, &ymap, c_y0, c_y1, 0, c_y3, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < (hbytes + ybytes) / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int main() {
  // 1) MMA layout
  static float X[MNT * KT], D[M * N];
  float *dX, *dD;
  cudaMalloc(&dX, sizeof(X));
  cudaMalloc(&dD, sizeof(D));
  cudaFuncSetAttribute(mma_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  srand(1);
  for (int i = 0; i < MNT * KT; ++i) X[i] = (float)(rand() % 7 - 3);
  cudaMemcpy(dX, X, sizeof(X), cudaMemcpyHostToDevice);
  const int var[2][2] = {{4096, 1024}, {1024, 4096}};
  for (int vi = 0; vi < 2; ++vi) {
    cudaMemset(dD, 0, sizeof(D));
    mma_kern<<<1, 128, 16384>>>(dX, dD, var[vi][0], var[vi][1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < KT; ++k) r += (double)X[m * KT + k] * X[n * KT + k];
        err = fmax(err, fabs(r - D[m * N + n]));
        mx = fmax(mx, fabs(D[m * N + n]));
      }
    printf("bf16 MN-major SW128 lbo=%d sbo=%d: max err %.3g (max |D| %.3g) %s\n", var[vi][0], var[vi][1], err, mx,
           cudaGetErrorString(e));
  }
  // 2) TMA boxes.  H: [units][K][2U] floats (U = 16, K = 32 per unit: FD
  // units of 32 antennas), 6 units; box {32 floats, 32 antennas, 4 units}.
  // Y: [n][T][C][2K] floats (n = 2 items, T = 14, C = 3 clusters of K = 32
  // antennas); box {68 floats, 1 cluster, 14, 2 items} at cluster 1.
  auto enc = get_encode();
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  const int U2 = 32, K = 32, NU = 6, T = 14, C = 3, NI = 2;
  const size_t hn = (size_t)NU * K * U2, yn = (size_t)NI * T * C * 2 * K;
  float* hH = (float*)malloc(hn * 4);
  float* hY = (float*)malloc(yn * 4);
  for (size_t i = 0; i < hn; ++i) hH[i] = (float)i;
  for (size_t i = 0; i < yn; ++i) hY[i] = (float)(1000000 + i);
  float *dH, *dY, *dO;
  cudaMalloc(&dH, hn * 4);
  cudaMalloc(&dY, yn * 4);
  cudaMalloc(&dO, 1 << 20);
  cudaMemcpy(dH, hH, hn * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, hY, yn * 4, cudaMemcpyHostToDevice);
  CUtensorMap hmap, ymap;
  {
    cuuint64_t dims[3] = {(cuuint64_t)U2, (cuuint64_t)K, (cuuint64_t)NU};
    cuuint64_t strides[2] = {(cuuint64_t)U2 * 4, (cuuint64_t)K * U2 * 4};
    cuuint32_t box[3] = {32, 32, 4}, es[3] = {1, 1, 1};
    CUresult r = enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dH, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("H map: %d\n", (int)r);
  }
  {
    // dims: {2K floats of the cluster, C, T, n}; strides {2K*4, C*2K*4, T*C*2K*4}
    cuuint64_t dims[4] = {(cuuint64_t)2 * K, (cuuint64_t)C, (cuuint64_t)T, (cuuint64_t)NI};
    cuuint64_t strides[3] = {(cuuint64_t)2 * K * 4, (cuuint64_t)C * 2 * K * 4, (cuuint64_t)T * C * 2 * K * 4};
    cuuint32_t box[4] = {68, 1, (cuuint32_t)T, 2}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dY, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("Y map: %d\n", (int)r);
  }
  const int hbytes = 32 * 32 * 4 * 4, ybytes = 68 * T * 2 * 4;
  cudaFuncSetAttribute(tma_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hbytes + ybytes);
  // H units 4..7 (units 6, 7 out of range -> zero fill); Y cluster 2 (the
  // padding floats 64..67 run past dim 0 -> zero fill)
  tma_kern<<<1, 128, hbytes + ybytes>>>(hmap, ymap, hbytes, ybytes, 0, 4, 0, 2, 0, dO);
  cudaError_t e = cudaDeviceSynchronize();
  printf("tma kernel: %s\n", cudaGetErrorString(e));
  float* o = (float*)malloc(hbytes + ybytes);
  cudaMemcpy(o, dO, hbytes + ybytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int q = 0; q < 4; ++q)
    for (int k = 0; k < 32; ++k)
      for (int f = 0; f < 32; ++f) {
        const int unit = 4 + q;
        const float want = unit < NU ? hH[((size_t)unit * K + k) * U2 + f] : 0.f;
        if (o[(q * 32 + k) * 32 + f] != want) ++bad;
      }
  printf("H box mismatches: %d\n", bad);
  bad = 0;
  const float* oy = o + hbytes / 4;
  for (int n = 0; n < 2; ++n)
    for (int t = 0; t < T; ++t)
      for (int x = 0; x < 68; ++x) {
        const int cl = 2;
        const float want = (x < 64) ? hY[(((size_t)n * T + t) * C + cl) * 2 * K + x] : 0.f;
        if (oy[(n * T + t) * 68 + x] != want) ++bad;
      }
  printf("Y box mismatches (cluster 2, pad zero-filled): %d\n", bad);
  tma_kern<<<1, 128, hbytes + ybytes>>>(hmap, ymap, hbytes, ybytes, 0, 0, 0, 0, 0, dO);
  cudaDeviceSynchronize();
  cudaMemcpy(o, dO, hbytes + ybytes, cudaMemcpyDeviceToHost);
  bad = 0;
  for (int n = 0; n < 2; ++n)
    for (int t = 0; t < T; ++t)
      for (int x = 0; x < 68; ++x) {
        const float want = (x < 64) ? hY[(((size_t)n * T + t) * C + 0) * 2 * K + x] : 0.f;
        if (oy[(n * T + t) * 68 + x] != want) ++bad;
      }
  printf("Y box mismatches (cluster 0, pad past dim 0 zero-filled): %d\n", bad);
  return 0;
}
