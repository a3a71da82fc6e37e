// On-device synthesis of uplink frames: the model of
// the reference's run_trial / transmit (montecarlo.py:154-160, model.py:
// 207-236) -- H ~ CN(0, 1/B), uniform symbol indices, y = H s + CN(0, N0) --
// generated on the GPU from a counter-based Philox4x32-10 stream, so the
// 25-50 GB inputs of cfg5 never cross PCIe and every item is reproducible
// from (seed, item index) alone, in any order, on any GPU.
//
// Counter mapping (documented contract; tests/test_synth_device.py restates it
// in NumPy): key = (seed_lo, seed_hi); counter = (n_lo, n_hi, stream, j) for
// item n (the global item index), stream 0 = H, 1 = symbols, 2 = noise, and
// block j:
//   H     : block j -> 4 uniforms -> Box-Muller -> entries 2j, 2j+1 of the
//           item's H[b][u] (row-major, b*U + u), real/imag parts
//   symbol: block j -> 4 x 32 bits -> indices of entries 4j..4j+3 of
//           S[t][u] (t*U + u), index = (x * M) >> 32
//   noise : block j -> entries 2j, 2j+1 of the item's noise[t][b] (t*B + b)
// Box-Muller: u1 = (x0 + 1) 2^-32, u2 = x1 2^-32, r = sqrt(-2 ln u1),
// (r cos 2 pi u2, r sin 2 pi u2) = (z0, z1) for the first complex value,
// (x2, x3) likewise for the second; scaled by sqrt(v/2).
#pragma once
#include "dbp_device.cuh"

namespace dbp {

__host__ __device__ inline void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)M0 * c[0];
    const uint64_t p1 = (uint64_t)M1 * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ void philox_block(uint64_t seed, int64_t n, uint32_t stream, uint32_t j, uint32_t out[4]) {
  out[0] = (uint32_t)n;
  out[1] = (uint32_t)((uint64_t)n >> 32);
  out[2] = stream;
  out[3] = j;
  philox4x32_10(out, (uint32_t)seed, (uint32_t)(seed >> 32));
}

// two CN(0, 2 * s^2) values (each real part N(0, s^2)) from one block
__device__ __forceinline__ void box_muller2(const uint32_t x[4], float s, float2& a, float2& b) {
  const float k = 2.3283064365386963e-10f;  // 2^-32
  {
    const float u1 = ((float)x[0] + 1.f) * k, u2 = (float)x[1] * k;
    const float r = s * sqrtf(-2.f * logf(u1));
    float sn, cs;
    sincospif(2.f * u2, &sn, &cs);
    a = make_float2(r * cs, r * sn);
  }
  {
    const float u1 = ((float)x[2] + 1.f) * k, u2 = (float)x[3] * k;
    const float r = s * sqrtf(-2.f * logf(u1));
    float sn, cs;
    sincospif(2.f * u2, &sn, &cs);
    b = make_float2(r * cs, r * sn);
  }
}

// One CTA per item (grid-stride): symbols into shared memory, then each
// thread generates whole rows b of H (written out), accumulates
// y[t][b] = sum_u H[b][u] s[t][u] in registers and adds the noise.
__global__ void synth_kernel(uint64_t seed, int64_t n_items, int64_t item0, int B, int U, int T,
                             const __grid_constant__ ConstParams cp, const float* __restrict__ n0_dev,
                             int64_t n0_group, float n0, float2* __restrict__ H, float2* __restrict__ Y,
                             uint8_t* __restrict__ sym) {
  __shared__ float2 s_sym[MAX_T * 64];
  const float hs = sqrtf(0.5f / (float)B);
  for (int64_t n = blockIdx.x; n < n_items; n += gridDim.x) {
    const int64_t gn = item0 + n;  // global item index: the counter
    __syncthreads();
    for (int j = threadIdx.x; 4 * j < T * U; j += blockDim.x) {
      uint32_t x[4];
      philox_block(seed, gn, 1u, (uint32_t)j, x);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = 4 * j + q;
        if (e < T * U) {
          const int idx = (int)(((uint64_t)x[q] * (uint32_t)cp.M) >> 32);
          s_sym[e] = cp.syms[idx];
          if (sym) sym[n * T * U + e] = (uint8_t)idx;
        }
      }
    }
    __syncthreads();
    const float nv = n0_dev ? n0_dev[gn / n0_group] : n0;
    const float ns = sqrtf(0.5f * nv);
    float2* Hn = H + n * (int64_t)B * U;
    float2* Yn = Y + n * (int64_t)T * B;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      float2 acc[MAX_T];
#pragma unroll
      for (int t = 0; t < MAX_T; ++t) acc[t] = make_float2(0.f, 0.f);
      // entries b*U + u, two per Philox block (U even)
      for (int u = 0; u < U; u += 2) {
        uint32_t x[4];
        philox_block(seed, gn, 0u, (uint32_t)((b * U + u) >> 1), x);
        float2 h0, h1;
        box_muller2(x, hs, h0, h1);
        *reinterpret_cast<float4*>(Hn + b * U + u) = make_float4(h0.x, h0.y, h1.x, h1.y);
#pragma unroll
        for (int t = 0; t < MAX_T; ++t) {
          if (t < T) {
            c_fma(acc[t], h0, s_sym[t * U + u]);
            c_fma(acc[t], h1, s_sym[t * U + u + 1]);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < MAX_T; ++t) {
        if (t < T) {
          // noise entry t*B + b: block (t*B + b)/2, half (t*B + b)&1 (B even)
          const int e = t * B + b;
          uint32_t x[4];
          philox_block(seed, gn, 2u, (uint32_t)(e >> 1), x);
          float2 z0, z1;
          box_muller2(x, ns, z0, z1);
          Yn[e] = c_add(acc[t], (e & 1) ? z1 : z0);
        }
      }
    }
  }
}

}  // namespace dbp
