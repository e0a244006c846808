// philox.cu -- Alg. 1 step 1: an m x l matrix Omega of iid
// N(0,1) entries, here l = k (reading A3).  Counter-based Philox4x64-10
// (Salmon et al., SC'11) keyed by (seed, 0); raw block j uses counter
// (j+1, 0, 0, 0) and yields normals 4j..4j+3 by Box-Muller in fp64, rounded to
// fp32 (reading A6).  Normal n of the global N x k matrix is entry (n / k, n % k).
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"

namespace {

__device__ __forceinline__ void philox4x64_10(uint64_t x[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    const uint64_t hi0 = __umul64hi(M0, x[0]), lo0 = M0 * x[0];
    const uint64_t hi1 = __umul64hi(M1, x[2]), lo1 = M1 * x[2];
    const uint64_t y0 = hi1 ^ x[1] ^ k0, y2 = hi0 ^ x[3] ^ k1;
    x[0] = y0; x[1] = lo1; x[2] = y2; x[3] = lo0;
  }
}

__device__ __forceinline__ void normals4(uint64_t seed, int64_t j, float z[4]) {
  uint64_t x[4] = {(uint64_t)(j + 1), 0, 0, 0};
  philox4x64_10(x, seed, 0);
  const double two_pi = 6.283185307179586476925286766559;
  const double inv53 = 1.0 / 9007199254740992.0;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const double u0 = ((double)(x[2 * p] >> 11) + 0.5) * inv53;
    const double u1 = ((double)(x[2 * p + 1] >> 11) + 0.5) * inv53;
    const double r = sqrt(-2.0 * log(u0));
    z[2 * p] = (float)(r * cos(two_pi * u1));
    z[2 * p + 1] = (float)(r * sin(two_pi * u1));
  }
}

// Row-major: out[n] = normal n.
__global__ void k_gauss(uint64_t seed, int64_t total, float* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (4 * j >= total) return;
  float z[4];
  normals4(seed, j, z);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int64_t n = 4 * j + t;
    if (n < total) out[n] = z[t];
  }
}

// Panels: block i (global blk0 + i) gets out[(i*k + c)*b + m] = Omega[(blk0+i)*b + m][c].
// k % 4 == 0, so normals 4j..4j+3 share a row: a thread owns (m, c..c+3) and a warp
// covers 32 consecutive m, i.e. every store instruction writes one 128-byte line.
// out16 (3xF16 twin, instead of out): 2^exp Omega in the tw_off layout (common.cuh) of out.
__global__ void k_gauss_panel(uint64_t seed, int64_t blk0, int b, int k, float* __restrict__ out,
                              uint16_t* __restrict__ out16, float sc) {
  const int local = blockIdx.x * blockDim.x + threadIdx.x;   // (c/4) * b + m
  if (local >= b * (k / 4)) return;
  const int m = local % b, c = 4 * (local / b);
  const int64_t i = blockIdx.y;
  const int64_t r = (blk0 + i) * b + m;
  float z[4];
  normals4(seed, r * (k / 4) + c / 4, z);
  const int64_t o = (i * k + c) * b + m;
  if (out16) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float x = z[t] * sc;
      const __half h = __float2half_rn(x);
      const __half l = __float2half_rn(x - __half2float(h));
      uint16_t* o16 = out16 + tw_off(o + (int64_t)t * b);
      o16[0] = __half_as_ushort(h);
      o16[TW_LO] = __half_as_ushort(l);
    }
    return;
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) out[o + (int64_t)t * b] = z[t];
}

}  // namespace

cudaError_t launch_omega_panels(uint64_t seed, int blk0, int nb, int b, int k, float* out, cudaStream_t s,
                                int* launches, uint16_t* out16, int exp) {
  const int per = b * (k / 4);
  k_gauss_panel<<<dim3((per + 255) / 256, nb), 256, 0, s>>>(seed, blk0, b, k, out, out16, ldexpf(1.f, exp));
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_gaussian_rowmajor(uint64_t seed, int rows, int cols, float* out, cudaStream_t s, int* launches) {
  const int64_t total = (int64_t)rows * cols;
  const int64_t nblk = (total + 3) / 4;
  k_gauss<<<(unsigned)((nblk + 255) / 256), 256, 0, s>>>(seed, total, out);
  ++*launches;
  return cudaGetLastError();
}
