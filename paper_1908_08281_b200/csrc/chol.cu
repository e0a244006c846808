// chol.cu -- the small k x k factorizations of CholeskyQR (Alg. 1 "compute its
// QR factorization"; CholeskyQR2 per north_star).
//
// Input: a Gram matrix G = Y^T Y (k x k, from the tensor-core GEMM).
// Output: L (lower, G = L L^T, so R = L^T) and Linv = L^-1 (lower), row-major
// with explicit zeros above the diagonal; the panel step then forms
// Q = Y R^-1 = Y Linv^T on the tensor cores.
//
// Second CholeskyQR pass: its Gram is I + E with max|E| tiny.  Then
//   L = I + low(E) + O(|E|^2),  Linv = I - low(E) + O(|E|^2),
// low(E) = strict lower part of E plus half its diagonal.  When max|E| <= 1e-4
// the O(|E|^2) <= 1e-8 remainder is below fp32 resolution and the factor is
// written by this first-order formula; otherwise the
// full factorization runs.  A pivot <= 0 flags HG_ST_CHOL_BREAKDOWN.
//
// One CTA (1024 threads) per block; the working matrix lives in shared memory
// for k <= 128 and in an L2-resident global scratch slab otherwise.
#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int NT = 1024;
constexpr float NEAR_ID_TOL = 1e-4f;

__global__ void __launch_bounds__(NT) k_cholinv(int k, const float* __restrict__ G, float* __restrict__ Lout,
                                                float* __restrict__ Linv, float* __restrict__ work, int smem_mat,
                                                int32_t* status) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red[NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t kk = (int64_t)k * k;
  const int64_t off = (int64_t)blockIdx.x * kk;
  float* A = smem_mat ? sm : work + off;
  float* colbuf = smem_mat ? sm + kk : sm;   // [32 warps][k]
  const float* Gb = G + off;
  float* Lb = Lout ? Lout + off : nullptr;
  float* Ib = Linv + off;

  // load + distance from identity
  float emax = 0.f;
  for (int64_t i = t; i < kk; i += NT) {
    const float g = Gb[i];
    A[i] = g;
    const int r = (int)(i / k), c = (int)(i % k);
    const float e = fabsf(g - (r == c ? 1.f : 0.f));
    emax = fmaxf(emax, isfinite(g) ? e : INFINITY);
  }
  for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  if (lane == 0) red[warp] = emax;
  __syncthreads();
  if (t < 32) {
    float v = red[t];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (t == 0) red[0] = v;
  }
  __syncthreads();
  const float E = red[0];
  if (!isfinite(E)) {
    if (t == 0) hg_flag(status, HGS_NONFINITE);
  }
  if (E <= NEAR_ID_TOL) {
    for (int64_t i = t; i < kk; i += NT) {
      const int r = (int)(i / k), c = (int)(i % k);
      float l, li;
      if (c > r) { l = 0.f; li = 0.f; }
      else if (c == r) { const float e = 0.5f * (A[i] - 1.f); l = 1.f + e; li = 1.f - e; }
      else { l = A[i]; li = -A[i]; }
      if (Lb) Lb[i] = l;
      Ib[i] = li;
    }
    return;
  }
  // ---- right-looking Cholesky, lower triangle of A
  for (int j = 0; j < k; ++j) {
    __syncthreads();
    float d = A[(int64_t)j * k + j];
    if (!(d > 0.f) || !isfinite(d)) {
      if (t == 0) hg_flag(status, HGS_CHOL_BREAKDOWN);
      d = 1.f;
    }
    const float s = sqrtf(d), inv = 1.0f / s;
    for (int i = j + 1 + t; i < k; i += NT) A[(int64_t)i * k + j] *= inv;
    __syncthreads();
    if (t == 0) A[(int64_t)j * k + j] = s;
    const int n = k - j - 1;
    for (int idx = t; idx < n * n; idx += NT) {
      const int i = j + 1 + idx / n, l = j + 1 + idx % n;
      if (l <= i) A[(int64_t)i * k + l] -= A[(int64_t)i * k + j] * A[(int64_t)l * k + j];
    }
  }
  __syncthreads();
  if (Lb)
    for (int64_t i = t; i < kk; i += NT) {
      const int r = (int)(i / k), c = (int)(i % k);
      Lb[i] = (c <= r) ? A[i] : 0.f;
    }
  // ---- Linv = L^-1 column by column (forward substitution), one warp per column
  float* x = colbuf + (int64_t)warp * k;
  for (int c = warp; c < k; c += NT / 32) {
    if (lane == 0) x[c] = 1.0f / A[(int64_t)c * k + c];
    __syncwarp();
    for (int i = c + 1; i < k; ++i) {
      float acc = 0.f;
      for (int j = c + lane; j < i; j += 32) acc = fmaf(A[(int64_t)i * k + j], x[j], acc);
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) x[i] = -acc / A[(int64_t)i * k + i];
      __syncwarp();
    }
    for (int i = lane; i < k; i += 32) Ib[(int64_t)i * k + c] = (i >= c) ? x[i] : 0.f;
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_cholinv(int nb, int k, const float* G, float* L, float* Linv, float* work, int32_t* status,
                           cudaStream_t s, int* launches) {
  const bool smem_mat = k <= 128;
  const size_t smem = ((smem_mat ? (size_t)k * k : 0) + (size_t)(NT / 32) * k) * sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_cholinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  k_cholinv<<<nb, NT, smem, s>>>(k, G, L, Linv, work, smem_mat ? 1 : 0, status);
  ++*launches;
  return cudaGetLastError();
}
