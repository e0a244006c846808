// finalize.cu -- Alg. 1 steps 5-6 epilogue and the Eq. 15 scale.
//
// Inputs per block: Vw_t = (B^T U~)^T and Uw_t = (S U~)^T (k x b, one row per
// singular triplet, unsorted).  sigma_j = ||B^T u~_j|| accumulated in fp64
// (the singular value of B for the eigenvector u~_j of B B^T), then the
// triplets are sorted non-increasing (ties by index), v_j = B^T u~_j / sigma_j,
// u_j = S u~_j, and the pair's sign is fixed so that the
// largest-|.| entry of u_j (first index on ties) is positive.
#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int NT = 256;

__global__ void __launch_bounds__(NT) k_colnorm(int b, const float* __restrict__ Vw_t, double* __restrict__ sig) {
  __shared__ double red[NT / 32];
  const int64_t row = blockIdx.x;               // blk*k + j
  const float* x = Vw_t + row * b;
  double acc = 0.0;
  for (int i = threadIdx.x; i < b; i += NT) {
    const double v = x[i];
    acc = fma(v, v, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    sig[row] = sqrt(s);
  }
}

// one CTA per block: rank of each sigma (descending, ties by index) -> perm, sigma_out
__global__ void k_rank(int k, const double* __restrict__ sig, int32_t* __restrict__ perm, float* __restrict__ sigma,
                       int32_t* status) {
  const int blk = blockIdx.x;
  const double* s = sig + (int64_t)blk * k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const double v = s[j];
    if (!isfinite(v)) hg_flag(status, HGS_NONFINITE);
    int r = 0;
    for (int l = 0; l < k; ++l) {
      const double w = s[l];
      r += (w > v) || (w == v && l < j);
    }
    perm[(int64_t)blk * k + r] = j;
    sigma[(int64_t)blk * k + r] = (float)v;
  }
}

// one CTA per (block, sorted index jj)
__global__ void __launch_bounds__(NT) k_rows(int b, int k, const float* __restrict__ Vw_t,
                                             const float* __restrict__ Uw_t, const int32_t* __restrict__ perm,
                                             const double* __restrict__ sig, float* __restrict__ Ut,
                                             float* __restrict__ Vt, int uv_bk, uint16_t* __restrict__ u16,
                                             float* __restrict__ vs_out) {
  __shared__ float bv[NT / 32];
  __shared__ int bi[NT / 32];
  const int blk = blockIdx.x / k, jj = blockIdx.x % k;
  const int j = perm[(int64_t)blk * k + jj];
  const int64_t src = ((int64_t)blk * k + j) * b, dst = ((int64_t)blk * k + jj) * b;
  const float* u = Uw_t + src;
  float best = -1.f;
  int arg = 0x7fffffff;
  for (int i = threadIdx.x; i < b; i += NT) {
    const float a = fabsf(u[i]);
    if (a > best) { best = a; arg = i; }        // i increases: first index kept on ties
  }
  for (int o = 16; o; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oi < arg)) { best = ob; arg = oi; }
  }
  if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = arg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w)
      if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) { bv[0] = bv[w]; bi[0] = bi[w]; }
  }
  __syncthreads();
  const float sgn = (u[bi[0]] < 0.f) ? -1.f : 1.f;
  const double sv = sig[(int64_t)blk * k + j];
  const double smax = sig[(int64_t)blk * k + perm[(int64_t)blk * k]];
  // v_j = B^T u_j / sigma_j; a zero (or noise-level) sigma_j of a rank-deficient block has no
  // defined v_j: write 0 instead of inf/NaN (the R1 apply flags such a sigma, k_inv_sigma)
  const float vs = (sv > 1e-7 * smax && sv > 0.0) ? (float)((double)sgn / sv) : 0.f;
  if (u16) {
    // hg_solve with the fused apply: U and V only feed that kernel -- write U's 3xF16 twin (unit vectors:
    // exponent 14, tw_off layout) and v_j's scale (the apply prep forms V's twin from Vw_t); no fp32 Ut / Vt
    if (threadIdx.x == 0) vs_out[(int64_t)blk * k + jj] = vs;
    for (int i = 4 * threadIdx.x; i < b; i += 4 * NT) {
      const float4 x = *reinterpret_cast<const float4*>(u + i);
      uint2 hv, lv;
      split4(x, sgn * 16384.f, hv, lv);
      uint16_t* o = u16 + tw_off(dst + i);
      *reinterpret_cast<uint2*>(o) = hv;
      *reinterpret_cast<uint2*>(o + TW_LO) = lv;
    }
    return;
  }
  const float* v = Vw_t + src;
  if (uv_bk) {   // HG_UV_BK: U, V [nb][b][k] (column jj of U_i, V_i)
    const int64_t ob = (int64_t)blk * b * k + jj;
    for (int i = threadIdx.x; i < b; i += NT) {
      Ut[ob + (int64_t)i * k] = sgn * u[i];
      Vt[ob + (int64_t)i * k] = v[i] * vs;
    }
    return;
  }
  for (int i = threadIdx.x; i < b; i += NT) {
    Ut[dst + i] = sgn * u[i];
    Vt[dst + i] = v[i] * vs;
  }
}

// sigma, rs: [nb][ld], the first k of each row used (ld > k: oversampled, truncated to rank k)
__global__ void k_inv_sigma(int nb, int k, int ld, const float* __restrict__ sigma, float scale,
                            float* __restrict__ rs, int32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * ld) return;
  const int64_t blk = i / ld;
  if (i % ld >= k) {
    rs[i] = 0.f;
    return;
  }
  const float s = sigma[i], s1 = sigma[blk * ld];
  if (!isfinite(s) || !(s > 1e-6f * s1)) {
    hg_flag(status, isfinite(s) ? HGS_SINGULAR_SIGMA : HGS_NONFINITE);
    rs[i] = 0.f;
    return;
  }
  rs[i] = scale / s;
}

// Reading R2: rs[i][j] = c sigma_j / ((1+mu) - sigma_j), the Woodbury
// weights of X_ii^-1 ~ I + U diag(sigma/((1+mu) - sigma)) U^T, times c = mu/(1+mu).
__global__ void k_woodbury_scale(int nb, int k, int ld, const float* __restrict__ sigma, float c, float opm,
                                 float* __restrict__ rs, int32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * ld) return;
  if (i % ld >= k) {
    rs[i] = 0.f;
    return;
  }
  const float s = sigma[i];
  const float d = opm - s;
  if (!isfinite(s) || !(d > 0.f)) {
    hg_flag(status, isfinite(s) ? HGS_SINGULAR_SIGMA : HGS_NONFINITE);
    rs[i] = 0.f;
    return;
  }
  rs[i] = c * s / d;
}

}  // namespace

cudaError_t launch_woodbury_scale(int nb, int k, int ld, const float* sigma, float c, float one_plus_mu, float* rs,
                                  int32_t* status, cudaStream_t s, int* launches) {
  const int64_t n = (int64_t)nb * ld;
  k_woodbury_scale<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nb, k, ld, sigma, c, one_plus_mu, rs, status);
  ++*launches;
  return cudaGetLastError();
}

// grid (nb, ceil(k/32)): a CTA normalises 32 columns of W_f and writes them as rows of Uk
__global__ void __launch_bounds__(NT) k_unit_columns_t(int k, const float* __restrict__ Wf, float* __restrict__ Uk) {
  __shared__ double part[NT / 32][32];
  __shared__ float inv[32];
  const int blk = blockIdx.x, j0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* W = Wf + (int64_t)blk * k * k;
  const int j = j0 + lane;
  double acc = 0.0;
  if (j < k)
    for (int r = w; r < k; r += NT / 32) {
      const double v = W[(int64_t)r * k + j];
      acc = fma(v, v, acc);
    }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    double s2 = 0.0;
    for (int i = 0; i < NT / 32; ++i) s2 += part[i][lane];
    inv[lane] = s2 > 0.0 ? (float)(1.0 / sqrt(s2)) : 0.f;
  }
  __syncthreads();
  float* U = Uk + (int64_t)blk * k * k;
  for (int jj = w; jj < 32 && j0 + jj < k; jj += NT / 32)
    for (int r = lane; r < k; r += 32) U[(int64_t)(j0 + jj) * k + r] = W[(int64_t)r * k + j0 + jj] * inv[jj];
}

cudaError_t launch_unit_columns_t(int nb, int k, const float* Wf, float* Uk, cudaStream_t s, int* launches) {
  k_unit_columns_t<<<dim3(nb, (k + 31) / 32), NT, 0, s>>>(k, Wf, Uk);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_finalize(int nb, int b, int k, const float* Vw_t, const float* Uw_t, float* Ut, float* sigma,
                            float* Vt, double* sig_raw, int32_t* perm, int32_t* status, cudaStream_t s,
                            int* launches, bool uv_bk, uint16_t* u16, float* vs_out) {
  k_colnorm<<<nb * k, NT, 0, s>>>(b, Vw_t, sig_raw);
  k_rank<<<nb, 256, 0, s>>>(k, sig_raw, perm, sigma, status);
  k_rows<<<nb * k, NT, 0, s>>>(b, k, Vw_t, Uw_t, perm, sig_raw, Ut, Vt, uv_bk ? 1 : 0, u16, vs_out);
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_inv_sigma(int nb, int k, int ld, const float* sigma, float scale, float* rs, int32_t* status,
                             cudaStream_t s, int* launches) {
  const int64_t n = (int64_t)nb * ld;
  k_inv_sigma<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nb, k, ld, sigma, scale, rs, status);
  ++*launches;
  return cudaGetLastError();
}
