// schur.cu -- NEXT-1: one level of the 2x2 Schur-complement inverse of
// PAPER.md:127-154 (Eqs. 11-14) over super-blocks of two adjacent diagonal blocks; the
// orchestration (GEMMs on the tcgen05 path, the rSVDs) is in abi.cu (hg_solve_schur).  This file
// holds the pieces that are not GEMMs or rSVDs:
//   k_theta_offblock  Eq. 1 off-diagonal block Theta_{2s,2s+1} from the sorted CSC of H
//   k_scale_rows      W_t[j][:] = d_j U_t[j][:]        (U diag(d) U^T = W_t^T U_t)
//   k_add_identity    A += I                            (Woodbury: I + U diag(d) U^T)
//   k_symmetrize      K = (K + K^T) / 2                 (Schur Gram K_Z, bitwise symmetric input
//                                                        for the rSVD, reading A12)
//   k_axpby           F = c (P + g Q)
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int OFF_ROWS = 8;   // rows (warps) per CTA of the off-diagonal assembly

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int lo, int hi, int x) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// grid (ns, b / OFF_ROWS): warp = row u of block 2s; for every hyperedge e of u (ascending e, the
// caller's CSR order) the members of e inside block 2s+1 (a contiguous range of the vertex-sorted
// CSC member list, found by binary search) get w_e/delta(e) added to a b-wide row accumulator in
// shared memory; entry (u, v) therefore sums its common edges in ascending e order (deterministic).
__global__ void __launch_bounds__(OFF_ROWS * 32) k_theta_offblock(int b, const int64_t* __restrict__ row_ptr,
                                                                  const int32_t* __restrict__ col,
                                                                  const int32_t* __restrict__ col_ptr,
                                                                  const int32_t* __restrict__ csc,
                                                                  const float* __restrict__ eval,
                                                                  const float* __restrict__ dvr,
                                                                  float* __restrict__ out) {
  extern __shared__ float acc[];   // [OFF_ROWS][b]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = blockIdx.x;
  const int ul = blockIdx.y * OFF_ROWS + warp;
  if (ul >= b) return;
  const int64_t u = (int64_t)(2 * s) * b + ul;
  const int v0 = (2 * s + 1) * b;
  float* a = acc + (size_t)warp * b;
  for (int j = lane; j < b; j += 32) a[j] = 0.f;
  __syncwarp();
  for (int64_t p = row_ptr[u]; p < row_ptr[u + 1]; ++p) {
    const int e = col[p];
    const float val = eval[e];
    const int lo = col_ptr[e], hi = col_ptr[e + 1];
    const int first = lower_bound_i32(csc, lo, hi, v0);
    const int last = lower_bound_i32(csc, first, hi, v0 + b);
    for (int q = first + lane; q < last; q += 32) a[csc[q] - v0] += val;
    __syncwarp();
  }
  const float ru = dvr[u];
  float* o = out + ((size_t)s * b + ul) * b;
  for (int j = lane; j < b; j += 32) o[j] = a[j] * ru * dvr[v0 + j];
}

__global__ void k_scale_rows(int64_t n, int k, int b, const float* __restrict__ d, const float* __restrict__ Ut,
                             float* __restrict__ Wt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / b;   // (block, j) flattened: d index = row
    Wt[i] = d[row] * Ut[i];
  }
}

__global__ void k_add_identity(int nb, int b, float* __restrict__ A) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * b) return;
  const int64_t blk = i / b, r = i % b;
  A[(blk * b + r) * b + r] += 1.f;
}

// K = (K + K^T)/2 per b x b block: CTA per pair of mirrored 32 x 32 tiles (ti <= tj), both staged in
// shared memory so every global access is a coalesced row segment
__global__ void __launch_bounds__(256) k_symmetrize(int b, float* __restrict__ K) {
  __shared__ float A[32][33], B[32][33];
  const int ti = blockIdx.x, tj = blockIdx.y;
  if (ti > tj) return;
  float* Kb = K + (size_t)blockIdx.z * b * b;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int gi = ti * 32 + r, gj = tj * 32 + r;
    A[r][tx] = (gi < b && tj * 32 + tx < b) ? Kb[(size_t)gi * b + tj * 32 + tx] : 0.f;   // tile (ti, tj)
    B[r][tx] = (gj < b && ti * 32 + tx < b) ? Kb[(size_t)gj * b + ti * 32 + tx] : 0.f;   // tile (tj, ti)
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int gi = ti * 32 + r, gj = tj * 32 + r;
    const float v = 0.5f * (A[r][tx] + B[tx][r]);      // (ti*32 + r, tj*32 + tx)
    const float u = 0.5f * (B[r][tx] + A[tx][r]);      // (tj*32 + r, ti*32 + tx)
    if (gi < b && tj * 32 + tx < b) Kb[(size_t)gi * b + tj * 32 + tx] = v;
    if (gj < b && ti * 32 + tx < b) Kb[(size_t)gj * b + ti * 32 + tx] = u;
  }
}

// F_s = c (P_s + g Q_s) for super-block s: rows [s * pitch_f, + b*T) of F, P, Q at their pitches
__global__ void k_axpby(int ns, int64_t len, float c, float g, const float* __restrict__ P, int64_t pp,
                        const float* __restrict__ Q, int64_t pq, float* __restrict__ F, int64_t pf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)ns * len;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / len, j = i % len;
    F[s * pf + j] = c * fmaf(g, Q[s * pq + j], P[s * pp + j]);
  }
}

// Node of the nested tessellation (2h x 2h, row-major) from its quadrants: top-left TL, bottom-right
// BR, top-right TR and bottom-left TR^T (the node inverse and the node Theta are symmetric).
__global__ void k_place_node(int nn, int h, const float* __restrict__ TL, int64_t sTL, const float* __restrict__ BR,
                             int64_t sBR, const float* __restrict__ TR, int64_t sTR, float* __restrict__ out) {
  const int64_t n = 2 * (int64_t)h, per = n * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn * per; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / per, rc = i % per, r = rc / n, c = rc % n;
    float v;
    if (r < h && c < h) v = TL[s * sTL + r * h + c];
    else if (r >= h && c >= h) v = BR[s * sBR + (r - h) * h + (c - h)];
    else if (r < h) v = TR[s * sTR + r * h + (c - h)];
    else v = TR[s * sTR + c * h + (r - h)];
    out[i] = v;
  }
}

}  // namespace

cudaError_t launch_theta_offblock(int ns, int b, const int64_t* row_ptr, const int32_t* col, const int32_t* col_ptr,
                                  const int32_t* csc, const float* eval, const float* dvr, float* out, cudaStream_t s,
                                  int* launches) {
  const size_t smem = (size_t)OFF_ROWS * b * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_theta_offblock, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid(ns, (b + OFF_ROWS - 1) / OFF_ROWS);
  k_theta_offblock<<<grid, OFF_ROWS * 32, smem, s>>>(b, row_ptr, col, col_ptr, csc, eval, dvr, out);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(int nb, int k, int b, const float* d, const float* Ut, float* Wt, cudaStream_t s,
                              int* launches) {
  const int64_t n = (int64_t)nb * k * b;
  k_scale_rows<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(n, k, b, d, Ut, Wt);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_add_identity(int nb, int b, float* A, cudaStream_t s, int* launches) {
  const int64_t n = (int64_t)nb * b;
  k_add_identity<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nb, b, A);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_symmetrize(int nb, int b, float* K, cudaStream_t s, int* launches) {
  const int nt = (b + 31) / 32;
  k_symmetrize<<<dim3(nt, nt, nb), 256, 0, s>>>(b, K);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_axpby(int ns, int64_t len, float c, float g, const float* P, int64_t pp, const float* Q, int64_t pq,
                         float* F, int64_t pf, cudaStream_t s, int* launches) {
  const int64_t n = (int64_t)ns * len;
  k_axpby<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(ns, len, c, g, P, pp, Q, pq, F, pf);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_place_node(int nn, int h, const float* TL, int64_t sTL, const float* BR, int64_t sBR, const float* TR,
                              int64_t sTR, float* out, cudaStream_t s, int* launches) {
  const int64_t n = (int64_t)nn * 4 * h * h;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 32);
  k_place_node<<<grid, 256, 0, s>>>(nn, h, TL, sTL, BR, sBR, TR, sTR, out);
  ++*launches;
  return cudaGetLastError();
}
