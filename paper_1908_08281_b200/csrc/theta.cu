// theta.cu -- degrees and diagonal-block assembly of X = I - Theta/(1+mu).
//
//   delta(e) = sum_v H(v,e),  delta(v) = sum_e w(e) H(v,e)
//   Theta_ii[u][v] = r_u r_v sum_{e ni u,v} w_e/delta(e),  r = delta(v)^-1/2   (Eq. 1)
//   X_ii = I - Theta_ii/(1+mu)
//
// Assembly: one CTA per (block, 128-row tile U, 64-column tile V).  The CTA
// hashes V's incidences (edge -> members of V, in shared memory); the thread
// owning row u walks u's CSR row in ascending edge order and adds w_e/delta(e)
// to acc[u][v] for every v of V sharing e.  Every (u,v) sum is therefore taken
// over the common edges in ascending edge order -- the same sequence for (v,u)
// -- so the written blocks are bitwise symmetric and run-to-run deterministic
// with no atomics on values.  Traffic: the b x b block is written once
// (4 b^2 bytes per block; HBM-write bound); CSR reads are ~2 nnz per tile row.
#include "common.cuh"
#include "kernels.cuh"

namespace {

__global__ void k_edge_count(int64_t nnz, const int32_t* __restrict__ col, int32_t* __restrict__ de) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&de[col[p]], 1);
}

__global__ void k_edge_val(int E, const int32_t* __restrict__ de, const float* __restrict__ w,
                           float* __restrict__ val, int32_t* status) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int c = de[e];
  if (c == 0) {
    hg_flag(status, HGS_EMPTY_EDGE);
    val[e] = 0.f;
    return;
  }
  float v = w[e] / (float)c;
  if (!isfinite(v)) hg_flag(status, HGS_NONFINITE);
  val[e] = v;
}

__global__ void k_vertex_deg(int N, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                             const float* __restrict__ w, float* __restrict__ dvr, int32_t* status) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N) return;
  float s = 0.f;
  for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) s += w[col[p]];
  if (!(s > 0.f)) {
    hg_flag(status, HGS_ISOLATED_VERTEX);
    dvr[v] = 0.f;
    return;
  }
  dvr[v] = 1.0f / sqrtf(s);
}

constexpr int TU = 128, TV = 64, NT = 256, HCAP = 4096, LCAP = 4096;

struct AsmSmem {
  float acc[TU][TV + 1];
  int hkey[HCAP];
  int hcnt[HCAP];
  int hoff[HCAP];
  unsigned short list[LCAP];
  int64_t vptr[TV + 1];
  int wsum[NT / 32];
};

__device__ __forceinline__ int hslot(int e) { return (int)(((unsigned)e * 2654435761u) >> 20) & (HCAP - 1); }

__global__ void __launch_bounds__(NT) k_assemble(int b, const int64_t* __restrict__ row_ptr,
                                                 const int32_t* __restrict__ col,
                                                 const float* __restrict__ eval, const float* __restrict__ dvr,
                                                 float inv1pmu, int raw, float* __restrict__ blocks) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  AsmSmem& S = *reinterpret_cast<AsmSmem*>(smem_raw);
  const int t = threadIdx.x;
  const int blk = blockIdx.z, u0 = blockIdx.y * TU, v0 = blockIdx.x * TV;
  const int64_t base = (int64_t)blk * b;
  const int nv = min(TV, b - v0), nu = min(TU, b - u0);

  for (int i = t; i < TU * (TV + 1); i += NT) (&S.acc[0][0])[i] = 0.f;
  for (int i = t; i <= nv; i += NT) S.vptr[i] = row_ptr[base + v0 + i];
  __syncthreads();
  const int64_t p_begin = S.vptr[0], p_end = S.vptr[nv];

  const int ul = t % TU, half = t / TU;   // thread owns row u0+ul, columns [32*half, 32*half+32)
  const bool urow = ul < nu;
  int64_t up0 = 0, up1 = 0;
  if (urow) { up0 = row_ptr[base + u0 + ul]; up1 = row_ptr[base + u0 + ul + 1]; }

  for (int64_t c0 = p_begin; c0 < p_end; c0 += LCAP) {       // chunks of V's incidences, in order
    const int cnt = (int)((p_end - c0) < LCAP ? (p_end - c0) : LCAP);
    for (int i = t; i < HCAP; i += NT) { S.hkey[i] = -1; S.hcnt[i] = 0; }
    __syncthreads();
    for (int i = t; i < cnt; i += NT) {
      const int e = col[c0 + i];
      int s = hslot(e);
      for (;;) {
        int old = atomicCAS(&S.hkey[s], -1, e);
        if (old == -1 || old == e) { atomicAdd(&S.hcnt[s], 1); break; }
        s = (s + 1) & (HCAP - 1);
      }
    }
    __syncthreads();
    // exclusive scan of hcnt -> hoff (NT threads x HCAP/NT entries)
    {
      constexpr int PER = HCAP / NT;
      int loc[PER], run = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) { loc[j] = run; run += S.hcnt[t * PER + j]; }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((t & 31) >= o) incl += y;
      }
      if ((t & 31) == 31) S.wsum[t >> 5] = incl;
      __syncthreads();
      int wbase = 0;
      for (int w = 0; w < (t >> 5); ++w) wbase += S.wsum[w];
      const int excl = wbase + incl - run;
#pragma unroll
      for (int j = 0; j < PER; ++j) S.hoff[t * PER + j] = excl + loc[j];
    }
    __syncthreads();
    for (int i = t; i < HCAP; i += NT) S.hcnt[i] = 0;
    __syncthreads();
    for (int i = t; i < cnt; i += NT) {
      const int64_t p = c0 + i;
      const int e = col[p];
      int lo = 0, hi = nv;                                      // v_local: vptr[lo] <= p < vptr[lo+1]
      while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (S.vptr[mid] <= p) lo = mid; else hi = mid; }
      int s = hslot(e);
      while (S.hkey[s] != e) s = (s + 1) & (HCAP - 1);
      const int pos = atomicAdd(&S.hcnt[s], 1);
      S.list[S.hoff[s] + pos] = (unsigned short)lo;
    }
    __syncthreads();
    if (urow) {
      for (int64_t p = up0; p < up1; ++p) {                   // ascending edge order
        const int e = col[p];
        int s = hslot(e);
        int key;
        while ((key = S.hkey[s]) != e && key != -1) s = (s + 1) & (HCAP - 1);
        if (key != e) continue;
        const float val = eval[e];
        const int o = S.hoff[s], n = S.hcnt[s];
        for (int j = 0; j < n; ++j) {
          const int vl = S.list[o + j];
          if ((vl >> 5) == half) S.acc[ul][vl] += val;
        }
      }
    }
    __syncthreads();
  }
  // X_ii[u][v] = delta_uv - (r_u r_v) acc / (1+mu), coalesced rows of TV
  float* out = blocks + (int64_t)blk * b * b;
  for (int i = t; i < nu * TV; i += NT) {
    const int r = i / TV, c = i % TV;
    if (c >= nv) continue;
    const int u = u0 + r, v = v0 + c;
    const float th = (dvr[base + u] * dvr[base + v]) * S.acc[r][c];
    out[(int64_t)u * b + v] = raw ? th : ((u == v ? 1.0f : 0.0f) - th * inv1pmu);
  }
}

}  // namespace

cudaError_t launch_degrees(int N, int E, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                               const float* w, int32_t* de_cnt, float* edge_val, float* dv_rsqrt, int32_t* status,
                               cudaStream_t s, int* launches) {
  cudaError_t e = cudaMemsetAsync(de_cnt, 0, sizeof(int32_t) * (size_t)E, s);
  if (e != cudaSuccess) return e;
  if (nnz > 0) {
    int grid = (int)((nnz + 255) / 256 < 148 * 16 ? (nnz + 255) / 256 : 148 * 16);
    k_edge_count<<<grid, 256, 0, s>>>(nnz, col_idx, de_cnt);
    ++*launches;
  }
  k_edge_val<<<(E + 255) / 256, 256, 0, s>>>(E, de_cnt, w, edge_val, status);
  k_vertex_deg<<<(N + 255) / 256, 256, 0, s>>>(N, row_ptr, col_idx, w, dv_rsqrt, status);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_assemble(int nb, int b, const int64_t* row_ptr, const int32_t* col_idx, const float* edge_val,
                            const float* dv_rsqrt, float mu, bool raw_theta, float* blocks, cudaStream_t s,
                            int* launches) {
  static bool attr = false;
  const int smem = (int)sizeof(AsmSmem);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((b + TV - 1) / TV, (b + TU - 1) / TU, nb);
  k_assemble<<<grid, NT, smem, s>>>(b, row_ptr, col_idx, edge_val, dv_rsqrt, 1.0f / (1.0f + mu), raw_theta ? 1 : 0,
                                    blocks);
  ++*launches;
  return cudaGetLastError();
}
