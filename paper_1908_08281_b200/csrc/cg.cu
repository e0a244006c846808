// cg.cu -- the paper's second approach: conjugate gradient on Eq. 5,
//   X f = theta/(1+theta) y,   X = I - Theta/(1+theta),   Theta = Dv^-1/2 H W De^-1 H^T Dv^-1/2
// (Eq. 1, Eq. 5, Eqs. 16-20), one independent CG
// per right-hand-side column of the N x T tag matrix.
//
// X is never formed: every iteration applies it matrix-free through the incidence H in two
// sparse gathers (B200 design):
//   edge phase    Q[e]  = (w_e/delta(e)) sum_{v in e} r_v P[v]          (H^T, CSC member lists)
//   vertex phase  XP[v] = P[v] - r_v/(1+theta) sum_{e ni v} Q[e]          (H, the caller's CSR)
// with r = delta(v)^-1/2.  Rows of P, Q, ... are column SLICES of TS = 4*LPR fp32 values (one
// float4 per lane of an LPR-lane group), stored slice-major [ns][rows][TS] so that a gathered
// row is one contiguous, aligned 128/256/512-byte run, and the grid's slowest dimension is the
// slice: the CTAs resident at any time gather from one slice of P (or Q), which stays in L2.
//
// Determinism: the CSC member lists are sorted by vertex (atomics only decide the fill order,
// the sort fixes it), edges with more than CH members are summed in CH-member chunks whose
// partials are added in chunk order, and every dot product is a fixed-order per-CTA partial
// followed by a fixed-order fp64 sum.  Results are bitwise reproducible run to run.
//
// Iteration control: per column, active while ||r|| > tol ||r_0|| and fewer than max_iter
// iterations were taken (reading C2, as oracle/hg_oracle.c:or_cg_solve).  In graph
// mode the iteration body sits in a CUDA-graph WHILE node whose condition the control kernel
// sets from the device (no host round trip); enqueued directly, max_iter bodies are enqueued
// and every kernel returns at once after the control kernel has cleared `running`.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int CH = 128;     // members per edge work item
constexpr int NT = 256;     // threads per CTA (8 warps)
constexpr int NW = NT / 32;
constexpr int VPG = 16;     // consecutive rows per lane group in the row kernels
constexpr int SORT_SMALL = 64;          // edges up to this size: warp rank sort
constexpr int BM_WORDS = 8192;          // bitmap chunk: 262144 vertex ids (32 KB)

__device__ __forceinline__ float4 f4_fma(float a, float4 x, float4 y) {
  return make_float4(fmaf(a, x.x, y.x), fmaf(a, x.y, y.y), fmaf(a, x.z, y.z), fmaf(a, x.w, y.w));
}

// ------------------------------------------------------------------ setup: CSC of H
// One CTA, exclusive scans over e of: delta(e) (CSC pointers), number of CH-chunks (work
// items), chunks of multi-chunk edges (partial slots), multi-chunk edge flag (big-edge list).
__global__ void __launch_bounds__(1024) k_cg_scan(int E, const int32_t* __restrict__ de, int32_t* __restrict__ col_ptr,
                                                  int32_t* __restrict__ item_ptr, int32_t* __restrict__ slot_ptr,
                                                  int32_t* __restrict__ big_ptr, int32_t* __restrict__ totals) {
  __shared__ int4 wsum[32];
  __shared__ int4 carry;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  if (t == 0) carry = make_int4(0, 0, 0, 0);
  __syncthreads();
  for (int base = 0; base < E; base += 1024) {
    const int e = base + t;
    int4 v = make_int4(0, 0, 0, 0);
    if (e < E) {
      const int n = de[e];
      const int nc = (n + CH - 1) / CH;
      v = make_int4(n, nc, nc > 1 ? nc : 0, nc > 1 ? 1 : 0);
    }
    int4 x = v;   // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(~0u, x.x, o), b = __shfl_up_sync(~0u, x.y, o);
      int c = __shfl_up_sync(~0u, x.z, o), d = __shfl_up_sync(~0u, x.w, o);
      if (lane >= o) { x.x += a; x.y += b; x.z += c; x.w += d; }
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int4 s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int a = __shfl_up_sync(~0u, s.x, o), b = __shfl_up_sync(~0u, s.y, o);
        int c = __shfl_up_sync(~0u, s.z, o), d = __shfl_up_sync(~0u, s.w, o);
        if (lane >= o) { s.x += a; s.y += b; s.z += c; s.w += d; }
      }
      wsum[lane] = s;   // inclusive over warps
    }
    __syncthreads();
    int4 pre = carry;
    if (wid > 0) { int4 w = wsum[wid - 1]; pre.x += w.x; pre.y += w.y; pre.z += w.z; pre.w += w.w; }
    if (e < E) {
      col_ptr[e] = pre.x + x.x - v.x;
      item_ptr[e] = pre.y + x.y - v.y;
      slot_ptr[e] = pre.z + x.z - v.z;
      big_ptr[e] = pre.w + x.w - v.w;
    }
    __syncthreads();
    if (t == 0) {
      int4 w = wsum[31];
      carry = make_int4(carry.x + w.x, carry.y + w.y, carry.z + w.z, carry.w + w.w);
    }
    __syncthreads();
  }
  if (t == 0) {
    col_ptr[E] = carry.x;
    totals[0] = carry.y;   // work items
    totals[1] = carry.w;   // multi-chunk edges
    totals[2] = carry.z;   // partial slots
  }
}

// csc_tmp[col_ptr[e] + i] = members of e in arbitrary order (the sort below fixes it)
__global__ void k_cg_fill(int N, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                          const int32_t* __restrict__ col_ptr, int32_t* __restrict__ cursor,
                          int32_t* __restrict__ csc_tmp) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x)
    for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
      const int e = col[p];
      csc_tmp[col_ptr[e] + atomicAdd(&cursor[e], 1)] = v;
    }
}

// Edges with <= SORT_SMALL members: one warp, rank = number of smaller members (ids are unique).
__global__ void k_cg_sort_small(int E, const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ tmp,
                                int32_t* __restrict__ csc) {
  const int lane = threadIdx.x & 31;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < E; e += (gridDim.x * blockDim.x) >> 5) {
    const int s = col_ptr[e], n = col_ptr[e + 1] - s;
    if (n > SORT_SMALL) continue;
    const int a = lane < n ? tmp[s + lane] : INT_MAX;
    const int b = lane + 32 < n ? tmp[s + lane + 32] : INT_MAX;
    int ra = 0, rb = 0;
    for (int j = 0; j < n; ++j) {
      const int x = __shfl_sync(~0u, j < 32 ? a : b, j & 31);
      ra += x < a;
      rb += x < b;
    }
    if (lane < n) csc[s + ra] = a;
    if (lane + 32 < n) csc[s + rb] = b;
  }
}

// Edges with > SORT_SMALL members: one CTA, members marked in a shared bitmap per chunk of
// 262144 vertex ids and written out in ascending order (a counting sort over the ids).
__global__ void __launch_bounds__(NT) k_cg_sort_big(int N, int E, const int32_t* __restrict__ col_ptr,
                                                    const int32_t* __restrict__ tmp, int32_t* __restrict__ csc) {
  __shared__ uint32_t bm[BM_WORDS];
  __shared__ int wsum[NW];
  __shared__ int s_base;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int WPT = BM_WORDS / NT;   // 32 consecutive words per thread
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const int s = col_ptr[e], n = col_ptr[e + 1] - s;
    if (n <= SORT_SMALL) continue;
    if (t == 0) s_base = 0;
    const int nchunks = (N + BM_WORDS * 32 - 1) / (BM_WORDS * 32);
    for (int c = 0; c < nchunks; ++c) {
      for (int i = t; i < BM_WORDS; i += NT) bm[i] = 0u;
      __syncthreads();
      for (int j = t; j < n; j += NT) {
        const int v = tmp[s + j];
        if ((v >> 18) == c) atomicOr(&bm[(v & 0x3ffff) >> 5], 1u << (v & 31));
      }
      __syncthreads();
      int cnt = 0;
      for (int i = 0; i < WPT; ++i) cnt += __popc(bm[t * WPT + i]);
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(~0u, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wid] = x;
      __syncthreads();
      int pre = s_base;
      for (int w = 0; w < wid; ++w) pre += wsum[w];
      pre += x - cnt;
      for (int i = 0; i < WPT; ++i) {
        uint32_t bits = bm[t * WPT + i];
        while (bits) {
          const int bpos = __ffs(bits) - 1;
          bits &= bits - 1;
          csc[s + pre++] = (c << 18) + (t * WPT + i) * 32 + bpos;
        }
      }
      __syncthreads();
      if (t == 0) {
        int tot = 0;
        for (int w = 0; w < NW; ++w) tot += wsum[w];
        s_base += tot;
      }
      __syncthreads();
    }
  }
}

// Work items: edge e's members [start, end) in chunks of CH; slot >= 0 for multi-chunk edges.
__global__ void k_cg_items(int E, const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ item_ptr,
                           const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ big_ptr,
                           int4* __restrict__ items, int4* __restrict__ bigs) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int s = col_ptr[e], t = col_ptr[e + 1], nc = (t - s + CH - 1) / CH;
    for (int j = 0; j < nc; ++j)
      items[item_ptr[e] + j] = make_int4(e, s + j * CH, min(s + (j + 1) * CH, t), nc > 1 ? slot_ptr[e] + j : -1);
    if (nc > 1) bigs[big_ptr[e]] = make_int4(e, slot_ptr[e], nc, 0);
  }
}

// ------------------------------------------------------------------ iteration kernels
struct CgDev {
  int N, E, T, ns, nparts;   // nparts = CTAs along rows of the row kernels (dot partials)
  float mu_c;                // theta/(1+theta)
  float inv1pmu;             // 1/(1+theta)
  float tol;
  int max_iter;
  const int64_t* row_ptr;
  const int32_t* col;
  const float* eval;         // w_e/delta(e)
  const float* dvr;          // delta(v)^-1/2
  const int32_t* csc;
  const int4* items;
  const int4* bigs;
  const int32_t* totals;     // [0] items, [1] big edges, [2] slots
  float *P, *R, *F, *XP, *Q, *part, *red;
  double *rr, *rr0;
  float *alpha, *beta;
  int32_t *active, *iters;
  int32_t* ctl;              // [0] running, [1] iteration, [2..] active count per iteration
  int32_t* status;
};

__device__ __forceinline__ bool cg_stopped(const CgDev& d) { return *(volatile const int32_t*)d.ctl == 0; }

// Q = edge phase (see header).  One LPR-lane group per work item; grid (items, slices).
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_edge(CgDev d) {
  if (cg_stopped(d)) return;
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const unsigned gmask = (LPR == 32) ? ~0u : (((1u << LPR) - 1u) << (grp * LPR));
  const int item = (blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp;
  if (item >= d.totals[0]) return;
  const int4 it = d.items[item];
  const int s = blockIdx.y;
  const float* P = d.P + (size_t)s * d.N * TS + 4 * gl;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = it.y; base < it.z; base += LPR) {
    const int j = base + gl;
    const int myv = j < it.z ? d.csc[j] : 0;
    const float myr = j < it.z ? d.dvr[myv] : 0.f;
    const int cnt = min(LPR, it.z - base);
    for (int u0 = 0; u0 < cnt; u0 += 8) {
      float4 x[8];
      float r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int src = (u0 + u) & (LPR - 1);
        const int v = __shfl_sync(gmask, myv, src, LPR);
        r[u] = __shfl_sync(gmask, myr, src, LPR);
        x[u] = (u0 + u < cnt) ? __ldg(reinterpret_cast<const float4*>(P + (size_t)v * TS))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = f4_fma(r[u], x[u], acc);
    }
  }
  float4* out;
  if (it.w < 0) {
    const float ev = d.eval[it.x];
    acc = make_float4(acc.x * ev, acc.y * ev, acc.z * ev, acc.w * ev);
    out = reinterpret_cast<float4*>(d.Q + ((size_t)s * d.E + it.x) * TS + 4 * gl);
  } else {
    const int nslots = d.totals[2];
    out = reinterpret_cast<float4*>(d.part + ((size_t)s * nslots + it.w) * TS + 4 * gl);
  }
  *out = acc;
}

// Multi-chunk edges: Q[e] = eval_e * sum of the chunk partials in chunk order.
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_edge_reduce(CgDev d) {
  if (cg_stopped(d)) return;
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const int bi = (blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp;
  if (bi >= d.totals[1]) return;
  const int4 b = d.bigs[bi];
  const int s = blockIdx.y, nslots = d.totals[2];
  const float4* part = reinterpret_cast<const float4*>(d.part + ((size_t)s * nslots + b.y) * TS + 4 * gl);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < b.z; ++j) {
    const float4 x = part[(size_t)j * LPR];
    acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
  }
  const float ev = d.eval[b.x];
  *reinterpret_cast<float4*>(d.Q + ((size_t)s * d.E + b.x) * TS + 4 * gl) =
      make_float4(acc.x * ev, acc.y * ev, acc.z * ev, acc.w * ev);
}

// CTA-wide fixed-order reduction of per-lane float4 column sums into red[s][cta][TS].
template <int LPR>
__device__ __forceinline__ void cta_column_partial(const CgDev& d, float4 v, float* sm) {
  constexpr int TS = 4 * LPR, G = 32 / LPR, NG = NW * G;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const int g = (threadIdx.x >> 5) * G + grp;   // group index in the CTA
  reinterpret_cast<float4*>(sm)[g * LPR + gl] = v;
  __syncthreads();
  if (threadIdx.x < TS) {
    float a = 0.f;
    for (int i = 0; i < NG; ++i) a += sm[i * TS + threadIdx.x];
    d.red[((size_t)blockIdx.y * d.nparts + blockIdx.x) * TS + threadIdx.x] = a;
  }
}

// XP = vertex phase (see header); partial p^T X p per column.  Group = VPG consecutive rows.
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_vertex(CgDev d) {
  if (cg_stopped(d)) return;
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  __shared__ __align__(16) float sm[NW * G * TS];
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const unsigned gmask = (LPR == 32) ? ~0u : (((1u << LPR) - 1u) << (grp * LPR));
  const int s = blockIdx.y;
  const int v0 = ((blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp) * VPG;
  const size_t so = (size_t)s * d.N * TS + 4 * gl;
  const float* Q = d.Q + (size_t)s * d.E * TS + 4 * gl;
  float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int v = v0; v < min(v0 + VPG, d.N); ++v) {
    const int64_t p0 = d.row_ptr[v], p1 = d.row_ptr[v + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t base = p0; base < p1; base += LPR) {
      const int64_t j = base + gl;
      const int mye = j < p1 ? d.col[j] : 0;
      const int cnt = (int)min((int64_t)LPR, p1 - base);
      for (int u0 = 0; u0 < cnt; u0 += 8) {
        float4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = __shfl_sync(gmask, mye, (u0 + u) & (LPR - 1), LPR);
          x[u] = (u0 + u < cnt) ? __ldg(reinterpret_cast<const float4*>(Q + (size_t)e * TS))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) { acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w; }
      }
    }
    const float c = -d.dvr[v] * d.inv1pmu;
    const float4 p = *reinterpret_cast<const float4*>(d.P + so + (size_t)v * TS);
    const float4 xp = f4_fma(c, acc, p);
    *reinterpret_cast<float4*>(d.XP + so + (size_t)v * TS) = xp;
    dot.x = fmaf(p.x, xp.x, dot.x); dot.y = fmaf(p.y, xp.y, dot.y);
    dot.z = fmaf(p.z, xp.z, dot.z); dot.w = fmaf(p.w, xp.w, dot.w);
  }
  cta_column_partial<LPR>(d, dot, sm);
}

// f += alpha p; r -= alpha Xp (Eqs. 16-17); partial r^T r.
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_axpy(CgDev d) {
  if (cg_stopped(d)) return;
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  __shared__ __align__(16) float sm[NW * G * TS];
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const int s = blockIdx.y;
  const int v0 = ((blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp) * VPG;
  const size_t so = (size_t)s * d.N * TS + 4 * gl;
  const float4 a = *reinterpret_cast<const float4*>(d.alpha + s * TS + 4 * gl);
  float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int v = v0; v < min(v0 + VPG, d.N); ++v) {
    const size_t o = so + (size_t)v * TS;
    const float4 p = *reinterpret_cast<const float4*>(d.P + o);
    const float4 xp = *reinterpret_cast<const float4*>(d.XP + o);
    float4 f = *reinterpret_cast<const float4*>(d.F + o);
    float4 r = *reinterpret_cast<const float4*>(d.R + o);
    f.x = fmaf(a.x, p.x, f.x); f.y = fmaf(a.y, p.y, f.y); f.z = fmaf(a.z, p.z, f.z); f.w = fmaf(a.w, p.w, f.w);
    r.x = fmaf(-a.x, xp.x, r.x); r.y = fmaf(-a.y, xp.y, r.y); r.z = fmaf(-a.z, xp.z, r.z); r.w = fmaf(-a.w, xp.w, r.w);
    *reinterpret_cast<float4*>(d.F + o) = f;
    *reinterpret_cast<float4*>(d.R + o) = r;
    dot.x = fmaf(r.x, r.x, dot.x); dot.y = fmaf(r.y, r.y, dot.y);
    dot.z = fmaf(r.z, r.z, dot.z); dot.w = fmaf(r.w, r.w, dot.w);
  }
  cta_column_partial<LPR>(d, dot, sm);
}

// p = r + beta p (Eq. 18)
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_pupdate(CgDev d) {
  if (cg_stopped(d)) return;
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const int s = blockIdx.y;
  const int v0 = ((blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp) * VPG;
  const size_t so = (size_t)s * d.N * TS + 4 * gl;
  const float4 b = *reinterpret_cast<const float4*>(d.beta + s * TS + 4 * gl);
  for (int v = v0; v < min(v0 + VPG, d.N); ++v) {
    const size_t o = so + (size_t)v * TS;
    const float4 r = *reinterpret_cast<const float4*>(d.R + o);
    float4 p = *reinterpret_cast<const float4*>(d.P + o);
    p.x = fmaf(b.x, p.x, r.x); p.y = fmaf(b.y, p.y, r.y); p.z = fmaf(b.z, p.z, r.z); p.w = fmaf(b.w, p.w, r.w);
    *reinterpret_cast<float4*>(d.P + o) = p;
  }
}

// f_0 = 0, r_0 = c y - X f_0 = c y, p_0 = r_0; partial r_0^T r_0.
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_init(CgDev d, const float* __restrict__ Y) {
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  __shared__ __align__(16) float sm[NW * G * TS];
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const int s = blockIdx.y;
  const int v0 = ((blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp) * VPG;
  const size_t so = (size_t)s * d.N * TS + 4 * gl;
  const int c0 = s * TS + 4 * gl;   // T % 4 == 0: a float4 is all in or all out
  float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int v = v0; v < min(v0 + VPG, d.N); ++v) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c0 < d.T) {
      const float4 y = *reinterpret_cast<const float4*>(Y + (size_t)v * d.T + c0);
      r = make_float4(d.mu_c * y.x, d.mu_c * y.y, d.mu_c * y.z, d.mu_c * y.w);
    }
    const size_t o = so + (size_t)v * TS;
    *reinterpret_cast<float4*>(d.R + o) = r;
    *reinterpret_cast<float4*>(d.P + o) = r;
    *reinterpret_cast<float4*>(d.F + o) = make_float4(0.f, 0.f, 0.f, 0.f);
    dot.x = fmaf(r.x, r.x, dot.x); dot.y = fmaf(r.y, r.y, dot.y);
    dot.z = fmaf(r.z, r.z, dot.z); dot.w = fmaf(r.w, r.w, dot.w);
  }
  cta_column_partial<LPR>(d, dot, sm);
}

// Per-column scalars from the CTA partials (fp64, fixed order).  grid = ns, 512 threads.
//   mode 0 (init):  rr = rr0 = r_0^T r_0; active = rr0 > 0 and tol < 1
//   mode 1 (alpha): alpha = rr / p^T X p (Eq. 19), 0 for inactive columns
//   mode 2 (beta):  beta = r_i^T r_i / rr (Eq. 20); iters++; deactivate on ||r_i|| <= tol ||r_0||
// Modes 0 and 2 add the slice's active-column count to ctl[2 + iteration].
template <int TS>
__global__ void __launch_bounds__(512) k_cg_scalars(CgDev d, int mode) {
  constexpr int RL = 512 / TS;
  __shared__ double sm[512];
  __shared__ int s_act;
  if (mode != 0 && cg_stopped(d)) return;
  const int t = threadIdx.x, c = t % TS, rl = t / TS, s = blockIdx.x;
  double a = 0.0;
  for (int i = rl; i < d.nparts; i += RL) a += (double)d.red[((size_t)s * d.nparts + i) * TS + c];
  sm[t] = a;
  if (t == 0) s_act = 0;
  __syncthreads();
  if (t < TS) {
    double tot = 0.0;
    for (int i = 0; i < RL; ++i) tot += sm[i * TS + t];
    const int gc = s * TS + t;
    const int it = d.ctl[1];
    if (mode == 0) {
      d.rr[gc] = tot;
      d.rr0[gc] = tot;
      d.iters[gc] = 0;
      const bool act = tot > 0.0 && !(d.tol >= 1.f);
      d.active[gc] = act;
      if (act) atomicAdd(&s_act, 1);
    } else if (mode == 1) {
      float al = 0.f;
      if (d.active[gc]) {
        if (!(tot > 0.0)) {
          hg_flag(d.status, HGS_CG_BREAKDOWN);
          d.active[gc] = 0;
        } else {
          al = (float)(d.rr[gc] / tot);
        }
      }
      d.alpha[gc] = al;
    } else {
      float be = 0.f;
      if (d.active[gc]) {
        d.iters[gc] += 1;
        be = (float)(tot / d.rr[gc]);
        d.rr[gc] = tot;
        if (!isfinite(tot)) hg_flag(d.status, HGS_NONFINITE);
        if (sqrt(tot) <= (double)d.tol * sqrt(d.rr0[gc]) || !isfinite(tot)) d.active[gc] = 0;
        else atomicAdd(&s_act, 1);
      }
      d.beta[gc] = be;
    }
    (void)it;
  }
  __syncthreads();
  if (t == 0 && mode != 1) atomicAdd(&d.ctl[2 + (mode == 0 ? 0 : d.ctl[1] + 1)], s_act);
}

// After the scalars: running = (any column active) and iterations < max_iter; advances the
// iteration counter; in graph mode sets the WHILE node's condition.
__global__ void k_cg_control(CgDev d, cudaGraphConditionalHandle h, int use_handle, int init) {
  int run = 0;
  if (init) {
    run = d.ctl[2] > 0 && d.max_iter > 0;
  } else if (d.ctl[0]) {
    const int it = d.ctl[1] + 1;   // iterations completed
    d.ctl[1] = it;
    run = d.ctl[2 + it] > 0 && it < d.max_iter;
  }
  d.ctl[0] = run;
  if (use_handle) cudaGraphSetConditional(h, run ? 1u : 0u);
}

// F out in the caller's [N][T] layout; iterations and ||r||/||r_0|| per column.
template <int LPR>
__global__ void __launch_bounds__(NT) k_cg_out(CgDev d, float* __restrict__ Fo, int32_t* __restrict__ iters_out,
                                               float* __restrict__ rel_out) {
  constexpr int TS = 4 * LPR, G = 32 / LPR;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const int s = blockIdx.y;
  const int v0 = ((blockIdx.x * NW + (threadIdx.x >> 5)) * G + grp) * VPG;
  const int c0 = s * TS + 4 * gl;
  if (c0 < d.T)
    for (int v = v0; v < min(v0 + VPG, d.N); ++v)
      *reinterpret_cast<float4*>(Fo + (size_t)v * d.T + c0) =
          *reinterpret_cast<const float4*>(d.F + (size_t)s * d.N * TS + (size_t)v * TS + 4 * gl);
  if (blockIdx.x == 0 && threadIdx.x < TS) {
    const int gc = s * TS + threadIdx.x;
    if (gc < d.T) {
      if (iters_out) iters_out[gc] = d.iters[gc];
      if (rel_out) rel_out[gc] = d.rr0[gc] > 0.0 ? (float)sqrt(d.rr[gc] / d.rr0[gc]) : 0.f;
    }
  }
}

// ------------------------------------------------------------------ NEXT-4
// Frozen-degree gradient of P(w) = sum_t f_t^T L f_t + kappa ||w||^2 (oracle or_weight_gradient):
//   grad_e = -(1/delta(e)) sum_t s_{e,t}^2 + 2 kappa w_e,   s_{e,t} = sum_{v in e} r_v F[v][t].
// One warp per CSC work item; columns in chunks of 128 (a float4 per lane) straight from the
// caller's [N][T] F.  Single-chunk edges finish here; chunks of larger edges go to partial
// slots [slot][Tp] that k_wgrad_big adds in chunk order before squaring (deterministic).
__global__ void __launch_bounds__(NT) k_wgrad_items(int T, int Tp, const float* __restrict__ F,
                                                    const float* __restrict__ dvr, const int32_t* __restrict__ csc,
                                                    const int4* __restrict__ items, const int32_t* __restrict__ totals,
                                                    float* __restrict__ part, double* __restrict__ sqpart) {
  // grid (items, column chunks of 128): the chunk is the slow dimension, so the CTAs in flight
  // gather rows of one 512-byte-wide column slice of F, which stays in L2
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * NW + (threadIdx.x >> 5);
  if (item >= totals[0]) return;
  const int4 it = items[item];
  const int c = blockIdx.y * 128 + 4 * lane;
  const bool on = c < T;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = it.y; base < it.z; base += 32) {
    const int j = base + lane;
    const int myv = j < it.z ? csc[j] : 0;
    const float myr = j < it.z ? dvr[myv] : 0.f;
    const int cnt = min(32, it.z - base);
    for (int u0 = 0; u0 < cnt; u0 += 8) {
      float4 x[8];
      float r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = __shfl_sync(~0u, myv, (u0 + u) & 31);
        r[u] = __shfl_sync(~0u, myr, (u0 + u) & 31);
        x[u] = (on && u0 + u < cnt) ? __ldg(reinterpret_cast<const float4*>(F + (size_t)v * T + c))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = f4_fma(r[u], x[u], acc);
    }
  }
  if (it.w >= 0) {
    if (on) *reinterpret_cast<float4*>(part + (size_t)it.w * Tp + c) = acc;
  } else {
    double sq = (double)acc.x * acc.x + (double)acc.y * acc.y + (double)acc.z * acc.z + (double)acc.w * acc.w;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(~0u, sq, o);
    if (lane == 0) sqpart[(size_t)it.x * gridDim.y + blockIdx.y] = sq;
  }
}

// single-chunk edges: grad_e from the per-chunk sums of squares, added in chunk order
__global__ void k_wgrad_small(int E, int nch, const int32_t* __restrict__ de, const float* __restrict__ w, float kappa,
                              const double* __restrict__ sqpart, float* __restrict__ grad) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    if (de[e] > CH || de[e] == 0) continue;   // multi-chunk edges: k_wgrad_big
    double sq = 0.0;
    for (int ch = 0; ch < nch; ++ch) sq += sqpart[(size_t)e * nch + ch];
    grad[e] = (float)(-sq / (double)de[e] + 2.0 * (double)kappa * (double)w[e]);
  }
}

__global__ void __launch_bounds__(NT) k_wgrad_big(int T, int Tp, const int4* __restrict__ bigs,
                                                  const int32_t* __restrict__ totals, const int32_t* __restrict__ de,
                                                  const float* __restrict__ w, float kappa,
                                                  const float* __restrict__ part, float* __restrict__ grad) {
  const int lane = threadIdx.x & 31;
  const int bi = blockIdx.x * NW + (threadIdx.x >> 5);
  if (bi >= totals[1]) return;
  const int4 b = bigs[bi];
  double sq = 0.0;
  for (int c = 4 * lane; c < T; c += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < b.z; ++j) {
      const float4 x = *reinterpret_cast<const float4*>(part + (size_t)(b.y + j) * Tp + c);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    sq += (double)acc.x * acc.x + (double)acc.y * acc.y + (double)acc.z * acc.z + (double)acc.w * acc.w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(~0u, sq, o);
  if (lane == 0) grad[b.x] = (float)(-sq / (double)de[b.x] + 2.0 * (double)kappa * (double)w[b.x]);
}

// One simplex-constrained steepest-descent step (oracle or_weight_step, reading N2), one
// CTA, fp64 fixed-order reductions: mean-free gradient over the free coordinates, w -= mu g,
// then clamp negative free coordinates to 0 (they join the active set) and remove the excess
// mass evenly from the remaining free ones, until none is negative.
__device__ double block_sum_d(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(~0u, v, o);
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sm[i];
  return t;
}

__global__ void __launch_bounds__(1024) k_weight_step(int E, float* __restrict__ w, int32_t* __restrict__ active,
                                                      const float* __restrict__ grad, float mu, int32_t* status) {
  __shared__ double sm[32];
  double gs = 0.0, nf = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (!active[e]) { gs += grad[e]; nf += 1.0; }
  gs = block_sum_d(gs, sm);
  nf = block_sum_d(nf, sm);
  if (nf == 0.0) {
    if (threadIdx.x == 0) hg_flag(status, HGS_SIMPLEX_DEGENERATE);
    return;
  }
  const double gm = gs / nf;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (!active[e]) w[e] = (float)((double)w[e] - (double)mu * ((double)grad[e] - gm));
  for (int round = 0; round < E + 1; ++round) {
    __syncthreads();
    double clamped = 0.0;
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      if (!active[e] && w[e] < 0.f) { w[e] = 0.f; active[e] = 1; clamped += 1.0; }
    clamped = block_sum_d(clamped, sm);
    if (clamped == 0.0) break;
    double sum = 0.0, fr = 0.0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) { sum += w[e]; if (!active[e]) fr += 1.0; }
    sum = block_sum_d(sum, sm);
    fr = block_sum_d(fr, sm);
    if (fr == 0.0) {
      if (threadIdx.x == 0) hg_flag(status, HGS_SIMPLEX_DEGENERATE);
      return;
    }
    const double ex = (sum - 1.0) / fr;
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      if (!active[e]) w[e] = (float)((double)w[e] - ex);
  }
}

// Start of the weight iteration on the simplex 1^T w = 1, w >= 0 (Eq. optprob):
// w_out = w / (1^T w), the sum in a fixed order in fp64.  A negative, non-finite or all-zero w flags
// HGS_SIMPLEX_DEGENERATE (w_out then = w).
__global__ void __launch_bounds__(1024) k_weight_normalize(int E, const float* __restrict__ w, float* __restrict__ wo,
                                                           int32_t* status) {
  __shared__ double sm[32];
  double s = 0.0, bad = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const float x = w[e];
    s += x;
    if (!(x >= 0.f) || !isfinite(x)) bad += 1.0;
  }
  s = block_sum_d(s, sm);
  bad = block_sum_d(bad, sm);
  const bool ok = bad == 0.0 && s > 0.0;
  if (!ok && threadIdx.x == 0) hg_flag(status, HGS_SIMPLEX_DEGENERATE);
  const double inv = ok ? 1.0 / s : 1.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) wo[e] = (float)((double)w[e] * inv);
}

// P(w) = ||F||^2 - sum_e (w_e/delta(e)) sum_t s_{e,t}^2 + kappa ||w||^2 from the gradient at the same
// w: w_e (2 kappa w_e - grad_e) = w_e sum_t s^2 / delta(e), so P = ||F||^2 + w^T grad - kappa ||w||^2.
// Fixed-order fp64 sums: per-CTA partials, then one CTA adds them in order.
__global__ void __launch_bounds__(256) k_wobj_partial(int64_t nF, const float* __restrict__ F, int E,
                                                      const float* __restrict__ w, const float* __restrict__ grad,
                                                      float kappa, double* __restrict__ part) {
  __shared__ double sm[8];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x)
    acc += (double)F[i] * (double)F[i];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    acc += (double)w[e] * (double)grad[e] - (double)kappa * (double)w[e] * (double)w[e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += sm[i];
    part[blockIdx.x] = t;
  }
}

__global__ void k_wobj_final(int n, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
  }
}

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

// ------------------------------------------------------------------ host side
int cg_lanes(int T) { return T > 64 ? 32 : (T > 32 ? 16 : 8); }

CgLayout cg_layout(int64_t N, int64_t E, int64_t nnz, int64_t T, int64_t max_iter) {
  CgLayout L;
  const int64_t TS = 4 * cg_lanes((int)T), ns = (T + TS - 1) / TS;
  const int64_t rb = (int64_t)NW * (32 / cg_lanes((int)T)) * VPG;
  const int64_t nparts = (N + rb - 1) / rb;
  const int64_t max_items = E + nnz / CH + 1, max_big = nnz / CH + 1, max_slots = 2 * (nnz / CH) + 2;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al256(bytes);
    return o;
  };
  L.TS = (int)TS;
  L.ns = (int)ns;
  L.nparts = (int)nparts;
  L.max_items = max_items;
  L.max_big = max_big;
  L.de = take(4 * E);
  L.eval = take(4 * E);
  L.dvr = take(4 * N);
  L.col_ptr = take(4 * (E + 1));
  L.item_ptr = take(4 * E);
  L.slot_ptr = take(4 * E);
  L.big_ptr = take(4 * E);
  L.cursor = take(4 * E);
  L.totals = take(16);
  L.csc_tmp = take(4 * (nnz > 0 ? nnz : 1));
  L.csc = take(4 * (nnz > 0 ? nnz : 1));
  L.items = take(16 * max_items);
  L.bigs = take(16 * max_big);
  const size_t vec = 4 * (size_t)ns * N * TS;
  L.P = take(vec);
  L.R = take(vec);
  L.F = take(vec);
  L.XP = take(vec);
  L.sqpart = take(8 * (size_t)E * ((T + 127) / 128));   // weight gradient: per-edge, per-chunk sums
  L.Q = take(4 * (size_t)ns * E * TS);
  L.part = take(4 * (size_t)ns * max_slots * TS);
  L.red = take(4 * (size_t)ns * nparts * TS);
  const size_t tp = (size_t)ns * TS;
  L.rr = take(8 * tp);
  L.rr0 = take(8 * tp);
  L.alpha = take(4 * tp);
  L.beta = take(4 * tp);
  L.active = take(4 * tp);
  L.iters = take(4 * tp);
  L.ctl = take(4 * (size_t)(max_iter + 3));
  L.status = take(4);
  L.total = off;
  return L;
}

namespace {
template <class T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

CgDev make_dev(const CgArgs& a, const CgLayout& L) {
  CgDev d;
  d.N = a.N; d.E = a.E; d.T = a.T; d.ns = L.ns; d.nparts = L.nparts;
  d.mu_c = a.mu / (1.0f + a.mu);
  d.inv1pmu = 1.0f / (1.0f + a.mu);
  d.tol = a.tol;
  d.max_iter = a.max_iter;
  d.row_ptr = a.row_ptr; d.col = a.col_idx;
  d.eval = at<float>(a.ws, L.eval); d.dvr = at<float>(a.ws, L.dvr);
  d.csc = at<int32_t>(a.ws, L.csc);
  d.items = at<int4>(a.ws, L.items); d.bigs = at<int4>(a.ws, L.bigs);
  d.totals = at<int32_t>(a.ws, L.totals);
  d.P = at<float>(a.ws, L.P); d.R = at<float>(a.ws, L.R); d.F = at<float>(a.ws, L.F);
  d.XP = at<float>(a.ws, L.XP); d.Q = at<float>(a.ws, L.Q); d.part = at<float>(a.ws, L.part);
  d.red = at<float>(a.ws, L.red);
  d.rr = at<double>(a.ws, L.rr); d.rr0 = at<double>(a.ws, L.rr0);
  d.alpha = at<float>(a.ws, L.alpha); d.beta = at<float>(a.ws, L.beta);
  d.active = at<int32_t>(a.ws, L.active); d.iters = at<int32_t>(a.ws, L.iters);
  d.ctl = at<int32_t>(a.ws, L.ctl);
  d.status = a.status;
  return d;
}

template <int LPR>
cudaError_t body(const CgDev& d, const CgLayout& L, cudaGraphConditionalHandle h, bool use_handle, cudaStream_t s,
                 int* launches) {
  constexpr int G = 32 / LPR;
  const dim3 gi((unsigned)((L.max_items + NW * G - 1) / (NW * G)), L.ns);
  const dim3 gb((unsigned)((L.max_big + NW * G - 1) / (NW * G)), L.ns);
  const dim3 gr(L.nparts, L.ns);
  k_cg_edge<LPR><<<gi, NT, 0, s>>>(d);
  k_cg_edge_reduce<LPR><<<gb, NT, 0, s>>>(d);
  k_cg_vertex<LPR><<<gr, NT, 0, s>>>(d);
  k_cg_scalars<4 * LPR><<<L.ns, 512, 0, s>>>(d, 1);
  k_cg_axpy<LPR><<<gr, NT, 0, s>>>(d);
  k_cg_scalars<4 * LPR><<<L.ns, 512, 0, s>>>(d, 2);
  k_cg_pupdate<LPR><<<gr, NT, 0, s>>>(d);
  k_cg_control<<<1, 1, 0, s>>>(d, h, use_handle ? 1 : 0, 0);
  *launches += 8;
  return cudaGetLastError();
}

// degrees (r = delta(v)^-1/2, w_e/delta(e)) and the sorted CSC of H with its CH-chunk work items
cudaError_t setup_csc(const CgArgs& a, const CgLayout& L, cudaStream_t s, int* launches) {
  void* ws = a.ws;
  cudaError_t e = launch_degrees(a.N, a.E, a.nnz, a.row_ptr, a.col_idx, a.w, at<int32_t>(ws, L.de),
                                 at<float>(ws, L.eval), at<float>(ws, L.dvr), a.status, s, launches);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(at<int32_t>(ws, L.cursor), 0, 4 * (size_t)a.E, s)) != cudaSuccess) return e;
  int32_t* col_ptr = at<int32_t>(ws, L.col_ptr);
  k_cg_scan<<<1, 1024, 0, s>>>(a.E, at<int32_t>(ws, L.de), col_ptr, at<int32_t>(ws, L.item_ptr),
                               at<int32_t>(ws, L.slot_ptr), at<int32_t>(ws, L.big_ptr), at<int32_t>(ws, L.totals));
  const int gN = (int)std::min<int64_t>((a.N + 255) / 256, 148 * 8);
  const int gE = (int)std::min<int64_t>((a.E + 255) / 256, 148 * 8);
  k_cg_fill<<<gN, 256, 0, s>>>(a.N, a.row_ptr, a.col_idx, col_ptr, at<int32_t>(ws, L.cursor),
                               at<int32_t>(ws, L.csc_tmp));
  k_cg_sort_small<<<(int)std::min<int64_t>((a.E + 7) / 8, 148 * 16), 256, 0, s>>>(
      a.E, col_ptr, at<int32_t>(ws, L.csc_tmp), at<int32_t>(ws, L.csc));
  k_cg_sort_big<<<(int)std::min<int64_t>(a.E, 148 * 4), NT, 0, s>>>(a.N, a.E, col_ptr, at<int32_t>(ws, L.csc_tmp),
                                                                     at<int32_t>(ws, L.csc));
  k_cg_items<<<gE, 256, 0, s>>>(a.E, col_ptr, at<int32_t>(ws, L.item_ptr), at<int32_t>(ws, L.slot_ptr),
                                at<int32_t>(ws, L.big_ptr), at<int4>(ws, L.items), at<int4>(ws, L.bigs));
  *launches += 6;
  return cudaGetLastError();
}

template <int LPR>
cudaError_t prologue(const CgArgs& a, const CgDev& d, const CgLayout& L, cudaStream_t s, int* launches) {
  cudaError_t e = cudaMemsetAsync(d.ctl, 0, 4 * (size_t)(a.max_iter + 3), s);
  if (e != cudaSuccess) return e;
  if ((e = setup_csc(a, L, s, launches)) != cudaSuccess) return e;
  const dim3 gr(L.nparts, L.ns);
  k_cg_init<LPR><<<gr, NT, 0, s>>>(d, a.Y);
  k_cg_scalars<4 * LPR><<<L.ns, 512, 0, s>>>(d, 0);
  *launches += 2;
  return cudaGetLastError();
}

template <int LPR>
cudaError_t run_cg_t(const CgArgs& a, const CgLayout& L, const CgGraphHook* hook, cudaStream_t s, int* launches) {
  const CgDev d = make_dev(a, L);
  cudaError_t e = prologue<LPR>(a, d, L, s, launches);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h = 0;
  if (hook) {
    // graph mode: the control kernel sets the WHILE condition before the loop; the body is
    // captured into the conditional node's graph.
    if ((e = hook->begin(hook->ctx, &h)) != cudaSuccess) return e;   // creates the handle only
    k_cg_control<<<1, 1, 0, s>>>(d, h, 1, 1);
    ++*launches;
    cudaStream_t bs = nullptr;
    if ((e = hook->open_body(hook->ctx, h, &bs)) != cudaSuccess) return e;
    if ((e = body<LPR>(d, L, h, true, bs, launches)) != cudaSuccess) return e;
    if ((e = hook->close_body(hook->ctx)) != cudaSuccess) return e;
  } else {
    k_cg_control<<<1, 1, 0, s>>>(d, 0, 0, 1);
    ++*launches;
    for (int i = 0; i < a.max_iter; ++i)
      if ((e = body<LPR>(d, L, 0, false, s, launches)) != cudaSuccess) return e;
  }
  const dim3 gr(L.nparts, L.ns);
  k_cg_out<LPR><<<gr, NT, 0, s>>>(d, a.F, a.iters_out, a.rel_out);
  ++*launches;
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_cg(const CgArgs& a, const CgGraphHook* hook, cudaStream_t s, int* launches) {
  const CgLayout L = cg_layout(a.N, a.E, a.nnz, a.T, a.max_iter);
  switch (L.TS / 4) {
    case 32: return run_cg_t<32>(a, L, hook, s, launches);
    case 16: return run_cg_t<16>(a, L, hook, s, launches);
    default: return run_cg_t<8>(a, L, hook, s, launches);
  }
}

// NEXT-4 entry points; a.F is the caller's F [N][T], a.ws a CG workspace.
cudaError_t launch_weight_gradient(const CgArgs& a, float kappa, float* grad, cudaStream_t s, int* launches) {
  const CgLayout L = cg_layout(a.N, a.E, a.nnz, a.T, 0);
  cudaError_t e = setup_csc(a, L, s, launches);
  if (e != cudaSuccess) return e;
  const int Tp = L.ns * L.TS;   // partial-slot pitch (the CG partial buffer holds max_slots x Tp)
  const int nch = (a.T + 127) / 128;
  double* sqpart = at<double>(a.ws, L.sqpart);   // [E][nch]
  k_wgrad_items<<<dim3((unsigned)((L.max_items + NW - 1) / NW), nch), NT, 0, s>>>(
      a.T, Tp, a.F, at<float>(a.ws, L.dvr), at<int32_t>(a.ws, L.csc), at<int4>(a.ws, L.items),
      at<int32_t>(a.ws, L.totals), at<float>(a.ws, L.part), sqpart);
  k_wgrad_small<<<(unsigned)std::min<int64_t>((a.E + 255) / 256, 148 * 8), 256, 0, s>>>(
      a.E, nch, at<int32_t>(a.ws, L.de), a.w, kappa, sqpart, grad);
  k_wgrad_big<<<(unsigned)((L.max_big + NW - 1) / NW), NT, 0, s>>>(
      a.T, Tp, at<int4>(a.ws, L.bigs), at<int32_t>(a.ws, L.totals), at<int32_t>(a.ws, L.de), a.w, kappa,
      at<float>(a.ws, L.part), grad);
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_weight_normalize(int E, const float* w, float* wo, int32_t* status, cudaStream_t s,
                                    int* launches) {
  k_weight_normalize<<<1, 1024, 0, s>>>(E, w, wo, status);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_weight_step(int E, float* w, int32_t* active, const float* grad, float mu, int32_t* status,
                               cudaStream_t s, int* launches) {
  k_weight_step<<<1, 1024, 0, s>>>(E, w, active, grad, mu, status);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_csc_setup(const CgArgs& a, cudaStream_t s, int* launches) {
  return setup_csc(a, cg_layout(a.N, a.E, a.nnz, a.T, 0), s, launches);
}

// out[0] = P(w) (fp64, device) from grad = the frozen-degree gradient at w; part: >= 296 doubles scratch
cudaError_t launch_weight_objective(int64_t nF, const float* F, int E, const float* w, const float* grad, float kappa,
                                    double* part, double* out, cudaStream_t s, int* launches) {
  constexpr int NB = 296;   // 2 CTAs per SM
  k_wobj_partial<<<NB, 256, 0, s>>>(nF, F, E, w, grad, kappa, part);
  k_wobj_final<<<1, 32, 0, s>>>(NB, part, out);
  *launches += 2;
  return cudaGetLastError();
}
