// theta.cu -- degrees and diagonal-block assembly of X = I - Theta/(1+mu).
//
//   delta(e) = sum_v H(v,e),  delta(v) = sum_e w(e) H(v,e)
//   Theta_ii[u][v] = r_u r_v sum_{e ni u,v} w_e/delta(e),  r = delta(v)^-1/2   (Eq. 1)
//   X_ii = I - Theta_ii/(1+mu)
//
// Assembly, default path: sorted per-block CSC keys + full-width row tiles
// (k_seg_sort, k_assemble_rows; see "Sorted-CSC assembly" below).  Fallback
// (blocks whose segments overflow shared memory, E*b >= 2^32, or HG_ASSEMBLE=tiles):
// k_assemble, one CTA per (block, 128-row tile U, 64-column tile V) that hashes V's
// incidences (edge -> members of V, in shared memory); the thread owning row u walks
// u's CSR row in ascending edge order and adds w_e/delta(e) to acc[u][v] for every v
// of V sharing e.  Both paths sum every (u,v) over the common edges in ascending edge
// order -- the same sequence for (v,u) -- so the written blocks are bitwise symmetric,
// identical between the paths and run-to-run deterministic with no atomics on values.
// Traffic: the b x b block is written once (4 b^2 bytes per block; HBM-write bound).
#include <cstdlib>

#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "gemm.cuh"

cudaError_t launch_assemble_tiles(int blk0, int nb, int b, const int64_t* row_ptr, const int32_t* col_idx,
                                  const float* edge_val, const float* dv_rsqrt, float mu, bool raw_theta,
                                  float* blocks, const int32_t* overflow, cudaStream_t s, int* launches);

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

__global__ void __launch_bounds__(NT) k_assemble(int blk0, int b, const int64_t* __restrict__ row_ptr,
                                                 const int32_t* __restrict__ col,
                                                 const float* __restrict__ eval, const float* __restrict__ dvr,
                                                 float inv1pmu, int raw, float* __restrict__ blocks,
                                                 const int32_t* __restrict__ overflow) {
  const int blk = blk0 + blockIdx.z;
  if (overflow && !overflow[blk]) return;     // block assembled by the sorted-CSC path
  extern __shared__ __align__(16) uint8_t smem_raw[];
  AsmSmem& S = *reinterpret_cast<AsmSmem*>(smem_raw);
  const int t = threadIdx.x;
  const int u0 = blockIdx.y * TU, v0 = blockIdx.x * TV;
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


// ---------------------------------------------------------------------------
// Sorted-CSC assembly (default path).
//   k_seg_sort: per (block, 512-vertex segment) the incidences (e, v) become
//   32-bit keys e*b + v_local, bitonic-sorted in shared memory and written back
//   at the segment's CSR range: each segment is then an edge-major list, so the
//   members of edge e inside the segment are one key range [e*b, (e+1)*b).
//   k_assemble_rows: one CTA per (block, TR rows) with the full b-wide fp32
//   accumulator in shared memory; a warp per row walks the row's edges in
//   ascending order (lanes binary-search their edge's key range in every
//   segment), then adds w_e/delta(e) to acc[u][v] for the members, one edge at
//   a time.  Each (u,v) therefore sums its common edges in ascending edge order
//   -- the same additions as k_assemble, bitwise -- so blocks stay bitwise
//   symmetric.  Output rows are written once, coalesced.
constexpr int SEG_V = 512;          // vertices per sorted segment
constexpr int SEG_CAP = 16384;      // keys per segment in shared memory (64 KB)
constexpr int NSEG_MAX = 4;         // b <= 4 SEG_V on the sorted path
constexpr int ROWS_NT = 512;        // k_assemble_rows: one warp per row
constexpr int TR_ROWS = ROWS_NT / 32;
constexpr int STAGE_KEYS = 512;     // per-warp member-key staging (2 KB)

__global__ void __launch_bounds__(1024) k_seg_sort(int blk0, int b, const int64_t* __restrict__ row_ptr,
                                                   const int32_t* __restrict__ col, uint32_t* __restrict__ keys,
                                                   int2* __restrict__ rng, int32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  int64_t* vp = reinterpret_cast<int64_t*>(smem_raw);                    // [SEG_V + 1]
  uint32_t* sk = reinterpret_cast<uint32_t*>(smem_raw + (SEG_V + 2) * 8);  // [SEG_CAP]
  const int blk = blk0 + blockIdx.x, seg = blockIdx.y, t = threadIdx.x;
  const int64_t vb = (int64_t)blk * b + (int64_t)seg * SEG_V;
  const int nv = min(SEG_V, b - seg * SEG_V);
  if (nv <= 0) return;
  for (int i = t; i <= nv; i += 1024) vp[i] = row_ptr[vb + i];
  __syncthreads();
  const int64_t p0 = vp[0];
  const int n = (int)(vp[nv] - p0);
  if (n > SEG_CAP) {
    if (t == 0) overflow[blk] = 1;
    return;
  }
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  for (int i = t; i < np2; i += 1024) {
    uint32_t key = 0xFFFFFFFFu;
    if (i < n) {
      const int64_t p = p0 + i;
      int lo = 0, hi = nv;                         // vertex: vp[lo] <= p < vp[lo+1]
      while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (vp[mid] <= p) lo = mid; else hi = mid; }
      key = (uint32_t)col[p] * (uint32_t)b + (uint32_t)(seg * SEG_V + lo);
    }
    sk[i] = key;
  }
  __syncthreads();
  for (int k2 = 2; k2 <= np2; k2 <<= 1) {          // bitonic sort, ascending
    for (int j = k2 >> 1; j > 0; j >>= 1) {
      for (int i = t; i < np2; i += 1024) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = sk[i], c = sk[ixj];
          const bool up = (i & k2) == 0;
          if ((a > c) == up) { sk[i] = c; sk[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = t; i < n; i += 1024) keys[p0 + i] = sk[i];
  // member ranges of every incidence (u, e) of the block inside this segment: keys of
  // edge e are [e b, (e+1) b); indices relative to the block's first incidence kb0
  const int64_t kb0 = row_ptr[(int64_t)blk * b], kb1 = row_ptr[(int64_t)(blk + 1) * b];
  const int s0 = (int)(p0 - kb0);
  for (int64_t p = kb0 + t; p < kb1; p += 1024) {
    const uint32_t e = (uint32_t)col[p];
    int lo = 0, hi = n;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (sk[mid] < e * (uint32_t)b) lo = mid + 1; else hi = mid; }
    int lo2 = lo, hi2 = n;
    while (lo2 < hi2) { const int mid = (lo2 + hi2) >> 1; if (sk[mid] < (e + 1) * (uint32_t)b) lo2 = mid + 1; else hi2 = mid; }
    rng[p * NSEG_MAX + seg] = make_int2(s0 + lo, s0 + lo2);
  }
}


// The row walk: one warp per row u, ascending edge order; for each edge e of the row the
// members in the block are the key runs rng[p][segment] (p = global CSR position of (u, e);
// run bounds relative to the block's first incidence, from k_seg_sort), read from
// global memory (coalesced runs).  Each (u, v) sums its common edges in ascending edge
// order.  The warp writes its row as soon as it is complete (rows are independent).
__device__ __forceinline__ void assemble_rows_walk(int b, int nu, int nseg, int64_t base, int u0,
                                                   const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                                   const uint32_t* __restrict__ K, const int2* __restrict__ rng,
                                                   const float* __restrict__ eval, const float* __restrict__ dvr,
                                                   float inv1pmu, int raw, float* __restrict__ out, float* acc,
                                                   uint32_t* stage, int lane, int warp) {
  for (int r = warp; r < nu; r += ROWS_NT / 32) {
    const int64_t u = base + u0 + r;
    const int64_t q0 = row_ptr[u], q1 = row_ptr[u + 1];
    float* arow = acc + (size_t)r * b;
    for (int64_t c0 = q0; c0 < q1; c0 += 32) {
      const int ne = (int)((q1 - c0) < 32 ? (q1 - c0) : 32);
      uint32_t e = 0;
      float val = 0.f;
      int2 rg[NSEG_MAX];
#pragma unroll
      for (int sg = 0; sg < NSEG_MAX; ++sg) rg[sg] = make_int2(0, 0);
      if (lane < ne) {
        e = (uint32_t)col[c0 + lane];
        val = eval[e];
        for (int sg = 0; sg < nseg; ++sg) rg[sg] = rng[(c0 + lane) * NSEG_MAX + sg];
      }
      // gather: lane j copies its edge's member runs into the warp's staging area (all
      // loads in flight together), then the scatter runs in ascending edge order from
      // shared memory -- one L2 round trip per row chunk instead of one per edge
      int len = 0;
#pragma unroll
      for (int sg = 0; sg < NSEG_MAX; ++sg)
        if (sg < nseg) len += rg[sg].y - rg[sg].x;
      int off = len;                               // inclusive warp scan of the run lengths
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, off, o);
        if (lane >= o) off += x;
      }
      const int total = __shfl_sync(0xffffffffu, off, 31);
      off -= len;                                  // exclusive
      if (total <= STAGE_KEYS) {
        if (lane < ne) {
          int d = off;
#pragma unroll
          for (int sg = 0; sg < NSEG_MAX; ++sg) {
            if (sg >= nseg) break;
            const int m0 = rg[sg].x, m1 = rg[sg].y;
            int m = m0;
            for (; m + 8 <= m1; m += 8) {   // eight independent loads in flight per lane
              uint32_t x[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) x[i] = K[m + i];
#pragma unroll
              for (int i = 0; i < 8; ++i) stage[d + i] = x[i];
              d += 8;
            }
            for (; m < m1; ++m) stage[d++] = K[m];
          }
        }
        __syncwarp();
        for (int j = 0; j < ne; ++j) {             // ascending edge order
          const float vj = __shfl_sync(0xffffffffu, val, j);
          const uint32_t ebj = __shfl_sync(0xffffffffu, e, j) * (uint32_t)b;
          const int o0 = __shfl_sync(0xffffffffu, off, j), n0 = __shfl_sync(0xffffffffu, len, j);
          for (int i = lane; i < n0; i += 32) arow[stage[o0 + i] - ebj] += vj;
          __syncwarp();
        }
      } else {
        for (int j = 0; j < ne; ++j) {             // ascending edge order (long rows: direct)
          const float vj = __shfl_sync(0xffffffffu, val, j);
          const uint32_t ebj = __shfl_sync(0xffffffffu, e, j) * (uint32_t)b;
#pragma unroll
          for (int sg = 0; sg < NSEG_MAX; ++sg) {
            if (sg >= nseg) break;
            const int l = __shfl_sync(0xffffffffu, rg[sg].x, j), h = __shfl_sync(0xffffffffu, rg[sg].y, j);
            for (int m = l + lane; m < h; m += 32) arow[K[m] - ebj] += vj;
          }
          __syncwarp();
        }
      }
    }
    const int uu = u0 + r;
    const float du = dvr[base + uu];
    float* orow = out + (int64_t)uu * b;
    for (int v = lane; v < b; v += 32) {
      const float th = (du * dvr[base + v]) * arow[v];
      orow[v] = raw ? th : ((uu == v ? 1.0f : 0.0f) - th * inv1pmu);
    }
  }
}

__global__ void __launch_bounds__(ROWS_NT) k_assemble_rows(int blk0, int b, const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ keys,
                                                          const int2* __restrict__ rng,
                                                          const float* __restrict__ eval,
                                                          const float* __restrict__ dvr, float inv1pmu, int raw,
                                                          float* __restrict__ blocks,
                                                          const int32_t* __restrict__ overflow) {
  const int blk = blk0 + blockIdx.x;
  if (overflow[blk]) return;                      // handled by the hashed-tile kernel
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float* acc = reinterpret_cast<float*>(smem_raw);   // [TR_ROWS][b]
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem_raw + (size_t)TR_ROWS * b * 4) + (threadIdx.x >> 5) * STAGE_KEYS;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t base = (int64_t)blk * b;
  const int u0 = blockIdx.y * TR_ROWS;
  const int nu = min(TR_ROWS, b - u0);
  const int nseg = (b + SEG_V - 1) / SEG_V;
  const int64_t kb0 = row_ptr[base];
  for (int i = t; i < TR_ROWS * b; i += ROWS_NT) acc[i] = 0.f;
  __syncthreads();
  assemble_rows_walk(b, nu, nseg, base, u0, row_ptr, col, keys + kb0, rng, eval, dvr, inv1pmu, raw,
                     blocks + (int64_t)blk * b * b, acc, stage, lane, warp);
}


// ---------------------------------------------------------------------------
// Per-block radix assembly (default when E < 2^17 and a block's incidences fit in shared
// memory; other blocks take the hashed-tile kernel, problems with E >= 2^17 the segmented path).
//   k_block_sort: one CTA per block.  The block's incidences (u, e) as keys e << 15 | idx
//   (idx = position in the block's CSR range) are stably radix-sorted by e (LSD, 3 passes of
//   6/6/5 bits, warp-ordered chunks, ranks by __match_any_sync: deterministic), so each edge's
//   members in the block become one run, in ascending vertex order.  Out: memb[p0 + j] = the
//   block-local vertex of sorted entry j; rng[p] = the run [start, end) (relative to p0) of the
//   members of incidence p's edge.
//   k_assemble_rows2: one CTA per (block, 16 rows), a warp per row u walks u's edges in
//   ascending order and adds w_e/delta(e) to acc[u][v] for the members v.  Heavy edges (>= 32
//   members in the block) with all lanes; a run of light edges as one batch of (edge, member)
//   pairs -- pairs with the same v are applied by one lane, in ascending edge order, to the
//   running acc[v]: every entry sees exactly the sequence of fp32 additions of the edge-by-edge
//   walk (bitwise equal to k_assemble and k_assemble_rows; blocks bitwise symmetric).
constexpr int BR_NT = 1024;
constexpr int BR_NW = BR_NT / 32;
constexpr int BR_IDXB = 15;                  // idx bits of a key
constexpr int BR_CAP = 25600;                // incidences per block (2 x 100 KB key buffers)
constexpr int R2_NT = 512;                   // k_assemble_rows2: one warp per row
constexpr int R2_ROWS = R2_NT / 32;
constexpr int HEAVY = 32;                    // members of an edge in the block for the all-lanes path

__global__ void __launch_bounds__(BR_NT, 1) k_block_sort(int blk0, int b, const int64_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col, uint32_t* __restrict__ memb,
                                                         int2* __restrict__ rng, int32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint32_t* kA = reinterpret_cast<uint32_t*>(smem_raw);                    // [BR_CAP]
  uint32_t* kB = kA + BR_CAP;                                              // [BR_CAP]
  int* vp = reinterpret_cast<int*>(kB + BR_CAP);                           // [b + 1] CSR offsets rel. p0
  int* hist = vp + 2049;                                                   // [64][BR_NW]
  int* wtot = hist + 64 * BR_NW;                                           // [BR_NW]
  const int blk = blk0 + blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t vb = (int64_t)blk * b;
  const int64_t p0 = row_ptr[vb];
  const int64_t n64 = row_ptr[vb + b] - p0;
  if (n64 > BR_CAP) {   // handled by the hashed-tile kernel
    if (t == 0) overflow[blk] = 1;
    return;
  }
  const int n = (int)n64;
  for (int i = t; i <= b; i += BR_NT) vp[i] = (int)(row_ptr[vb + i] - p0);
  for (int i = t; i < n; i += BR_NT) kA[i] = ((uint32_t)col[p0 + i] << BR_IDXB) | (uint32_t)i;
  __syncthreads();
  // LSD passes over the edge bits [15, 21), [21, 27), [27, 32)
  const int chunk = (n + BR_NW - 1) / BR_NW;
  const int c0 = warp * chunk, c1 = min(n, c0 + chunk);
  uint32_t* src = kA;
  uint32_t* dst = kB;
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = BR_IDXB + 6 * pass, nb = pass < 2 ? 64 : 32;
    for (int i = t; i < 64 * BR_NW; i += BR_NT) hist[i] = 0;
    __syncthreads();
    for (int g = c0; g < c1; g += 32) {   // per-warp digit counts (no atomics: one leader per digit)
      const int i = g + lane;
      const unsigned act = __ballot_sync(0xffffffffu, i < c1);
      if (i < c1) {
        const int dg = (int)((src[i] >> shift) & (nb - 1));
        const unsigned m = __match_any_sync(act, dg);
        if (lane == __ffs(m) - 1) hist[dg * BR_NW + warp] += __popc(m);
      }
      __syncwarp();
    }
    __syncthreads();
    // exclusive scan over (digit, warp) in digit-major order: 2048 entries, 2 per thread
    {
      const int i0 = 2 * t;
      const int a0 = hist[i0], a1 = hist[i0 + 1];
      int s = a0 + a1, x = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wtot[warp] = x;
      __syncthreads();
      int pre = 0;
      for (int w = 0; w < warp; ++w) pre += wtot[w];
      const int ex = pre + x - s;
      hist[i0] = ex;
      hist[i0 + 1] = ex + a0;
    }
    __syncthreads();
    for (int g = c0; g < c1; g += 32) {   // stable scatter
      const int i = g + lane;
      const unsigned act = __ballot_sync(0xffffffffu, i < c1);
      int dg = 0, pos = 0;
      unsigned m = 0;
      uint32_t key = 0;
      if (i < c1) {
        key = src[i];
        dg = (int)((key >> shift) & (nb - 1));
        m = __match_any_sync(act, dg);
        pos = hist[dg * BR_NW + warp] + __popc(m & ((1u << lane) - 1u));
      }
      __syncwarp();
      if (i < c1) {
        dst[pos] = key;
        if (lane == __ffs(m) - 1) hist[dg * BR_NW + warp] += __popc(m);
      }
      __syncwarp();
    }
    __syncthreads();
    uint32_t* tmp = src; src = dst; dst = tmp;
  }
  // src: sorted.  Runs of equal edge: start flags, then per entry its run [rs, re) by a block max-scan
  // of starts (forward) and min-scan of ends (backward); contiguous chunks per thread.
  const int per = (n + BR_NT - 1) / BR_NT;
  const int j0 = t * per, j1 = min(n, j0 + per);
  int last_start = -1;                 // the last run start within this thread's chunk
  for (int j = j0; j < j1; ++j)
    if (j == 0 || (src[j] >> BR_IDXB) != (src[j - 1] >> BR_IDXB)) last_start = j;
  int first_start = n;                 // the first run start strictly after this thread's chunk start
  for (int j = j1 - 1; j >= j0; --j)
    if (j == 0 || (src[j] >> BR_IDXB) != (src[j - 1] >> BR_IDXB)) first_start = j;
  // inclusive max-scan of last_start over threads, exclusive min-scan (from the right) of first_start
  int mx = last_start, mn = first_start;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, mx, o);
    if (lane >= o) mx = max(mx, y);
    const int z = __shfl_down_sync(0xffffffffu, mn, o);
    if (lane + o < 32) mn = min(mn, z);
  }
  __syncthreads();   // hist / wtot reuse below
  int* wmax = hist;
  int* wmin = hist + BR_NW;
  if (lane == 31) wmax[warp] = mx;
  if (lane == 0) wmin[warp] = mn;
  __syncthreads();
  int before = -1, after = n;   // last start before my chunk / first start after my chunk
  for (int w = 0; w < warp; ++w) before = max(before, wmax[w]);
  for (int w = warp + 1; w < BR_NW; ++w) after = min(after, wmin[w]);
  {
    const int xm = __shfl_up_sync(0xffffffffu, mx, 1);
    if (lane > 0) before = max(before, xm);
    const int xn = __shfl_down_sync(0xffffffffu, mn, 1);
    if (lane < 31) after = min(after, xn);
  }
  // walk the chunk: rs = current run start, re = next run start
  int rs = before;
  int re_next = after;   // first start after the chunk
  // ends: for j in chunk, re = the next start > j: scan backward
  for (int j = j1 - 1; j >= j0; --j) {
    const bool st = (j == 0 || (src[j] >> BR_IDXB) != (src[j - 1] >> BR_IDXB));
    dst[j] = (uint32_t)re_next;        // run end of entry j (dst is free now)
    if (st) re_next = j;
  }
  for (int j = j0; j < j1; ++j) {
    const uint32_t key = src[j];
    if (j == 0 || (key >> BR_IDXB) != (src[j - 1] >> BR_IDXB)) rs = j;
    const int idx = (int)(key & ((1u << BR_IDXB) - 1u));
    int lo = 0, hi = b;                // vertex of incidence idx: vp[lo] <= idx < vp[lo + 1]
    while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (vp[mid] <= idx) lo = mid; else hi = mid; }
    memb[p0 + j] = (uint32_t)lo;
    rng[p0 + idx] = make_int2(rs, (int)dst[j]);
  }
}

__global__ void __launch_bounds__(R2_NT) k_assemble_rows2(int blk0, int b, const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ memb,
                                                          const int2* __restrict__ rng,
                                                          const float* __restrict__ eval,
                                                          const float* __restrict__ dvr, float inv1pmu, int raw,
                                                          float* __restrict__ blocks,
                                                          const int32_t* __restrict__ overflow) {
  const int blk = blk0 + blockIdx.x;
  if (overflow[blk]) return;                      // handled by the hashed-tile kernel
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float* acc = reinterpret_cast<float*>(smem_raw);   // [R2_ROWS][b]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float* stc = reinterpret_cast<float*>(smem_raw + (size_t)R2_ROWS * b * 4) + warp * 32;   // per-warp pair values
  const int64_t base = (int64_t)blk * b;
  const int u0 = blockIdx.y * R2_ROWS;
  const int uu = u0 + warp;
  for (int i = t; i < R2_ROWS * b; i += R2_NT) acc[i] = 0.f;
  __syncthreads();
  if (uu >= b) return;
  const int64_t p0 = row_ptr[base];
  const uint32_t* M = memb + p0;
  float* arow = acc + (size_t)warp * b;
  const int64_t q0 = row_ptr[base + uu], q1 = row_ptr[base + uu + 1];
  for (int64_t c0 = q0; c0 < q1; c0 += 32) {
    const int ne = (int)((q1 - c0) < 32 ? (q1 - c0) : 32);
    float val = 0.f;
    int rs = 0, len = 0;
    if (lane < ne) {
      const int2 r = rng[c0 + lane];
      rs = r.x;
      len = r.y - r.x;
      val = eval[col[c0 + lane]];
    }
    const unsigned heavy = __ballot_sync(0xffffffffu, lane < ne && len >= HEAVY);
    int i = 0;
    while (i < ne) {
      if ((heavy >> i) & 1u) {   // heavy edge: all lanes, distinct members
        const float c = __shfl_sync(0xffffffffu, val, i);
        const int s = __shfl_sync(0xffffffffu, rs, i), l = __shfl_sync(0xffffffffu, len, i);
        int m = lane;
        for (; m + 96 < l; m += 128) {   // four loads in flight
          const uint32_t v0 = M[s + m], v1 = M[s + m + 32], v2 = M[s + m + 64], v3 = M[s + m + 96];
          arow[v0] += c;
          arow[v1] += c;
          arow[v2] += c;
          arow[v3] += c;
        }
        for (; m < l; m += 32) arow[M[s + m]] += c;
        __syncwarp();
        ++i;
        continue;
      }
      // a run of light edges [i, i1): (edge, member) pairs in ascending edge order
      const unsigned hv = heavy & ~((2u << i) - 1u);   // heavy edges after i
      const int i1 = hv ? (__ffs(hv) - 1) : ne;
      const int ln = (lane >= i && lane < i1) ? len : 0;
      int incl = ln;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int q0p = 0; q0p < total; q0p += 32) {
        const int q = q0p + lane;
        // edge of pair q: the first lane with incl > q (binary search over the lanes' prefixes)
        int lo = 0;
#pragma unroll
        for (int st = 16; st; st >>= 1) {
          const int y = __shfl_sync(0xffffffffu, incl, lo + st - 1);
          if (y <= q) lo += st;
        }
        const int ex = __shfl_sync(0xffffffffu, incl - ln, lo & 31);
        const int s = __shfl_sync(0xffffffffu, rs, lo & 31);
        const float c = __shfl_sync(0xffffffffu, val, lo & 31);
        const bool act = q < total;
        const uint32_t v = act ? M[s + (q - ex)] : 0xffffffffu;
        stc[lane] = c;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        __syncwarp();
        if (act) {
          const unsigned m = __match_any_sync(am, v);
          if (lane == __ffs(m) - 1) {   // leader: this v's pairs in ascending edge order
            float x = arow[v];
            unsigned mm = m;
            while (mm) {
              const int l = __ffs(mm) - 1;
              mm &= mm - 1;
              x += stc[l];
            }
            arow[v] = x;
          }
        }
        __syncwarp();
      }
      i = i1;
    }
  }
  __syncwarp();
  const float du = dvr[base + uu];
  float* orow = blocks + (int64_t)blk * b * b + (int64_t)uu * b;
  const float* dv = dvr + base;
  for (int v4 = lane; v4 < b / 4; v4 += 32) {
    const float4 a = *reinterpret_cast<const float4*>(arow + 4 * v4);
    const float4 r = *reinterpret_cast<const float4*>(dv + 4 * v4);
    const int v = 4 * v4;
    float4 o;
    o.x = (du * r.x) * a.x;
    o.y = (du * r.y) * a.y;
    o.z = (du * r.z) * a.z;
    o.w = (du * r.w) * a.w;
    if (!raw) {
      o.x = ((uu == v + 0) ? 1.0f : 0.0f) - o.x * inv1pmu;
      o.y = ((uu == v + 1) ? 1.0f : 0.0f) - o.y * inv1pmu;
      o.z = ((uu == v + 2) ? 1.0f : 0.0f) - o.z * inv1pmu;
      o.w = ((uu == v + 3) ? 1.0f : 0.0f) - o.w * inv1pmu;
    }
    *reinterpret_cast<float4*>(orow + v) = o;
  }
}


// ---------------------------------------------------------------------------
// Grouped assembly (default when nb * E <= GRP_MAX): the incidences of all blocks are grouped
// by (block, edge) once per solve, before the stream parts fork:
//   k_grp_count   cnt[blk][e] = |e n block|                      (atomic counts, thread per vertex)
//   k_grp_scan    start[blk][e] = p0(blk) + sum_{e' < e} cnt[blk][e']  (CTA per block; the block's
//                 members land in its own CSR range), cur = start
//   k_grp_fill    memb[atomicAdd(cur[blk][e], 1)] = block-local vertex   (after it: cur = end)
// so the members of edge e in block blk are memb[start .. cur).  The order inside a run is not
// deterministic and does not matter: an edge contributes one addition to each (u, v), and the
// row walk orders the contributions to one (u, v) by edge (k_assemble_rows3 = k_assemble_rows2
// with these runs).
constexpr int64_t GRP_MAX = 1ll << 26;       // nb * E counters per array

// warp per vertex, lane per incidence
__global__ void k_grp_count(int N, int b, int E, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                            int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < N; v += (gridDim.x * blockDim.x) >> 5) {
    int32_t* cb = cnt + (int64_t)(v / b) * (E + 1);
    const int64_t p1 = row_ptr[v + 1];
    for (int64_t p = row_ptr[v] + lane; p < p1; p += 32) atomicAdd(&cb[col[p]], 1);
  }
}

// CTA per block: exclusive scan of cnt[blk][0..E) (coalesced: warp w scans the w-th contiguous
// segment in 32-entry chunks with a carry), offset by the block's first incidence; rows of E + 1
// entries, the last = the block's end (so edge e's run is [start[e], start[e + 1]))
__global__ void __launch_bounds__(1024) k_grp_scan(int b, int E, const int64_t* __restrict__ row_ptr,
                                                   int32_t* __restrict__ start, int32_t* __restrict__ cur) {
  __shared__ int wsum[32];
  const int blk = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int32_t* st = start + (int64_t)blk * (E + 1);
  int32_t* cu = cur + (int64_t)blk * (E + 1);
  if (t == 0) st[E] = (int)row_ptr[(int64_t)(blk + 1) * b];
  const int seg = (E + 31) / 32;
  const int s0 = warp * seg, s1 = min(E, s0 + seg);
  int tot = 0;
  for (int e = s0 + lane; e < s1; e += 32) tot += st[e];
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0) wsum[warp] = tot;
  __syncthreads();
  int carry = (int)row_ptr[(int64_t)blk * b];
  for (int w = 0; w < warp; ++w) carry += wsum[w];
  for (int e0 = s0; e0 < s1; e0 += 32) {
    const int e = e0 + lane;
    const int c = e < s1 ? st[e] : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (e < s1) {
      st[e] = carry + x - c;
      cu[e] = carry + x - c;
    }
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

// warp per vertex, lane per incidence: memb[cursor++] = the vertex; rng[p] = its edge's run in the block
__global__ void k_grp_fill(int N, int b, int E, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                           const int32_t* __restrict__ start, int32_t* __restrict__ cur, uint32_t* __restrict__ memb,
                           int2* __restrict__ rng) {
  const int lane = threadIdx.x & 31;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < N; v += (gridDim.x * blockDim.x) >> 5) {
    const int64_t off = (int64_t)(v / b) * (E + 1);
    const uint32_t vl = (uint32_t)(v % b);
    const int64_t p1 = row_ptr[v + 1];
    for (int64_t p = row_ptr[v] + lane; p < p1; p += 32) {
      const int e = col[p];
      HG_DCHECK(e >= 0 && e < E);
      const int pos = atomicAdd(&cur[off + e], 1);
      HG_DCHECK(pos < start[off + e + 1]);
      memb[pos] = vl;
      rng[p] = make_int2(start[off + e], start[off + e + 1]);
    }
  }
}

// delta(e) = sum over blocks of |e n block| (no hot-address atomics), w_e / delta(e)
__global__ void k_grp_degree(int nb, int E, const int32_t* __restrict__ cnt, const float* __restrict__ w,
                             int32_t* __restrict__ de, float* __restrict__ val, int32_t* status) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int c = 0;
  for (int i = 0; i < nb; ++i) c += cnt[(int64_t)i * (E + 1) + e];
  de[e] = c;
  if (c == 0) {
    hg_flag(status, HGS_EMPTY_EDGE);
    val[e] = 0.f;
    return;
  }
  const float v = w[e] / (float)c;
  if (!isfinite(v)) hg_flag(status, HGS_NONFINITE);
  val[e] = v;
}

__global__ void __launch_bounds__(R2_NT) k_assemble_rows3(int blk0, int b, const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ memb,
                                                          const int2* __restrict__ rng,
                                                          const float* __restrict__ eval,
                                                          const float* __restrict__ dvr, float inv1pmu, int raw,
                                                          float* __restrict__ blocks, uint16_t* __restrict__ x16) {
  const int blk = blk0 + blockIdx.x;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float* acc = reinterpret_cast<float*>(smem_raw);                                  // [R2_ROWS][b]
  float* dvs = acc + (size_t)R2_ROWS * b;                                           // [b]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float* stc = dvs + b + warp * 32;                                                 // per-warp pair values
  const int64_t base = (int64_t)blk * b;
  const int u0 = blockIdx.y * R2_ROWS;
  const int uu = u0 + warp;
  for (int i = t; i < R2_ROWS * b; i += R2_NT) acc[i] = 0.f;
  for (int i = t; i < b; i += R2_NT) dvs[i] = dvr[base + i];
  __syncthreads();
  if (uu >= b) return;
  float* arow = acc + (size_t)warp * b;
  const int64_t q0 = row_ptr[base + uu], q1 = row_ptr[base + uu + 1];
  for (int64_t c0 = q0; c0 < q1; c0 += 32) {
    const int ne = (int)((q1 - c0) < 32 ? (q1 - c0) : 32);
    float val = 0.f;
    int rs = 0, len = 0;
    if (lane < ne) {
      const int2 r = rng[c0 + lane];
      rs = r.x;
      len = r.y - r.x;
      val = eval[col[c0 + lane]];
    }
    const unsigned heavy = __ballot_sync(0xffffffffu, lane < ne && len >= HEAVY);
    int i = 0;
    while (i < ne) {
      if ((heavy >> i) & 1u) {   // heavy edge: all lanes, distinct members
        const float c = __shfl_sync(0xffffffffu, val, i);
        const int s = __shfl_sync(0xffffffffu, rs, i), l = __shfl_sync(0xffffffffu, len, i);
        const uint32_t* Ms = memb + s;
        HG_DCHECK(s >= row_ptr[base] && s + l <= row_ptr[base + b]);
        int m = lane;
        for (; m + 96 < l; m += 128) {   // four loads in flight
          const uint32_t v0 = Ms[m], v1 = Ms[m + 32], v2 = Ms[m + 64], v3 = Ms[m + 96];
          arow[v0] += c;
          arow[v1] += c;
          arow[v2] += c;
          arow[v3] += c;
        }
        for (; m < l; m += 32) {
          HG_DCHECK(Ms[m] < (uint32_t)b);
          arow[Ms[m]] += c;
        }
        __syncwarp();
        ++i;
        continue;
      }
      // a run of light edges [i, i1): (edge, member) pairs in ascending edge order; the pairs of one
      // v are applied by one lane in that order (the same fp32 additions as edge by edge)
      const unsigned hv = heavy & ~((2u << i) - 1u);
      const int i1 = hv ? (__ffs(hv) - 1) : ne;
      const int ln = (lane >= i && lane < i1) ? len : 0;
      int incl = ln;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int qb = 0; qb < total; qb += 32) {
        const int q = qb + lane;
        int lo = 0;   // the first lane with incl > q
#pragma unroll
        for (int st = 16; st; st >>= 1) {
          const int y = __shfl_sync(0xffffffffu, incl, lo + st - 1);
          if (y <= q) lo += st;
        }
        const int ex = __shfl_sync(0xffffffffu, incl - ln, lo & 31);
        const int s = __shfl_sync(0xffffffffu, rs, lo & 31);
        const float c = __shfl_sync(0xffffffffu, val, lo & 31);
        const bool act = q < total;
        const uint32_t v = act ? memb[s + (q - ex)] : 0xffffffffu;
        HG_DCHECK(!act || (v < (uint32_t)b && s + (q - ex) < row_ptr[base + b]));
        stc[lane] = c;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        __syncwarp();
        if (act) {
          const unsigned mk = __match_any_sync(am, v);
          if (lane == __ffs(mk) - 1) {
            float x = arow[v];
            unsigned mm = mk;
            while (mm) {
              const int l = __ffs(mm) - 1;
              mm &= mm - 1;
              x += stc[l];
            }
            arow[v] = x;
          }
        }
        __syncwarp();
      }
      i = i1;
    }
  }
  __syncwarp();
  const float du = dvs[uu];
  const int64_t ooff = (int64_t)blk * b * b + (int64_t)uu * b;
  float* orow = blocks ? blocks + ooff : nullptr;
#pragma unroll 4
  for (int v4 = lane; v4 < b / 4; v4 += 32) {
    const float4 a = *reinterpret_cast<const float4*>(arow + 4 * v4);
    const float4 r = *reinterpret_cast<const float4*>(dvs + 4 * v4);
    const int v = 4 * v4;
    float4 o;
    o.x = (du * r.x) * a.x;
    o.y = (du * r.y) * a.y;
    o.z = (du * r.z) * a.z;
    o.w = (du * r.w) * a.w;
    if (!raw) {
      o.x = ((uu == v + 0) ? 1.0f : 0.0f) - o.x * inv1pmu;
      o.y = ((uu == v + 1) ? 1.0f : 0.0f) - o.y * inv1pmu;
      o.z = ((uu == v + 2) ? 1.0f : 0.0f) - o.z * inv1pmu;
      o.w = ((uu == v + 3) ? 1.0f : 0.0f) - o.w * inv1pmu;
    }
    if (orow) *reinterpret_cast<float4*>(orow + v) = o;
    if (x16) {   // the 3xF16 twin (tw_off layout), exponent 14 (|X_ij|, |Theta_ij| <= 1)
      const __half2 h01 = __floats2half2_rn(o.x * 16384.f, o.y * 16384.f);
      const __half2 h23 = __floats2half2_rn(o.z * 16384.f, o.w * 16384.f);
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      const __half2 l01 = __floats2half2_rn(o.x * 16384.f - f01.x, o.y * 16384.f - f01.y);
      const __half2 l23 = __floats2half2_rn(o.z * 16384.f - f23.x, o.w * 16384.f - f23.y);
      uint2 hv, lv;
      hv.x = *reinterpret_cast<const uint32_t*>(&h01); hv.y = *reinterpret_cast<const uint32_t*>(&h23);
      lv.x = *reinterpret_cast<const uint32_t*>(&l01); lv.y = *reinterpret_cast<const uint32_t*>(&l23);
      uint16_t* o16 = x16 + tw_off(ooff + v);
      *reinterpret_cast<uint2*>(o16) = hv;
      *reinterpret_cast<uint2*>(o16 + TW_LO) = lv;
    }
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

// keys [nnz] u32 | overflow [nb] i32 | member ranges [nnz][NSEG_MAX] int2 | grouped path: run
// starts [nb][E] i32, run ends [nb][E] i32 (256-byte aligned parts)
static size_t al256(size_t x) { return (x + 255) / 256 * 256; }
bool assemble_grouped(int nb, int E) {
  const char* force = getenv("HG_ASSEMBLE");
  return (int64_t)nb * E <= GRP_MAX && !(force && force[0] != 'g');
}
static size_t grp_off(int64_t nnz, int nb) {
  return al256((size_t)nnz * 4) + al256((size_t)nb * 4) + al256((size_t)nnz * NSEG_MAX * sizeof(int2));
}
size_t assemble_keys_bytes(int64_t nnz, int nb, int E) {
  size_t g = (int64_t)nb * E <= GRP_MAX ? 2 * al256((size_t)nb * (E + 1) * 4) : 0;   // whatever HG_ASSEMBLE says
  return grp_off(nnz, nb) + g + 256;
}

static int32_t* grp_start(void* keys_ws, int64_t nnz, int nb) {
  return reinterpret_cast<int32_t*>(static_cast<char*>(keys_ws) + grp_off(nnz, nb));
}
static int32_t* grp_cur(void* keys_ws, int64_t nnz, int nb, int E) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<char*>(grp_start(keys_ws, nnz, nb)) +
                                    al256((size_t)nb * (E + 1) * 4));
}

// Grouped path: degrees and the (block, edge) grouping of all nb_total blocks, once per
// solve before the stream parts fork (replaces launch_degrees when assemble_grouped(nb_total, E))
cudaError_t launch_degrees_grouped(int nb_total, int b, int E, int64_t nnz, const int64_t* row_ptr,
                                   const int32_t* col_idx, const float* w, int32_t* de_cnt, float* edge_val,
                                   float* dv_rsqrt, int32_t* status, void* keys_ws, cudaStream_t s, int* launches) {
  uint32_t* memb = reinterpret_cast<uint32_t*>(keys_ws);
  int2* rng = reinterpret_cast<int2*>(static_cast<char*>(keys_ws) + al256((size_t)nnz * 4) + al256((size_t)nb_total * 4));
  int32_t* gstart = grp_start(keys_ws, nnz, nb_total);
  int32_t* gcur = grp_cur(keys_ws, nnz, nb_total, E);
  const int N = nb_total * b;
  cudaError_t e = cudaMemsetAsync(gstart, 0, (size_t)nb_total * (E + 1) * 4, s);
  if (e != cudaSuccess) return e;
  const int grid = (int)(((int64_t)N * 32 + 255) / 256 < 148 * 32 ? ((int64_t)N * 32 + 255) / 256 : 148 * 32);
  k_grp_count<<<grid, 256, 0, s>>>(N, b, E, row_ptr, col_idx, gstart);
  k_grp_degree<<<(E + 255) / 256, 256, 0, s>>>(nb_total, E, gstart, w, de_cnt, edge_val, status);
  k_vertex_deg<<<(N + 255) / 256, 256, 0, s>>>(N, row_ptr, col_idx, w, dv_rsqrt, status);
  k_grp_scan<<<nb_total, 1024, 0, s>>>(b, E, row_ptr, gstart, gcur);
  k_grp_fill<<<grid, 256, 0, s>>>(N, b, E, row_ptr, col_idx, gstart, gcur, memb, rng);
  *launches += 5;
  return cudaGetLastError();
}

// keys: nnz uint32 + nb int32 overflow flags (workspace).  E*b must be < 2^32 for the
// sorted path (32-bit keys); otherwise every block takes the hashed-tile kernel.
cudaError_t launch_assemble(int blk0, int nb, int nb_total, int b, int E, int64_t nnz, const int64_t* row_ptr,
                            const int32_t* col_idx, const float* edge_val, const float* dv_rsqrt, float mu,
                            bool raw_theta, float* blocks, void* keys_ws, cudaStream_t s, int* launches,
                            uint16_t* x16, bool skip_f32) {
  uint32_t* keys = reinterpret_cast<uint32_t*>(keys_ws);
  int32_t* overflow = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(keys_ws) + al256((size_t)nnz * 4));
  int2* rng = reinterpret_cast<int2*>(reinterpret_cast<char*>(keys_ws) + al256((size_t)nnz * 4) +
                                      al256((size_t)nb_total * 4));
  // HG_ASSEMBLE=tiles forces the hashed-tile kernel (verification: both paths are bit-identical)
  const char* force = getenv("HG_ASSEMBLE");
  const bool tiles = force && force[0] == 't';
  if (assemble_grouped(nb_total, E)) {   // grouped by launch_degrees_grouped: the row walk only
    const size_t smem = (size_t)R2_ROWS * b * 4 + (size_t)b * 4 + (size_t)R2_ROWS * 32 * 4;
    static size_t attr4 = 0;
    if (smem > attr4) {
      cudaError_t e = cudaFuncSetAttribute(k_assemble_rows3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr4 = smem;
    }
    k_assemble_rows3<<<dim3(nb, (b + R2_ROWS - 1) / R2_ROWS), R2_NT, smem, s>>>(
        blk0, b, row_ptr, col_idx, keys, rng, edge_val, dv_rsqrt, 1.0f / (1.0f + mu), raw_theta ? 1 : 0,
        (x16 && skip_f32) ? nullptr : blocks, x16);
    ++*launches;
    return cudaGetLastError();
  }
  const bool radix_ok = E < (1 << 17) && b <= 2048 && !tiles && !(force && force[0] == 's');
  const bool sorted_ok = (uint64_t)E * (uint64_t)b < (1ull << 32) && b <= 4 * SEG_V && !tiles;
  cudaError_t e = cudaMemsetAsync(overflow + blk0, (radix_ok || sorted_ok) ? 0 : 1, sizeof(int32_t) * nb, s);
  if (e != cudaSuccess) return e;
  if (radix_ok) {
    // per-block radix sort + batched row walk (HG_ASSEMBLE=segments: the segmented path below)
    const size_t ssmem = (size_t)2 * BR_CAP * 4 + 2049 * 4 + 64 * BR_NW * 4 + BR_NW * 4;
    static bool attr0 = false;
    if (!attr0) {
      e = cudaFuncSetAttribute(k_block_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
      if (e != cudaSuccess) return e;
      attr0 = true;
    }
    k_block_sort<<<nb, BR_NT, ssmem, s>>>(blk0, b, row_ptr, col_idx, keys, rng, overflow);
    const size_t smem = (size_t)R2_ROWS * b * 4 + (size_t)R2_ROWS * 32 * 4;
    static size_t attr3 = 0;
    if (smem > attr3) {
      e = cudaFuncSetAttribute(k_assemble_rows2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr3 = smem;
    }
    k_assemble_rows2<<<dim3(nb, (b + R2_ROWS - 1) / R2_ROWS), R2_NT, smem, s>>>(
        blk0, b, row_ptr, col_idx, keys, rng, edge_val, dv_rsqrt, 1.0f / (1.0f + mu), raw_theta ? 1 : 0, blocks,
        overflow);
    *launches += 2;
  } else if (sorted_ok) {
    const int nseg = (b + SEG_V - 1) / SEG_V;
    const size_t ssmem = (size_t)(SEG_V + 2) * 8 + (size_t)SEG_CAP * 4;
    static bool attr1 = false;
    if (!attr1) {
      e = cudaFuncSetAttribute(k_seg_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
      if (e != cudaSuccess) return e;
      attr1 = true;
    }
    k_seg_sort<<<dim3(nb, nseg), 1024, ssmem, s>>>(blk0, b, row_ptr, col_idx, keys, rng, overflow);
    const size_t smem = (size_t)TR_ROWS * b * 4 + (size_t)(ROWS_NT / 32) * STAGE_KEYS * 4;
    static size_t attr2 = 0;
    if (smem > attr2) {
      e = cudaFuncSetAttribute(k_assemble_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr2 = smem;
    }
    k_assemble_rows<<<dim3(nb, (b + TR_ROWS - 1) / TR_ROWS), ROWS_NT, smem, s>>>(
        blk0, b, row_ptr, col_idx, keys, rng, edge_val, dv_rsqrt, 1.0f / (1.0f + mu), raw_theta ? 1 : 0, blocks,
        overflow);
    *launches += 2;
  }
  e = launch_assemble_tiles(blk0, nb, b, row_ptr, col_idx, edge_val, dv_rsqrt, mu, raw_theta, blocks, overflow, s,
                            launches);
  if (e != cudaSuccess || !x16) return e;
  // the other assembly paths write fp32 only: split the part's blocks into the twin afterwards
  const int64_t off = (int64_t)blk0 * b * b;
  ++*launches;
  return launch_f16_split(blocks + off, (int64_t)nb * b, b, b, 14, x16 + 2 * off, s);
}

cudaError_t launch_assemble_tiles(int blk0, int nb, int b, const int64_t* row_ptr, const int32_t* col_idx,
                                  const float* edge_val, const float* dv_rsqrt, float mu, bool raw_theta,
                                  float* blocks, const int32_t* overflow, cudaStream_t s, int* launches) {
  static bool attr = false;
  const int smem = (int)sizeof(AsmSmem);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((b + TV - 1) / TV, (b + TU - 1) / TU, nb);
  k_assemble<<<grid, NT, smem, s>>>(blk0, b, row_ptr, col_idx, edge_val, dv_rsqrt, 1.0f / (1.0f + mu), raw_theta ? 1 : 0,
                                    blocks, overflow);
  ++*launches;
  return cudaGetLastError();
}
