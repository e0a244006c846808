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

#include "common.cuh"
#include "kernels.cuh"

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

// keys [nnz] u32 | overflow [nb] i32 | member ranges [nnz][NSEG_MAX] int2 (256-byte aligned parts)
static size_t al256(size_t x) { return (x + 255) / 256 * 256; }
size_t assemble_keys_bytes(int64_t nnz, int nb) {
  return al256((size_t)nnz * 4) + al256((size_t)nb * 4) + (size_t)nnz * NSEG_MAX * sizeof(int2) + 256;
}

// keys: nnz uint32 + nb int32 overflow flags (workspace).  E*b must be < 2^32 for the
// sorted path (32-bit keys); otherwise every block takes the hashed-tile kernel.
cudaError_t launch_assemble(int blk0, int nb, int nb_total, int b, int E, int64_t nnz, const int64_t* row_ptr,
                            const int32_t* col_idx, const float* edge_val, const float* dv_rsqrt, float mu,
                            bool raw_theta, float* blocks, void* keys_ws, cudaStream_t s, int* launches) {
  uint32_t* keys = reinterpret_cast<uint32_t*>(keys_ws);
  int32_t* overflow = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(keys_ws) + al256((size_t)nnz * 4));
  int2* rng = reinterpret_cast<int2*>(reinterpret_cast<char*>(keys_ws) + al256((size_t)nnz * 4) +
                                      al256((size_t)nb_total * 4));
  // HG_ASSEMBLE=tiles forces the hashed-tile kernel (verification: both paths are bit-identical)
  const char* force = getenv("HG_ASSEMBLE");
  const bool sorted_ok = (uint64_t)E * (uint64_t)b < (1ull << 32) && b <= 4 * SEG_V && !(force && force[0] == 't');
  cudaError_t e = cudaMemsetAsync(overflow + blk0, sorted_ok ? 0 : 1, sizeof(int32_t) * nb, s);
  if (e != cudaSuccess) return e;
  if (sorted_ok) {
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
  return launch_assemble_tiles(blk0, nb, b, row_ptr, col_idx, edge_val, dv_rsqrt, mu, raw_theta, blocks, overflow, s,
                               launches);
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
