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
// Full path: one CTA (32 warps) per block, the lower triangle held as 32x32
// tiles (row pitch 36: 16-byte aligned rows read as float4 broadcasts) in
// shared memory for k <= 256 (L2-resident global scratch beyond):
//   right-looking tile Cholesky with one-panel lookahead: per panel p, TRSM(i,p) |
//   trailing update, during which warp 0 updates tile (p+1,p+1) first and factors it
//   (POTRF) -- two barriers per panel; tile products are register-blocked half tiles;
//   in-place tile TRTRI (LAPACK trtri order): invert diagonal tiles, then for
//   block columns j = nt-2..0: L_ij <- -(sum_{m=j+1..i} Linv_im L_mj) Linv_jj.
//   (Recursive doubling -- B <- -C^-1 (B A^-1) per 2m x 2m tile block, log2(nt) levels of
//   two register-held product phases -- measured the same 82k cycles at k = 256, not adopted.)
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int NT = 512, NWARP = NT / 32;   // 128 registers/thread: tile rows stay in registers
constexpr int TS = 32, LDT = 36, TILE = TS * LDT;   // 16-byte rows: float4 row broadcasts
constexpr float NEAR_ID_TOL = 1e-4f;

__device__ unsigned long long g_chol_dbg[2];   // [0] near-identity factorizations, [1] full ones
__device__ long long g_chol_clk[64];           // phase timestamps of block 0's last full factorization
#define CHOL_CLK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_chol_clk[i] = clock64(); } while (0)

__device__ __forceinline__ int tidx(int i, int j) { return i * (i + 1) / 2 + j; }   // i >= j

// warp: Cholesky of a 32x32 SPD tile in place (lower triangle); lane = row, the
// row lives in registers and column c is broadcast by shuffles (no smem round trips)
__device__ void tile_potrf(float* T, int lane, int32_t* status, bool& bad) {
  float a[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) a[t] = T[lane * LDT + t];
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float d = __shfl_sync(0xffffffffu, a[c], c);
    if (!(d > 0.f) || !isfinite(d)) {
      bad = true;
      d = 1.f;
    }
    // 1/sqrt(d) from MUFU.RSQ + one Newton step (~1 ulp; the IEEE __fsqrt_rn /
    // __frcp_rn sequences made the 32-step chain ~3x longer), sqrt(d) = d / sqrt(d)
    float inv = rsqrtf(d);
    inv = inv * fmaf(-0.5f * d * inv, inv, 1.5f);
    const float s = d * inv;
    if (lane == c) a[c] = s;
    if (lane > c) a[c] *= inv;
#pragma unroll 31
    for (int l = c + 1; l < TS; ++l) {
      const float v = __shfl_sync(0xffffffffu, a[c], l);   // L[l][c]
      if (lane >= l) a[l] = fmaf(-a[c], v, a[l]);
    }
  }
#pragma unroll
  for (int t = 0; t < TS; ++t) T[lane * LDT + t] = a[t];
  __syncwarp();
  (void)status;
}

// warp: A <- A L^-T (L lower 32x32), lane = row of A (row staged in registers)
__device__ void tile_trsm(float* A, const float* L, int lane) {
  float a[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) a[t] = A[lane * LDT + t];
  const float rd = __frcp_rn(L[lane * LDT + lane]);     // lane c: 1 / L[c][c]
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float x[4] = {a[c], 0.f, 0.f, 0.f};   // four independent chains (fixed order)
#pragma unroll
    for (int t = 0; t < c; ++t) x[t & 3] = fmaf(-a[t], L[c * LDT + t], x[t & 3]);
    a[c] = ((x[0] + x[1]) + (x[2] + x[3])) * __shfl_sync(0xffffffffu, rd, c);
  }
#pragma unroll
  for (int t = 0; t < TS; ++t) A[lane * LDT + t] = a[t];
  __syncwarp();
}

// Register-blocked warp products on 16-row halves of 32x32 tiles (pitch LDT = 36).
// Lane = (rg, cg) = (lane >> 2, lane & 3) owns rows r0 + rg + 8i (i < 2).  Rows are
// interleaved so that the eight row groups fall in distinct 16-byte bank groups
// ((row * 36 / 4) mod 8 = row mod 8): every float4 operand load is conflict-free.
// C[r][c] -= sum_t A[r][t] B[c][t]; lane columns c = cg + 4j (j < 8), B rows float4 over t.
__device__ void tile_sub_abt_h(float* C, const float* A, const float* B, int lane, int r0) {
  const int rg = lane >> 2, cg = lane & 3;
  float acc[2][8];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll 2
  for (int t = 0; t < TS; t += 4) {
    float4 a[2], b[8];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = *reinterpret_cast<const float4*>(A + (r0 + rg + 8 * i) * LDT + t);
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const float4*>(B + (cg + 4 * j) * LDT + t);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[i][j] = fmaf(a[i].x, b[j].x, acc[i][j]);
        acc[i][j] = fmaf(a[i].y, b[j].y, acc[i][j]);
        acc[i][j] = fmaf(a[i].z, b[j].z, acc[i][j]);
        acc[i][j] = fmaf(a[i].w, b[j].w, acc[i][j]);
      }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) C[(r0 + rg + 8 * i) * LDT + cg + 4 * j] -= acc[i][j];
  __syncwarp();
}

// acc[r][c] += sum_t A[r][t] B[t][c] for the lane's rows r0 + rg + 8i and columns
// 8 cg .. 8 cg + 7 (B rows as two float4: the four column groups hit distinct bank groups)
__device__ __forceinline__ void tile_ab_acc_h(float (&acc)[2][8], const float* A, const float* B, int lane, int r0) {
  const int rg = lane >> 2, cg = lane & 3;
#pragma unroll 2
  for (int t = 0; t < TS; t += 4) {
    float4 a[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = *reinterpret_cast<const float4*>(A + (r0 + rg + 8 * i) * LDT + t);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 b0 = *reinterpret_cast<const float4*>(B + (t + u) * LDT + 8 * cg);
      const float4 b1 = *reinterpret_cast<const float4*>(B + (t + u) * LDT + 8 * cg + 4);
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float av = u == 0 ? a[i].x : u == 1 ? a[i].y : u == 2 ? a[i].z : a[i].w;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av, bb[j], acc[i][j]);
      }
    }
  }
}

__device__ __forceinline__ void tile_store_h(float* C, const float (&v)[2][8], int lane, int r0) {
  const int rg = lane >> 2, cg = lane & 3;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float* row = C + (r0 + rg + 8 * i) * LDT + 8 * cg;
    *reinterpret_cast<float4*>(row) = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
    *reinterpret_cast<float4*>(row + 4) = make_float4(v[i][4], v[i][5], v[i][6], v[i][7]);
  }
}

// warp: lower-triangular 32x32 tile inverse in place, as the TRSM above applied to the
// identity: lane r solves row r of I L^-T, i.e. column r of L^-1 (the former column-by-column
// substitution with lane-dependent branches took ~32k cycles per tile, 10x this)
__device__ void tile_trtri(float* T, int lane) {
  float a[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) a[t] = 0.f;
  const float rd = __frcp_rn(T[lane * LDT + lane]);     // lane c: 1 / L[c][c]
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float x[4] = {c == lane ? 1.f : 0.f, 0.f, 0.f, 0.f};   // four independent chains (fixed order)
#pragma unroll
    for (int t = 0; t < c; ++t) x[t & 3] = fmaf(-a[t], T[c * LDT + t], x[t & 3]);
    a[c] = ((x[0] + x[1]) + (x[2] + x[3])) * __shfl_sync(0xffffffffu, rd, c);
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < TS; ++c) T[c * LDT + lane] = a[c];   // L^-1[c][lane]; zero above the diagonal
  __syncwarp();
}

// warps write the full k x k row-major matrix (zeros above the diagonal) from the
// lower tiles: float4 rows when k % 4 == 0 (17.0k cycles at k = 256 vs 18.4k for the
// scalar form); else warp per (tile row, tile column, 8-row slab), lanes = columns
__device__ void store_lower(float* out, const float* tiles, int k, int nt, int warp, int lane) {
  if ((k & 3) == 0) {   // float4 rows: lane covers columns 4 lane .. 4 lane + 3 of a 128-column slab
    const int nq = (k + 127) / 128;
    for (int task = warp; task < k * nq; task += NWARP) {
      const int r = task / nq, c = (task % nq) * 128 + 4 * lane;
      if (c >= k) continue;
      const int i = r / TS, j = c / TS;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j <= i) {
        v = *reinterpret_cast<const float4*>(tiles + (int64_t)tidx(i, j) * TILE + (r % TS) * LDT + c % TS);
        if (c + 0 > r) v.x = 0.f;
        if (c + 1 > r) v.y = 0.f;
        if (c + 2 > r) v.z = 0.f;
        if (c + 3 > r) v.w = 0.f;
      }
      *reinterpret_cast<float4*>(out + (int64_t)r * k + c) = v;
    }
    return;
  }
  for (int task = warp; task < nt * nt * 4; task += NWARP) {
    const int tl = task >> 2, rq = (task & 3) * 8;
    const int i = tl / nt, j = tl % nt;
    const int c = j * TS + lane;
    if (c >= k) continue;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = i * TS + rq + u;
      if (r < k) out[(int64_t)r * k + c] = (c <= r) ? tiles[(int64_t)tidx(i, j) * TILE + (rq + u) * LDT + lane] : 0.f;
    }
  }
}

// SMEM (template): tiles in shared memory (k <= 256) or in the L2 scratch, a compile-time
// choice so that the shared-memory instantiation's tile pointers are provably shared.
template <bool SMEM>
__global__ void __maxnreg__(128) k_cholinv(int k, const float* __restrict__ G, float* __restrict__ Lout,
                                           float* __restrict__ Linv, float* __restrict__ work, int32_t* status,
                                           int opts) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red[NWARP];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nt = (k + TS - 1) / TS;
  const int ntiles = nt * (nt + 1) / 2;
  const int64_t kk = (int64_t)k * k;
  const int64_t off = (int64_t)blockIdx.x * kk;
  const float* Gb = G + off;
  float* Lb = Lout ? Lout + off : nullptr;
  float* Ib = Linv ? Linv + off : nullptr;   // null: factor only (no TRTRI)

  // distance from the identity (near-identity path for the second CholeskyQR pass)
  float emax = 0.f;
  for (int r = warp; r < k; r += NWARP)             // warp per row, lanes over columns (no divisions)
    for (int c = lane; c <= r; c += 32) {           // lower triangle (G symmetric; the Gram GEMM
                                                    // may leave tiles above the diagonal unset)
      const float g = Gb[(int64_t)r * k + c];
      const float e = fabsf(g - (r == c ? 1.f : 0.f));
      emax = fmaxf(emax, isfinite(g) ? e : INFINITY);
    }
  for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  if (lane == 0) red[warp] = emax;
  __syncthreads();
  if (t < 32) {
    float v = t < NWARP ? red[t] : 0.f;   // red holds NWARP partial maxima
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (t == 0) red[0] = v;
  }
  __syncthreads();
  const float E = red[0];
  if (!isfinite(E) && t == 0) hg_flag(status, HGS_NONFINITE);
  if (t == 0) atomicAdd(&g_chol_dbg[E <= NEAR_ID_TOL ? 0 : 1], 1ull);
  if (E <= NEAR_ID_TOL) {
    for (int r = warp; r < k; r += NWARP)
      for (int c = lane; c < k; c += 32) {
        const int64_t i = (int64_t)r * k + c;
        const float g = Gb[i];
        float l, li;
        if (c > r) { l = 0.f; li = 0.f; }
        else if (c == r) { const float e = 0.5f * (g - 1.f); l = 1.f + e; li = 1.f - e; }
        else { l = g; li = -g; }
        if (Lb) Lb[i] = l;
        if (Ib) Ib[i] = li;
      }
    return;
  }

  CHOL_CLK(0);
  float* tiles = SMEM ? sm : work + (int64_t)blockIdx.x * ((int64_t)ntiles * TILE);
  float* temp = SMEM ? sm + (int64_t)ntiles * TILE : sm;   // [nt-1] tiles in shared memory
  auto T = [&](int i, int j) {
    HG_DCHECK(i >= 0 && j >= 0 && j <= i && i < nt);
    return tiles + (int64_t)tidx(i, j) * TILE;
  };

  // Shifted retry (shifted CholeskyQR): if a pivot is <= 0 -- the fp32 Gram of an
  // ill-conditioned Y (e.g. X Omega with k = b, cond ~ 1e4) is numerically
  // indefinite -- factor G + s I with s = 1e-5 max_i G_ii instead.  R_s^T R_s = G + sI
  // keeps span(Y R_s^-1) = span(Y) with cond(Y R_s^-1) <~ sqrt(1/1e-5); the caller's
  // further CholeskyQR passes make it orthonormal.  Only a failed shifted attempt
  // flags HG_ST_CHOL_BREAKDOWN.
  __shared__ int s_bad;
  __shared__ float s_shift;
  for (int attempt = 0; attempt < 2; ++attempt) {
  if (t == 0) {
    s_bad = 0;
    float dmax = 0.f;
    if (attempt == 1)
      for (int i = 0; i < k; ++i) dmax = fmaxf(dmax, Gb[(int64_t)i * k + i]);
    s_shift = attempt == 1 ? 1e-5f * dmax : 0.f;
  }
  __syncthreads();
  const float shift = s_shift;
  // load the lower tiles (padding beyond k = identity): warp per (tile, 8-row slab),
  // lanes = columns, 8 independent coalesced loads in flight per lane
  for (int task = warp; task < ntiles * 4; task += NWARP) {
    const int tl = task >> 2, rq = (task & 3) * 8;
    int i = 0;
    while ((i + 1) * (i + 2) / 2 <= tl) ++i;
    const int j = tl - i * (i + 1) / 2;
    const int c = j * TS + lane;
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = i * TS + rq + u;
      v[u] = (r < k && c < k) ? Gb[(int64_t)r * k + c] + (r == c ? shift : 0.f) : (r == c ? 1.f : 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) tiles[(int64_t)tl * TILE + (rq + u) * LDT + lane] = v[u];
  }
  __syncthreads();

  // ---- right-looking tile Cholesky
  CHOL_CLK(1);
  bool bad = false;
  // one-panel lookahead: warp 0 updates the next diagonal tile first and factors it
  // while the other warps finish the trailing update
  if (warp == 0) {
    tile_potrf(T(0, 0), lane, status, bad);
    if (bad && lane == 0) s_bad = 1;
  }
  __syncthreads();
  for (int p = 0; p < nt; ++p) {
    CHOL_CLK(2 + 3 * p);
    for (int i = p + 1 + warp; i < nt; i += NWARP) tile_trsm(T(i, p), T(p, p), lane);
    __syncthreads();
    CHOL_CLK(3 + 3 * p);
    const int m = nt - p - 1;                       // trailing tiles (i,j), p < j <= i
    if (m > 0) {
      if (warp == 0) {                              // lookahead: tile (p+1, p+1), then POTRF
        tile_sub_abt_h(T(p + 1, p + 1), T(p + 1, p), T(p + 1, p), lane, 0);
        tile_sub_abt_h(T(p + 1, p + 1), T(p + 1, p), T(p + 1, p), lane, 16);
        if (p < 2) CHOL_CLK(30 + 2 * p);
        tile_potrf(T(p + 1, p + 1), lane, status, bad);
        if (p < 2) CHOL_CLK(31 + 2 * p);
        if (bad && lane == 0) s_bad = 1;
      } else {
        const int ntask = (m * (m + 1) / 2 - 1) * 2;  // half tiles, diagonal (p+1, p+1) excluded
        // warps on warp 0's SM sub-partition (warp % 4 == 0) skip the trailing update when
        // opts & 1, so the lookahead POTRF chain does not share its scheduler with them
        const int nw = (opts & 1) ? NWARP - NWARP / 4 : NWARP - 1;
        const int tw = (opts & 1) ? warp - (warp >> 2) - 1 : warp - 1;
        for (int task = ((opts & 1) && (warp & 3) == 0) ? ntask : tw; task < ntask; task += nw) {
          const int w = (task >> 1) + 1;
          int a = 0;
          while ((a + 1) * (a + 2) / 2 <= w) ++a;
          const int b = w - a * (a + 1) / 2;
          const int i = p + 1 + a, j = p + 1 + b;
          tile_sub_abt_h(T(i, j), T(i, p), T(j, p), lane, (task & 1) * 16);
        }
      }
    }
    __syncthreads();
    CHOL_CLK(4 + 3 * p);
  }
  __syncthreads();
  if (!s_bad) break;
  if (attempt == 1 && t == 0) hg_flag(status, HGS_CHOL_BREAKDOWN);
  __syncthreads();
  }

  if (Lb) store_lower(Lb, tiles, k, nt, warp, lane);
  if (!Ib) return;
  // ---- in-place tile TRTRI
  CHOL_CLK(40);
  for (int d = warp; d < nt; d += NWARP) tile_trtri(T(d, d), lane);
  __syncthreads();
  CHOL_CLK(41);
  for (int j = nt - 2; j >= 0; --j) {
    const int dn = nt - 1 - j;
    for (int task = warp; task < dn * 2; task += NWARP) {   // temp[w] = sum_{m=j+1..i} Linv_im L_mj
      const int w = task >> 1, i = j + 1 + w, r0 = (task & 1) * 16;
      float acc[2][8] = {};
      for (int m = j + 1; m <= i; ++m) tile_ab_acc_h(acc, T(i, m), T(m, j), lane, r0);
      tile_store_h(temp + (int64_t)w * TILE, acc, lane, r0);
    }
    __syncthreads();
    for (int task = warp; task < dn * 2; task += NWARP) {   // L_ij <- -temp Linv_jj
      const int w = task >> 1, i = j + 1 + w, r0 = (task & 1) * 16;
      float acc[2][8] = {};
      tile_ab_acc_h(acc, temp + (int64_t)w * TILE, T(j, j), lane, r0);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[a][c] = -acc[a][c];
      tile_store_h(T(i, j), acc, lane, r0);
    }
    __syncthreads();
    CHOL_CLK(42 + (nt - 2 - j));
  }
  CHOL_CLK(60);
  store_lower(Ib, tiles, k, nt, warp, lane);
  __syncthreads();
  CHOL_CLK(61);
}

// ================================================================== k_cholinv2 (k <= 256)
// All 16 warps share every phase (no single-warp tile loops on the critical path):
//   per panel p:  warp 0 factors the diagonal tile (row per lane, the pivot column broadcast
//                 through a double-buffered shared column -- no shuffle chains);
//                 L_ip = A_ip L_pp^-T by forward substitution, a panel row per thread (i > p), then the trailing
//                 update A_ij -= L_ip L_jp^T -- 16-row half-tile units, 4 x 4 outputs per lane,
//                 float4 operand rows (8 LDS.128 per 64 FMA, conflict-free);
//   triangular inverse: D_i = L_ii^-1 (a warp per tile, in parallel), X_ii = D_i, then block columns j = nt-2 .. 0: T_i = sum_{m=j+1..i} X_im L_mj
//                 into the (then free) D area, X_ij = -T_i D_j -- the LAPACK trtri order, in place.
constexpr int NT2 = 512, NW2 = NT2 / 32;

// out[r][c] (op)= sum_t A[r][t] * B[c][t] over one 16-row half tile (rows r0 .. r0 + 15); lane = (rg, cg):
// rows r0 + rg + 4 ii, columns cg + 8 jj.  mode 0: out = acc, 1: out -= acc.  Operands may alias out
// (every lane computes before any lane stores).
__device__ __forceinline__ void half_abt(float* out, const float* A, const float* B, int lane, int r0, int mode) {
  const int rg = lane >> 3, cg = lane & 7;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 2
  for (int t = 0; t < TS; t += 4) {
    float4 a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(A + (r0 + rg + 4 * i) * LDT + t);
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const float4*>(B + (cg + 8 * j) * LDT + t);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][j] = fmaf(a[i].x, b[j].x, acc[i][j]);
        acc[i][j] = fmaf(a[i].y, b[j].y, acc[i][j]);
        acc[i][j] = fmaf(a[i].z, b[j].z, acc[i][j]);
        acc[i][j] = fmaf(a[i].w, b[j].w, acc[i][j]);
      }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float* o = out + (r0 + rg + 4 * i) * LDT + cg + 8 * j;
      *o = mode ? *o - acc[i][j] : acc[i][j];
    }
  __syncwarp();
}

// acc[r][c] += sum_t A[r][t] * B[t][c] over a 16-row half tile; lane = (rg, cg): rows r0 + rg + 4 ii,
// columns 4 cg .. 4 cg + 3 (B rows read as float4: 8 lanes cover one 128-byte row)
__device__ __forceinline__ void half_ab_acc(float (&acc)[4][4], const float* A, const float* B, int lane, int r0) {
  const int rg = lane >> 3, cg = lane & 7;
#pragma unroll 2
  for (int t = 0; t < TS; t += 4) {
    float4 a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(A + (r0 + rg + 4 * i) * LDT + t);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 bv = *reinterpret_cast<const float4*>(B + (t + u) * LDT + 4 * cg);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float av = u == 0 ? a[i].x : u == 1 ? a[i].y : u == 2 ? a[i].z : a[i].w;
        acc[i][0] = fmaf(av, bv.x, acc[i][0]);
        acc[i][1] = fmaf(av, bv.y, acc[i][1]);
        acc[i][2] = fmaf(av, bv.z, acc[i][2]);
        acc[i][3] = fmaf(av, bv.w, acc[i][3]);
      }
    }
  }
}

__device__ __forceinline__ void half_store(float* out, const float (&acc)[4][4], int lane, int r0, float sign) {
  const int rg = lane >> 3, cg = lane & 7;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<float4*>(out + (r0 + rg + 4 * i) * LDT + 4 * cg) =
        make_float4(sign * acc[i][0], sign * acc[i][1], sign * acc[i][2], sign * acc[i][3]);
}

// warp: Cholesky of the 32 x 32 tile T in place (lower; zeros written above the diagonal); the reciprocal
// diagonal 1 / L_cc goes to rdiag[c].  Row per lane; the scaled pivot column is published through colbuf
// (two 32-float buffers, alternating) and read back as float4 broadcasts.
__device__ void diag_potrf(float* T, float* rdiag, float* colbuf, int lane, bool& bad) {
  float a[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) a[t] = T[lane * LDT + t];
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float d = __shfl_sync(0xffffffffu, a[c], c);
    if (!(d > 0.f) || !isfinite(d)) {
      bad = true;
      d = 1.f;
    }
    float inv = rsqrtf(d);
    inv = inv * fmaf(-0.5f * d * inv, inv, 1.5f);
    if (lane == c) {
      a[c] = d * inv;
      rdiag[c] = inv;
    }
    if (lane > c) a[c] *= inv;
    float* cb = colbuf + (c & 1) * TS;
    cb[lane] = a[c];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TS / 4; ++q) {
      if (4 * q + 3 <= c) continue;   // compile-time (c unrolled): only the quads past the pivot
      const float4 v = *reinterpret_cast<const float4*>(cb + 4 * q);
      const float cv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int l = 4 * q + u;
        if (l > c && lane >= l) a[l] = fmaf(-a[c], cv[u], a[l]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < TS; ++t) T[lane * LDT + t] = (t <= lane) ? a[t] : 0.f;
  __syncwarp();
}

// warp: Dt = L^-1 of the factored 32 x 32 tile T (lower, zeros above): lane r solves row r of I L^-T =
// column r of L^-1 (four independent FMA chains)
__device__ void diag_inverse(const float* T, float* Dt, int lane) {
  float x[TS];
  const float rd = __frcp_rn(T[lane * LDT + lane]);
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float y[4] = {c == lane ? 1.f : 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < c; ++t) y[t & 3] = fmaf(-x[t], T[c * LDT + t], y[t & 3]);
    x[c] = ((y[0] + y[1]) + (y[2] + y[3])) * __shfl_sync(0xffffffffu, rd, c);
  }
#pragma unroll
  for (int c = 0; c < TS; ++c) Dt[c * LDT + lane] = x[c];   // D[c][lane]; zero above the diagonal
  __syncwarp();
}

// thread: row A (32 floats, in place) <- A L^-T for the factored lower tile L (forward substitution along the
// row: x_c = (a_c - sum_{t<c} x_t L_ct) / L_cc; L rows are warp-wide broadcasts, four FMA chains per entry)
__device__ __forceinline__ void row_trsm(float* A, const float* L, const float* rdiag) {
  float x[TS];
#pragma unroll
  for (int q = 0; q < TS / 4; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(A + 4 * q);
    x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float y[4] = {x[c], 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; 4 * q < c; ++q) {
      const float4 l = *reinterpret_cast<const float4*>(L + c * LDT + 4 * q);
      const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (4 * q + u < c) y[u] = fmaf(-x[4 * q + u], lv[u], y[u]);
    }
    x[c] = ((y[0] + y[1]) + (y[2] + y[3])) * rdiag[c];
  }
#pragma unroll
  for (int q = 0; q < TS / 4; ++q)
    *reinterpret_cast<float4*>(A + 4 * q) = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
}

__global__ void __launch_bounds__(NT2, 1) k_cholinv2(int k, const float* __restrict__ G, float* __restrict__ Lout,
                                                     float* __restrict__ Linv, int32_t* status) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red[NW2];
  __shared__ __align__(16) float colbuf[2 * TS];
  __shared__ float rdiag[TS];
  __shared__ int s_bad;
  __shared__ float s_shift;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nt = (k + TS - 1) / TS;
  const int ntiles = nt * (nt + 1) / 2;
  const int64_t off = (int64_t)blockIdx.x * k * k;
  const float* Gb = G + off;
  float* Lb = Lout ? Lout + off : nullptr;
  float* Ib = Linv ? Linv + off : nullptr;
  float* tiles = sm;                                   // [ntiles][TILE] lower tiles
  float* dti = sm + (int64_t)ntiles * TILE;            // [nt][TILE]: D_p, then the trtri temporaries
  auto T = [&](int i, int j) { return tiles + (int64_t)tidx(i, j) * TILE; };
  auto D = [&](int i) { return dti + (int64_t)i * TILE; };
  CHOL_CLK(0);

  for (int attempt = 0; attempt < 2; ++attempt) {
    if (t == 0) {
      s_bad = 0;
      float dmax = 0.f;
      if (attempt == 1)
        for (int i = 0; i < k; ++i) dmax = fmaxf(dmax, Gb[(int64_t)i * k + i]);
      s_shift = attempt == 1 ? 1e-5f * dmax : 0.f;
    }
    __syncthreads();
    const float shift = s_shift;
    // load the lower tiles as float4 rows (identity padding beyond k) and measure max|G - I|
    float emax = 0.f;
    for (int task = t; task < ntiles * TS * 8; task += NT2) {
      const int tl = task >> 8, r = (task >> 3) & 31, c4 = task & 7;
      int i = 0;
      while ((i + 1) * (i + 2) / 2 <= tl) ++i;
      const int j = tl - i * (i + 1) / 2;
      const int R = i * TS + r, C = j * TS + 4 * c4;
      float4 v;
      if (R < k && C < k) {
        v = *reinterpret_cast<const float4*>(Gb + (int64_t)R * k + C);
      } else {
        v = make_float4(R == C ? 1.f : 0.f, R == C + 1 ? 1.f : 0.f, R == C + 2 ? 1.f : 0.f, R == C + 3 ? 1.f : 0.f);
      }
      const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (C + u <= R && R < k) {
          const float e = fabsf(e4[u] - (R == C + u ? 1.f : 0.f));
          emax = fmaxf(emax, isfinite(e4[u]) ? e : INFINITY);
        }
      if (shift != 0.f) {
        if (R == C) v.x += shift;
        if (R == C + 1) v.y += shift;
        if (R == C + 2) v.z += shift;
        if (R == C + 3) v.w += shift;
      }
      *reinterpret_cast<float4*>(tiles + (int64_t)tl * TILE + r * LDT + 4 * c4) = v;
    }
    if (attempt == 0) {
      for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
      if (lane == 0) red[warp] = emax;
      __syncthreads();
      float E = 0.f;
#pragma unroll
      for (int w = 0; w < NW2; ++w) E = fmaxf(E, red[w]);
      if (!isfinite(E) && t == 0) hg_flag(status, HGS_NONFINITE);
      if (t == 0) atomicAdd(&g_chol_dbg[E <= NEAR_ID_TOL ? 0 : 1], 1ull);
      if (E <= NEAR_ID_TOL) {   // second CholeskyQR pass: first-order factor from the tiles
        for (int task = t; task < k * (k / 4); task += NT2) {
          const int r = task / (k / 4), c = 4 * (task % (k / 4));
          const int i = r / TS, j = c / TS;
          float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
          if (j <= i) g = *reinterpret_cast<const float4*>(T(i, j) + (r % TS) * LDT + c % TS);
          const float gv[4] = {g.x, g.y, g.z, g.w};
          float l[4], li[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cc = c + u;
            if (cc > r) { l[u] = 0.f; li[u] = 0.f; }
            else if (cc == r) { const float e = 0.5f * (gv[u] - 1.f); l[u] = 1.f + e; li[u] = 1.f - e; }
            else { l[u] = gv[u]; li[u] = -gv[u]; }
          }
          if (Lb) *reinterpret_cast<float4*>(Lb + (int64_t)r * k + c) = make_float4(l[0], l[1], l[2], l[3]);
          if (Ib) *reinterpret_cast<float4*>(Ib + (int64_t)r * k + c) = make_float4(li[0], li[1], li[2], li[3]);
        }
        return;
      }
    }
    __syncthreads();
    CHOL_CLK(1);

    // ---- right-looking Cholesky, panel width 32
    bool bad = false;
    for (int p = 0; p < nt; ++p) {
      CHOL_CLK(2 + 3 * p);
      if (warp == 0) {
        diag_potrf(T(p, p), rdiag, colbuf, lane, bad);
        if (bad && lane == 0) s_bad = 1;
      }
      __syncthreads();
      CHOL_CLK(3 + 3 * p);
      const int m = nt - 1 - p;
      // L_ip = A_ip L_pp^-T by forward substitution, one panel row per thread (no diagonal inverse on the
      // panel chain: the eight D_i the triangular inverse needs are formed in parallel after the loop)
      if (t < m * TS) row_trsm(T(p + 1 + (t >> 5), p) + (t & 31) * LDT, T(p, p), rdiag);
      __syncthreads();
      CHOL_CLK(4 + 3 * p);
      const int nu = m * (m + 1);                  // half tiles of the trailing lower tiles
      for (int u = warp; u < nu; u += NW2) {
        const int w = u >> 1;
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= w) ++a;
        const int b = w - a * (a + 1) / 2;
        const int i = p + 1 + a, j = p + 1 + b;
        half_abt(T(i, j), T(i, p), T(j, p), lane, (u & 1) * 16, 1);
      }
      __syncthreads();
    }
    if (!s_bad) break;
    if (attempt == 1 && t == 0) hg_flag(status, HGS_CHOL_BREAKDOWN);
    __syncthreads();
  }
  CHOL_CLK(40);

  if (Lb) store_lower(Lb, tiles, k, nt, warp, lane);
  if (!Ib) return;
  // ---- D_i = L_ii^-1, one warp per diagonal tile
  for (int i = warp; i < nt; i += NW2) diag_inverse(T(i, i), D(i), lane);
  __syncthreads();
  // ---- triangular inverse in place: X_ii = D_i; columns j = nt-2 .. 0
  for (int task = t; task < nt * TS * 8; task += NT2) {
    const int i = task >> 8, r = (task >> 3) & 31, c4 = task & 7;
    *reinterpret_cast<float4*>(T(i, i) + r * LDT + 4 * c4) = *reinterpret_cast<const float4*>(D(i) + r * LDT + 4 * c4);
  }
  __syncthreads();
  CHOL_CLK(41);
  for (int j = nt - 2; j >= 0; --j) {
    const int dn = nt - 1 - j;
    for (int u = warp; u < 2 * dn; u += NW2) {     // T_i = sum_{m=j+1..i} X_im L_mj  -> D area
      const int i = j + 1 + (u >> 1), r0 = (u & 1) * 16;
      float acc[4][4] = {};
      for (int mm = j + 1; mm <= i; ++mm) half_ab_acc(acc, T(i, mm), T(mm, j), lane, r0);
      half_store(D(i - j - 1), acc, lane, r0, 1.f);
    }
    __syncthreads();
    for (int u = warp; u < 2 * dn; u += NW2) {     // X_ij = -T_i X_jj
      const int i = j + 1 + (u >> 1), r0 = (u & 1) * 16;
      float acc[4][4] = {};
      half_ab_acc(acc, D(i - j - 1), T(j, j), lane, r0);
      half_store(T(i, j), acc, lane, r0, -1.f);
    }
    __syncthreads();
  }
  CHOL_CLK(60);
  store_lower(Ib, tiles, k, nt, warp, lane);
  CHOL_CLK(61);
}

}  // namespace

cudaError_t chol_clocks(long long* out) { return cudaMemcpyFromSymbol(out, g_chol_clk, sizeof(g_chol_clk)); }

cudaError_t chol_debug(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_chol_dbg, sizeof(g_chol_dbg));
  if (e == cudaSuccess && reset) {
    unsigned long long z[2] = {0, 0};
    e = cudaMemcpyToSymbol(g_chol_dbg, z, sizeof z);
  }
  return e;
}

size_t cholinv_work_floats(int k) {
  const int nt = (k + TS - 1) / TS;
  return (size_t)nt * (nt + 1) / 2 * TILE;
}

cudaError_t launch_cholinv(int nb, int k, const float* G, float* L, float* Linv, float* work, int32_t* status,
                           cudaStream_t s, int* launches) {
  const int nt = (k + TS - 1) / TS;
  const size_t tiles_bytes = cholinv_work_floats(k) * sizeof(float);
  const size_t temp_bytes = (size_t)(nt > 1 ? nt - 1 : 1) * TILE * sizeof(float);
  const bool smem_tiles = tiles_bytes + temp_bytes <= 200 * 1024;
  const size_t smem = (smem_tiles ? tiles_bytes : 0) + temp_bytes;
  static size_t attr[2] = {0, 0};
  if (smem > 48 * 1024 && smem > attr[smem_tiles]) {
    cudaError_t e = smem_tiles
                        ? cudaFuncSetAttribute(k_cholinv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                        : cudaFuncSetAttribute(k_cholinv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[smem_tiles] = smem;
  }
  // k <= 256: the all-warps kernel (HG_CHOL_V1=1: the single-warp-tile kernel below)
  static const bool v1 = getenv("HG_CHOL_V1") && getenv("HG_CHOL_V1")[0] == '1';
  if (nt <= 8 && !v1) {
    const size_t sm2 = (size_t)(nt * (nt + 1) / 2 + nt) * TILE * sizeof(float);
    static size_t attr2 = 0;
    if (sm2 > 48 * 1024 && sm2 > attr2) {
      cudaError_t e = cudaFuncSetAttribute(k_cholinv2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      if (e != cudaSuccess) return e;
      attr2 = sm2;
    }
    k_cholinv2<<<nb, NT2, sm2, s>>>(k, G, L, Linv, status);
    ++*launches;
    return cudaGetLastError();
  }
  // opts bit 0 (HG_CHOL_OPTS, default 1): lookahead warp alone on its sub-partition (see the panel loop)
  static const int dbg = getenv("HG_CHOL_OPTS") ? atoi(getenv("HG_CHOL_OPTS")) : 1;
  if (smem_tiles) k_cholinv<true><<<nb, NT, smem, s>>>(k, G, L, Linv, work, status, dbg);
  else k_cholinv<false><<<nb, NT, smem, s>>>(k, G, L, Linv, work, status, dbg);
  ++*launches;
  return cudaGetLastError();
}
