// eig.cu -- eigen-preconditioner of the one-sided Jacobi SVD (Alg. 1 step 5).
//
// The Jacobi of jacobi_blk.cu orthogonalises the columns of W = L (B B^T = L L^T):
// W J = U~ Sigma.  Started from W = L it needs 8-9 sweeps on the configs, because
// the singular values of B are tightly clustered (sigma(X_ii) in [theta/(1+theta), 1],
// the top k of them within ~2%: SURVEY.md App. A).  Started from W0 = L J0, where J0
// is an orthogonal approximation of the eigenvectors of A = L^T L (the right singular
// vectors of L), the columns of W0 are already orthogonal to ~fp32 rounding and one
// sweep (a check that rotates little or nothing) finishes ("Jacobi
// preconditioner"; the mixed-precision Jacobi idea: an SVD computed cheaply in
// lower accuracy preconditions the accurate one-sided Jacobi).  The preconditioner
// only changes where the Jacobi starts, not what it converges to: the result is the
// Jacobi's, whatever the quality of J0, as long as J0 is orthogonal -- which the
// CholeskyQR2 after these kernels guarantees (abi.cu).
//
// J0 here (all fp32; deviations from exactness only cost Jacobi rotations):
//   k_sytrd_eig  one CTA per block: Householder tridiagonalisation Q^T A Q = T with
//                the lower triangle of A in shared-memory 32x32 tiles; eigenvalues of T
//                by Sturm bisection; eigenvectors Z of T by inverse iteration (thread
//                per eigenvalue);
//   k_orgtr      Q = H_0 H_1 ... H_{k-3} formed explicitly (stored transposed);
//   then (abi.cu) J0^T = diag(s) (Q Z)^T on the tensor cores, CholeskyQR2.
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int INV_IT = 3;         // inverse iterations per eigenvector

__device__ long long g_eig_clk[32];  // debug: phase clock stamps of block 0 (hg_debug_eig_clocks)
#define EIG_CLK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_eig_clk[i] = clock64(); } while (0)
// steps 0, 64, 128, 192 of the tridiagonalisation: stamps at (b), after (b), after (c), after (c2), after (d)
#define EIG_SCLK(i) do { if ((j & 63) == 0 && j < 256) EIG_CLK(8 + 5 * (j >> 6) + (i)); } while (0)

__host__ __device__ inline int tix(int I, int J) { return I * (I + 1) / 2 + J; }   // lower tile (I >= J)

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic start vector of the inverse iteration for eigenvalue i, in [-1, 1)
__device__ __forceinline__ float start_vec(int r, int i) {
  uint32_t h = (uint32_t)r * 0x9E3779B1u ^ ((uint32_t)i * 0x85EBCA77u + 0x165667B1u);
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  return (float)(h >> 8) * (2.0f / 16777216.0f) - 1.0f;
}

// Number of eigenvalues of the (normalised) tridiagonal T below x: sign changes of the Sturm
// sequence p_0 = 1, p_1 = d_0 - x, p_{i+1} = (d_i - x) p_i - e_{i-1}^2 p_{i-1} (Golub & Van Loan
// §8.4.1), in the division-free three-term form; |d|, e^2 <= ~1 after normalisation, so |p| grows
// by at most ~3^8 between the exact power-of-two rescalings every 8 steps.  An exact zero p_i
// counts one change over the pair (p_{i-1}, p_i, p_{i+1} = -e^2 p_{i-1}) whichever its sign bit.
// d, e2s: shared, 16-byte aligned, e2s[i] = e_{i-1}^2 (e2s[0] = 0), zero-padded to a multiple of 8.
__device__ __forceinline__ int sturm_count(const float* __restrict__ d, const float* __restrict__ e2s, int k, float x) {
  float p0 = 0.f, p1 = 1.f;   // p_{-1}, p_0
  int cnt = 0;
  for (int i0 = 0; i0 < k; i0 += 8) {
    const int n = min(8, k - i0);
    const float4 da = *reinterpret_cast<const float4*>(d + i0), db = *reinterpret_cast<const float4*>(d + i0 + 4);
    const float4 ea = *reinterpret_cast<const float4*>(e2s + i0), eb = *reinterpret_cast<const float4*>(e2s + i0 + 4);
    const float dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
    const float ev[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < n) {
        const float p2 = fmaf(dv[q] - x, p1, -ev[q] * p0);
        cnt += (__float_as_uint(p2) ^ __float_as_uint(p1)) >> 31;
        p0 = p1;
        p1 = p2;
      }
    }
    const float m = fmaxf(fabsf(p0), fabsf(p1));
    const int ex = ((__float_as_int(m) >> 23) & 0xff) - 127;
    if (ex > 48 || (ex < -48 && m != 0.f)) {
      const float sc = __int_as_float((127 - ex) << 23);
      p0 *= sc;
      p1 *= sc;
    }
  }
  return cnt;
}

// ---------------------------------------------------------------- tridiagonalisation
// One CTA per block, 2 tiles of 32x32 per warp held in registers (lane = tile row): the lower
// triangle of A never leaves the register file.  Householder tridiagonalisation (Golub & Van Loan
// Alg. 8.3.1, unblocked, LAPACK sytd2 form: x = A[j+1:, j]; H_j = I - tau v v^T, H_j x = beta e1;
// p = tau A22 v; w = p - (tau/2)(p^T v) v; A22 -= v w^T + w v^T), four block barriers per step:
//   (b) y' = A22 z on the raw column z = A[j+1:, j] (A22 v = s (A22 z - beta A22 e_1), s = 1/(alpha -
//       beta), so the product need not wait for the norm): row part per tile, and for strictly lower
//       tiles the transposed part by a butterfly reduce-scatter across the lanes;
//   (c) Householder scalars (every thread), v, y = A22 v, y^T v;      (c2) w;
//   (d) rank-2 update in registers; the owners of the next two columns publish them (and the next
//       column's norm partials) to shared memory.
// Tiles are listed by tile column J descending, so the trailing tiles of a step are a prefix of the
// list; tile p lives in slot p / NWT of warp p % NWT (the longest-lived tiles spread over all warps).
constexpr int NSLOT = 2;

__host__ __device__ inline int sytrd_warps(int ntl) {
  const int nt = ntl * (ntl + 1) / 2;
  return (nt + NSLOT - 1) / NSLOT;
}

struct TrdSmem {   // offsets in 4-byte words
  int zs, xs2, vs, ws, ys, yrow, ycol, nrm, red, dsc, tl, total;
};
__host__ __device__ inline TrdSmem trd_smem(int ntl) {
  TrdSmem S;
  int off = 0;
  const int nt = ntl * (ntl + 1) / 2, KP = 32 * ntl;
  S.zs = off; off += KP;
  S.xs2 = off; off += KP;
  S.vs = off; off += KP;
  S.ws = off; off += KP;
  S.ys = off; off += KP;
  S.yrow = off; off += nt * 32;
  S.ycol = off; off += nt * 32;
  S.nrm = off; off += 8;
  S.red = off; off += 32;
  S.dsc = off; off += 4;
  S.tl = off; off += nt;
  S.total = off;
  return S;
}

__device__ __forceinline__ float sel32(const float* a, int c) {   // a[c], c warp-uniform, static register indices
  float v = a[0];
#pragma unroll
  for (int i = 1; i < 32; ++i) v = (c == i) ? a[i] : v;
  return v;
}

__global__ void __launch_bounds__(576, 1) k_sytrd(int k, int ntl, const float* __restrict__ A, float* __restrict__ Hv,
                                                  float* __restrict__ tau_out, float* __restrict__ d_out,
                                                  float* __restrict__ e_out) {
  extern __shared__ __align__(16) float sm[];
  const TrdSmem S = trd_smem(ntl);
  float* zs = sm + S.zs;     // column j, rows > j (0 elsewhere)
  float* xs2 = sm + S.xs2;   // column j + 1, rows >= j + 1
  float* vs = sm + S.vs;
  float* ws = sm + S.ws;
  float* ys = sm + S.ys;
  float* yrow = sm + S.yrow;
  float* ycol = sm + S.ycol;
  float* nrm = sm + S.nrm;   // partial sums of squares of column j, rows >= j + 2, per tile row
  float* red = sm + S.red;
  float* dsc = sm + S.dsc;   // A(j, j)
  int* tl = reinterpret_cast<int*>(sm + S.tl);
  const int blk = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int NT = blockDim.x, NWT = NT >> 5;
  const int KP = 32 * ntl, nt = ntl * (ntl + 1) / 2;
  const float* Ab = A + (int64_t)blk * k * k;
  float* Hb = Hv + (int64_t)blk * k * k;
  float* tb = tau_out + (int64_t)blk * k;
  EIG_CLK(0);
  if (t == 0) {
    int a = 0;
    for (int J = ntl - 1; J >= 0; --J)
      for (int I = J; I < ntl; ++I) tl[a++] = I | (J << 8);
  }
  for (int i = t; i < KP; i += NT) { zs[i] = 0.f; xs2[i] = 0.f; vs[i] = 0.f; ws[i] = 0.f; ys[i] = 0.f; }
  if (t < 32) red[t] = 0.f;
  if (t < 8) nrm[t] = 0.f;
  __syncthreads();
  // registers: slot s = tile p = warp + NWT s
  float a[NSLOT][32];
  int tI[NSLOT], tJ[NSLOT];
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    const int p = warp + NWT * s;
    HG_DCHECK(NWT * NSLOT >= nt);
    tI[s] = p < nt ? (tl[p] & 0xff) : 0;
    tJ[s] = p < nt ? (tl[p] >> 8) : 0;
    const int r = 32 * tI[s] + lane;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int cc = 32 * tJ[s] + c;
      float v = 0.f;
      if (p < nt && r < k && cc < k) v = (r >= cc) ? Ab[(int64_t)r * k + cc] : Ab[(int64_t)cc * k + r];
      a[s][c] = v;
    }
  }
  // publish column jn (rows > jn, its diagonal, its norm partials over rows >= jn + 2) and column
  // jn + 1 (rows >= jn + 1) from the registers of the tiles holding them
  auto emit = [&](int jn, int nact) {
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const int p = warp + NWT * s;
      if (p >= nact) continue;
      const int r = 32 * tI[s] + lane;
      if (tJ[s] == (jn >> 5)) {
        const float v = sel32(a[s], jn & 31);
        zs[r] = (r > jn && r < k) ? v : 0.f;
        if (r == jn) dsc[0] = v;
        const float x = (r >= jn + 2 && r < k) ? v : 0.f;
        const float q = warp_sum_f(x * x);
        if (lane == 0) nrm[tI[s]] = q;
      }
      if (jn + 1 < k && tJ[s] == ((jn + 1) >> 5)) {
        const float v = sel32(a[s], (jn + 1) & 31);
        xs2[r] = (r >= jn + 1 && r < k) ? v : 0.f;
      }
    }
  };
  emit(0, nt);
  __syncthreads();
  EIG_CLK(1);

  for (int j = 0; j + 2 < k; ++j) {
    const int t0 = (j + 1) >> 5, ntr = ntl - t0;
    const int nrow = ntr * (ntr + 1) / 2;
    EIG_SCLK(0);
    // (b) y' = A22 z
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const int p = warp + NWT * s;
      if (p >= nrow) continue;
      const int I = tI[s], J = tJ[s], ti = tix(I, J);
      HG_DCHECK(J <= I && I < ntl && ti < nt);
      const float* zJ = zs + 32 * J;
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 z4 = *reinterpret_cast<const float4*>(zJ + 4 * c4);
        acc0 = fmaf(a[s][4 * c4 + 0], z4.x, acc0);
        acc1 = fmaf(a[s][4 * c4 + 1], z4.y, acc1);
        acc0 = fmaf(a[s][4 * c4 + 2], z4.z, acc0);
        acc1 = fmaf(a[s][4 * c4 + 3], z4.w, acc1);
      }
      yrow[ti * 32 + lane] = acc0 + acc1;
      if (I > J) {   // transposed half: lane L <- sum_r a[r][L] z_r (butterfly reduce-scatter)
        const float zl = zs[32 * I + lane];
        float h16[16], h8[8], h4[4], h2[2];
        {
          const bool up = lane & 16;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float lo = a[s][i] * zl, hi = a[s][i + 16] * zl;
            h16[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
          }
        }
        {
          const bool up = lane & 8;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            h8[i] = (up ? h16[i + 8] : h16[i]) + __shfl_xor_sync(0xffffffffu, up ? h16[i] : h16[i + 8], 8);
        }
        {
          const bool up = lane & 4;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            h4[i] = (up ? h8[i + 4] : h8[i]) + __shfl_xor_sync(0xffffffffu, up ? h8[i] : h8[i + 4], 4);
        }
        {
          const bool up = lane & 2;
#pragma unroll
          for (int i = 0; i < 2; ++i)
            h2[i] = (up ? h4[i + 2] : h4[i]) + __shfl_xor_sync(0xffffffffu, up ? h4[i] : h4[i + 2], 2);
        }
        const bool up = lane & 1;
        ycol[ti * 32 + lane] = (up ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, up ? h2[0] : h2[1], 1);
      }
    }
    __syncthreads();
    EIG_SCLK(1);
    // (c) Householder scalars (every thread, fp32), v, y = A22 v, y^T v partials
    float xn2 = 0.f;
    {   // nrm[0..7]: independent loads, tile rows < (j + 2) / 32 masked
      const float4 n0 = *reinterpret_cast<const float4*>(nrm), n1 = *reinterpret_cast<const float4*>(nrm + 4);
      const int i0 = (j + 2) >> 5;
      xn2 = ((i0 <= 0 ? n0.x : 0.f) + (i0 <= 1 ? n0.y : 0.f)) + ((i0 <= 2 ? n0.z : 0.f) + (i0 <= 3 ? n0.w : 0.f)) +
            (((i0 <= 4 && ntl > 4) ? n1.x : 0.f) + ((i0 <= 5 && ntl > 5) ? n1.y : 0.f)) +
            (((i0 <= 6 && ntl > 6) ? n1.z : 0.f) + ((i0 <= 7 && ntl > 7) ? n1.w : 0.f));
    }
    const float alpha = zs[j + 1];
    float beta = alpha, tau = 0.f, scal = 0.f;
    if (xn2 > 0.f) {
      beta = -copysignf(sqrtf(fmaf(alpha, alpha, xn2)), alpha);
      tau = __fdividef(beta - alpha, beta);
      scal = __fdividef(1.f, alpha - beta);
    }
    float dot = 0.f;
    for (int r = t; r < KP; r += NT) {
      float v = 0.f, y = 0.f;
      if (r > j && r < k) {
        const int I = r >> 5, rr = r & 31;
        float yq[16];   // independent loads (static bounds, predicated), then a fixed-order sum
#pragma unroll
        for (int J = 0; J < 8; ++J) yq[J] = (J >= t0 && J <= I) ? yrow[tix(I, J) * 32 + rr] : 0.f;
#pragma unroll
        for (int I2 = 1; I2 < 8; ++I2) yq[7 + I2] = (I2 > I && I2 < ntl) ? ycol[tix(I2, I) * 32 + rr] : 0.f;
        yq[15] = 0.f;
#pragma unroll
        for (int h = 8; h; h >>= 1)
#pragma unroll
          for (int i = 0; i < h; ++i) yq[i] += yq[i + h];
        const float yp = yq[0];
        v = (r == j + 1) ? 1.f : zs[r] * scal;
        y = scal * fmaf(-beta, xs2[r], yp);
      }
      vs[r] = v;
      ys[r] = y;
      if (r < k) Hb[(int64_t)j * k + r] = v;
      dot = fmaf(y, v, dot);
    }
    if (t == 0) {
      d_out[(int64_t)blk * k + j] = dsc[0];
      e_out[(int64_t)blk * k + j] = beta;
      tb[j] = tau;
    }
    dot = warp_sum_f(dot);
    if (lane == 0) red[warp] = dot;
    __syncthreads();
    EIG_SCLK(2);
    if (tau == 0.f) {   // H_j = I (uniform): no update; publish the next columns of A as it is
      emit(j + 1, nrow);
      __syncthreads();
      continue;
    }
    float yv = 0.f;
#pragma unroll
    for (int w4 = 0; w4 < 20; w4 += 4) {   // <= 18 warps; red[NWT..19] are zero
      const float4 q = *reinterpret_cast<const float4*>(red + w4);
      yv += (q.x + q.y) + (q.z + q.w);
    }
    const float Kc = 0.5f * tau * tau * yv;   // w = tau y - (tau^2 / 2)(y^T v) v, formed on the fly below
    EIG_SCLK(3);
    // (d) A22 -= v w^T + w v^T (no FMA contraction: the two products are summed in either order, so
    //     diagonal tiles stay exactly symmetric); publish columns j + 1, j + 2
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const int p = warp + NWT * s;
      if (p >= nrow) continue;
      const int I = tI[s], J = tJ[s];
      const float vr = vs[32 * I + lane], wr = fmaf(tau, ys[32 * I + lane], -Kc * vr);
      const float* vJ = vs + 32 * J;
      const float* yJ = ys + 32 * J;
      auto wq = [&](const float4& v4, const float4& y4) {
        return make_float4(fmaf(tau, y4.x, -Kc * v4.x), fmaf(tau, y4.y, -Kc * v4.y), fmaf(tau, y4.z, -Kc * v4.z),
                           fmaf(tau, y4.w, -Kc * v4.w));
      };
      if (I == J) {
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 v4 = *reinterpret_cast<const float4*>(vJ + 4 * c4);
          const float4 w4 = wq(v4, *reinterpret_cast<const float4*>(yJ + 4 * c4));
          a[s][4 * c4 + 0] = __fsub_rn(a[s][4 * c4 + 0], __fadd_rn(__fmul_rn(vr, w4.x), __fmul_rn(wr, v4.x)));
          a[s][4 * c4 + 1] = __fsub_rn(a[s][4 * c4 + 1], __fadd_rn(__fmul_rn(vr, w4.y), __fmul_rn(wr, v4.y)));
          a[s][4 * c4 + 2] = __fsub_rn(a[s][4 * c4 + 2], __fadd_rn(__fmul_rn(vr, w4.z), __fmul_rn(wr, v4.z)));
          a[s][4 * c4 + 3] = __fsub_rn(a[s][4 * c4 + 3], __fadd_rn(__fmul_rn(vr, w4.w), __fmul_rn(wr, v4.w)));
        }
      } else {   // strictly lower tile: no symmetry to keep, two FMAs per entry
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 v4 = *reinterpret_cast<const float4*>(vJ + 4 * c4);
          const float4 w4 = wq(v4, *reinterpret_cast<const float4*>(yJ + 4 * c4));
          a[s][4 * c4 + 0] = fmaf(-vr, w4.x, fmaf(-wr, v4.x, a[s][4 * c4 + 0]));
          a[s][4 * c4 + 1] = fmaf(-vr, w4.y, fmaf(-wr, v4.y, a[s][4 * c4 + 1]));
          a[s][4 * c4 + 2] = fmaf(-vr, w4.z, fmaf(-wr, v4.z, a[s][4 * c4 + 2]));
          a[s][4 * c4 + 3] = fmaf(-vr, w4.w, fmaf(-wr, v4.w, a[s][4 * c4 + 3]));
        }
      }
    }
    emit(j + 1, nrow);
    __syncthreads();
    EIG_SCLK(4);
  }
  // the last 2x2 (or 1x1) block: d_{k-2}, e_{k-2}, d_{k-1}
  if (t == 0) {
    float* db = d_out + (int64_t)blk * k;
    float* eb = e_out + (int64_t)blk * k;
    const int j = k >= 2 ? k - 2 : 0;
    db[j] = dsc[0];
    if (k >= 2) {
      eb[k - 2] = zs[k - 1];
      db[k - 1] = xs2[k - 1];
      tb[k - 2] = 0.f;
    }
    eb[k - 1] = 0.f;
    tb[k - 1] = 0.f;
  }
  EIG_CLK(2);
}

// ---------------------------------------------------------------- tridiagonalisation, 256 < k <= 512
// The same algorithm as k_sytrd with the lower tiles of A in global scratch (L2-resident; 136 tiles of
// 32 x 32 at k = 512 do not fit in one SM's registers or shared memory): 1024 threads, task lists by
// tile column as in k_sytrd, the transposed half of the product by column tasks (lane = tile column,
// coalesced), the rank-2 update with lane = tile column (coalesced stores).  Vectors in shared memory.
constexpr int BIG_NT = 1024;
constexpr int BIG_NW = BIG_NT / 32;
constexpr int BIG_MAXNTL = 16;

struct BigSmem {   // offsets in 4-byte words
  int vs, ys, yrow, ycol, nrm, red, tl_incl, tl_strict, total;
};
__host__ __device__ inline BigSmem big_smem(int ntl) {
  BigSmem S;
  int off = 0;
  const int nt = ntl * (ntl + 1) / 2, KP = 32 * ntl;
  S.vs = off; off += KP;
  S.ys = off; off += KP;
  S.yrow = off; off += nt * 32;
  S.ycol = off; off += nt * 32;
  S.nrm = off; off += BIG_MAXNTL;
  S.red = off; off += BIG_NW;
  S.tl_incl = off; off += nt;
  S.tl_strict = off; off += nt;
  S.total = off;
  return S;
}

__global__ void __launch_bounds__(BIG_NT, 1) k_sytrd_big(int k, int ntl, const float* __restrict__ A,
                                                         float* __restrict__ tiles, float* __restrict__ Hv,
                                                         float* __restrict__ tau_out, float* __restrict__ d_out,
                                                         float* __restrict__ e_out) {
  extern __shared__ __align__(16) float sm[];
  const BigSmem S = big_smem(ntl);
  float* vs = sm + S.vs;
  float* ys = sm + S.ys;
  float* yrow = sm + S.yrow;
  float* ycol = sm + S.ycol;
  float* nrm = sm + S.nrm;
  float* red = sm + S.red;
  int* tl_incl = reinterpret_cast<int*>(sm + S.tl_incl);
  int* tl_strict = reinterpret_cast<int*>(sm + S.tl_strict);
  const int blk = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int KP = 32 * ntl, nt = ntl * (ntl + 1) / 2;
  const float* Ab = A + (int64_t)blk * k * k;
  float* T = tiles + (int64_t)blk * nt * 1024;   // tile ti at T + ti * 1024, row-major 32 x 32
  float* Hb = Hv + (int64_t)blk * k * k;
  float* tb = tau_out + (int64_t)blk * k;
  EIG_CLK(0);
  auto At = [&](int r, int c) -> float& {   // element (r, c), r >= c or inside a diagonal tile
    return T[tix(r >> 5, c >> 5) * 1024 + (r & 31) * 32 + (c & 31)];
  };
  for (int idx = t; idx < nt * 1024; idx += BIG_NT) {
    const int ti = idx >> 10, rr = (idx >> 5) & 31, cc = idx & 31;
    int I = 0;
    while (tix(I + 1, 0) <= ti) ++I;
    const int J = ti - tix(I, 0);
    const int r = 32 * I + rr, c = 32 * J + cc;
    float v = 0.f;
    if (r < k && c < k) v = (r >= c) ? Ab[(int64_t)r * k + c] : Ab[(int64_t)c * k + r];
    T[idx] = v;
  }
  if (t == 0) {
    int a = 0, b = 0;
    for (int J = ntl - 1; J >= 0; --J)
      for (int I = J; I < ntl; ++I) {
        tl_incl[a++] = I | (J << 8);
        if (I > J) tl_strict[b++] = I | (J << 8);
      }
  }
  for (int i = t; i < KP; i += BIG_NT) { vs[i] = 0.f; ys[i] = 0.f; }
  if (t < BIG_MAXNTL) nrm[t] = 0.f;
  __syncthreads();
  if (warp < ntl) {   // norm partials of column 0 (rows >= 2), one per tile row
    const int r = 32 * warp + lane;
    const float x = (r >= 2 && r < k) ? At(r, 0) : 0.f;
    const float s = warp_sum_f(x * x);
    if (lane == 0) nrm[warp] = s;
  }
  __syncthreads();
  EIG_CLK(1);
  for (int j = 0; j + 2 < k; ++j) {
    const int t0 = (j + 1) >> 5, ntr = ntl - t0, jt = j >> 5, cj = j & 31;
    const int nrow = ntr * (ntr + 1) / 2, nstr = ntr * (ntr - 1) / 2;
    // (b) y' = A22 z, z = column j masked to rows > j
    for (int task = warp; task < nrow + nstr; task += BIG_NW) {
      const bool rowmode = task < nrow;
      const int ij = rowmode ? tl_incl[task] : tl_strict[task - nrow];
      const int I = ij & 0xff, J = ij >> 8, ti = tix(I, J);
      HG_DCHECK(J <= I && I < ntl);
      const float* Tt = T + ti * 1024;
      const int zr = 32 * (rowmode ? J : I) + lane;
      const float zl = (zr > j && zr < k) ? T[tix(zr >> 5, jt) * 1024 + lane * 32 + cj] : 0.f;
      float acc0 = 0.f, acc1 = 0.f;
      if (rowmode) {
        const float* row = Tt + lane * 32;
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          acc0 = fmaf(row[c], __shfl_sync(0xffffffffu, zl, c), acc0);
          acc1 = fmaf(row[c + 1], __shfl_sync(0xffffffffu, zl, c + 1), acc1);
        }
        yrow[ti * 32 + lane] = acc0 + acc1;
      } else {
#pragma unroll
        for (int r = 0; r < 32; r += 2) {
          acc0 = fmaf(Tt[r * 32 + lane], __shfl_sync(0xffffffffu, zl, r), acc0);
          acc1 = fmaf(Tt[(r + 1) * 32 + lane], __shfl_sync(0xffffffffu, zl, r + 1), acc1);
        }
        ycol[ti * 32 + lane] = acc0 + acc1;
      }
    }
    __syncthreads();
    // (c) Householder scalars, v, y = A22 v, y^T v
    float xn2 = 0.f;
    for (int I = (j + 2) >> 5; I < ntl; ++I) xn2 += nrm[I];
    const float alpha = At(j + 1, j);
    float beta = alpha, tau = 0.f, scal = 0.f;
    if (xn2 > 0.f) {
      beta = -copysignf(sqrtf(fmaf(alpha, alpha, xn2)), alpha);
      tau = __fdividef(beta - alpha, beta);
      scal = __fdividef(1.f, alpha - beta);
    }
    float dot = 0.f;
    for (int r = t; r < KP; r += BIG_NT) {
      float v = 0.f, y = 0.f;
      if (r > j && r < k) {
        const int I = r >> 5, rr = r & 31;
        float yp = 0.f;
        for (int J = t0; J <= I; ++J) yp += yrow[tix(I, J) * 32 + rr];
        for (int I2 = I + 1; I2 < ntl; ++I2) yp += ycol[tix(I2, I) * 32 + rr];
        v = (r == j + 1) ? 1.f : At(r, j) * scal;
        y = scal * fmaf(-beta, At(r, j + 1), yp);
      }
      vs[r] = v;
      ys[r] = y;
      if (r < k) Hb[(int64_t)j * k + r] = v;
      dot = fmaf(y, v, dot);
    }
    if (t == 0) {
      d_out[(int64_t)blk * k + j] = At(j, j);
      e_out[(int64_t)blk * k + j] = beta;
      tb[j] = tau;
    }
    dot = warp_sum_f(dot);
    if (lane == 0) red[warp] = dot;
    __syncthreads();
    const int J1 = t0, c1 = (j + 1) & 31;
    if (tau == 0.f) {   // H_j = I: no update; the next column's norm from A as it is
      if (warp < ntl) {
        const int r = 32 * warp + lane;
        const float x = (r >= j + 3 && r < k && warp >= J1) ? At(r, j + 1) : 0.f;
        const float s = warp_sum_f(x * x);
        if (lane == 0) nrm[warp] = s;
      }
      __syncthreads();
      continue;
    }
    float yv = 0.f;
    for (int w = 0; w < BIG_NW; ++w) yv += red[w];
    const float Kc = 0.5f * tau * tau * yv;
    // (d) A22 -= v w^T + w v^T, lane = tile column (coalesced); w = tau y - Kc v formed on the fly; the
    //     warps on tile column J1 accumulate the norm partials of column j + 1 (rows >= j + 3)
    for (int task = warp; task < nrow; task += BIG_NW) {
      const int ij = tl_incl[task];
      const int I = ij & 0xff, J = ij >> 8;
      float* Tt = T + tix(I, J) * 1024;
      const int cg = 32 * J + lane;
      const float vc = vs[cg], wc = fmaf(tau, ys[cg], -Kc * vc);
      float part = 0.f;
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        const int rg = 32 * I + r;
        const float vr = vs[rg], wr = fmaf(tau, ys[rg], -Kc * vr);
        const float a = __fsub_rn(Tt[r * 32 + lane], __fadd_rn(__fmul_rn(vr, wc), __fmul_rn(wr, vc)));
        Tt[r * 32 + lane] = a;
        if (J == J1 && lane == c1 && rg >= j + 3 && rg < k) part = fmaf(a, a, part);
      }
      if (J == J1) {
        const float s = warp_sum_f(part);
        if (lane == 0) nrm[I] = s;
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    float* db = d_out + (int64_t)blk * k;
    float* eb = e_out + (int64_t)blk * k;
    if (k >= 2) {
      db[k - 2] = At(k - 2, k - 2);
      eb[k - 2] = At(k - 1, k - 2);
      tb[k - 2] = 0.f;
    }
    db[k - 1] = At(k - 1, k - 1);
    eb[k - 1] = 0.f;
    tb[k - 1] = 0.f;
  }
  EIG_CLK(2);
}

// ---------------------------------------------------------------- eigenpairs of T
// CTAs of EIG_NT threads, ceil(k / EIG_NT) per block, thread per eigenvalue.  (1) T / tn (tn = max
// |Gershgorin bound|): the division-free Sturm counts stay in range; eigenvectors are unchanged.
// (2) Eigenvalues: two scans of NSCAN Sturm counts (4 points per thread) narrow the interval holding
// the spectrum and bracket every eigenvalue, then each thread bisects to fp32 resolution.
// (3) Eigenvectors: INV_IT steps of inverse iteration from a pseudo-random start (LAPACK gttrf/gtts2
// elimination with partial pivoting, branch-free), the iterate in shared memory, the U rows
// recomputed per SEG-row segment from checkpoints of the forward elimination.
// Out: Z [nb][k][k], column i = the unit eigenvector of the i-th smallest eigenvalue; scale = 1.
constexpr int EIG_NT = 64;
constexpr int SEG = 16;           // inverse iteration: rows per checkpoint segment
constexpr int NSCAN = 256;        // Sturm-count scan points (4 per thread)

struct TdSmem {   // offsets in 4-byte words
  int d, e, e2, cnt, red, ck, xs, total;
};
__host__ __device__ inline TdSmem td_smem(int k) {
  TdSmem S;
  int off = 0;
  const int kp = (k + 7) / 8 * 8, nseg = (k - 1 + SEG - 1) / SEG + 1;
  S.d = off; off += kp;
  S.e = off; off += kp;
  S.e2 = off; off += kp;
  S.cnt = off; off += NSCAN;
  S.red = off; off += 8;
  S.ck = off; off += nseg * 3 * EIG_NT;
  S.xs = off; off += k * EIG_NT;
  S.total = off;
  return S;
}

// Sturm counts at 4 points (shared loads of d, e2s amortised over the points)
__device__ __forceinline__ void sturm_count4(const float* __restrict__ d, const float* __restrict__ e2s, int k,
                                             const float x[4], int cnt[4]) {
  float p0[4], p1[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) { p0[u] = 0.f; p1[u] = 1.f; cnt[u] = 0; }
  for (int i0 = 0; i0 < k; i0 += 8) {
    const int n = min(8, k - i0);
    const float4 da = *reinterpret_cast<const float4*>(d + i0), db = *reinterpret_cast<const float4*>(d + i0 + 4);
    const float4 ea = *reinterpret_cast<const float4*>(e2s + i0), eb = *reinterpret_cast<const float4*>(e2s + i0 + 4);
    const float dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
    const float ev[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < n) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float p2 = fmaf(dv[q] - x[u], p1[u], -ev[q] * p0[u]);
          cnt[u] += (__float_as_uint(p2) ^ __float_as_uint(p1[u])) >> 31;
          p0[u] = p1[u];
          p1[u] = p2;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float m = fmaxf(fabsf(p0[u]), fabsf(p1[u]));
      const int ex = ((__float_as_int(m) >> 23) & 0xff) - 127;
      if (ex > 48 || (ex < -48 && m != 0.f)) {
        const float sc = __int_as_float((127 - ex) << 23);
        p0[u] *= sc;
        p1[u] *= sc;
      }
    }
  }
}

__global__ void __launch_bounds__(EIG_NT) k_trideig(int k, const float* __restrict__ d_in, const float* __restrict__ e_in,
                                                    float* __restrict__ Z, float* __restrict__ scale_out) {
  extern __shared__ __align__(16) float tsm[];
  const TdSmem S = td_smem(k);
  float* d = tsm + S.d;
  float* e = tsm + S.e;
  float* e2 = tsm + S.e2;   // e2[i] = e_{i-1}^2 (the Sturm recurrence's shifted layout), e2[0] = 0
  int* cnt = reinterpret_cast<int*>(tsm + S.cnt);
  float* red = tsm + S.red;
  const int blk = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ev_i = blockIdx.y * EIG_NT + t;   // this thread's eigenvalue index
  const int kp = (k + 7) / 8 * 8;
  for (int i = t; i < kp; i += EIG_NT) {
    d[i] = i < k ? d_in[(int64_t)blk * k + i] : 0.f;
    e[i] = i < k - 1 ? e_in[(int64_t)blk * k + i] : 0.f;
  }
  __syncthreads();
  EIG_CLK(3);
  float gmin = FLT_MAX, gmax = -FLT_MAX;
  for (int i = t; i < k; i += EIG_NT) {
    const float em = i > 0 ? fabsf(e[i - 1]) : 0.f, ep = i < k - 1 ? fabsf(e[i]) : 0.f;
    gmin = fminf(gmin, d[i] - em - ep);
    gmax = fmaxf(gmax, d[i] + em + ep);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    gmin = fminf(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  }
  if (lane == 0) { red[warp] = gmin; red[4 + warp] = gmax; }
  __syncthreads();
  gmin = fminf(red[0], red[1]);
  gmax = fmaxf(red[4], red[5]);
  float tn = fmaxf(fabsf(gmin), fabsf(gmax));
  if (!(tn > 0.f) || !isfinite(tn)) tn = 1.f;
  const float itn = 1.f / tn;
  for (int i = t; i < kp; i += EIG_NT) {
    const float em = (i > 0 && i < k) ? e_in[(int64_t)blk * k + i - 1] * itn : 0.f;
    e2[i] = em * em;
  }
  __syncthreads();
  for (int i = t; i < kp; i += EIG_NT) {
    d[i] *= itn;
    e[i] *= itn;
  }
  __syncthreads();
  const float pad = 4.f * FLT_EPSILON;
  float glo = gmin * itn - pad, ghi = gmax * itn + pad;
  auto pt = [&](float lo_, float hi_, int m) { return lo_ + (hi_ - lo_) * (float)(m + 1) / (float)(NSCAN + 1); };
  for (int pass = 0; pass < 2; ++pass) {
    float xq[4];
    int cq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xq[u] = pt(glo, ghi, 4 * t + u);
    sturm_count4(d, e2, k, xq, cq);
#pragma unroll
    for (int u = 0; u < 4; ++u) cnt[4 * t + u] = cq[u];
    __syncthreads();
    if (pass == 1) break;
    // occupied part: from the last point with count 0 to the first with count k (counts are
    // non-decreasing in x up to rounding; binary searches)
    int a = 0, b = NSCAN;
    while (a < b) { const int m = (a + b) >> 1; if (cnt[m] > 0) b = m; else a = m + 1; }
    const int f0 = a;
    a = 0; b = NSCAN;
    while (a < b) { const int m = (a + b) >> 1; if (cnt[m] >= k) b = m; else a = m + 1; }
    const int fk = a;
    const float nlo = f0 > 0 ? pt(glo, ghi, f0 - 1) : glo;
    const float nhi = fk < NSCAN ? pt(glo, ghi, fk) : ghi;
    __syncthreads();
    glo = nlo;
    ghi = nhi;
  }
  if (ev_i >= k) return;   // no barrier below
  float lo, hi;
  {
    int a = 0, b = NSCAN;   // first scan point with count > ev_i
    while (a < b) { const int m = (a + b) >> 1; if (cnt[m] > ev_i) b = m; else a = m + 1; }
    lo = a > 0 ? pt(glo, ghi, a - 1) : glo;
    hi = a < NSCAN ? pt(glo, ghi, a) : ghi;
  }
  for (int it = 0; it < 40; ++it) {
    const float mid = 0.5f * (lo + hi);
    if (!(mid > lo && mid < hi)) break;   // fp32 resolution
    if (sturm_count(d, e2, k, mid) > ev_i) hi = mid;
    else lo = mid;
  }
  const float lam = 0.5f * (lo + hi);
  EIG_CLK(4);

  // Inverse iteration.  The iterate lives in shared memory (xs[row][thread]); the forward elimination
  // keeps a checkpoint of its working row (w0, w1, rhs) every SEG rows and the back substitution walks
  // the segments from the last, recomputing each segment's U rows into registers.  A segment reads
  // the right-hand sides of rows base + 1 .. base + SEG, the first of the next segment's rows (already
  // overwritten by the new iterate) is carried over in a register.
  const float eps_piv = FLT_EPSILON;   // replaces an exactly zero pivot (T normalised: ||T|| ~ 1)
  float* xs = tsm + S.xs + t;          // xs[r * EIG_NT]
  HG_DCHECK(S.xs + (k - 1) * EIG_NT + EIG_NT <= S.total);
  float* ck = tsm + S.ck + t;          // [seg][3][EIG_NT]
  // one elimination step on rows (r, r + 1) (branch-free partial pivoting): working row (w0, w1 | rw)
  // against row r + 1 (e_r, d_{r+1} - lam, e_{r+1} | ra); returns the U row (1/u0, u1, u2, ru)
  auto elim = [&](int r, float& w0, float& w1, float& rw, float ra) {
    const float a0 = e[r], a1 = d[r + 1] - lam, a2 = e[r + 1];
    const bool pv = fabsf(w0) >= fabsf(a0);
    float den = pv ? w0 : a0;
    if (den == 0.f) den = eps_piv;
    const float inv = __fdividef(1.f, den);
    const float l = (pv ? a0 : w0) * inv;
    const float4 f = make_float4(inv, pv ? w1 : a1, pv ? 0.f : a2, pv ? rw : ra);
    const float n0 = fmaf(-l, pv ? w1 : a1, pv ? a1 : w1);
    const float n1 = pv ? a2 : -l * a2;
    rw = fmaf(-l, pv ? rw : ra, pv ? ra : rw);
    w0 = n0;
    w1 = n1;
    return f;
  };
  for (int r = 0; r < k; ++r) xs[r * EIG_NT] = start_vec(r, ev_i);
  const int nseg = (k - 1 + SEG - 1) / SEG;
  float rscale = 1.f;
  for (int it = 0; it < INV_IT; ++it) {
    float w0 = d[0] - lam, w1 = k > 1 ? e[0] : 0.f, rw = xs[0] * rscale;
    for (int sg = 0; sg < nseg; ++sg) {
      const int base = sg * SEG;
      ck[sg * 3 * EIG_NT] = w0;
      ck[sg * 3 * EIG_NT + EIG_NT] = w1;
      ck[sg * 3 * EIG_NT + 2 * EIG_NT] = rw;
#pragma unroll
      for (int q = 0; q < SEG; ++q)
        if (base + q + 1 < k) elim(base + q, w0, w1, rw, xs[(base + q + 1) * EIG_NT] * rscale);
    }
    if (w0 == 0.f) w0 = eps_piv;
    float x1 = rw / w0, x2 = 0.f;   // x_{r+1}, x_{r+2}
    const float xlast = x1;
    float nrm2 = x1 * x1;
    const int top = (nseg - 1) * SEG + SEG;
    float carry = top < k ? xs[top * EIG_NT] * rscale : 0.f;
    for (int sg = nseg - 1; sg >= 0; --sg) {
      const int base = sg * SEG;
      float rb[SEG];
#pragma unroll
      for (int q = 0; q < SEG - 1; ++q) rb[q] = (base + q + 1 < k) ? xs[(base + q + 1) * EIG_NT] * rscale : 0.f;
      rb[SEG - 1] = carry;
      carry = xs[base * EIG_NT] * rscale;   // row base's right-hand side, for segment sg - 1
      float u0[SEG], u1[SEG], u2[SEG], ru[SEG];
      float sw0 = ck[sg * 3 * EIG_NT], sw1 = ck[sg * 3 * EIG_NT + EIG_NT], srw = ck[sg * 3 * EIG_NT + 2 * EIG_NT];
#pragma unroll
      for (int q = 0; q < SEG; ++q) {
        if (base + q + 1 < k) {
          const float4 f = elim(base + q, sw0, sw1, srw, rb[q]);
          u0[q] = f.x; u1[q] = f.y; u2[q] = f.z; ru[q] = f.w;
        }
      }
#pragma unroll
      for (int q = SEG - 1; q >= 0; --q) {
        const int r = base + q;
        if (r + 1 < k) {
          const float x = (ru[q] - u1[q] * x1 - u2[q] * x2) * u0[q];
          xs[r * EIG_NT] = x;
          nrm2 = fmaf(x, x, nrm2);
          x2 = x1;
          x1 = x;
        }
      }
    }
    xs[(k - 1) * EIG_NT] = xlast;
    rscale = nrm2 > 0.f ? rsqrtf(nrm2) : 0.f;
    EIG_CLK(5 + it);
  }
  float* Zb = Z + (int64_t)blk * k * k;   // [row][k]: column ev_i = this eigenvector
  for (int r = 0; r < k; ++r) Zb[(int64_t)r * k + ev_i] = xs[r * EIG_NT] * rscale;
  scale_out[(int64_t)blk * k + ev_i] = 1.f;
}

// Q^T with Q = H_0 H_1 ... H_{k-3} (LAPACK orgtr, backward accumulation): column c of Q is
// H_0 ... H_{c-1} e_c (H_j e_c = e_c for j >= c), applied from the inside out.  Warp per CPW columns
// (lane = rows lane + 32 s), no block barrier; out[c][r] = Q[r][c].
template <int RPL, int CPW>
__global__ void __launch_bounds__(128) k_orgtr(int k, const float* __restrict__ Hv, const float* __restrict__ tau,
                                               float* __restrict__ Qt) {
  const int blk = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = (blockIdx.y * 4 + warp) * CPW;
  if (c0 >= k) return;
  const float* Hb = Hv + (int64_t)blk * k * k;
  const float* tb = tau + (int64_t)blk * k;
  float z[RPL][CPW];
#pragma unroll
  for (int s = 0; s < RPL; ++s)
#pragma unroll
    for (int q = 0; q < CPW; ++q) z[s][q] = (lane + 32 * s == c0 + q) ? 1.f : 0.f;
  const int jtop = min(k - 3, c0 + CPW - 2);   // the largest j < the warp's largest column
  float vn[RPL];
  auto loadv = [&](int j, float* v) {
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
      v[s] = (j >= 0 && r < k) ? Hb[(int64_t)j * k + r] : 0.f;
    }
  };
  loadv(jtop, vn);
  for (int j = jtop; j >= 0; --j) {
    float v[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) v[s] = vn[s];
    loadv(j - 1, vn);   // prefetch
    const float tj = tb[j];
    if (tj == 0.f) continue;
    const int s0 = (j + 1) >> 5;   // rows <= j: v = 0
    float dot[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) dot[q] = 0.f;
#pragma unroll
    for (int s = 0; s < RPL; ++s)
      if (s >= s0)
#pragma unroll
        for (int q = 0; q < CPW; ++q) dot[q] = fmaf(v[s], z[s][q], dot[q]);
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int q = 0; q < CPW; ++q) dot[q] += __shfl_xor_sync(0xffffffffu, dot[q], o);
#pragma unroll
    for (int q = 0; q < CPW; ++q) dot[q] *= -tj;
#pragma unroll
    for (int s = 0; s < RPL; ++s)
      if (s >= s0)
#pragma unroll
        for (int q = 0; q < CPW; ++q) z[s][q] = fmaf(dot[q], v[s], z[s][q]);
  }
  float* ob = Qt + (int64_t)blk * k * k;
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    if (c0 + q >= k) continue;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
      if (r < k) ob[(int64_t)(c0 + q) * k + r] = z[s][q];
    }
  }
}

}  // namespace

extern "C" int hg_debug_eig_clocks(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_eig_clk, sizeof(g_eig_clk));
}

// per block: tau [k], scale [k], d [k], e [k] (a multiple of 4 floats: 16-byte aligned per part), and for
// k > 256 the lower tiles of A for k_sytrd_big (nt x 32 x 32)
static int big_ntl(int k) { return k > 256 ? (k + 31) / 32 : 0; }
size_t eig_scratch_floats(int k) {
  const size_t ntl = big_ntl(k);
  return ((size_t)4 * k + 3) / 4 * 4 + ntl * (ntl + 1) / 2 * 1024;
}

bool eig_precond_supported(int k) { return k >= 1 && k <= 512; }

cudaError_t launch_eig_precond(int nb, int k, const float* A, float* Hv, float* Z, float* scratch, float* Qt,
                               const float** scale, cudaStream_t s, int* launches) {
  if (!eig_precond_supported(k)) return cudaErrorInvalidValue;
  const int ntl = (k + 31) / 32;
  float* tau = scratch;                         // [nb][k]
  float* sc = scratch + (size_t)nb * k;         // [nb][k]
  float* dd = scratch + (size_t)2 * nb * k;     // [nb][k]
  float* ee = scratch + (size_t)3 * nb * k;     // [nb][k]
  *scale = sc;
  cudaError_t e;
  if (ntl <= 8) {   // k <= 256: register-resident tiles
    const TrdSmem S = trd_smem(ntl);
    k_sytrd<<<nb, 32 * sytrd_warps(ntl), (size_t)S.total * 4, s>>>(k, ntl, A, Hv, tau, dd, ee);
  } else {          // 256 < k <= 512: tiles in (L2-resident) global scratch after d, e
    const size_t smem = (size_t)big_smem(ntl).total * 4;
    e = cudaFuncSetAttribute(k_sytrd_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    float* tiles = scratch + ((size_t)4 * nb * k + 3) / 4 * 4;
    k_sytrd_big<<<nb, BIG_NT, smem, s>>>(k, ntl, A, tiles, Hv, tau, dd, ee);
  }
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t td_bytes = (size_t)td_smem(k).total * 4;
  e = cudaFuncSetAttribute(k_trideig, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)td_bytes);
  if (e != cudaSuccess) return e;
  k_trideig<<<dim3(nb, (k + EIG_NT - 1) / EIG_NT), EIG_NT, td_bytes, s>>>(k, dd, ee, Z, sc);
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const dim3 grid(nb, (k + 31) / 32), grid16(nb, (k + 15) / 16);
  switch (ntl) {
    case 1: k_orgtr<1, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 2: k_orgtr<2, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 3: k_orgtr<3, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 4: k_orgtr<4, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 5: k_orgtr<5, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 6: k_orgtr<6, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 7: k_orgtr<7, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 8: k_orgtr<8, 8><<<grid, 128, 0, s>>>(k, Hv, tau, Qt); break;
    case 9: case 10: case 11: case 12: k_orgtr<12, 4><<<grid16, 128, 0, s>>>(k, Hv, tau, Qt); break;
    default: k_orgtr<16, 4><<<grid16, 128, 0, s>>>(k, Hv, tau, Qt); break;
  }
  ++*launches;
  return cudaGetLastError();
}
