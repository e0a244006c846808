// jacobi_blk.cu -- Alg. 1 step 5: one-sided (Hestenes) Jacobi on
// W = L^T (k x k, B B^T = L L^T), organised in column blocks.
//
// Same rotations as the scalar cyclic method (jacobi.cu): every column pair
// (p, q) is visited once per sweep and rotated by the angle that zeroes its 2x2
// Gram [[a_pp, a_pq], [a_pq, a_qq]] while |a_pq| > tol sqrt(a_pp a_qq); the
// sweep loop stops after a sweep without rotations.  What changes is the data
// movement.  Columns are grouped in blocks of BW; an outer round pairs blocks
// (I, J) by a round-robin tournament (nblk - 1 rounds), plus one "diagonal"
// round for the pairs inside each block:
//   1. each CTA of the cluster forms, for every block pair, the PW x PW
//      (PW = 2 BW) partial Gram [W_I W_J]^T [W_I W_J] of row chunks of its row
//      slab (register-blocked 4x4 tiles, fixed chunk order: deterministic);
//   2. the pair's owner CTA sums the partials (DSMEM) and runs the scalar
//      rotations on that small fp64 Gram -- BW rounds of BW disjoint cross pairs
//      (p in I, q in J), or BW-1 tournament rounds inside I and J -- applying
//      each to the Gram (two-sided) and accumulating them in a PW x PW Q;
//   3. every CTA applies [W_I W_J] <- [W_I W_J] Q to its rows.
// Cluster rounds per sweep: k/BW instead of k - 1; the Gram and the update are
// register-blocked products instead of per-pair dot products.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int NT = 512;
constexpr int MAX_SWEEPS = 40;
constexpr size_t SMEM_CAP = 220 * 1024;

__device__ unsigned long long g_jb_dbg[3];   // [0] max sweeps, [1] total sweeps, [2] blocks
__device__ long long g_jb_clk[16];           // block 0 / rank 0 / thread 0: sweep 1, outer rounds 0-3
#define JB_CLK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0 && sweep == 1 && ro < 4) g_jb_clk[(i) + 4 * ro] = clock64(); } while (0)

__device__ __forceinline__ void cluster_barrier_jb() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// round-robin tournament on n players (n even): round r, pair i
__device__ __forceinline__ void tourn(int r, int i, int n, int& p, int& q) {
  const int n1 = n - 1;
  if (i == 0) { p = 0; q = 1 + r; return; }
  int x = r + i, y = r - i + n1;
  if (x >= n1) x -= n1;
  if (y >= n1) y -= n1;
  p = 1 + x;
  q = 1 + y;
}

__device__ __forceinline__ uint32_t mapa(const void* local, int rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
__device__ __forceinline__ void st_cluster_f32(float* local_addr, int rank, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(mapa(local_addr, rank)), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_s32(int* local_addr, int rank, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(mapa(local_addr, rank)), "r"(v) : "memory");
}
__device__ __forceinline__ float4 ld_cluster_f4(const float* local_addr, int rank) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(mapa(local_addr, rank))
               : "memory");
  return v;
}

template <int BW>
struct JB {
  static constexpr int PW = 2 * BW;                  // pair width
  static constexpr int LDQ = PW + 4;                 // 16-byte rows
  static constexpr int PACK = PW * (PW + 1) / 2;     // upper-packed PW x PW
  static constexpr int N4 = PW / 4;                  // 4x4 tiles per dimension
  static constexpr int UT = N4 * (N4 + 1) / 2;       // upper 4x4 tiles
  static constexpr int MAXOWN = 8;
  static constexpr int NQB = 4;                      // Q matrices staged per apply chunk
  __host__ __device__ static int pk(int a, int b) { return a * PW - (a * (a - 1)) / 2 + (b - a); }   // a <= b
};

struct Layout {
  int K2, nblk, Pb, R, nch, rch, ldw, nown, gs;
  size_t offW, offGp, offG, offQ, offQb, offJ, offF, total;
};

template <int BW>
__host__ __device__ inline Layout make_layout(int k, int C) {
  using P = JB<BW>;
  Layout L;
  L.K2 = (k + P::PW - 1) / P::PW * P::PW;
  L.nblk = L.K2 / BW;
  L.Pb = L.nblk / 2;
  L.R = ((k + C - 1) / C + 3) / 4 * 4;
  L.ldw = L.K2 + 4;
  L.nown = (L.Pb + C - 1) / C;
  int np2 = 1;
  while (np2 < L.nown) np2 <<= 1;
  L.gs = NT / np2;                                   // threads per owned pair
  // partial Grams over row chunks of 32 (more Gram tasks); one chunk if shared memory is short
  for (int pass = 0; pass < 2; ++pass) {
    L.rch = pass == 0 ? 32 : L.R;
    L.nch = (L.R + L.rch - 1) / L.rch;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) / 16 * 16; return o; };
    L.offW = take((size_t)L.R * L.ldw * 4);
    L.offGp = take((size_t)C * L.nch * L.nown * P::PACK * 4);
    L.offG = take((size_t)L.nown * P::PW * P::LDQ * 8);   // fp64 inner Gram
    L.offQ = take((size_t)L.nown * P::PW * P::LDQ * 4);
    L.offQb = take((size_t)P::NQB * P::PW * P::LDQ * 4);
    L.offJ = take((size_t)P::MAXOWN * P::PW * 16);
    L.offF = take((size_t)128 * 4);
    L.total = off;
    if (L.total <= SMEM_CAP) break;
  }
  return L;
}

template <int BW>
__global__ void __launch_bounds__(NT, 1) k_jacobi_blk(int k, int C, double tol, const float* __restrict__ L,
                                                      float* __restrict__ Wf, int32_t* status, int w_is_l) {
  using P = JB<BW>;
  constexpr int PW = P::PW, LDQ = P::LDQ, PACK = P::PACK, N4 = P::N4, UT = P::UT, NQB = P::NQB;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const Layout Lo = make_layout<BW>(k, C);
  int rank = 0;
  if (C > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int blk = blockIdx.x / C;
  const int nblk = Lo.nblk, Pb = Lo.Pb, R = Lo.R, ldw = Lo.ldw, nown = Lo.nown, nch = Lo.nch, rch = Lo.rch;
  const int GS = Lo.gs;
  const int r0 = rank * R;
  const int nr = max(0, min(R, k - r0));
  float* W = reinterpret_cast<float*>(smem_raw + Lo.offW);
  float* Gp = reinterpret_cast<float*>(smem_raw + Lo.offGp);     // [C][nch][nown][PACK]
  double* Gw = reinterpret_cast<double*>(smem_raw + Lo.offG);    // [nown][PW][LDQ]
  float* Qw = reinterpret_cast<float*>(smem_raw + Lo.offQ);      // [nown][PW][LDQ]
  float* Qb = reinterpret_cast<float*>(smem_raw + Lo.offQb);     // [NQB][PW][LDQ]
  int* Jp = reinterpret_cast<int*>(smem_raw + Lo.offJ);          // [MAXOWN][PW] partner
  float* Jd = reinterpret_cast<float*>(Jp + P::MAXOWN * PW);     // [MAXOWN][PW] J[a][a]
  float* Jo = Jd + P::MAXOWN * PW;                               // [MAXOWN][PW] J[partner][a]
  int* Jact = reinterpret_cast<int*>(Jo + P::MAXOWN * PW);       // [MAXOWN]
  int* flag = reinterpret_cast<int*>(smem_raw + Lo.offF);        // [Pb] rotated-this-round
  const int t = threadIdx.x;
  const double tol2 = tol * tol;
  const float* Lb = L + (int64_t)blk * k * k;

  for (int i = t; i < R * ldw; i += NT) {
    const int rl = i / ldw, c = i % ldw;
    W[i] = (rl < nr && c < k) ? Lb[w_is_l ? (int64_t)(r0 + rl) * k + c : (int64_t)c * k + (r0 + rl)] : 0.f;
  }
  __syncthreads();

  auto colof = [&](int a, int I, int J) { return a < BW ? BW * I + a : BW * J + (a - BW); };
  auto blocks_of = [&](int ro, int g, int& I, int& J) {
    if (ro == nblk - 1) { I = 2 * g; J = 2 * g + 1; }   // diagonal round: within-block pairs
    else tourn(ro, g, nblk, I, J);
  };

  int sweep = 0;
  bool converged = false;
  for (; sweep < MAX_SWEEPS && !converged; ++sweep) {
    int any = 0;
    for (int ro = 0; ro < nblk; ++ro) {
      const bool diag = (ro == nblk - 1);
      JB_CLK(0);
      // ---- 1. partial Grams: (pair, upper 4x4 tile, row chunk) -> owner's Gp[rank][chunk][slot]
      for (int task = t; task < Pb * UT * nch; task += NT) {
        const int ch = task % nch, pt = task / nch;
        const int g = pt / UT;
        int tt = pt % UT, ta = 0;
        while (tt >= N4 - ta) { tt -= N4 - ta; ++ta; }
        const int tb = ta + tt;
        int I, J;
        blocks_of(ro, g, I, J);
        const int ca = colof(4 * ta, I, J), cb = colof(4 * tb, I, J);
        float acc[4][4] = {};
        const int rend = min(nr, (ch + 1) * rch);
        for (int rl = ch * rch; rl < rend; ++rl) {
          const float4 x = *reinterpret_cast<const float4*>(W + rl * ldw + ca);
          const float4 y = *reinterpret_cast<const float4*>(W + rl * ldw + cb);
          const float xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xa[i], ya[j], acc[i][j]);
        }
        const int owner = g % C, slot = g / C;
        float* dst = Gp + (((size_t)rank * nch + ch) * nown + slot) * PACK;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int a = 4 * ta + i, b = 4 * tb + j;
            if (a > b) continue;
            if (owner == rank) dst[P::pk(a, b)] = acc[i][j];
            else st_cluster_f32(dst + P::pk(a, b), owner, acc[i][j]);
          }
      }
      if (C > 1) cluster_barrier_jb(); else __syncthreads();
      JB_CLK(1);

      // ---- 2. owners: sum partials, rotate on the PW x PW Gram, accumulate Q
      const int gi = t / GS, tg = t % GS;
      if (gi < nown) {
        const int g = gi * C + rank;
        if (g < Pb) {
          double* G = Gw + (size_t)gi * PW * LDQ;
          float* Q = Qw + (size_t)gi * PW * LDQ;
          int* jp = Jp + gi * PW;
          float* jd = Jd + gi * PW;
          float* jo = Jo + gi * PW;
          const int bar_id = 1 + gi;
          for (int e = tg; e < PW * PW; e += GS) {
            const int a = e / PW, b = e % PW;
            const int lo = min(a, b), hi = max(a, b);
            double s = 0.0;
            for (int c = 0; c < C; ++c)
              for (int ch = 0; ch < nch; ++ch) s += Gp[(((size_t)c * nch + ch) * nown + gi) * PACK + P::pk(lo, hi)];
            G[a * LDQ + b] = s;
            Q[a * LDQ + b] = (a == b) ? 1.f : 0.f;
          }
          int rot_any = 0;
          const int nin = diag ? BW - 1 : BW;
          // thread tg owns column b = tg % PW, rows a = tg / PW + (GS / PW) u
          const int bq = tg % PW, a0 = tg / PW, astep = GS / PW;
          const int nu = PW / astep;                    // entries per thread
          if (tg == 0) Jact[gi] = 0;
          group_bar(bar_id, GS);
          for (int ri = 0; ri < nin; ++ri) {
            if (tg < BW) {
              int p, q;
              if (diag) {
                const int h = BW / 2;
                if (tg < h) { tourn(ri, tg, BW, p, q); }
                else { tourn(ri, tg - h, BW, p, q); p += BW; q += BW; }
              } else {
                p = tg;
                q = BW + ((tg + ri) % BW);
              }
              const double app = G[p * LDQ + p], aqq = G[q * LDQ + q], apq = G[p * LDQ + q];
              float c = 1.f, s = 0.f;
              if (apq * apq > tol2 * app * aqq) {
                // approximate angle (fast fp32 intrinsics: any angle near the optimum still
                // annihilates a_pq to first order); (c, s) orthogonal to fp32 rounding:
                // c = (1+t^2)^-1/2 from rsqrtf refined by one fp64 Newton step
                const float zeta = __fdividef((float)(aqq - app), (float)(2.0 * apq));
                const float az = fabsf(zeta);   // zeta = 0 -> t = 1; huge zeta -> t = 0
                const float tf = copysignf(__fdividef(1.0f, az + sqrtf(fmaf(az, az, 1.0f))), zeta);
                const double td = tf;
                const double xx = fma(td, td, 1.0);
                double cd = (double)rsqrtf((float)xx);
                cd = cd * fma(-0.5 * xx * cd, cd, 1.5);
                c = (float)cd;
                s = (float)(cd * td);
                Jact[gi] = ri + 1;   // never reset: "== ri + 1" means this round rotates
              }
              // col_p' = c col_p - s col_q ; col_q' = s col_p + c col_q
              jp[p] = q; jd[p] = c; jo[p] = -s;
              jp[q] = p; jd[q] = c; jo[q] = s;
            }
            group_bar(bar_id, GS);
            if (Jact[gi] != ri + 1) continue;   // no pair of this inner round rotates
            rot_any = 1;
            double gn[8];
            float qn[8];
            const int pb = jp[bq];
            const double db = jd[bq], ob = jo[bq];
            const bool bact = ob != 0.0;
            unsigned touched = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (u >= nu) break;
              const int a = a0 + astep * u;
              const int pa = jp[a];
              const double da = jd[a], oa = jo[a];
              if (!bact && oa == 0.0) continue;   // neither row nor column rotates: unchanged
              touched |= 1u << u;
              // G' = J^T G J : G'[a][b] = sum_{x in {a,pa}, y in {b,pb}} J[x][a] G[x][y] J[y][b]
              gn[u] = da * (db * G[a * LDQ + bq] + ob * G[a * LDQ + pb]) +
                      oa * (db * G[pa * LDQ + bq] + ob * G[pa * LDQ + pb]);
              // Q' = Q J : Q'[a][b] = Q[a][b] J[b][b] + Q[a][pb] J[pb][b]
              qn[u] = bact ? (float)db * Q[a * LDQ + bq] + (float)ob * Q[a * LDQ + pb] : Q[a * LDQ + bq];
            }
            group_bar(bar_id, GS);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (u >= nu) break;
              if (!(touched >> u & 1)) continue;
              G[(a0 + astep * u) * LDQ + bq] = gn[u];
              Q[(a0 + astep * u) * LDQ + bq] = qn[u];
            }
            group_bar(bar_id, GS);
          }
          if (tg == 0) {
            for (int cr = 0; cr < C; ++cr) {
              if (cr == rank) flag[g] = rot_any;
              else st_cluster_s32(flag + g, cr, rot_any);
            }
          }
        }
      }
      if (C > 1) cluster_barrier_jb(); else __syncthreads();
      JB_CLK(2);

      // ---- 3. apply [W_I W_J] <- [W_I W_J] Q, NQB pairs at a time
      for (int g0 = 0; g0 < Pb; g0 += NQB) {
        const int npair = min(NQB, Pb - g0);
        constexpr int F4 = PW / 4;
        for (int e = t; e < npair * PW * F4; e += NT) {   // fetch Q (owner's smem) as float4 rows
          const int pp = e / (PW * F4), rem = e % (PW * F4), a = rem / F4, c4 = rem % F4;
          const int g = g0 + pp;
          if (!flag[g]) continue;
          const int owner = g % C, slot = g / C;
          const float* src = Qw + (size_t)slot * PW * LDQ + a * LDQ + 4 * c4;
          const float4 v = (owner == rank) ? *reinterpret_cast<const float4*>(src) : ld_cluster_f4(src, owner);
          *reinterpret_cast<float4*>(Qb + (size_t)pp * PW * LDQ + a * LDQ + 4 * c4) = v;
        }
        __syncthreads();
        const int rq_n = (nr + 3) / 4;
        const int ntask = npair * rq_n * F4;
        float out[2][4][4];
        int tk[2];
        int nt_mine = 0;
        for (int task = t; task < ntask && nt_mine < 2; task += NT, ++nt_mine) {
          tk[nt_mine] = task;
          const int pp = task / (rq_n * F4), rem = task % (rq_n * F4), rq = rem / F4, cq = rem % F4;
          const int g = g0 + pp;
          if (!flag[g]) continue;
          int I, J;
          blocks_of(ro, g, I, J);
          const float* Qp = Qb + (size_t)pp * PW * LDQ;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) out[nt_mine][i][j] = 0.f;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int cbase = half ? BW * J : BW * I;
#pragma unroll
            for (int t4 = 0; t4 < BW / 4; ++t4) {
              float xr[4][4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 x = *reinterpret_cast<const float4*>(W + (4 * rq + i) * ldw + cbase + 4 * t4);
                xr[i][0] = x.x; xr[i][1] = x.y; xr[i][2] = x.z; xr[i][3] = x.w;
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float4 qv = *reinterpret_cast<const float4*>(Qp + (BW * half + 4 * t4 + u) * LDQ + 4 * cq);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  out[nt_mine][i][0] = fmaf(xr[i][u], qv.x, out[nt_mine][i][0]);
                  out[nt_mine][i][1] = fmaf(xr[i][u], qv.y, out[nt_mine][i][1]);
                  out[nt_mine][i][2] = fmaf(xr[i][u], qv.z, out[nt_mine][i][2]);
                  out[nt_mine][i][3] = fmaf(xr[i][u], qv.w, out[nt_mine][i][3]);
                }
              }
            }
          }
        }
        __syncthreads();
        for (int m = 0; m < nt_mine; ++m) {
          const int task = tk[m];
          const int pp = task / (rq_n * F4), rem = task % (rq_n * F4), rq = rem / F4, cq = rem % F4;
          const int g = g0 + pp;
          if (!flag[g]) continue;
          int I, J;
          blocks_of(ro, g, I, J);
          const int col = colof(4 * cq, I, J);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<float4*>(W + (4 * rq + i) * ldw + col) =
                make_float4(out[m][i][0], out[m][i][1], out[m][i][2], out[m][i][3]);
        }
        __syncthreads();
      }
      for (int g = 0; g < Pb; ++g) any |= flag[g];
      JB_CLK(3);
    }
    converged = (any == 0);
  }
  if (!converged && t == 0 && rank == 0) hg_flag(status, HGS_JACOBI_CAP);
  if (t == 0 && rank == 0) {
    atomicMax(&g_jb_dbg[0], (unsigned long long)sweep);
    atomicAdd(&g_jb_dbg[1], (unsigned long long)sweep);
    atomicAdd(&g_jb_dbg[2], 1ull);
  }
  float* out = Wf + (int64_t)blk * k * k;
  for (int i = t; i < nr * k; i += NT) {
    const int rl = i / k, c = i % k;
    out[(int64_t)(r0 + rl) * k + c] = W[rl * ldw + c];
  }
  if (C > 1) cluster_barrier_jb();
}

template <int BW>
cudaError_t launch_bw(int nb, int k, const float* L, float* Wf, int32_t* status, cudaStream_t s, double tol,
                      int w_is_l) {
  // rows per CTA: 128 up to k = 256 (one CTA per SM for configs[3]), 64 beyond
  const int rt = k <= 256 ? 128 : 64;
  const int C = (k + rt - 1) / rt;
  if (C > 8) return cudaErrorInvalidValue;
  const Layout Lo = make_layout<BW>(k, C);
  if (Lo.nown > JB<BW>::MAXOWN || Lo.Pb > 128 || Lo.total > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_jacobi_blk<BW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lo.total);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb * C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = Lo.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_jacobi_blk<BW>, k, C, tol, L, Wf, status, w_is_l);
}

}  // namespace

cudaError_t jacobi_blk_clocks(long long* out) { return cudaMemcpyFromSymbol(out, g_jb_clk, sizeof(g_jb_clk)); }

cudaError_t jacobi_blk_debug(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_jb_dbg, sizeof(g_jb_dbg));
  if (e == cudaSuccess && reset) {
    unsigned long long z[3] = {0, 0, 0};
    e = cudaMemcpyToSymbol(g_jb_dbg, z, sizeof z);
  }
  return e;
}

double jacobi_tol(int k);

// Block width 16 (32 x 32 inner problems) by default; HG_JACOBI_BW=8 selects 8 columns
// (measured slower at configs[3]: 12.4 vs 8.4 ms -- inner rounds are latency-bound, so
// halving their size does not pay for doubling the number of outer rounds).
cudaError_t launch_jacobi_blk(int nb, int k, const float* L, float* Wf, int32_t* status, cudaStream_t s,
                              int* launches) {
  static const int bw = [] {
    const char* v = getenv("HG_JACOBI_BW");
    return v ? atoi(v) : 16;
  }();
  ++*launches;
  const int wl = jacobi_on_l() ? 1 : 0;
  if (bw == 8) return launch_bw<8>(nb, k, L, Wf, status, s, jacobi_tol(k), wl);
  return launch_bw<16>(nb, k, L, Wf, status, s, jacobi_tol(k), wl);
}
