// jacobi_blk.cu -- Alg. 1 step 5: one-sided (Hestenes) Jacobi on
// W = L^T (k x k, B B^T = L L^T), organised in column blocks.
//
// Same rotations as the scalar cyclic method (jacobi.cu): every column pair
// (p, q) is visited once per sweep and rotated by the angle that zeroes its 2x2
// Gram [[a_pp, a_pq], [a_pq, a_qq]] while |a_pq| > tol sqrt(a_pp a_qq); the
// sweep loop stops after a sweep in which no |a_pq| / sqrt(a_pp a_qq) exceeded
// 4 tol (its rotations above tol are still applied; reading A16 in DESIGN.md).  What changes is the data
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
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int NT = 512;   // 4 owner warps per owned pair (nown <= 4)
constexpr int MAX_SWEEPS = 40;

__device__ unsigned long long g_jb_dbg[3];   // [0] max sweeps, [1] total sweeps, [2] blocks
__device__ long long g_jb_clk[16];           // block 0 / rank 0 / thread 0: sweep 1, outer rounds 0-1
__device__ long long g_jb_iclk[48];          // inner rounds 0-3 of block 0, pair 0, sweep 1, outer round 0
__device__ int g_jb_iclk_on;                 // set by the caller of the stamps (debug)
// debug (build with -DHG_JB_SWEEPMAX, tools/jacobi_sweepmax.py): per block and sweep, the largest
// a_pq^2 / (a_pp a_qq) seen (float bits); compiled out otherwise
__device__ unsigned g_jb_smax[64 * 40];
__device__ int g_jb_smax_on;
__device__ __forceinline__ void jb_meas(unsigned* slot, double apq, double app, double aqq) {
#ifdef HG_JB_SWEEPMAX
  if (slot) atomicMax(slot, __float_as_uint((float)(apq * apq / (app * aqq))));
#endif
}
#define JB_CLK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0 && sweep == 1 && ro < 2) g_jb_clk[(i) + 8 * ro] = clock64(); } while (0)

__device__ __forceinline__ void cluster_barrier_jb() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// An owned pair's fp64 Gram entry (a, b) read straight from the C packed fp32 partials
// (one per cluster CTA, summed in rank order): the inner sweeps load their registers
// from here, no separate fp64 Gram pass.
template <int BW>
struct GramSrc {
  const float* Gp;   // partials of this pair: Gp[c * stride + pk(lo, hi)]
  int C, stride;
  __device__ __forceinline__ double operator()(int a, int b) const {
    const int idx = JB<BW>::pk(min(a, b), max(a, b));
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += Gp[(size_t)c * stride + idx];
    return s;
  }
};

// Q layout in shared memory (pitch LDQ): element (a, j) at a * LDQ + (j ^ qsw(a)).  The
// XOR stays inside aligned groups of 4 (float4 rows stay float4 rows, permuted) and
// makes the lane-per-row column accesses of the inner rounds bank-conflict free.
__device__ __forceinline__ int qsw(int a) { return (a >> 3) & 3; }

// Rotation of the 2x2 Gram [[app, apq], [apq, aqq]] (Golub & Van Loan sym.schur2) with
// an approximate angle from fast fp32 intrinsics (any angle near the optimum still
// annihilates a_pq to first order); (c, s) orthogonal to fp32 rounding: c = (1+t^2)^-1/2
// from rsqrtf refined by one fp64 Newton step.  Returns the new diagonal entries.
__device__ __forceinline__ void jrot(double app, double aqq, double apq, float& c, float& s, double& dp, double& dq) {
  const float zeta = __fdividef((float)(aqq - app), (float)(2.0 * apq));
  const float az = fabsf(zeta);
  const float tf = copysignf(__fdividef(1.0f, az + sqrtf(fmaf(az, az, 1.0f))), zeta);
  const double td = tf;
  const double xx = fma(td, td, 1.0);
  double cd = (double)rsqrtf((float)xx);
  cd = cd * fma(-0.5 * xx * cd, cd, 1.5);
  c = (float)cd;
  s = (float)(cd * td);
  const double c2 = (double)c, s2 = (double)s;
  const double x = 2.0 * c2 * s2 * apq;
  dp = c2 * c2 * app - x + s2 * s2 * aqq;     // G'[p][p] = c^2 a_pp - 2cs a_pq + s^2 a_qq
  dq = s2 * s2 * app + x + c2 * c2 * aqq;     // G'[q][q] = s^2 a_pp + 2cs a_pq + c^2 a_qq
}

// Diagonal-round inner sweep: the pairs inside one column block (columns base ..
// base + BW - 1 of the PW x PW problem) never touch the other block, so each block is
// an independent BW x BW problem, solved by one warp (lane = row, lanes >= BW idle).
// Round-robin by the circle method: slot 0 holds column 0, slot s >= 1 holds column
// 1 + (s - 1 + r) % (BW - 1), pairs are slots (i, BW - 1 - i); after each round slots
// 1..BW-1 rotate by one, so register indices are compile-time constants inside the
// runtime round loop.  G <- J^T G J (columns lane-locally with (c, s) broadcast through
// shared memory, rows by shuffles), Q <- Q J on the block's columns.  Q rows of the
// block are (re)initialised here to the identity over all PW columns.
template <int BW>
__device__ __forceinline__ int diag_col(int s, int r) { return s == 0 ? 0 : 1 + (s - 1 + r) % (BW - 1); }

template <int BW>
__device__ int inner_sweep_diag(const GramSrc<BW>& G, float* Q, int base, double tol2, double stop2, double2* cs,
                                int lane, unsigned* smax) {
  constexpr int PW = 2 * BW, LDQ = JB<BW>::LDQ;
  const bool act = lane < BW;
  const int row = base + (act ? lane : 0);
  const int sw = qsw(row);
  float* qrow = Q + row * LDQ;
  double g[BW];
#pragma unroll
  for (int j = 0; j < BW; ++j) g[j] = act ? G(row, base + j) : 0.0;   // round 0: slot j = column j
  if (act) {
#pragma unroll
    for (int j = 0; j < PW; ++j) qrow[j ^ sw] = (j == row) ? 1.f : 0.f;
  }
  double d = act ? G(row, row) : 1.0;
  {  // no pair of the block above the threshold: nothing can rotate, skip
    int need = 0;
#pragma unroll
    for (int j = 0; j < BW; ++j) {
      const double dj = __shfl_sync(0xffffffffu, d, j);
      need |= act && j != lane && g[j] * g[j] > tol2 * d * dj;
    }
    if (__ballot_sync(0xffffffffu, need) == 0u) return 0;
  }
  int rot_any = 0, big = 0;
#pragma unroll 1
  for (int r = 0; r < BW - 1; ++r) {
    int pa = lane, pj = 0, pslot = 0;
    bool first = false;
    if (act) {
      const int sl = lane == 0 ? 0 : 1 + ((lane - 1 - r) % (BW - 1) + (BW - 1)) % (BW - 1);
      const int ps = BW - 1 - sl;
      pa = diag_col<BW>(ps, r);
      first = sl < ps;
      pj = min(sl, ps);
      pslot = ps;
    }
    double apq = 0.0;   // G[lane][pa] = g[pslot]
#pragma unroll
    for (int j = 0; j < BW; ++j) apq = (j == pslot) ? g[j] : apq;
    const double aqq = __shfl_sync(0xffffffffu, d, pa);
    float c = 1.f, s = 0.f;
    double dp = d, dq = aqq;
    if (first) jb_meas(smax, apq, d, aqq);
    big |= first && apq * apq > stop2 * d * aqq;
    if (first && apq * apq > tol2 * d * aqq) jrot(d, aqq, apq, c, s, dp, dq);
    const float c_o = __shfl_sync(0xffffffffu, c, pa);
    const float s_o = __shfl_sync(0xffffffffu, s, pa);
    const double dq_o = __shfl_sync(0xffffffffu, dq, pa);
    if (first) d = dp;
    else if (act) { c = c_o; s = s_o; d = dq_o; }
    if (__ballot_sync(0xffffffffu, first && s != 0.f) != 0u) {
      rot_any = 1;
      if (first) cs[pj] = make_double2((double)c, (double)s);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < BW / 2; ++i) {   // columns: slots (i, BW - 1 - i)
        const double2 v = cs[i];
        const double gp = g[i], gq = g[BW - 1 - i];
        g[i] = fma(v.x, gp, -v.y * gq);
        g[BW - 1 - i] = fma(v.y, gp, v.x * gq);
        if (act) {
          const int cp = base + diag_col<BW>(i, r), cq = base + diag_col<BW>(BW - 1 - i, r);
          const float cf = (float)v.x, sf = (float)v.y;
          const float qp = qrow[cp ^ sw], qq = qrow[cq ^ sw];
          qrow[cp ^ sw] = fmaf(cf, qp, -sf * qq);
          qrow[cq ^ sw] = fmaf(sf, qp, cf * qq);
        }
      }
      const double cd = c, sd = first ? -(double)s : (double)s;   // rows
#pragma unroll
      for (int j = 0; j < BW; ++j) {
        const double o = __shfl_sync(0xffffffffu, g[j], pa);
        g[j] = fma(sd, o, cd * g[j]);
      }
      __syncwarp();   // cs is rewritten next round
    }
    const double t0 = g[1];   // advance the slot assignment to round r + 1
#pragma unroll
    for (int j = 1; j < BW - 1; ++j) g[j] = g[j + 1];
    g[BW - 1] = t0;
  }
  return rot_any | (__ballot_sync(0xffffffffu, big) != 0u ? 2 : 0);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Cross rounds of the inner sweep (BW rounds, pairs (j, BW + (j + r) % BW)) by the
// four warps h = 0..3 of an owner group (128 threads, named barrier bar_id).  Warp h
// holds register slots j and BW + j for j in [h QW, (h+1) QW) of row `lane` of G
// (fp64) and of Q (fp32).  Register slots, not columns, are paired, so register
// indices are compile-time constants inside the runtime round loop: slot j (< BW)
// holds column j, slot BW + j holds column BW + (j + r) % BW, pairs are slots
// (j, BW + j) = columns (j, BW + (j + r) % BW).  After each round the J-half slots
// (of G and of Q) rotate by one, one value per thread passing to the neighbouring
// warp through shared memory; after BW rounds the slots are back in column order.
// One warp of the group (aw, spread over the SMSPs by the caller) computes all BW
// angles of a round from a_pq values the holders staged in shared memory together
// with the slot exchange (2 barriers per round; the second ORs "anything rotated").
// Rotation arithmetic: jrot.
struct Cross4Scratch {
  double* dsm;    // [PW] diagonal of G
  double* apq;    // [BW] a_pq of the next round's pairs
  double* xg;     // [4][32] G slot exchange
  double2* csd;   // [BW] (c, s) fp64
  float* xq;      // [4][32] Q slot exchange
  float2* csf;    // [BW] (c, s) fp32
  int* flags;     // [2] "round rotates" (by round parity) | [4] per-warp "needs a sweep" | [1] "above stop"
};

template <int BW>
__device__ int inner_sweep_cross4(const GramSrc<BW>& G, float* Q, double tol2, const Cross4Scratch& S, int lane, int h,
                                  int aw, int bar_id, int npass, double stop2, unsigned* smax) {
  constexpr int PW = 2 * BW, LDQ = JB<BW>::LDQ, QW = BW / 4;
  const int j0 = h * QW;
  const bool act = lane < PW;
  double gI[QW], gJ[QW];
  float qI[QW], qJ[QW];
#pragma unroll
  for (int i = 0; i < QW; ++i) {
    gI[i] = act ? G(lane, j0 + i) : 0.0;
    gJ[i] = act ? G(lane, BW + j0 + i) : 0.0;
    qI[i] = (lane == j0 + i) ? 1.f : 0.f;
    qJ[i] = (lane == BW + j0 + i) ? 1.f : 0.f;
  }
  if (h == 0 && act) S.dsm[lane] = G(lane, lane);
  if (lane < BW && lane / QW == h) S.apq[lane] = gJ[lane - j0];   // round 0: pair a = slot (a, BW + a)
  if (h == 0 && lane == 0) S.flags[6] = 0;                        // "a measure above the stop threshold"
  named_bar(bar_id, 128);
  // no cross entry above the threshold: no round can rotate (G never changes), skip
  int need = 0;
  if (lane < BW) {
    const double da = S.dsm[lane];
#pragma unroll
    for (int i = 0; i < QW; ++i) {
      need |= gJ[i] * gJ[i] > tol2 * da * S.dsm[BW + j0 + i];
      jb_meas(smax, gJ[i], da, S.dsm[BW + j0 + i]);
    }
  }
  need = __ballot_sync(0xffffffffu, need) != 0u;
  if (lane == 0) S.flags[2 + h] = need;
  named_bar(bar_id, 128);
  int rot_any = 0;
  if (S.flags[2] | S.flags[3] | S.flags[4] | S.flags[5]) {
    const bool stamp = g_jb_iclk_on && blockIdx.x == 0 && bar_id == 1 && lane == 0;
    auto ICLK = [&](int r, int i) {
      if (stamp && r < 4) g_jb_iclk[12 * r + 3 * i + (h == aw ? 0 : (h == ((aw + 1) & 3) ? 1 : 2))] = clock64();
    };
#pragma unroll 1
    for (int r = 0; r < BW * npass; ++r) {   // npass inner sweeps; slots return to column order every BW rounds
      ICLK(r, 0);
      // angles (warp aw, lane = pair a: rows a and pa = BW + (a + r) % BW)
      int rot = 0;
      if (h == aw && lane < BW) {
        const int pa = BW + (lane + r) % BW;
        const double apq = S.apq[lane], app = S.dsm[lane], aqq = S.dsm[pa];
        float c = 1.f, sn = 0.f;
        if (r < BW) jb_meas(smax, apq, app, aqq);
        if (r < BW && apq * apq > stop2 * app * aqq) S.flags[6] = 1;
        if (apq * apq > tol2 * app * aqq) {
          double dp, dq;
          jrot(app, aqq, apq, c, sn, dp, dq);
          S.dsm[lane] = dp;
          S.dsm[pa] = dq;
          rot = sn != 0.f;
        }
        S.csd[lane] = make_double2((double)c, (double)sn);
        S.csf[lane] = make_float2(c, sn);
      }
      if (h == aw) {   // plain barrier + a flag word: bar.red.or measured ~400 cycles slower
        const unsigned any = __ballot_sync(0xffffffffu, rot);
        if (lane == 0) S.flags[r & 1] = any != 0u;
      }
      ICLK(r, 1);
      named_bar(bar_id, 128);
      if (S.flags[r & 1]) {
        ICLK(r, 2);
        rot_any = 1;
#pragma unroll
        for (int i = 0; i < QW; ++i) {   // columns of G and Q: slot pair (j, BW + j)
          const double2 v = S.csd[j0 + i];
          const float2 vf = S.csf[j0 + i];
          const double gp = gI[i], gq = gJ[i];
          gI[i] = fma(v.x, gp, -v.y * gq);
          gJ[i] = fma(v.y, gp, v.x * gq);
          const float qp = qI[i], qq = qJ[i];
          qI[i] = fmaf(vf.x, qp, -vf.y * qq);
          qJ[i] = fmaf(vf.y, qp, vf.x * qq);
        }
        int pa = lane, pj = 0;   // rows of G: row_p' = c row_p - s row_q ; row_q' = s row_p + c row_q
        bool first = false;
        if (lane < BW) { pa = BW + (lane + r) % BW; pj = lane; first = true; }
        else if (act) { pa = ((lane - BW - r) % BW + BW) % BW; pj = pa; }
        const double2 v = S.csd[pj];
        const double cd = act ? v.x : 1.0, sd = act ? (first ? -v.y : v.y) : 0.0;
#pragma unroll
        for (int i = 0; i < QW; ++i) {
          const double oI = __shfl_sync(0xffffffffu, gI[i], pa);
          const double oJ = __shfl_sync(0xffffffffu, gJ[i], pa);
          gI[i] = fma(sd, oI, cd * gI[i]);
          gJ[i] = fma(sd, oJ, cd * gJ[i]);
        }
      }
      // slot rotation: new slot BW + j = old slot BW + j + 1 (wrapping inside the J half);
      // the holder of old slot BW + a + 1 stages a_pq of round r + 1's pair a
      S.xg[h * 32 + lane] = gJ[0];
      S.xq[h * 32 + lane] = qJ[0];
      if (lane < BW) {
        const int sl = (lane + 1) % BW;   // old J slot index of round r + 1's partner of row a
        if (sl / QW == h) {
          double v = gJ[0];
#pragma unroll
          for (int i = 1; i < QW; ++i) v = (sl - j0 == i) ? gJ[i] : v;
          S.apq[lane] = v;
        }
      }
      ICLK(r, 3);
      named_bar(bar_id, 128);
      const double ng = S.xg[((h + 1) & 3) * 32 + lane];
      const float nq = S.xq[((h + 1) & 3) * 32 + lane];
#pragma unroll
      for (int i = 0; i < QW - 1; ++i) {
        gJ[i] = gJ[i + 1];
        qJ[i] = qJ[i + 1];
      }
      gJ[QW - 1] = ng;
      qJ[QW - 1] = nq;
    }
  }
  if (act) {   // slots are back in column order: write Q (swizzled, see qsw)
    const int sw = qsw(lane);
    float* qrow = Q + lane * LDQ;
#pragma unroll
    for (int i = 0; i < QW; ++i) {
      qrow[(j0 + i) ^ sw] = qI[i];
      qrow[(BW + j0 + i) ^ sw] = qJ[i];
    }
  }
  return rot_any | (S.flags[6] ? 2 : 0);
}

// per-owned-pair scratch (doubles): dsm [PW] | apq [BW] | xg [4 x 32] | csd [BW x 2] |
// xq [4 x 32 floats] | csf [BW x 2 floats] | flags [6 ints]  (the diagonal round reuses
// csd as its cs and the start of xg as its two "rotated" flags)
template <int BW>
__host__ __device__ constexpr int jscr() { return 2 * BW + BW + 4 * 32 + 2 * BW + (4 * 32 + 2 * BW) / 2 + 4; }
template <int BW>
__device__ __forceinline__ Cross4Scratch cross4_scratch(double* js) {
  Cross4Scratch S;
  S.dsm = js;
  S.apq = js + 2 * BW;
  S.xg = js + 3 * BW;
  S.csd = reinterpret_cast<double2*>(js + 3 * BW + 128);
  S.xq = reinterpret_cast<float*>(js + 5 * BW + 128);
  S.csf = reinterpret_cast<float2*>(S.xq + 128);
  S.flags = reinterpret_cast<int*>(S.csf + BW);
  return S;
}

struct Layout {
  int K2, nblk, Pb, R, nch, rch, ldw, nown;
  size_t offW, offGp, offQ, offQb, offJ, offF, total;
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
  // partial Grams: one per (CTA, owned pair) -- the row split is inside the CTA (phase 1)
  L.rch = L.R;
  L.nch = 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) / 16 * 16; return o; };
  L.offW = take((size_t)L.R * L.ldw * 4);
  L.offGp = take((size_t)C * L.nown * P::PACK * 4);
  L.offQ = take((size_t)L.nown * P::PW * P::LDQ * 4);
  L.offQb = take((size_t)P::NQB * P::PW * P::LDQ * 4);   // apply-phase Q staging
  L.offJ = take((size_t)L.nown * jscr<BW>() * 8);          // inner-round scratch per owned pair
  L.offF = take((size_t)128 * 4);
  L.total = off;
  return L;
}

template <int BW>
__global__ void __launch_bounds__(NT, 1) k_jacobi_blk(int k, int C, double tol, const float* __restrict__ L,
                                                      float* __restrict__ Wf, int32_t* status, int w_is_l, int npass,
                                                      double stop_f) {
  using P = JB<BW>;
  constexpr int PW = P::PW, LDQ = P::LDQ, PACK = P::PACK, N4 = P::N4, UT = P::UT, NQB = P::NQB;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const Layout Lo = make_layout<BW>(k, C);
  int rank = 0;
  if (C > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int blk = blockIdx.x / C;
  const int nblk = Lo.nblk, Pb = Lo.Pb, R = Lo.R, ldw = Lo.ldw, nown = Lo.nown;
  const int r0 = rank * R;
  const int nr = max(0, min(R, k - r0));
  float* W = reinterpret_cast<float*>(smem_raw + Lo.offW);
  float* Gp = reinterpret_cast<float*>(smem_raw + Lo.offGp);     // [C][nch][nown][PACK]
  float* Qw = reinterpret_cast<float*>(smem_raw + Lo.offQ);      // [nown][PW][LDQ]
  float* Qb = reinterpret_cast<float*>(smem_raw + Lo.offQb);     // [NQB][PW][LDQ]
  double* JS = reinterpret_cast<double*>(smem_raw + Lo.offJ);    // [nown][JSCR]: cs | dsm | xch
  int* flag = reinterpret_cast<int*>(smem_raw + Lo.offF);        // [Pb] rotated-this-round
  const int t = threadIdx.x;
  const double tol2 = tol * tol, stop2 = tol2 * stop_f * stop_f;
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
#ifdef HG_JB_SWEEPMAX
    unsigned* smax = (g_jb_smax_on && blk < 64 && sweep < 40) ? &g_jb_smax[blk * 40 + sweep] : nullptr;
#else
    unsigned* smax = nullptr;
#endif
    for (int ro = 0; ro < nblk; ++ro) {
      const bool diag = (ro == nblk - 1);
      JB_CLK(0);
      // ---- 1. partial Grams: (pair, upper 4x4 tile) over this CTA's rows -> owner's Gp[rank][slot]
      //         (measured faster at configs[3] than 8x8 tiles with in-CTA row splits: 15k vs
      //         18-21k cycles per outer round)
      for (int task = t; task < Pb * UT; task += NT) {
        const int g = task / UT;
        int tt = task % UT, ta = 0;
        while (tt >= N4 - ta) { tt -= N4 - ta; ++ta; }
        const int tb = ta + tt;
        int I, J;
        blocks_of(ro, g, I, J);
        const int ca = colof(4 * ta, I, J), cb = colof(4 * tb, I, J);
        // two-level fp32 sum: FMA over chunks of 16 rows, then the chunk sums.  One running
        // fp32 sum over nr rows carries noise near the stopping threshold, and the sweeps it
        // adds only rotate noise: measured at configs[3], 12.3 mean / 14 max sweeps per
        // block with one sum, 11.0 / 13 two-level (10.8 / 13 with fp64 chunk sums, which
        // cost 5k cycles more per round than they save)
        float accd[4][4] = {};
        for (int r0 = 0; r0 < nr; r0 += 16) {
          float acc[4][4] = {};
          auto row = [&](int rl) {
            const float4 x = *reinterpret_cast<const float4*>(W + rl * ldw + ca);
            const float4 y = *reinterpret_cast<const float4*>(W + rl * ldw + cb);
            const float xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xa[i], ya[j], acc[i][j]);
          };
          if (r0 + 16 <= nr) {
#pragma unroll 4
            for (int rl = r0; rl < r0 + 16; ++rl) row(rl);
          } else {
            for (int rl = r0; rl < nr; ++rl) row(rl);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) accd[i][j] += acc[i][j];
        }
        const int owner = g % C, slot = g / C;
        HG_DCHECK(slot < nown && owner < C);
        float* dst = Gp + ((size_t)rank * nown + slot) * PACK;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int a = 4 * ta + i, b = 4 * tb + j;
            if (a > b) continue;
            const float v = accd[i][j];
            if (owner == rank) dst[P::pk(a, b)] = v;
            else st_cluster_f32(dst + P::pk(a, b), owner, v);
          }
      }
      if (C > 1) cluster_barrier_jb(); else __syncthreads();
      JB_CLK(1);

      // ---- 2. owners: 4 warps per owned pair run the inner sweep in registers, loading the
      //         fp64 Gram straight from the packed partials (inner_sweep_cross4; diagonal
      //         round: inner_sweep_diag on blocks I and J)
      JB_CLK(2);
      {
        const int warp = t >> 5, lane = t & 31;
        const int gi = warp >> 2, h = warp & 3;   // owner group of 4 warps per owned pair
        const int g = gi * C + rank;
        if (gi < nown && g < Pb) {
          double* js = JS + (size_t)gi * jscr<BW>();
          const Cross4Scratch S = cross4_scratch<BW>(js);
          const GramSrc<BW> Gsrc{Gp + (size_t)gi * PACK, C, nown * PACK};
          int rot_any = 0;
          if (!diag) {
            rot_any = inner_sweep_cross4<BW>(Gsrc, Qw + (size_t)gi * PW * LDQ, tol2, S, lane, h, gi & 3, 1 + gi,
                                             npass, stop2, smax);
          } else if (h < 2) {   // diagonal round: block I by warp 0, block J by warp 1
            int* rflag = reinterpret_cast<int*>(S.xg);
            const int rh = inner_sweep_diag<BW>(Gsrc, Qw + (size_t)gi * PW * LDQ, h * BW, tol2, stop2,
                                                S.csd + h * (BW / 2), lane, smax);
            if (lane == 0) rflag[h] = rh;
            named_bar(1 + gi, 64);
            rot_any = rflag[0] | rflag[1];
          }
          JB_CLK(3);
          if (h == 0 && lane == 0) {
            for (int cr = 0; cr < C; ++cr) {
              if (cr == rank) flag[g] = rot_any;
              else st_cluster_s32(flag + g, cr, rot_any);
            }
          }
        }
      }
      if (C > 1) cluster_barrier_jb(); else __syncthreads();
      JB_CLK(4);

      // ---- 3. apply [W_I W_J] <- [W_I W_J] Q, qb <= NQB pairs at a time (<= 2 tasks per thread)
      constexpr int F4 = PW / 4;
      const int qb = min(NQB, (2 * NT) / (((nr + 3) / 4) * F4));
      for (int g0 = 0; g0 < Pb; g0 += qb) {
        const int npair = min(qb, Pb - g0);
        for (int e = t; e < npair * PW * F4; e += NT) {   // fetch Q (owner's smem) as float4 rows
          const int pp = e / (PW * F4), rem = e % (PW * F4), a = rem / F4, c4 = rem % F4;
          const int g = g0 + pp;
          if (!(flag[g] & 1)) continue;
          const int owner = g % C, slot = g / C;
          HG_DCHECK(slot < nown && pp < NQB && a < PW);
          const float* src = Qw + (size_t)slot * PW * LDQ + a * LDQ + 4 * c4;
          const float4 v = (owner == rank) ? *reinterpret_cast<const float4*>(src) : ld_cluster_f4(src, owner);
          const int sw = qsw(a);   // un-swizzle (see qsw): out[i] = v[i ^ sw]
          float4 o = v;
          if (sw & 1) o = make_float4(o.y, o.x, o.w, o.z);
          if (sw & 2) o = make_float4(o.z, o.w, o.x, o.y);
          *reinterpret_cast<float4*>(Qb + (size_t)pp * PW * LDQ + a * LDQ + 4 * c4) = o;
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
          if (!(flag[g] & 1)) continue;
          int I, J;
          blocks_of(ro, g, I, J);
          HG_DCHECK(4 * rq + 3 < R && BW * J + BW <= ldw && BW * I + BW <= ldw && pp < NQB);
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
          if (!(flag[g] & 1)) continue;
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
      for (int g = 0; g < Pb; ++g) any |= flag[g] >> 1;   // a measure above the stop threshold
      JB_CLK(5);
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

thread_local int g_rows_hint = 0;

template <int BW>
cudaError_t launch_bw(int nb, int k, const float* L, float* Wf, int32_t* status, cudaStream_t s, double tol,
                      int w_is_l) {
  // rows per CTA: 128 up to k = 256 (one CTA per SM for configs[3]), 64 beyond; a caller's
  // hint (jacobi_rows_hint) overrides it for one launch (wider clusters: shorter per-block latency)
  const int rt = g_rows_hint > 0 ? g_rows_hint : (k <= 256 ? 128 : 64);
  const int C = (k + rt - 1) / rt;
  if (C > 8) return cudaErrorInvalidValue;
  const Layout Lo = make_layout<BW>(k, C);
  if (Lo.nown > JB<BW>::MAXOWN || Lo.nown > NT / 128 || Lo.Pb > 128 || Lo.total > 227 * 1024 ||
      ((Lo.R + 3) / 4) * (JB<BW>::PW / 4) > 2 * NT)
    return cudaErrorInvalidValue;
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
  static const int npass = [] {   // inner sweeps per outer round (HG_JACOBI_INNER, default 1)
    const char* v = getenv("HG_JACOBI_INNER");
    const int x = v ? atoi(v) : 1;
    return x < 1 ? 1 : (x > 4 ? 4 : x);
  }();
  // stop rule: the sweep loop ends after a sweep whose largest rotation measure
  // |a_pq| / sqrt(a_pp a_qq) is <= stop_f * tol (HG_JACOBI_STOP = stop_f, default 4; 1 = "a sweep
  // without rotations").  Measured at configs[3] (tools/jacobi_sweepmax.py): the per-sweep maximum
  // falls 2e-3 ... 4e-5, 2e-6, then sits at 5.0-5.3e-7 -- the fp32 Gram noise floor, just above
  // tol = 5e-7 -- for the last 2-3 sweeps, which only rotate noise: 10.2 -> 8.1 sweeps, F and sigma
  // errors unchanged (6.2e-6 / 6.1e-7)
  static const double stop_f = [] {
    const char* v = getenv("HG_JACOBI_STOP");
    const double x = v ? atof(v) : 4.0;
    return x < 1.0 ? 1.0 : x;
  }();
  return cudaLaunchKernelEx(&cfg, k_jacobi_blk<BW>, k, C, tol, L, Wf, status, w_is_l, npass, stop_f);
}

}  // namespace

cudaError_t jacobi_blk_clocks(long long* out) { return cudaMemcpyFromSymbol(out, g_jb_clk, sizeof(g_jb_clk)); }
cudaError_t jacobi_blk_inner_clocks(long long* out, int enable) {
  cudaError_t e = cudaMemcpyToSymbol(g_jb_iclk_on, &enable, sizeof(int));
  if (e != cudaSuccess || !out) return e;
  return cudaMemcpyFromSymbol(out, g_jb_iclk, sizeof(g_jb_iclk));
}

cudaError_t jacobi_blk_debug(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_jb_dbg, sizeof(g_jb_dbg));
  if (e == cudaSuccess && reset) {
    unsigned long long z[3] = {0, 0, 0};
    e = cudaMemcpyToSymbol(g_jb_dbg, z, sizeof z);
  }
  return e;
}

double jacobi_tol(int k);

void jacobi_rows_hint(int rows) { g_rows_hint = rows; }

// debug: switch the per-sweep maximum rotation measure on (and clear it) / read it
extern "C" int hg_debug_jacobi_sweepmax(float* out, int on) {
  if (out) return (int)cudaMemcpyFromSymbol(out, g_jb_smax, sizeof(g_jb_smax));
  static unsigned z[64 * 40] = {};
  cudaError_t e = cudaMemcpyToSymbol(g_jb_smax, z, sizeof z);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_jb_smax_on, &on, sizeof(int));
  return (int)e;
}

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
