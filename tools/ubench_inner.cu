// Micro-benchmark of the block-Jacobi inner sweep (cross rounds) in isolation:
// one CTA, NG owner groups of 4 warps, a random symmetric 32x32 fp64 Gram per group
// with off-diagonal entries far above the threshold (every round rotates).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1908_08281_b200/csrc \
//        tools/ubench_inner.cu -o /tmp/ubench_inner && /tmp/ubench_inner
#include "../paper_1908_08281_b200/csrc/jacobi_blk.cu"

#include <cstdio>

// the library symbols the included file references (not used here)
bool jacobi_on_l() { return true; }
double jacobi_tol(int) { return 3e-7; }

namespace {

template <int BW, int MODE>
__device__ int cross4_var(const double* G, float* Q, double tol2, const Cross4Scratch& S, int lane, int h,
                                  int aw, int bar_id) {
  constexpr int PW = 2 * BW, LDQ = JB<BW>::LDQ, QW = BW / 4;
  const int j0 = h * QW;
  const bool act = lane < PW;
  double gI[QW], gJ[QW];
  float qI[QW], qJ[QW];
#pragma unroll
  for (int i = 0; i < QW; ++i) {
    gI[i] = act ? G[lane * LDQ + j0 + i] : 0.0;
    gJ[i] = act ? G[lane * LDQ + BW + j0 + i] : 0.0;
    qI[i] = (lane == j0 + i) ? 1.f : 0.f;
    qJ[i] = (lane == BW + j0 + i) ? 1.f : 0.f;
  }
  if (h == 0 && act) S.dsm[lane] = G[lane * LDQ + lane];
  if (lane < BW && lane / QW == h) S.apq[lane] = gJ[lane - j0];   // round 0: pair a = slot (a, BW + a)
  named_bar(bar_id, 128);
  // no cross entry above the threshold: no round can rotate (G never changes), skip
  int need = 0;
  if (lane < BW) {
    const double da = S.dsm[lane];
#pragma unroll
    for (int i = 0; i < QW; ++i) need |= gJ[i] * gJ[i] > tol2 * da * S.dsm[BW + j0 + i];
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
    for (int r = 0; r < BW; ++r) {
      ICLK(r, 0);
      // angles (warp aw, lane = pair a: rows a and pa = BW + (a + r) % BW)
      int rot = 0;
      if (h == aw && lane < BW) {
        const int pa = BW + (lane + r) % BW;
        const double apq = S.apq[lane], app = S.dsm[lane], aqq = S.dsm[pa];
        float c = 1.f, sn = 0.f;
        if (apq * apq > tol2 * app * aqq) {
          double dp, dq;
          if (MODE & 1) { c = 0.8f; sn = 0.6f; dp = app; dq = aqq; } else
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
          if (MODE & 2) break;
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
          if (MODE & 4) break;
          const double oI = __shfl_sync(0xffffffffu, gI[i], pa);
          const double oJ = __shfl_sync(0xffffffffu, gJ[i], pa);
          gI[i] = fma(sd, oI, cd * gI[i]);
          gJ[i] = fma(sd, oJ, cd * gJ[i]);
        }
      }
      // slot rotation: new slot BW + j = old slot BW + j + 1 (wrapping inside the J half);
      // the holder of old slot BW + a + 1 stages a_pq of round r + 1's pair a
      if (!(MODE & 8)) S.xg[h * 32 + lane] = gJ[0];
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
      const double ng = (MODE & 8) ? gJ[0] : S.xg[((h + 1) & 3) * 32 + lane];
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
  return rot_any;
}


template <int MODE>
__global__ void __launch_bounds__(512, 1) k_ubench(int ng, int reps, long long* cyc) {
  constexpr int BW = 16, PW = 32, LDQ = JB<BW>::LDQ;
  __shared__ double G[4][PW * LDQ];
  __shared__ float Q[4][PW * LDQ];
  __shared__ double scr[4][jscr<BW>()];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gi = warp >> 2, h = warp & 3;
  for (int i = t; i < 4 * PW * LDQ; i += blockDim.x) {
    const int g = i / (PW * LDQ), e = i % (PW * LDQ), a = e / LDQ, b = e % LDQ;
    const unsigned x = (unsigned)(min(a, b) * 131 + max(a, b) * 17 + g * 7) * 2654435761u;
    G[g][e] = (a == b) ? 1.0 + 0.01 * a : 0.05 * ((double)(x >> 8) / 16777216.0 - 0.5);
  }
  __syncthreads();
  long long t0 = clock64();
  int any = 0;
  if (gi < ng) {
    const Cross4Scratch S = cross4_scratch<BW>(scr[gi]);
    for (int r = 0; r < reps; ++r) any |= cross4_var<BW, MODE>(G[gi], Q[gi], 1e-14, S, lane, h, gi & 3, 1 + gi);
  }
  __syncthreads();
  long long t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  if (t == 0) cyc[1] = any;
}

}  // namespace

template <int MODE>
void run(const char* name, long long* d) {
  for (int ng = 1; ng <= 4; ng *= 3) {
    k_ubench<MODE><<<1, 512>>>(ng, 2, d);
    k_ubench<MODE><<<1, 512>>>(ng, 20, d);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s groups %d: %6.0f cycles per round\n", name, ng, h[0] / 20.0 / 16.0);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<0>("full", d);
  run<1>("no angle math", d);
  run<2>("no column update", d);
  run<4>("no row update", d);
  run<8>("no slot exchange", d);
  run<1 | 2 | 4 | 8>("barriers + flags only", d);
  run<2 | 4>("no col/row update", d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
