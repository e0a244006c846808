// apply.cu -- the fused Sigma^-1 scale + apply-to-RHS kernel.
//
//   F_i = c V_i Sigma_i^-1 U_i^T Y_i      (Eq. 3 with PAPER.md:160-163 Eq. 15)
//
// One launch per stream part, one CTA per (block i, 128 RHS columns t0..t0+127):
//   1. Z^T = Y_i^T U_i                (128 x k, K = b)   tcgen05 kind::f16, 3xF16, accumulators in TMEM
//   2. Z^T *= c / sigma_j  (column scale, c / sigma from sigma in the prologue: no k_inv_sigma launch),
//      re-split into fp16 hi | lo with a CTA-local power-of-two exponent and written to shared memory
//      as the K-major B operand of the second product -- the k x T intermediate never leaves the SM
//   3. F_i[m-tile] = V_i[m-tile] Z    (128 x 128, K = k) for the b/128 row tiles, TMEM double-buffered
//      so tile mt's drain + store overlaps tile mt+1's MMAs.
// Operands: U as the 3xF16 twin (common.cuh tw_off) of Ut [k][b] (K-major B of product 1), V as the twin
// of V [b][k] (K-major operand of product 2) -- both TMA-loaded into 128-byte SWIZZLE_128B rows
// [hi 32 k | lo 32 k] and read by the MMAs as they stand; Y tiles land as fp32 [32 rows][32 columns]
// chunks and are split in place into the same row layout by the 8 epilogue warps (a transposing split);
// Z is written in that layout too.  (64-byte SWIZZLE_64B rows halve the tensor core's operand fetch
// rate, gemm.cu.)  Exponents: 2^e_y from max|Y_i| per block (k_absmax, so results do not depend on the
// part / shard split), 2^14 for orthonormal U, V inside hg_solve (from max|U_i|, max|V_i| for
// caller-provided factors).
// Precision is that of the other 3xF16 products: 22 significant bits per operand, fp32 accumulation
// in chunks of 24 MMAs summed in registers.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

bool hg_tma_map_f32(CUtensorMap* m, const float* ptr, int64_t inner, int64_t outer, int64_t batch, int64_t ld,
                    int64_t bs, int box_outer, bool mn_major, bool f16_split);
bool hg_tma_map_twin(CUtensorMap* m, const uint16_t* tw, int64_t K, int64_t rows, int64_t batch, int64_t ld,
                     int64_t bs, int box_rows);

namespace {

constexpr int TN = 128;   // RHS columns per CTA = MMA M of product 1, N of product 2
constexpr int BK = 32;    // K elements per pipeline stage (128-byte rows: 32 hi | 32 lo fp16, SWIZZLE_128B)
constexpr int NEPI = 256, NTHREADS = NEPI + 64;
constexpr int S1 = 4, S2 = 4;   // both rings are latency-bound: as many bytes in flight as shared memory holds

template <int KP>
struct ACfg {
  static constexpr int A1 = TN * BK * 4;                 // Y tile: fp32 landing = hi | lo fp16 after the split
  static constexpr int B1 = KP * BK * 4;                 // U twin: KP rows [hi | lo]
  static constexpr int STAGE1 = A1 + B1;
  static constexpr int ZS = TN * KP * 4;                 // Z as hi | lo fp16 k-blocks
  static constexpr int A2 = 128 * BK * 4;                // V twin tile: 128 rows [hi | lo]
  // one ring: product 1 uses S1 stages of it; afterwards Z sits in its first ZS bytes and the V tiles
  // of product 2 cycle through S2 stages behind Z
  static constexpr int RING = S1 * STAGE1 > ZS + S2 * A2 ? S1 * STAGE1 : ZS + S2 * A2;
  static constexpr int SMEM = RING + 1024;
  static constexpr int NKB2 = KP / BK;
  static constexpr int NCH2 = (NKB2 + 3) / 4;            // TMEM chunks of product 2 (24 MMAs each)
  static constexpr int HALF = KP / 2;                    // Z columns per epilogue thread
  static_assert(HALF % 32 == 0, "a thread's Z columns are whole k-blocks");
};

struct ApplyArgs {
  int T, b, k, ldk;
  const float* sigma;         // [nb][ldk]
  float scale;
  float* F;                   // [nb*b][T]
  int32_t* status;
  const uint32_t* amax;       // [3][amax_ld]: bits of max|Y_i|, max|U_i|, max|V_i| per block
  int amax_ld;
};

__device__ __forceinline__ uint32_t idesc_f16(int n) {   // D f32, A/B fp16 K-major, M = 128, N = n
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// exponent e <= cap with 2^e m < 2^15 (below the fp16 maximum); 0 for m = 0 or non-finite m.
// U, V use cap 14: every factor with |entries| < 2 gets the exponent of the unit bound, so measured
// maxima (caller-provided factors) and the unit bound (inside hg_solve) give the same bits.
__device__ __forceinline__ int f16_exp_of(float m, int cap = 100) {
  if (!(m > 0.f) || !isfinite(m)) return 0;
  const int e = 14 - ilogbf(m);
  return e > cap ? cap : e;   // (cap 100, denormal-scale data: 2^e and its inverse stay finite)
}

__device__ __forceinline__ void split8(const float* x, float sc, uint4& hv, uint4& lv) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float a = x[2 * j] * sc, c = x[2 * j + 1] * sc;
    const __half2 hh = __floats2half2_rn(a, c);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(a - hf.x, c - hf.y);
    h[j] = *reinterpret_cast<const uint32_t*>(&hh);
    l[j] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hv = make_uint4(h[0], h[1], h[2], h[3]);
  lv = make_uint4(l[0], l[1], l[2], l[3]);
}

#ifdef HG_APPLY_CLK
// debug build (-DHG_APPLY_CLK): %globaltimer stamps of the phases of the first 160 CTAs
__device__ unsigned long long g_aclk[160 * 32];
__device__ __forceinline__ void aclk(int slot) {
  const int c = blockIdx.y * gridDim.x + blockIdx.x;
  if (c < 160 && slot < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_aclk[c * 32 + slot] = t;
  }
}
#define ACLK(cond, slot) do { if (cond) aclk(slot); } while (0)
#else
#define ACLK(cond, slot) do { } while (0)
#endif

template <int KP>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_apply_fused(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmU,
                  const __grid_constant__ CUtensorMap tmV, ApplyArgs aa) {
  using C = ACfg<KP>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full1[S1], conv1[S1], empty1[S1], tfull1[2], tempty1[2];
  __shared__ __align__(8) uint64_t zs_bar, p1_bar, full2[S2], empty2[S2], tfull2[2], tempty2[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float rs_sh[KP];
  __shared__ float red_sh[NEPI / 32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * TN, g = blockIdx.y;
  ACLK(threadIdx.x == 0, 0);
  const int nkb1 = (aa.b + BK - 1) / BK, nch1 = (nkb1 + 3) / 4;
  const int nmt = (aa.b + 127) / 128;

  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* r2 = base + C::ZS;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmY);
    tma_prefetch(&tmU);
    tma_prefetch(&tmV);
    for (int s = 0; s < S1; ++s) {
      mbar_init(&full1[s], 1);
      mbar_init(&conv1[s], NEPI / 32);
      mbar_init(&empty1[s], 1);
    }
    for (int s = 0; s < S2; ++s) {
      mbar_init(&full2[s], 1);
      mbar_init(&empty2[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull1[i], 1);
      mbar_init(&tempty1[i], NEPI / 32);
      mbar_init(&tfull2[i], 1);
      mbar_init(&tempty2[i], NEPI / 32);
    }
    mbar_init(&zs_bar, NEPI / 32);
    mbar_init(&p1_bar, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(&tmem_base_sh);
  // Eq. 15 weights c / sigma_j (reading A14: sigma_j <= 1e-6 sigma_1 is flagged and dropped)
  for (int j = threadIdx.x; j < KP; j += NTHREADS) {
    float r = 0.f;
    if (j < aa.k) {
      const float s = aa.sigma[(int64_t)g * aa.ldk + j], s1 = aa.sigma[(int64_t)g * aa.ldk];
      if (!isfinite(s) || !(s > 1e-6f * s1)) {
        if (blockIdx.x == 0) hg_flag(aa.status, isfinite(s) ? HGS_SINGULAR_SIGMA : HGS_NONFINITE);
      } else {
        r = aa.scale / s;
      }
    }
    rs_sh[j] = r;
  }
  const float ymax = __uint_as_float(aa.amax[g]);
  const float umax = __uint_as_float(aa.amax[aa.amax_ld + g]);
  const float vmax = __uint_as_float(aa.amax[2 * aa.amax_ld + g]);
  if (blockIdx.x == 0 && threadIdx.x == 0 && !(isfinite(ymax) && isfinite(umax) && isfinite(vmax)))
    hg_flag(aa.status, HGS_NONFINITE);
  const int ey = f16_exp_of(ymax), eu = f16_exp_of(umax, 14), ev = f16_exp_of(vmax, 14);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sbase = smem_u32(base);
  ACLK(threadIdx.x == 0, 1);

  if (warp == 8) {
    // ---------------- TMA producer (converged warp, one elected lane issues)
    for (int kb = 0; kb < nkb1; ++kb) {
      const int s = kb % S1;
      const uint32_t ph = (kb / S1) & 1;
      if (kb >= S1) mbar_wait(&empty1[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = base + s * C::STAGE1;
        mbar_arrive_expect_tx(&full1[s], C::STAGE1);
#pragma unroll
        for (int c = 0; c < TN / 32; ++c) tma_load_3d(st + c * 4096, &tmY, &full1[s], t0 + 32 * c, kb * BK, g);
        tma_load_3d(st + C::A1, &tmU, &full1[s], 2 * kb * BK, 0, g);
      }
      __syncwarp();
    }
    // the V ring reuses product-1 stage memory: wait until every product-1 MMA has read its operands
    // (a barrier of its own: a parity wait on tfull1 is only exact for a waiter that follows every phase)
    mbar_wait(&p1_bar, 0);
    int idx = 0;
    for (int mt = 0; mt < nmt; ++mt)
      for (int kb2 = 0; kb2 < C::NKB2; ++kb2, ++idx) {
        const int s = idx % S2;
        const uint32_t ph = (idx / S2) & 1;
        if (idx >= S2) mbar_wait(&empty2[s], ph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&full2[s], C::A2);
          tma_load_3d(r2 + s * C::A2, &tmV, &full2[s], 2 * kb2 * BK, mt * 128, g);
        }
        __syncwarp();
      }
  } else if (warp == 9) {
    // ---------------- MMA issuer (converged warp, one elected lane issues)
    // every operand: K-major SWIZZLE_128B rows [hi 32 k | lo 32 k], 8-row groups 1024 B apart (SBO),
    // K-step 16 = +32 B in the row, the lo half at +64 B
    // product 1: A = Y tile (128 rows t, split in place), B = U twin tile (KP rows j)
    const uint32_t idesc1 = idesc_f16(KP);
    const uint32_t hiw = umma_desc_hi(1024, 2);
    for (int kb = 0; kb < nkb1; ++kb) {
      const int s = kb % S1;
      const uint32_t ph = (kb / S1) & 1;
      const int c = kb >> 2, buf = c & 1;
      const bool first = (kb & 3) == 0;
      if (first && c >= 2) {
        mbar_wait(&tempty1[buf], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      mbar_wait(&conv1[s], ph);
      tc_fence_after();
      const bool last_in_chunk = (kb & 3) == 3 || kb == nkb1 - 1;
      if (elect_one()) {
        ACLK(kb == 0, 2);
        ACLK(kb == nkb1 - 1, 3);
        const uint32_t d = tmem + (uint32_t)(buf * KP);
        const uint32_t st0 = sbase + s * C::STAGE1;
        const uint32_t a0 = umma_desc_lo(st0, 16), b0 = umma_desc_lo(st0 + C::A1, 16);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint64_t dah = umma_desc2(a0 + kk * 2, hiw), dal = umma_desc2(a0 + 4 + kk * 2, hiw);
          const uint64_t dbh = umma_desc2(b0 + kk * 2, hiw), dbl = umma_desc2(b0 + 4 + kk * 2, hiw);
          mma_f16(d, dal, dbh, idesc1, (first && kk == 0) ? 0u : 1u);
          mma_f16(d, dah, dbl, idesc1, 1);
          mma_f16(d, dah, dbh, idesc1, 1);
        }
        mma_commit(&empty1[s]);
        if (last_in_chunk) mma_commit(&tfull1[buf]);
        if (kb == nkb1 - 1) mma_commit(&p1_bar);
      }
      __syncwarp();
    }
    // product 2: Z k-block kb2 (128 rows t) in the product-1 ring's memory and the V twin tile (128 rows m)
    mbar_wait(&zs_bar, 0);
    tc_fence_after();
    ACLK(lane == 0, 5);
    const uint32_t idesc2 = idesc_f16(TN);
    int idx = 0;
    for (int mt = 0; mt < nmt; ++mt) {
      const int buf2 = mt & 1;
      if (mt >= 2) {
        mbar_wait(&tempty2[buf2], ((mt >> 1) - 1) & 1);
        tc_fence_after();
      }
      for (int kb2 = 0; kb2 < C::NKB2; ++kb2, ++idx) {
        const int s = idx % S2;
        const uint32_t ph = (idx / S2) & 1;
        mbar_wait(&full2[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t d = tmem + (uint32_t)(buf2 * 256 + (kb2 >> 2) * 128);
          // F^T tile: lanes = RHS column t (A = Z^T k-block), TMEM columns = row m of the tile (B = V tile):
          // a warp's 32 lanes then store 32 consecutive t of one F row, 128 contiguous bytes
          const uint32_t b0 = umma_desc_lo(sbase + C::ZS + s * C::A2, 16);
          const uint32_t a0 = umma_desc_lo(sbase + kb2 * (TN * BK * 4), 16);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint64_t dah = umma_desc2(a0 + kk * 2, hiw), dal = umma_desc2(a0 + 4 + kk * 2, hiw);
            const uint64_t dbh = umma_desc2(b0 + kk * 2, hiw), dbl = umma_desc2(b0 + 4 + kk * 2, hiw);
            mma_f16(d, dal, dbh, idesc2, ((kb2 & 3) == 0 && kk == 0) ? 0u : 1u);
            mma_f16(d, dah, dbl, idesc2, 1);
            mma_f16(d, dah, dbh, idesc2, 1);
          }
          mma_commit(&empty2[s]);
          if (kb2 == C::NKB2 - 1) mma_commit(&tfull2[buf2]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- warps 0-7: Y split, product-1 drains, Z scale + re-split, F drains and stores
    const int t = threadIdx.x;
    const int q = warp & 3, h = warp >> 2;   // TMEM lane quarter, column half
    const float ysc = ldexpf(1.0f, ey);
    float acc[C::HALF];
#pragma unroll
    for (int j = 0; j < C::HALF; ++j) acc[j] = 0.f;
    auto drain = [&](int dch) {
      const int buf = dch & 1;
      mbar_wait(&tfull1[buf], (dch >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * KP + h * C::HALF);
#pragma unroll
      for (int j0 = 0; j0 < C::HALF; j0 += 16) {
        float v[16];
        tmem_ld16(ta + j0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[j0 + i] += v[i];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty1[buf]);
    };
    int drained = 0;
    for (int kb = 0; kb < nkb1; ++kb) {
      const int s = kb % S1;
      const uint32_t ph = (kb / S1) & 1;
      mbar_wait(&full1[s], ph);
      // the tile landed as 4 chunks [32 rows kk][32 columns t] (128-byte rows, SWIZZLE_128B); thread
      // units (t row r, 4 consecutive kk) are read transposed, then written as K-major rows t of
      // [hi 32 kk | lo 32 kk] (128 bytes, SWIZZLE_128B: 16-byte unit u of row r at u ^ (r & 7))
      uint8_t* reg = base + s * C::STAGE1;
      float4 x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = t + i * NEPI, kq = u >> 7, r = u & 127;
        const uint8_t* col = reg + (r >> 5) * 4096 + (r & 3) * 4;
        const int ch = (r & 31) >> 2;
        float e[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int kk = 4 * kq + j;
          e[j] = *reinterpret_cast<const float*>(col + kk * 128 + ((ch ^ (kk & 7)) << 4)) * ysc;
        }
        x[i] = make_float4(e[0], e[1], e[2], e[3]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NEPI) : "memory");
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = t + i * NEPI, kq = u >> 7, r = u & 127;
        uint2 hv, lv;
        split4(x[i], 1.0f, hv, lv);
        uint8_t* row = reg + r * 128 + ((kq & 1) << 3);
        *reinterpret_cast<uint2*>(row + (((kq >> 1) ^ (r & 7)) << 4)) = hv;
        *reinterpret_cast<uint2*>(row + (((4 + (kq >> 1)) ^ (r & 7)) << 4)) = lv;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv1[s]);
      while (drained < nch1 - 1 && kb >= (drained + 1) * 4 + 1) drain(drained++);
    }
    while (drained < nch1) drain(drained++);
    ACLK(t == 0, 4);

    // Z^T[t][j] = acc * c / sigma_j * 2^-(e_y + e_u); CTA-local exponent e_z from max|Z|
    const float a1 = ldexpf(1.0f, -(ey + eu));
    float zmax = 0.f;
#pragma unroll
    for (int j = 0; j < C::HALF; ++j) {
      acc[j] *= rs_sh[h * C::HALF + j] * a1;
      zmax = fmaxf(zmax, isfinite(acc[j]) ? fabsf(acc[j]) : INFINITY);
    }
    for (int o = 16; o; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    if (lane == 0) red_sh[warp] = zmax;
    // every warp is past its last drain here: the product-1 MMAs have finished reading the ring
    asm volatile("bar.sync 1, %0;" ::"n"(NEPI) : "memory");
#pragma unroll
    for (int w = 0; w < NEPI / 32; ++w) zmax = fmaxf(zmax, red_sh[w]);
    if (t == 0 && !isfinite(zmax)) hg_flag(aa.status, HGS_NONFINITE);
    const int ez = f16_exp_of(zmax) - 1;   // 2^e_z max|Z| in [2^13, 2^14)
    const float zsc = isfinite(zmax) && zmax > 0.f ? ldexpf(1.0f, ez) : 1.0f;
    {
      const int r = q * 32 + lane;
      const int sw = r & 7;
#pragma unroll
      for (int kbl = 0; kbl < C::HALF / 32; ++kbl) {
        uint8_t* zb = base + (h * (C::HALF / 32) + kbl) * (TN * BK * 4) + r * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 hv, lv;
          split8(&acc[kbl * 32 + u * 8], zsc, hv, lv);
          *reinterpret_cast<uint4*>(zb + ((u ^ sw) << 4)) = hv;
          *reinterpret_cast<uint4*>(zb + (((4 + u) ^ sw) << 4)) = lv;
        }
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&zs_bar);

    // F tiles: drain, rescale by 2^-(e_v + e_z), store (a warp instruction = 128 contiguous bytes of one F row)
    const float a2 = (isfinite(zmax) && zmax > 0.f) ? ldexpf(1.0f, -(ev + ez)) : ldexpf(1.0f, -ev);
    for (int mt = 0; mt < nmt; ++mt) {
      const int buf2 = mt & 1;
      mbar_wait(&tfull2[buf2], (mt >> 1) & 1);
      tc_fence_after();
      ACLK(t == 0, 6 + 2 * mt);
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf2 * 256 + h * 64);
      float v[64];
#pragma unroll
      for (int j0 = 0; j0 < 64; j0 += 16) {
        float w[16];
        tmem_ld16(ta + j0, w);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[j0 + i] = w[i];
        if (C::NCH2 == 2) {
          tmem_ld16(ta + 128 + j0, w);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[j0 + i] += w[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty2[buf2]);
      ACLK(t == 0, 22 + mt);
      // thread = RHS column tt, v[j] = F[row mt*128 + h*64 + j][tt]
      const int tt = t0 + q * 32 + lane;
      if (tt < aa.T) {
        float* fcol = aa.F + ((int64_t)g * aa.b + mt * 128 + h * 64) * aa.T + tt;
        const int mrows = min(64, aa.b - (mt * 128 + h * 64));
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (j < mrows) fcol[(int64_t)j * aa.T] = v[j] * a2;
      }
      ACLK(t == 0, 7 + 2 * mt);
    }
  }
  tc_fence_before();
  __syncthreads();
  ACLK(threadIdx.x == 0, 31);
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ prep kernels
// out[g] = bits of max |x| over block g's n4 float4 (non-negative floats order like their bits; out zeroed
// by the caller; a NaN sets the exponent bits so the consumer flags it)
__global__ void __launch_bounds__(256) k_absmax(const float* __restrict__ x, int64_t n4, uint32_t* __restrict__ out) {
  __shared__ uint32_t red[8];
  const float4* p = reinterpret_cast<const float4*>(x) + (int64_t)blockIdx.y * n4;
  uint32_t m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = p[i];
    m = max(max(m, __float_as_uint(v.x) & 0x7fffffffu), __float_as_uint(v.y) & 0x7fffffffu);
    m = max(max(m, __float_as_uint(v.z) & 0x7fffffffu), __float_as_uint(v.w) & 0x7fffffffu);
  }
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = max(m, red[w]);
    atomicMax(out + blockIdx.y, m);
  }
}

// out[p * ld + i] = v for the planes p < 2, i < n
__global__ void k_fill_bits(uint32_t* out, int n, int ld, uint32_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 2 * n) out[(i / n) * ld + i % n] = v;
}

// U twin (tw_off layout) of x [nb][rows][b]: fp16(2^e x), e from amax[g]
__global__ void __launch_bounds__(256) k_split_rows(const float* __restrict__ x, int64_t per_block8,
                                                    const uint32_t* __restrict__ amax, uint16_t* __restrict__ out16) {
  const int g = blockIdx.y;
  const float sc = ldexpf(1.0f, f16_exp_of(__uint_as_float(amax[g]), 14));
  const int64_t base = (int64_t)g * per_block8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_block8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(x)[2 * (base + i)];
    const float4 c = reinterpret_cast<const float4*>(x)[2 * (base + i) + 1];
    const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    uint4 hv, lv;
    split8(v, sc, hv, lv);
    uint16_t* o = out16 + tw_off(8 * (base + i));
    *reinterpret_cast<uint4*>(o) = hv;
    *reinterpret_cast<uint4*>(o + TW_LO) = lv;
  }
}

// V twin, transposed: src Vt [nb][ldk][b] (row j = singular vector j) -> the twin (tw_off layout) of
// V [nb][b][k], fp16(2^e V[i][j]); grid (ceil(b/32), k/32, nb), 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(256) k_split_t(const float* __restrict__ Vt, int b, int k, int ldk,
                                                 const uint32_t* __restrict__ amax, uint16_t* __restrict__ out16,
                                                 const int32_t* __restrict__ perm, const float* __restrict__ vs) {
  __shared__ float tile[32][33];
  const int g = blockIdx.z, i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float sc = ldexpf(1.0f, f16_exp_of(__uint_as_float(amax[g]), 14));
#pragma unroll
  for (int jj = w; jj < 32; jj += 8) {
    const int j = j0 + jj, i = i0 + lane;
    float x = 0.f;
    if (j < k && i < b) {
      // perm: row j of V^T is row perm[j] of the unsorted B^T U~ panel times sign_j / sigma_j (finalize.cu)
      const int js = perm ? perm[(int64_t)g * ldk + j] : j;
      x = Vt[((int64_t)g * ldk + js) * b + i] * (perm ? vs[(int64_t)g * ldk + j] * sc : sc);
    }
    tile[jj][lane] = x;
  }
  __syncthreads();
  const int i = threadIdx.x >> 3, jq = threadIdx.x & 7;   // row i of the tile, 4 consecutive j
  if (i0 + i < b && j0 + 4 * jq < k) {
    const float x0 = tile[4 * jq][i], x1 = tile[4 * jq + 1][i], x2 = tile[4 * jq + 2][i], x3 = tile[4 * jq + 3][i];
    uint2 hv, lv;
    split4(make_float4(x0, x1, x2, x3), 1.0f, hv, lv);
    uint16_t* o = out16 + tw_off(((int64_t)g * b + i0 + i) * k + j0 + 4 * jq);
    *reinterpret_cast<uint2*>(o) = hv;
    *reinterpret_cast<uint2*>(o + TW_LO) = lv;
  }
}

template <int KP>
cudaError_t launch_fused(const CUtensorMap& tY, const CUtensorMap& tU, const CUtensorMap& tV, const ApplyArgs& aa,
                         int nb, cudaStream_t s) {
  using C = ACfg<KP>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_apply_fused<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((aa.T + TN - 1) / TN, nb);
  k_apply_fused<KP><<<grid, NTHREADS, C::SMEM, s>>>(tY, tU, tV, aa);
  return cudaGetLastError();
}

}  // namespace

#ifdef HG_APPLY_CLK
extern "C" int hg_debug_apply_clk(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_aclk, sizeof(unsigned long long) * (size_t)n);
}
#endif

bool apply_fused_supported(int b, int k, int ldk, int T, const void* Ut, const void* Vt, const void* Y, const void* F) {
  static const bool off = [] {
    const char* v = getenv("HG_APPLY_FUSED");
    return v && v[0] == '0';
  }();
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return !off && k >= 32 && k <= 256 && (k % 32) == 0 && (b % 32) == 0 && (T % 4) == 0 && T > 0 && ldk >= k &&
         al16(Ut) && al16(Vt) && al16(Y) && al16(F);
}

size_t apply_fused_amax_bytes(int nb) { return sizeof(uint32_t) * 3 * (size_t)nb; }

// Apply prep: the exponent words and the operand twins of the fused kernel.
// Ut, Vt [nb][ldk][b] fp32; u16, v16: the twins (tw_off layout) of Ut [nb][ldk][b] and of V [nb][b][k];
// amax: [3][amax_ld] words, this part's first block at [0].  uv_unit: |U|, |V| <= 1
// (exponent 14, no max pass); otherwise the per-block maxima are measured.
cudaError_t launch_apply_prep(const float* Ut, const float* Vt, int nb, int b, int k, int ldk, const float* Y, int T,
                              uint16_t* u16, uint16_t* v16, uint32_t* amax, int amax_ld, bool uv_unit,
                              cudaStream_t s, int* launches, const int32_t* perm, const float* vs) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(amax, 0, sizeof(uint32_t) * nb, s)) != cudaSuccess) return e;
  const int64_t y4 = (int64_t)b * T / 4;
  const int gx = (int)std::min<int64_t>((y4 + 255) / 256, std::max(1, 148 * 8 / nb));
  k_absmax<<<dim3(gx, nb), 256, 0, s>>>(Y, y4, amax);
  ++*launches;
  const int64_t u4 = (int64_t)ldk * b / 4;
  const int gu = (int)std::min<int64_t>((u4 + 255) / 256, std::max(1, 148 * 8 / nb));
  if (uv_unit) {
    k_fill_bits<<<(2 * nb + 255) / 256, 256, 0, s>>>(amax + amax_ld, nb, amax_ld, 0x3f800000u);
    ++*launches;
  } else {
    if ((e = cudaMemsetAsync(amax + amax_ld, 0, sizeof(uint32_t) * nb, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(amax + 2 * amax_ld, 0, sizeof(uint32_t) * nb, s)) != cudaSuccess) return e;
    k_absmax<<<dim3(gu, nb), 256, 0, s>>>(Ut, u4, amax + amax_ld);
    k_absmax<<<dim3(gu, nb), 256, 0, s>>>(Vt, u4, amax + 2 * amax_ld);
    *launches += 2;
  }
  if (!perm) {
    k_split_rows<<<dim3(gu, nb), 256, 0, s>>>(Ut, (int64_t)ldk * b / 8, amax + amax_ld, u16);
    ++*launches;
  }
  k_split_t<<<dim3((b + 31) / 32, (k + 31) / 32, nb), 256, 0, s>>>(Vt, b, k, ldk, amax + 2 * amax_ld, v16, perm, vs);
  ++*launches;
  return cudaGetLastError();
}

// The fused kernel on the twins and exponent words of launch_apply_prep; sigma [nb][ldk], Y, F [nb*b][T].
cudaError_t launch_apply_fused(const float* sigma, int nb, int b, int k, int ldk, const float* Y, int T, float scale,
                               float* F, int32_t* status, const uint16_t* u16, const uint16_t* v16,
                               const uint32_t* amax, int amax_ld, cudaStream_t s, int* launches) {
  CUtensorMap tY, tU, tV;
  const int KP = k <= 64 ? 64 : (k <= 128 ? 128 : 256);
  bool ok = hg_tma_map_f32(&tY, Y, T, b, nb, T, (int64_t)b * T, 32, true, true);
  ok = ok && hg_tma_map_twin(&tU, u16, b, k, nb, b, (int64_t)ldk * b, KP);
  ok = ok && hg_tma_map_twin(&tV, v16, k, b, nb, k, (int64_t)b * k, 128);
  if (!ok) return cudaErrorInvalidValue;
  ApplyArgs aa{T, b, k, ldk, sigma, scale, F, status, amax, amax_ld};
  ++*launches;
  if (KP == 64) return launch_fused<64>(tY, tU, tV, aa, nb, s);
  if (KP == 128) return launch_fused<128>(tY, tU, tV, aa, nb, s);
  return launch_fused<256>(tY, tU, tV, aa, nb, s);
}
