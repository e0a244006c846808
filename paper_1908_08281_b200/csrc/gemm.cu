// gemm.cu -- batched FP32 GEMM on the 5th-generation tensor cores via 3xTF32.
//
// Every dense contraction of the path runs here:
//   power products  Y = X_ii S       (X_ii^T S = X_ii S, reading A12)
//   Gram matrices   G = P^T P        (CholeskyQR2)
//   Q-formation     Q = P L^-T       (CholeskyQR2)
//   B = S^T X_ii, V = B^T U~, U = S U~, and the Eq. 15 apply
//
// Design (sm_100a):
//   * one CTA per 128 x BN output tile, 10 warps: warps 0-7 split each TMA-landed
//     fp32 tile into tf32 hi (in place) and lo (second buffer), drain finished
//     TMEM chunks and run the epilogue; warp 8 issues TMA (cp.async.bulk.tensor);
//     warp 9 allocates TMEM and one lane issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8).
//   * 3xTF32: D += A_lo B_hi + A_hi B_lo + A_hi B_hi, hi = x as read by the tensor
//     core (tf32 truncation), lo = x - trunc_tf32(x) written by the split warps
//     (HG_TF32_SPLIT=rna: hi = rna_tf32(x), lo = rna_tf32(x - hi)); reading A13.
//   * operands may be K-major or MN-major in global memory (both legal for
//     kind::tf32); the mbarrier ring is full(TMA) -> conv(split) -> empty(commit).
//   * accumulation: TMEM chunks of K = 64, ping-pong, summed in fp32 registers
//     (see gemm_tc_kernel); epilogue: scaled, coalesced stores (a warp owns 32
//     consecutive rows m, so a transposed store D[n][m] is one 128-byte line).
//   * 3xF16 (GemmDesc::prec = 1): the same pipeline on kind::f16 (twice the tf32 MMA rate):
//     hi = fp16_rn(2^e x), lo = fp16_rn(2^e x - hi) -- 22 significant bits like the tf32 pair,
//     the power-of-two prescale 2^e (from the caller's bound on |x|) keeps the pair inside the
//     fp16 exponent range.  Operands the producer stored as twins (GemmDesc::A16 / B16, the tw_off
//     layout of common.cuh) are TMA-loaded straight into 128-byte SWIZZLE_128B rows [hi | lo] and feed
//     the MMAs as they stand (PRE kernels: the epilogue warps only drain); fp32 operands are split in
//     place (fp32 landing tile -> K-major SWIZZLE_64B hi | lo halves, both majors).
//     TMEM chunks of K = 128 (24 MMAs per chunk, the same truncation bound as the tf32 path).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm.cuh"

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte swizzle row

struct EpiArgs {
  int M, N, K;
  float* D;
  int64_t ldd, sd;
  int d_trans;
  float alpha;
  const float* rs;
  int64_t srs;
  const float* cs;
  int64_t scs;
  int a_mn, b_mn;
  int trunc_hi;   // 1: hi = the raw fp32 tile (tensor core truncates to tf32), lo = x - trunc(x)
  int lower;      // skip tiles entirely above the diagonal (GemmDesc::lower)
  const float* C; // residual (row-major D only): D += beta * C
  int64_t ldc, sc;
  float beta;
  int b_upper;    // B(kk, n) = 0 for kk > n (GemmDesc::b_upper): per k-block, MMAs over n >= kk only
  // 3xF16 only
  float a_sc, b_sc;   // 2^a_exp, 2^b_exp: prescale of the in-kernel split
  // optional pre-split copy of the (transposed) output for a later 3xF16 GEMM: hi / lo planes of
  // fp16_rn(2^d_exp D) in the twin layout (tw_off) of D[g*sd + n*ldd + m] (both precisions)
  uint16_t* D16;
  float d_sc;
  int d16_only;   // store only the twin
};

constexpr int NEPI = 256;            // converter / epilogue threads (8 warps)
constexpr int NTHREADS = NEPI + 64;  // + TMA warp + MMA warp

template <int BN, bool F16>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;   // 16 KB (3xF16: the fp32 tile, then hi | lo fp16 halves)
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = F16 ? A_BYTES + B_BYTES : 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (STAGE_BYTES * 4 <= 200 * 1024) ? 4 : (STAGE_BYTES * 3 <= 200 * 1024 ? 3 : 2);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr uint32_t TX = (uint32_t)(BM + BN) * BK * 4;
  static constexpr int HALF = BN / 2;           // columns per epilogue warp
  static constexpr int CHUNK = F16 ? 4 : 2;     // k-blocks per TMEM chunk: 24 MMAs either way
  static_assert(8 * 32 * (HALF + 4) * 4 <= STAGES * STAGE_BYTES, "epilogue staging must fit the pipeline smem");
  static_assert(8 * HALF * 36 * 4 <= STAGES * STAGE_BYTES, "transposed staging must fit the pipeline smem");
};

// kind::tf32 instruction descriptor: D f32, A/B tf32, M = 128, N = BN.
__device__ __forceinline__ uint32_t make_idesc(int bn, int a_mn, int b_mn) {
  uint32_t d = 0;
  d |= 1u << 4;                      // c_format = F32
  d |= 2u << 7;                      // a_format = TF32
  d |= 2u << 10;                     // b_format = TF32
  d |= (uint32_t)(a_mn & 1) << 15;   // a_major
  d |= (uint32_t)(b_mn & 1) << 16;   // b_major
  d |= (uint32_t)(bn >> 3) << 17;    // n_dim
  d |= (uint32_t)(BM >> 4) << 24;    // m_dim
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B fp16 (format 0), both K-major, M = 128, N = bn.
__device__ __forceinline__ uint32_t make_idesc_f16(int bn) {
  return (1u << 4) | ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float trunc_lo(float x) {   // x - trunc_tf32(x), exact in fp32
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ float4 split_hi(float4& x) {
  float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
  float4 l = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z), tf32_rna(x.w - h.w));
  x = h;
  return l;
}

// Accumulation: the tensor pipe's fp32 adder truncates, so an accumulator that
// absorbs all K/8 * 3 MMAs loses accuracy linearly in K (measured 7e-6 relative
// at K = 1024).  The MMAs of each K-chunk of 64 go to a fresh TMEM buffer (two
// buffers, ping-pong); the epilogue warps drain finished chunks and sum them in
// fp32 round-to-nearest registers, bounding the truncation to 24 MMAs.
// PRE (3xF16 with both operands pre-split): each 128-byte shared-memory row holds the hi fp16 of the
// k-block's 32 K elements in bytes 0-63 and their lo in bytes 64-127 (SWIZZLE_128B K-major rows of 64
// "elements"; the TMA box is (32 k, {hi, lo}, rows)).  The hi K-steps sit at +0 / +32 B of the row, the
// lo ones at +64 / +96 B.  The tensor core fetches 64-byte-row (SWIZZLE_64B) operands at half rate
// (two rows of every 8-row core matrix share their banks: ~250 instead of 128 cycles per 128 x 256 x 16
// MMA, measured), so only the in-kernel-split 3xF16 paths -- whose 128-byte fp32 landing rows become a
// 64-byte hi and a 64-byte lo row in place -- keep that layout.
template <int BN, bool F16, bool PRE = false>
__global__ void __launch_bounds__(NTHREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   EpiArgs ea) {
  static_assert(!PRE || F16, "pre-split operands are 3xF16 only");
  using C = Cfg<BN, F16>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[C::STAGES], conv_bar[C::STAGES], empty_bar[C::STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, g = blockIdx.z;
  if (ea.lower && n0 >= m0 + BM) return;   // tile above the diagonal (uniform: before any setup)
  const int num_kb = (ea.K + BK - 1) / BK;
  const int nchunks = (num_kb + C::CHUNK - 1) / C::CHUNK;
  constexpr bool pre_ab = PRE;   // twin operands: no in-kernel split at all

  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto sA_hi = [&](int s) { return base + s * C::STAGE_BYTES; };
  auto sA_lo = [&](int s) { return base + s * C::STAGE_BYTES + C::A_BYTES; };
  // 3xF16: [A tile | B tile] per stage (each split in place); 3xTF32: [A hi | A lo | B hi | B lo]
  auto sB_hi = [&](int s) { return base + s * C::STAGE_BYTES + (F16 ? 1 : 2) * C::A_BYTES; };
  auto sB_lo = [&](int s) { return base + s * C::STAGE_BYTES + 2 * C::A_BYTES + C::B_BYTES; };

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&conv_bar[s], NEPI / 32);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], NEPI / 32);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<C::TMEM_COLS>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 8) {
    // ---------------- TMA producer: converged warp, one elected lane issues
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % C::STAGES;
      const uint32_t ph = (kb / C::STAGES) & 1;
      if (kb >= C::STAGES) mbar_wait(&empty_bar[s], ph ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full_bar[s], C::TX);
        const int k0 = kb * BK;
        if (PRE) {
          tma_load_3d(sA_hi(s), &tmA, &full_bar[s], 2 * k0, m0, g);   // rows of [hi 32 k | lo 32 k]
          tma_load_3d(sB_hi(s), &tmB, &full_bar[s], 2 * k0, n0, g);
        } else if (!ea.a_mn) {
          tma_load_3d(sA_hi(s), &tmA, &full_bar[s], k0, m0, g);
        } else {
#pragma unroll
          for (int c = 0; c < BM / 32; ++c) tma_load_3d(sA_hi(s) + c * 4096, &tmA, &full_bar[s], m0 + 32 * c, k0, g);
        }
        if (PRE) {
        } else if (!ea.b_mn) {
          tma_load_3d(sB_hi(s), &tmB, &full_bar[s], k0, n0, g);
        } else {
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) tma_load_3d(sB_hi(s) + c * 4096, &tmB, &full_bar[s], n0 + 32 * c, k0, g);
        }
      }
      __syncwarp();
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer: the warp stays converged, one elected lane issues (under
    // `if (lane == 0)` every UTCHMMA sat in a per-lane R2UR loop); descriptors from 32-bit words
    const uint32_t sbase = smem_u32(base);
    // 3xF16 twins (PRE): K-major SWIZZLE_128B rows [hi 32 k | lo 32 k], 8-row groups 1024 B apart (SBO),
    // K-step 16 = +32 B in the row, the lo half at +64 B.
    // 3xF16 split in the kernel: K-major SWIZZLE_64B fp16, 1 KB groups of 8 hi rows (64 B each) + 8 lo
    // rows (SBO 1024, lo at +512); K-step 16 = +32 B in the row.
    // 3xTF32, K-major (SWIZZLE_128B): 8-row groups 1024 B apart (SBO), K-step = +32 B in the row.
    // MN-major (SWIZZLE_128B_BASE32B): 32-element chunks BK*128 B apart (LBO),
    // 4-row groups 512 B apart (SBO), K-step = +1024 B (8 rows).
    const uint32_t idesc = F16 ? make_idesc_f16(BN) : make_idesc(BN, ea.a_mn, ea.b_mn);
    const uint32_t a_lbo = (!F16 && ea.a_mn) ? BK * 128 : 16, b_lbo = (!F16 && ea.b_mn) ? BK * 128 : 16;
    const uint32_t a_hiw = PRE ? umma_desc_hi(1024, 2)
                         : F16 ? umma_desc_hi(1024, 4) : umma_desc_hi(ea.a_mn ? 512 : 1024, ea.a_mn ? 1 : 2);
    const uint32_t b_hiw = PRE ? umma_desc_hi(1024, 2)
                         : F16 ? umma_desc_hi(1024, 4) : umma_desc_hi(ea.b_mn ? 512 : 1024, ea.b_mn ? 1 : 2);
    // offsets (in 16-byte units) of the lo operands from the hi ones and of a K-step; bytes per B row n
    const uint32_t a_lo_off = (PRE ? 64 : F16 ? 512 : C::A_BYTES) >> 4;
    const uint32_t b_lo_off = (PRE ? 64 : F16 ? 512 : C::B_BYTES) >> 4;
    const uint32_t a_kstep = (F16 ? 32 : (ea.a_mn ? 1024 : 32)) >> 4, b_kstep = (F16 ? 32 : (ea.b_mn ? 1024 : 32)) >> 4;
    const uint32_t b_row = 128;
    constexpr int KSTEPS = F16 ? BK / 16 : BK / 8;
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % C::STAGES;
      const uint32_t ph = (kb / C::STAGES) & 1;
      const int c = kb / C::CHUNK, buf = c & 1;
      const bool first = (kb % C::CHUNK) == 0;
      if (first && c >= 2) {
        mbar_wait(&tempty_bar[buf], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      // both operands pre-split: the TMA-landed tile is the MMA operand as it stands -- wait for
      // the TMA itself (the epilogue warps only drain)
      mbar_wait(pre_ab ? &full_bar[s] : &conv_bar[s], ph);
      tc_fence_after();
      // b_upper: columns n < kb * BK of this k-block are zero in B -- the MMAs cover
      // n >= nlo only (N = BN - nlo, TMEM columns and B rows offset by nlo, a multiple of 16);
      // the drain masks what a chunk never wrote
      const int nlo = ea.b_upper ? (max(0, kb * BK - n0) & ~15) : 0;
      const bool last_in_chunk = (kb % C::CHUNK) == C::CHUNK - 1 || kb == num_kb - 1;
      if (elect_one()) {
        if (nlo < BN) {
          const uint32_t idk = nlo ? (F16 ? make_idesc_f16(BN - nlo) : make_idesc(BN - nlo, ea.a_mn, ea.b_mn)) : idesc;
          const uint32_t d = tmem + (uint32_t)(buf * BN + nlo);
          const uint32_t st0 = sbase + s * C::STAGE_BYTES;
          const uint32_t a0 = umma_desc_lo(st0, a_lbo);
          const uint32_t b0 = umma_desc_lo(st0 + (F16 ? 1 : 2) * C::A_BYTES + nlo * b_row, b_lbo);
#pragma unroll
          for (int kk = 0; kk < KSTEPS; ++kk) {
            const uint64_t dah = umma_desc2(a0 + kk * a_kstep, a_hiw), dal = umma_desc2(a0 + a_lo_off + kk * a_kstep, a_hiw);
            const uint64_t dbh = umma_desc2(b0 + kk * b_kstep, b_hiw), dbl = umma_desc2(b0 + b_lo_off + kk * b_kstep, b_hiw);
            if constexpr (F16) {
              mma_f16(d, dal, dbh, idk, (first && kk == 0) ? 0u : 1u);
              mma_f16(d, dah, dbl, idk, 1);
              mma_f16(d, dah, dbh, idk, 1);
            } else {
              mma_tf32(d, dal, dbh, idk, (first && kk == 0) ? 0u : 1u);
              mma_tf32(d, dah, dbl, idk, 1);
              mma_tf32(d, dah, dbh, idk, 1);
            }
          }
        }
        mma_commit(&empty_bar[s]);
        if (last_in_chunk) mma_commit(&tfull_bar[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- warps 0-7: tf32 hi/lo split, chunk drains, epilogue
    const int t = threadIdx.x;
    const int q = warp & 3, h = warp >> 2;          // TMEM lane quarter, column half
    float acc[C::HALF];
#pragma unroll
    for (int j = 0; j < C::HALF; ++j) acc[j] = 0.f;
    auto drain = [&](int dch) {
      const int buf = dch & 1;
      mbar_wait(&tfull_bar[buf], (dch >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + h * C::HALF);
      // b_upper: tile columns below the chunk's first k-block's nlo were never written by it
      const int clo = ea.b_upper ? min(BN, max(0, dch * C::CHUNK * BK - n0) & ~15) - h * C::HALF : 0;
#pragma unroll
      for (int j0 = 0; j0 < C::HALF; j0 += 16) {
        float v[16];
        tmem_ld16(ta + j0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[j0 + i] += (j0 + i >= clo) ? v[i] : 0.f;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[buf]);
    };
    int drained = 0;
    for (int kb = pre_ab ? num_kb : 0; kb < num_kb; ++kb) {
      const int s = kb % C::STAGES;
      const uint32_t ph = (kb / C::STAGES) & 1;
      mbar_wait(&full_bar[s], ph);
      if constexpr (F16) {
        // In-place 3xF16 split into 8-row groups of 1 KB -- the group's 8 hi rows (64 B each,
        // SWIZZLE_64B), then its 8 lo rows: exactly the bytes its 8 fp32 rows occupied.
        // K-major tiles: a warp converts whole groups (2 float4 per lane, __syncwarp, store),
        // no CTA barrier.  MN-major tiles (32-row chunks [32 k][32 rows], SWIZZLE_128B) are
        // read transposed (4 rows k of one column per unit): all threads load, barrier, store.
        auto conv_k = [&](uint8_t* reg, int R, float sc) {
          for (int gi = warp; gi < R / 8; gi += NEPI / 32) {
            uint8_t* gb = reg + gi * 1024;
            float4 x[2];
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int u = lane + 32 * h2, rr = u >> 3, kq = u & 7;
              const float4 v = *reinterpret_cast<const float4*>(gb + rr * 128 + ((kq ^ rr) << 4));
              x[h2] = make_float4(v.x * sc, v.y * sc, v.z * sc, v.w * sc);
            }
            __syncwarp();
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int u = lane + 32 * h2;
              f16_split_store(gb, gb + 512, u >> 3, u & 7, x[h2]);
            }
          }
        };
        auto conv_mn = [&](uint8_t* reg, int R, float sc) {
          constexpr int UMAX = BN > BM ? BN * 8 / NEPI : BM * 8 / NEPI;
          float4 x[UMAX];
          const int nu = R * 8 / NEPI;
#pragma unroll
          for (int i = 0; i < UMAX; ++i) {
            if (i >= nu) break;
            const int u = t + i * NEPI, kq = u / R, r = u % R;
            const uint8_t* col = reg + (r >> 5) * 4096 + (r & 3) * 4;
            const int ch = (r & 31) >> 2;
            float e[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int kk = 4 * kq + j;
              e[j] = *reinterpret_cast<const float*>(col + kk * 128 + ((ch ^ (kk & 7)) << 4)) * sc;
            }
            x[i] = make_float4(e[0], e[1], e[2], e[3]);
          }
          asm volatile("bar.sync 1, %0;" ::"n"(NEPI) : "memory");
#pragma unroll
          for (int i = 0; i < UMAX; ++i) {
            if (i >= nu) break;
            const int u = t + i * NEPI, kq = u / R, r = u % R;
            uint8_t* gb = reg + (r >> 3) * 1024;
            f16_split_store(gb, gb + 512, r & 7, kq, x[i]);
          }
        };
        if (ea.a_mn) conv_mn(sA_hi(s), BM, ea.a_sc); else conv_k(sA_hi(s), BM, ea.a_sc);
        if (ea.b_mn) conv_mn(sB_hi(s), BN, ea.b_sc); else conv_k(sB_hi(s), BN, ea.b_sc);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_bar[s]);
        while (drained < nchunks - 1 && kb >= (drained + 1) * C::CHUNK + 1) drain(drained++);
        continue;
      }
      float4* ah = reinterpret_cast<float4*>(sA_hi(s));
      float4* al = reinterpret_cast<float4*>(sA_lo(s));
      float4* bh = reinterpret_cast<float4*>(sB_hi(s));
      float4* bl = reinterpret_cast<float4*>(sB_lo(s));
      // b_upper: B rows (n) below this k-block's nlo are never read by the MMAs -- not split
      const int b0 = ea.b_upper ? min(BN, max(0, kb * BK - n0) & ~15) * (BK / 4) : 0;
      if (ea.trunc_hi) {
#pragma unroll
        for (int i = t; i < BM * BK / 4; i += NEPI) {
          const float4 x = ah[i];
          al[i] = make_float4(trunc_lo(x.x), trunc_lo(x.y), trunc_lo(x.z), trunc_lo(x.w));
        }
#pragma unroll
        for (int i = b0 + t; i < BN * BK / 4; i += NEPI) {
          const float4 x = bh[i];
          bl[i] = make_float4(trunc_lo(x.x), trunc_lo(x.y), trunc_lo(x.z), trunc_lo(x.w));
        }
      } else {
#pragma unroll
        for (int i = t; i < BM * BK / 4; i += NEPI) {
          float4 x = ah[i];
          float4 l = split_hi(x);
          ah[i] = x;
          al[i] = l;
        }
#pragma unroll
        for (int i = b0 + t; i < BN * BK / 4; i += NEPI) {
          float4 x = bh[i];
          float4 l = split_hi(x);
          bh[i] = x;
          bl[i] = l;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv_bar[s]);
      // drain chunk d once the MMAs of chunk d+1 are under way
      while (drained < nchunks - 1 && kb >= (drained + 1) * C::CHUNK + 1) drain(drained++);
    }
    while (drained < nchunks) drain(drained++);
    // epilogue: scale and store.  Transposed output D[n][m]: a warp's 32 rows m are
    // one 128-byte line per column n, stored straight from registers.  Row-major
    // output D[m][n]: each warp stages its 32 x HALF sub-tile in the (now idle)
    // pipeline shared memory and writes it back row by row (128 bytes per store
    // instruction instead of 32 scattered rows).
    const int mrow = q * 32 + lane;
    const int m = m0 + mrow;
    const float rsv = (m < ea.M) ? ea.alpha * (ea.rs ? ea.rs[(int64_t)g * ea.srs + m] : 1.0f) : 0.f;
    float* Dg = ea.D + (int64_t)g * ea.sd;
    const int nb0 = n0 + h * C::HALF;
    if (ea.d_trans) {
      const int mw0 = m0 + q * 32;   // this warp's 32 rows m
      const bool fast = !ea.cs && (ea.ldd & 3) == 0 && ((reinterpret_cast<uintptr_t>(Dg) & 15) == 0) &&
                        mw0 + 32 <= ea.M;
      if (fast) {
        // stage the warp's HALF x 32 block transposed (st[j][lane], pitch 36), then store
        // D[n][m] rows as float4: 8 lanes cover one row's 32 m, four rows per instruction
        constexpr int TP = 36;
        float* st = reinterpret_cast<float*>(base) + warp * C::HALF * TP;
#pragma unroll
        for (int j = 0; j < C::HALF; ++j) st[j * TP + lane] = acc[j] * rsv;
        __syncwarp();
        const int l4 = lane & 7;
        float* dcol = Dg + mw0 + 4 * l4;
        for (int j = lane >> 3; j < C::HALF; j += 4) {
          const int n = nb0 + j;
          if (n < ea.N) {
            HG_DCHECK(mw0 + 4 * l4 + 3 < ea.ldd);
            const float4 v = *reinterpret_cast<const float4*>(st + j * TP + 4 * l4);
            if (!ea.d16_only) *reinterpret_cast<float4*>(dcol + (int64_t)n * ea.ldd) = v;
            if (ea.D16) {
              uint2 hv, lv;
              split4(v, ea.d_sc, hv, lv);
              uint16_t* d16 = ea.D16 + tw_off((int64_t)g * ea.sd + (int64_t)n * ea.ldd + mw0 + 4 * l4);
              *reinterpret_cast<uint2*>(d16) = hv;
              *reinterpret_cast<uint2*>(d16 + TW_LO) = lv;
            }
          }
        }
      } else if (m < ea.M) {
#pragma unroll
        for (int j = 0; j < C::HALF; ++j) {
          const int n = nb0 + j;
          if (n < ea.N) {
            float val = acc[j] * rsv;
            if (ea.cs) val *= ea.cs[(int64_t)g * ea.scs + n];
            if (!ea.d16_only) Dg[(int64_t)n * ea.ldd + m] = val;
            if (ea.D16) {
              const float x = val * ea.d_sc;
              const __half hh = __float2half_rn(x);
              const __half ll = __float2half_rn(x - __half2float(hh));
              uint16_t* d16 = ea.D16 + tw_off((int64_t)g * ea.sd + (int64_t)n * ea.ldd + m);
              d16[0] = *reinterpret_cast<const uint16_t*>(&hh);
              d16[TW_LO] = *reinterpret_cast<const uint16_t*>(&ll);
            }
          }
        }
      }
    } else {
      // pitch HALF + 4: float4 writes of 8 lanes per phase hit disjoint banks
      constexpr int LDS = C::HALF + 4;
      float* st = reinterpret_cast<float*>(base) + warp * 32 * LDS;
#pragma unroll
      for (int j = 0; j < C::HALF; j += 4)
        *reinterpret_cast<float4*>(st + lane * LDS + j) =
            make_float4(acc[j] * rsv, acc[j + 1] * rsv, acc[j + 2] * rsv, acc[j + 3] * rsv);
      __syncwarp();
      const int mrows = min(32, ea.M - (m0 + q * 32));
      const bool vec = ((ea.ldd & 3) == 0) && ((reinterpret_cast<uintptr_t>(Dg) & 15) == 0);
      constexpr int CW = C::HALF < 128 ? C::HALF : 128;   // columns per warp instruction
      for (int r = 0; r < mrows; ++r) {
        float* drow = Dg + (int64_t)(m0 + q * 32 + r) * ea.ldd;
#pragma unroll
        for (int c = 0; c < C::HALF; c += CW) {
          const int cl = c + 4 * lane;
          if (cl >= C::HALF) continue;
          const int n = nb0 + cl;
          float4 v = *reinterpret_cast<const float4*>(st + r * LDS + cl);
          if (ea.cs) {
            const float* csg = ea.cs + (int64_t)g * ea.scs;
            if (n < ea.N) v.x *= csg[n];
            if (n + 1 < ea.N) v.y *= csg[n + 1];
            if (n + 2 < ea.N) v.z *= csg[n + 2];
            if (n + 3 < ea.N) v.w *= csg[n + 3];
          }
          if (ea.C) {
            const float* crow = ea.C + (int64_t)g * ea.sc + (int64_t)(m0 + q * 32 + r) * ea.ldc;
            if (vec && n + 3 < ea.N) {
              const float4 cv = *reinterpret_cast<const float4*>(crow + n);
              v.x = fmaf(ea.beta, cv.x, v.x); v.y = fmaf(ea.beta, cv.y, v.y);
              v.z = fmaf(ea.beta, cv.z, v.z); v.w = fmaf(ea.beta, cv.w, v.w);
            } else {
              if (n < ea.N) v.x = fmaf(ea.beta, crow[n], v.x);
              if (n + 1 < ea.N) v.y = fmaf(ea.beta, crow[n + 1], v.y);
              if (n + 2 < ea.N) v.z = fmaf(ea.beta, crow[n + 2], v.z);
              if (n + 3 < ea.N) v.w = fmaf(ea.beta, crow[n + 3], v.w);
            }
          }
          if (vec && n + 3 < ea.N) {
            *reinterpret_cast<float4*>(drow + n) = v;
          } else {
            if (n < ea.N) drow[n] = v.x;
            if (n + 1 < ea.N) drow[n + 1] = v.y;
            if (n + 2 < ea.N) drow[n + 2] = v.z;
            if (n + 3 < ea.N) drow[n + 3] = v.w;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ SIMT fp32 (verification)
__global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A, int a_mn, int64_t lda,
                                                        int64_t sa, const float* __restrict__ B, int b_mn,
                                                        int64_t ldb, int64_t sb, EpiArgs ea) {
  __shared__ float As[16][64 + 1], Bs[16][64 + 1];
  const int g = blockIdx.z, m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const float* Ag = A + (int64_t)g * sa;
  const float* Bg = B + (int64_t)g * sb;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < ea.K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i / 64, mm = i % 64;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < ea.M && k < ea.K) ? Ag[a_mn ? (int64_t)k * lda + m : (int64_t)m * lda + k] : 0.f;
      const int n = n0 + mm;
      Bs[kk][mm] = (n < ea.N && k < ea.K) ? Bg[b_mn ? (int64_t)k * ldb + n : (int64_t)n * ldb + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Bs[kk][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
  float* Dg = ea.D + (int64_t)g * ea.sd;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < ea.M && n < ea.N) {
        float v = acc[i][j] * ea.alpha;
        if (ea.rs) v *= ea.rs[(int64_t)g * ea.srs + m];
        if (ea.cs) v *= ea.cs[(int64_t)g * ea.scs + n];
        if (ea.C) v = fmaf(ea.beta, ea.C[(int64_t)g * ea.sc + (int64_t)m * ea.ldc + n], v);
        if (ea.d_trans)
          Dg[(int64_t)n * ea.ldd + m] = v;
        else
          Dg[(int64_t)m * ea.ldd + n] = v;
      }
    }
}

// ------------------------------------------------------------------ pre-split producer
// The 3xF16 twin (common.cuh tw_off) of a dense rows x cols fp32 matrix (row pitch ld, cols % 32 == 0):
// hi = fp16_rn(2^e x), lo = fp16_rn(2^e x - hi); 8 elements per thread (16-byte fp16 stores).
__global__ void __launch_bounds__(256) k_f16_split(const float* __restrict__ x, int64_t rows, int cols, int64_t ld,
                                                   float sc, uint16_t* __restrict__ out16) {
  const int c8 = cols / 8;
  const int64_t n = rows * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / c8;
    const int c = (int)(i % c8) * 8;
    const float4 a = *reinterpret_cast<const float4*>(x + r * ld + c);
    const float4 b = *reinterpret_cast<const float4*>(x + r * ld + c + 4);
    const float v[8] = {a.x * sc, a.y * sc, a.z * sc, a.w * sc, b.x * sc, b.y * sc, b.z * sc, b.w * sc};
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __half2 hh = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
      const float2 hf = __half22float2(hh);
      const __half2 ll = __floats2half2_rn(v[2 * j] - hf.x, v[2 * j + 1] - hf.y);
      h[j] = *reinterpret_cast<const uint32_t*>(&hh);
      l[j] = *reinterpret_cast<const uint32_t*>(&ll);
    }
    uint16_t* o = out16 + tw_off(r * cols + c);
    *reinterpret_cast<uint4*>(o) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(o + TW_LO) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3D map: (inner, outer, batch), row pitch ld elements, batch pitch bs elements; box (32, box_outer, 1).
// MN-major fp32 tiles use 32-byte swizzle atoms for the tf32 MMA (its only legal MN-major form),
// plain SWIZZLE_128B when the 3xF16 split reads them (f16_split = true).
bool make_map(CUtensorMap* m, const float* ptr, int64_t inner, int64_t outer, int64_t batch, int64_t ld,
              int64_t bs, int box_outer, bool mn_major, bool f16_split = false) {
  auto enc = get_encode();
  if (!enc) return false;
  if (batch <= 1) bs = ld * outer;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(batch < 1 ? 1 : batch)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)bs * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)box_outer, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (mn_major && !f16_split) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3xF16 twin operand (common.cuh tw_off): logical [batch][rows][K] (row pitch ld, batch pitch bs, in
// logical elements, multiples of 32) is [batch][rows][2 ld] fp16; box (64, box_rows, 1) at inner
// coordinate 2 k0 lands as 128-byte rows [hi 32 k | lo 32 k], SWIZZLE_128B.
bool make_map_twin(CUtensorMap* m, const uint16_t* tw, int64_t K, int64_t rows, int64_t batch, int64_t ld,
                   int64_t bs, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  if (batch <= 1) bs = ld * rows;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * K), (cuuint64_t)rows, (cuuint64_t)(batch < 1 ? 1 : batch)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)bs * 4};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(tw), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool F16, bool PRE = false>
cudaError_t launch_tc(const GemmDesc& g, const EpiArgs& ea, cudaStream_t stream) {
  using C = Cfg<BN, F16>;
  static bool attr_set = false;  // per-instantiation; set once per process
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, F16, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  CUtensorMap ta, tb;
  bool ok;
  if (PRE)
    ok = make_map_twin(&ta, g.A16, g.K, g.M, g.batch, g.lda, g.sa, BM);
  else
    ok = g.a_mn ? make_map(&ta, g.A, g.M, g.K, g.batch, g.lda, g.sa, 32, true, F16)
                : make_map(&ta, g.A, g.K, g.M, g.batch, g.lda, g.sa, BM, false);
  if (PRE)
    ok = ok && make_map_twin(&tb, g.B16, g.K, g.N, g.batch, g.ldb, g.sb, BN);
  else
    ok = ok && (g.b_mn ? make_map(&tb, g.B, g.N, g.K, g.batch, g.ldb, g.sb, 32, true, F16)
                       : make_map(&tb, g.B, g.K, g.N, g.batch, g.ldb, g.sb, BN, false));
  if (!ok) return cudaErrorInvalidValue;
  dim3 grid((g.M + BM - 1) / BM, (g.N + BN - 1) / BN, g.batch);
  gemm_tc_kernel<BN, F16, PRE><<<grid, NTHREADS, C::SMEM, stream>>>(ta, tb, ea);
  return cudaGetLastError();
}

}  // namespace

bool hg_tma_map_f32(CUtensorMap* m, const float* ptr, int64_t inner, int64_t outer, int64_t batch, int64_t ld,
                    int64_t bs, int box_outer, bool mn_major, bool f16_split) {
  return make_map(m, ptr, inner, outer, batch, ld, bs, box_outer, mn_major, f16_split);
}
bool hg_tma_map_twin(CUtensorMap* m, const uint16_t* tw, int64_t K, int64_t rows, int64_t batch, int64_t ld,
                     int64_t bs, int box_rows) {
  return make_map_twin(m, tw, K, rows, batch, ld, bs, box_rows);
}

static int prec_env() {   // HG_GEMM_PREC=f16 | tf32: the precision of GEMMs that leave GemmDesc::prec = -1
  static const int p = [] {
    const char* v = getenv("HG_GEMM_PREC");
    return (v && v[0] == 'f') ? 1 : 0;
  }();
  return p;
}

int gemm_prec(const GemmDesc& g) { return g.prec >= 0 ? g.prec : prec_env(); }

const char* gemm_check(const GemmDesc& g) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return "gemm: non-positive size";
  if (g.batch > 65535) return "gemm: batch > 65535";
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool pa = g.A16 != nullptr, pb = g.B16 != nullptr;
  if ((pa || pb) && gemm_prec(g) != 1) return "gemm: 3xF16 twin operands need prec = 1";
  if (pa != pb) return "gemm: 3xF16 twin operands come in pairs (A16 and B16)";
  if (pa ? (!al16(g.A16) || (g.lda & 31) || (g.batch > 1 && (g.sa & 31)) || g.lda < g.K) : (!g.A || !al16(g.A)))
    return pa ? "gemm: twin A needs 16-byte alignment, lda and sa multiples of 32, lda >= K"
              : "gemm: A must be non-null and 16-byte aligned";
  if (pb ? (!al16(g.B16) || (g.ldb & 31) || (g.batch > 1 && (g.sb & 31)) || g.ldb < g.K) : (!g.B || !al16(g.B)))
    return pb ? "gemm: twin B needs 16-byte alignment, ldb and sb multiples of 32, ldb >= K"
              : "gemm: B must be non-null and 16-byte aligned";
  if ((!pa && (g.lda & 3)) || (!pb && (g.ldb & 3))) return "gemm: lda/ldb must be multiples of 4";
  if (g.batch > 1 && ((!pa && (g.sa & 3)) || (!pb && (g.sb & 3)))) return "gemm: batch strides must be multiples of 4";
  if (!pa && (g.a_mn ? g.lda < g.M : g.lda < g.K)) return "gemm: lda too small";
  if (!pb && (g.b_mn ? g.ldb < g.N : g.ldb < g.K)) return "gemm: ldb too small";
  if (g.C && (g.d_trans || g.ldc < g.N)) return "gemm: residual C needs row-major D and ldc >= N";
  if (g.a_exp < -40 || g.a_exp > 40 || g.b_exp < -40 || g.b_exp > 40 || g.d_exp < -40 || g.d_exp > 40)
    return "gemm: |a_exp|, |b_exp|, |d_exp| must be <= 40";
  if (g.D16 && (!g.d_trans || !al16(g.D16) || (g.ldd & 31) || (g.batch > 1 && (g.sd & 31))))
    return "gemm: the twin output D16 needs d_trans, 16-byte alignment, ldd and sd multiples of 32";
  return nullptr;
}

cudaError_t launch_gemm(const GemmDesc& g, cudaStream_t stream, bool simt) {
  // Default split: hi = the fp32 operand as the tensor core reads it (tf32 truncation),
  // lo = x - trunc_tf32(x) (exact).  Versus hi = rna(x), lo = rna(x - hi) this drops one
  // shared-memory write per element: 5-10% faster GEMMs (measured) for 7.8e-7 instead
  // of 4.7e-7 relative error at K = 1024.  HG_TF32_SPLIT=rna selects the rounded split.
  static const int trunc_hi = [] {
    const char* v = getenv("HG_TF32_SPLIT");
    return (v && v[0] == 'r') ? 0 : 1;
  }();
  const bool f16 = !simt && gemm_prec(g) == 1;
  const float alpha = f16 ? ldexpf(g.alpha, -(g.a_exp + g.b_exp)) : g.alpha;
  EpiArgs ea{g.M, g.N, g.K, g.D, g.ldd, g.sd, g.d_trans ? 1 : 0, alpha, g.rs, g.srs, g.cs, g.scs,
             g.a_mn ? 1 : 0, g.b_mn ? 1 : 0, trunc_hi, g.lower ? 1 : 0, g.C, g.ldc, g.sc, g.beta,
             (g.b_upper && (f16 || !g.b_mn)) ? 1 : 0,
             ldexpf(1.0f, g.a_exp), ldexpf(1.0f, g.b_exp), g.D16, ldexpf(1.0f, g.d_exp),
             (g.D16 && g.d16_only) ? 1 : 0};
  if (simt) {
    if (g.A16 || g.B16) return cudaErrorInvalidValue;
    dim3 grid((g.M + 63) / 64, (g.N + 63) / 64, g.batch);
    gemm_simt_kernel<<<grid, 256, 0, stream>>>(g.A, ea.a_mn, g.lda, g.sa, g.B, ea.b_mn, g.ldb, g.sb, ea);
    return cudaGetLastError();
  }
  const int n = g.N < g.bn_max ? g.N : g.bn_max;
  if (f16 && g.A16 && g.B16) {
    if (n <= 32) return launch_tc<32, true, true>(g, ea, stream);
    if (n <= 64) return launch_tc<64, true, true>(g, ea, stream);
    if (n <= 128) return launch_tc<128, true, true>(g, ea, stream);
    return launch_tc<256, true, true>(g, ea, stream);
  }
  if (f16) {
    if (n <= 32) return launch_tc<32, true>(g, ea, stream);
    if (n <= 64) return launch_tc<64, true>(g, ea, stream);
    if (n <= 128) return launch_tc<128, true>(g, ea, stream);
    return launch_tc<256, true>(g, ea, stream);
  }
  if (n <= 32) return launch_tc<32, false>(g, ea, stream);
  if (n <= 64) return launch_tc<64, false>(g, ea, stream);
  if (n <= 128) return launch_tc<128, false>(g, ea, stream);
  return launch_tc<256, false>(g, ea, stream);
}

cudaError_t launch_f16_split(const float* x, int64_t rows, int cols, int64_t ld, int exp, uint16_t* out16,
                             cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if ((cols & 31) || (ld & 3)) return cudaErrorInvalidValue;
  const int64_t n = rows * (cols / 8);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_f16_split<<<grid, 256, 0, stream>>>(x, rows, cols, ld, ldexpf(1.0f, exp), out16);
  return cudaGetLastError();
}
