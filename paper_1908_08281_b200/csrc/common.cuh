// common.cuh -- device helpers shared by the hgrsvd kernels (sm_100a only).
//
// Status words, error plumbing and the raw PTX wrappers for mbarrier, TMA
// (cp.async.bulk.tensor) and tcgen05 (MMA, TMEM alloc/ld, commit).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/hg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "hgrsvd targets sm_100a only"
#endif

// Device status word codes (bit flags OR-ed into *d_status; 0 = ok).  The ABI
// maps any non-zero word to HG_ERR_NUMERICAL and names the first flag.
enum : int32_t {
  HGS_ISOLATED_VERTEX = 1 << 0,   // delta(v) == 0
  HGS_EMPTY_EDGE = 1 << 1,        // delta(e) == 0
  HGS_CHOL_BREAKDOWN = 1 << 2,    // non-positive pivot in CholeskyQR
  HGS_JACOBI_CAP = 1 << 3,        // Jacobi sweep cap hit
  HGS_SINGULAR_SIGMA = 1 << 4,    // sigma_j <= sigma_1 * 1e-6 at apply
  HGS_NONFINITE = 1 << 5,         // NaN/Inf
  HGS_CG_BREAKDOWN = 1 << 6,      // CG: p^T X p <= 0 (X is SPD, so only on corrupt input)
  HGS_SIMPLEX_DEGENERATE = 1 << 7,  // weight step: every hyperedge weight clamped to 0
};

// Bounds checks of the HG_BOUNDS_CHECK build (libhgrsvd_check.so): a violated index condition prints
// its location and traps (the CUDA context reports an illegal instruction); compiled out otherwise.
#ifdef HG_BOUNDS_CHECK
#define HG_DCHECK(c)                                                                    \
  do {                                                                                  \
    if (!(c)) {                                                                         \
      printf("HG_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                        \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define HG_DCHECK(c) \
  do {               \
  } while (0)
#endif

__device__ __forceinline__ void hg_flag(int32_t* st, int32_t f) {
  if (st) atomicOr(st, f);
}

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Pure polling wait (mbarrier.test_wait, no suspend): for waits on a pipeline's critical chain, where
// the wake-up of a suspended try_wait would add to every stage's latency.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "SPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SPIN_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// 3D tiled TMA load global -> shared, completing on an mbarrier.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 4D tiled TMA load (used for the pre-split fp16 hi/lo operand pairs: dims (K, rows, hi|lo, batch)).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ------------------------------------------------------------------ tcgen05
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::tf32, one CTA.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (fp16 operands, fp32 accumulator), one CTA.
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued MMAs of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 bits, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// One lane of a converged warp (elect.sync): the warp runs its role loop with uniform control flow
// and only the tcgen05 / TMA instructions sit under this predicate, so their operands stay in
// uniform registers (under `if (lane == 0)` every UTCHMMA was wrapped in a per-lane R2UR loop and
// the single issuing thread, not the tensor pipe, bounded the main loop).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// 3xF16 twin layout of a dense [rows][K] fp32 array (K % 32 == 0): every 32 consecutive elements o..o+31
// (o % 32 == 0) become 64 fp16 -- the 32 hi halves fp16_rn(2^e x), then the 32 lo halves
// fp16_rn(2^e x - hi) -- so a TMA box of 64 fp16 x R rows with SWIZZLE_128B lands as 128-byte
// shared-memory rows [hi 32 k | lo 32 k]: the K-major SWIZZLE_128B operand layout the tensor core reads
// at full rate.  Element o's hi half sits at tw_off(o), its lo half TW_LO further.
__host__ __device__ __forceinline__ int64_t tw_off(int64_t o) { return 2 * o - (o & 31); }
constexpr int TW_LO = 32;

// UMMA shared-memory descriptor (sm100 version bits); start, lbo, sbo in bytes
// (encoded >> 4).  layout: 2 = SWIZZLE_128B (16-byte atoms, 8-row period; the
// K-major form), 1 = SWIZZLE_128B_BASE32B (32-byte atoms, 4-row period; the
// only MN-major form legal for 32-bit operands), 4 = SWIZZLE_64B (16-byte atoms XOR-ed with address
// bits 7-8: 64-byte rows, 8-row / 512-byte period; the K-major fp16 form of the 3xF16 GEMM).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// The same descriptor from its two 32-bit words: lo = (start >> 4) | (lbo >> 4) << 16 (the start
// field advances by bytes >> 4 with no carry inside shared memory), hi = (sbo >> 4) | version | layout.
__device__ __forceinline__ uint32_t umma_desc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr >> 4) & 0x3FFF) | (((lbo >> 4) & 0x3FFF) << 16);
}
__device__ __forceinline__ uint32_t umma_desc_hi(uint32_t sbo, uint32_t layout) {
  return ((sbo >> 4) & 0x3FFF) | (1u << 14) | ((layout & 7) << 29);
}
__device__ __forceinline__ uint64_t umma_desc2(uint32_t lo, uint32_t hi) {
  return ((uint64_t)hi << 32) | lo;
}

// tf32 rounding (round-to-nearest, ties away): value stays an fp32 bit pattern.
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 3xF16 split of 4 consecutive k of one row into the K-major SWIZZLE_64B hi | lo planes:
// row r is 64 bytes (32 fp16), 16-byte unit u = kq / 2 sits at u ^ ((r >> 1) & 3).
__device__ __forceinline__ void f16_split_store(uint8_t* hi, uint8_t* lo, int r, int kq, float4 x) {
  const __half2 h01 = __floats2half2_rn(x.x, x.y), h23 = __floats2half2_rn(x.z, x.w);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(x.x - f01.x, x.y - f01.y), l23 = __floats2half2_rn(x.z - f23.x, x.w - f23.y);
  const int off = r * 64 + ((((kq >> 1) ^ (r >> 1)) & 3) << 4) + ((kq & 1) << 3);
  uint2 hv, lv;
  hv.x = *reinterpret_cast<const uint32_t*>(&h01); hv.y = *reinterpret_cast<const uint32_t*>(&h23);
  lv.x = *reinterpret_cast<const uint32_t*>(&l01); lv.y = *reinterpret_cast<const uint32_t*>(&l23);
  *reinterpret_cast<uint2*>(hi + off) = hv;
  *reinterpret_cast<uint2*>(lo + off) = lv;
}

__device__ __forceinline__ void split4(float4 x, float sc, uint2& hv, uint2& lv) {
  x = make_float4(x.x * sc, x.y * sc, x.z * sc, x.w * sc);
  const __half2 h01 = __floats2half2_rn(x.x, x.y), h23 = __floats2half2_rn(x.z, x.w);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(x.x - f01.x, x.y - f01.y), l23 = __floats2half2_rn(x.z - f23.x, x.w - f23.y);
  hv.x = *reinterpret_cast<const uint32_t*>(&h01); hv.y = *reinterpret_cast<const uint32_t*>(&h23);
  lv.x = *reinterpret_cast<const uint32_t*>(&l01); lv.y = *reinterpret_cast<const uint32_t*>(&l23);
}
