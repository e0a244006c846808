// gemm.cuh -- batched GEMM descriptor shared by the orchestration code.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// D_g(m,n) = alpha * rs_g[m] * cs_g[n] * sum_kk A_g(m,kk) B_g(kk,n) [+ beta * C_g(m,n)],  g < batch
//   A_g(m,kk) = A[g*sa + (a_mn ? kk*lda + m : m*lda + kk)]   (a_mn: "M-major" storage)
//   B_g(kk,n) = B[g*sb + (b_mn ? kk*ldb + n : n*ldb + kk)]
//   d_trans ? D[g*sd + n*ldd + m] : D[g*sd + m*ldd + n]
struct GemmDesc {
  int M = 0, N = 0, K = 0, batch = 1;
  const float* A = nullptr;
  bool a_mn = false;
  int64_t lda = 0, sa = 0;
  const float* B = nullptr;
  bool b_mn = false;
  int64_t ldb = 0, sb = 0;
  float* D = nullptr;
  bool d_trans = false;
  int64_t ldd = 0, sd = 0;
  float alpha = 1.0f;
  const float* rs = nullptr;
  int64_t srs = 0;
  const float* cs = nullptr;
  int64_t scs = 0;
  int bn_max = 256;   // widest N tile to use (smaller tiles = more CTAs for small outputs)
  bool lower = false; // symmetric result, consumer reads the lower triangle: skip output tiles
                      // entirely above the diagonal (n0 >= m0 + 128); those entries are left unset
  // residual (row-major output only): D += beta * C_g, C_g(m,n) = C[g*sc + m*ldc + n]
  const float* C = nullptr;
  int64_t ldc = 0, sc = 0;
  float beta = 0.f;
  // B(kk, n) = 0 for kk > n (e.g. B = Linv^T): the tensor-core kernel skips the zero
  // part of each k-block's MMAs (K-major B only; ignored otherwise -- still correct)
  bool b_upper = false;
  // Precision: -1 = the process default (HG_GEMM_PREC, 3xTF32 unless "f16"), 0 = 3xTF32,
  // 1 = 3xF16 (hi = fp16_rn(2^exp x), lo = fp16_rn(2^exp x - hi); the caller picks a_exp / b_exp
  // from a bound on |A| / |B| so that 2^exp max|x| < 65504 -- the result is rescaled by
  // 2^-(a_exp + b_exp) in the epilogue).
  int prec = -1;
  int a_exp = 0, b_exp = 0;
  // 3xF16 twin operands (prec 1 only, K-major, both or neither): A16 / B16 are the twins (common.cuh
  // tw_off layout: per 32 K elements the 32 hi then the 32 lo fp16) of logical arrays
  // A[g*sa + m*lda + kk] / B[g*sb + n*ldb + kk], already scaled by 2^a_exp / 2^b_exp; lda, ldb, sa, sb
  // multiples of 32.  When set, A / a_mn / B / b_mn are ignored.
  const uint16_t* A16 = nullptr;
  const uint16_t* B16 = nullptr;
  // Optional twin of a transposed output (d_trans only, either precision): fp16_rn(2^d_exp D) in the twin
  // layout of D[g*sd + n*ldd + m] -- the B16 / A16 form of a later 3xF16 GEMM that reads D K-major.
  uint16_t* D16 = nullptr;
  int d_exp = 0;
  bool d16_only = false;   // with D16: the fp32 D is not stored (nothing reads it), D may be null
};

// Enqueue the GEMM; returns cudaSuccess or the launch error.  `simt` selects the
// CUDA-core fp32 verification kernel instead of the tcgen05 3xTF32 kernel.
cudaError_t launch_gemm(const GemmDesc& g, cudaStream_t stream, bool simt);
// Validation used by the ABI (alignment/stride requirements of TMA); returns a
// static message or nullptr.
const char* gemm_check(const GemmDesc& g);
// The precision launch_gemm will use for g (0 = 3xTF32, 1 = 3xF16).
int gemm_prec(const GemmDesc& g);
// Twin producer for 3xF16 operands: out16 = the twin (common.cuh tw_off) of the dense rows x cols fp32
// matrix x (row pitch ld, cols % 32 == 0), scaled by 2^exp.
cudaError_t launch_f16_split(const float* x, int64_t rows, int cols, int64_t ld, int exp, uint16_t* out16,
                             cudaStream_t stream);
