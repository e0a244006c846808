// abi.cu -- the C ABI (include/hg.h): validation, workspace carving and the
// stage sequencing of the block randomized SVD path.
//
//   hg_build_theta          degrees -> Eq. 1 blocks
//   hg_block_rsvd           Alg. 1 per block
//   hg_block_apply_inverse  Eq. 3 with Eq. 15
//   hg_solve(_host)         the three in sequence
//
// Panels (b x k per block) are stored transposed, [nb][k][b], so that each of
// the k columns is contiguous; every GEMM below reads/writes that layout
// directly (see gemm.cu for the operand-major conventions).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hg.h"
#include "gemm.cuh"
#include "kernels.cuh"

#include <nvtx3/nvToolsExt.h>

// A part's side stream (defined next to the part streams below): side_fork makes the side stream of the
// current part wait for everything enqueued on `main` so far and returns it (or `main` itself when the
// streams cannot be made); side_join makes `main` wait for the side stream.  Plain graph edges under capture.
static cudaStream_t side_fork(cudaStream_t main_s);
static void side_join(cudaStream_t main_s, cudaStream_t side);

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

// ---------------------------------------------------------------- stage profiler
// When enabled (hg_profile_enable), every launch group is bracketed by a pair of
// CUDA events on the launching stream; hg_profile_collect sums the elapsed times
// per stage.  Off by default: no events are recorded on the hot path.
enum Stage { ST_DEGREES, ST_ASSEMBLE, ST_OMEGA, ST_GEMM_POWER, ST_GEMM_GRAM, ST_GEMM_QFORM, ST_GEMM_SVD,
             ST_GEMM_APPLY, ST_CHOLINV, ST_JACOBI, ST_FINALIZE, ST_INV_SIGMA, ST_CG, ST_EIG, ST_COUNT };
const char* const kStageNames[ST_COUNT] = {"degrees", "assemble", "omega", "gemm_power", "gemm_gram",
                                           "gemm_qform", "gemm_svd", "gemm_apply", "cholinv", "jacobi",
                                           "finalize", "inv_sigma", "cg", "eig_precond"};
struct ProfRec {
  int stage, part;
  cudaEvent_t a, b;
};
thread_local bool g_prof_on = false;
thread_local int g_prof_mode = 0;                 // 1: per-stage totals (parts in sequence), 2: timeline
thread_local int g_cur_part = 0;
thread_local cudaEvent_t g_t0 = nullptr;          // timeline origin (first solve since the last collect)
thread_local bool g_t0_set = false;
thread_local std::vector<ProfRec> g_prof;
thread_local std::vector<cudaEvent_t> g_evpool;

cudaEvent_t prof_event() {
  if (!g_evpool.empty()) {
    cudaEvent_t e = g_evpool.back();
    g_evpool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
// record a profiling event; inside a stream capture it must be an external record node
// (a plain record there only expresses a dependency inside the graph)
inline void prof_record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

// NVTX (SURVEY.md §5 tracing): with HG_NVTX=1 every stage's enqueue is an NVTX range named after the stage
// ("gemm_power[part 3]"), visible in Nsight Systems / ncu --nvtx when the kernels are enqueued directly
// (HG_NO_GRAPH=1; a replayed CUDA graph has no host-side enqueue to annotate).  Header-only NVTX 3: no link
// dependency, a no-op without an attached tool.
static bool nvtx_on() {
  static const bool on = [] {
    const char* v = getenv("HG_NVTX");
    return v && v[0] == '1';
  }();
  return on;
}

struct ProfScope {
  bool on;
  bool nv;
  cudaStream_t s;
  ProfRec r;
  ProfScope(int stage, cudaStream_t st) : on(g_prof_on), nv(nvtx_on()), s(st) {
    if (nv) {
      char name[48];
      snprintf(name, sizeof name, "%s[part %d]", kStageNames[stage], g_cur_part);
      nvtxRangePushA(name);
    }
    if (!on) return;
    r.stage = stage;
    r.part = g_cur_part;
    r.a = prof_event();
    r.b = prof_event();
    prof_record(r.a, s);
  }
  ~ProfScope() {
    if (on) {
      prof_record(r.b, s);
      g_prof.push_back(r);
    }
    if (nv) nvtxRangePop();
  }
};

hg_status fail(hg_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
hg_status fail(hg_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

hg_status cuda_fail(cudaError_t e, const char* where) {
  return fail(HG_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define HG_CU(expr, where)                      \
  do {                                          \
    cudaError_t e_ = (expr);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

constexpr size_t ALIGN = 256;

struct Layout {
  size_t de = 0, eval = 0, dvr = 0, keys = 0, blocks = 0, P[4] = {0, 0, 0, 0}, Ut = 0, Vt = 0;
  size_t X16 = 0, P16[4] = {0, 0, 0, 0};   // 3xF16 pre-split twins of the blocks and the panels (hi | lo planes)
  size_t G = 0, L = 0, Linv = 0, Wf = 0, Uk = 0, work = 0, eig = 0, sig = 0, sigma = 0, sigl = 0, rs = 0, Z = 0,
         Yp = 0, Fp = 0, amax = 0, status = 0;
  size_t h_rowptr = 0, h_col = 0, h_w = 0, h_Y = 0, h_F = 0;
  size_t total = 0;
};

Layout layout(int64_t N, int64_t E, int64_t nnz, int64_t b, int64_t k, int64_t T) {
  Layout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + ALIGN - 1) / ALIGN * ALIGN;
    return o;
  };
  const int64_t nb = N / b;
  L.de = take(4 * E);
  L.eval = take(4 * E);
  L.dvr = take(4 * N);
  L.keys = take(assemble_keys_bytes(nnz, (int)nb, (int)E));
  L.blocks = take(4 * nb * b * b);
  for (int i = 0; i < 4; ++i) L.P[i] = take(4 * nb * k * b);
  L.X16 = take(4 * nb * b * b);
  for (int i = 0; i < 4; ++i) L.P16[i] = take(4 * nb * k * b);
  L.Ut = take(4 * nb * k * b);
  L.Vt = take(4 * nb * k * b);
  L.G = take(4 * nb * k * k);
  L.L = take(4 * nb * k * k);
  L.Linv = take(4 * nb * k * k);
  L.Wf = take(4 * nb * k * k);
  L.Uk = take(4 * nb * k * k);
  L.work = take(4 * nb * k * k);
  L.eig = take(eig_precond_supported((int)k) ? 4 * nb * eig_scratch_floats((int)k) : 0);   // Jacobi preconditioner
  L.sig = take(8 * nb * k + 4 * nb * k);
  L.sigma = take(4 * nb * k);
  L.sigl = take(4 * nb * k);   // internal sigma of an oversampled (l = k + p) factorisation
  L.rs = take(4 * nb * k);
  const int64_t T4 = (T + 3) / 4 * 4;   // T % 4 != 0: Y, F go through 16-byte-pitched copies
  L.Z = take(4 * nb * k * (T > 0 ? T4 : 1));
  if (T % 4) {
    L.Yp = take(4 * N * T4);
    L.Fp = take(4 * N * T4);
  }
  L.amax = take(apply_fused_amax_bytes((int)nb));   // fused apply: per-block max|Y_i|, max|U_i|, max|V_i|
  L.status = take(4);
  L.h_rowptr = take(8 * (N + 1));
  L.h_col = take(4 * (nnz > 0 ? nnz : 1));
  L.h_w = take(4 * E);
  L.h_Y = take(4 * N * (T > 0 ? T : 1));
  L.h_F = take(4 * N * (T > 0 ? T : 1));
  L.total = off;
  return L;
}

template <class T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

hg_status check_sizes(int64_t N, int64_t b, int64_t k, int64_t q, int64_t T) {
  if (N <= 0 || b <= 0) return fail(HG_ERR_INVALID, "need N > 0 and b > 0 (N=%lld, b=%lld)", (long long)N, (long long)b);
  if (N % b) return fail(HG_ERR_INVALID, "N %% b != 0 (N=%lld, b=%lld); ragged blocks are not supported", (long long)N, (long long)b);
  if (b % 4) return fail(HG_ERR_INVALID, "b must be a multiple of 4 (b=%lld)", (long long)b);
  if (k < 1 || k > b) return fail(HG_ERR_INVALID, "need 1 <= k <= b (k=%lld, b=%lld)", (long long)k, (long long)b);
  if (k % 4) return fail(HG_ERR_INVALID, "k must be a multiple of 4 (k=%lld)", (long long)k);
  if (k > 512) return fail(HG_ERR_INVALID, "k > 512 is not supported (k=%lld)", (long long)k);
  if (q < 0) return fail(HG_ERR_INVALID, "q must be >= 0 (q=%lld)", (long long)q);
  if (T < 0) return fail(HG_ERR_INVALID, "T must be >= 0 (T=%lld)", (long long)T);
  if (N / b > 65535) return fail(HG_ERR_INVALID, "more than 65535 blocks");
  return HG_OK;
}

hg_status check_ws(const void* ws, size_t ws_bytes, size_t need) {
  if (!ws) return fail(HG_ERR_INVALID, "workspace is NULL");
  if (reinterpret_cast<uintptr_t>(ws) % ALIGN) return fail(HG_ERR_INVALID, "workspace must be 256-byte aligned");
  if (ws_bytes < need)
    return fail(HG_ERR_INVALID, "workspace too small: %zu bytes given, %zu needed", ws_bytes, need);
  return HG_OK;
}

hg_status gemm(const GemmDesc& g, cudaStream_t s, bool simt, const char* what, int stage = ST_GEMM_SVD) {
  if (const char* m = gemm_check(g)) return fail(HG_ERR_INVALID, "%s: %s", what, m);
  ProfScope ps(stage, s);
  cudaError_t e = launch_gemm(g, s, simt);
  ++g_launches;
  if (e != cudaSuccess) return cuda_fail(e, what);
  return HG_OK;
}

// ---------------------------------------------------------------- stages
// N-tile cap per GEMM role (HG_BN_POWER / HG_BN_GRAM / HG_BN_QFORM; 256 = widest).  The
// per-part chains are latency-bound while the GPU has idle SMs, so narrower tiles (more
// CTAs for the same MACs) can shorten a launch.
static int bn_env(const char* name, int dflt) {
  const char* v = getenv(name);
  const int x = v ? atoi(v) : dflt;
  return x >= 256 ? 256 : x >= 128 ? 128 : x >= 64 ? 64 : 32;
}

// 3xF16 bookkeeping of the rSVD panels: which fp32 panels carry a
// valid pre-split twin (hi | lo fp16 planes), the power-of-two exponent it was scaled by, and a
// bound on its column 2-norms.  Products X P have |(X P)_ij| <= ||x_i|| ||p_j|| <= cb(P) since
// ||X||_2 <= 1 (X = I - Theta/(1+mu), 0 <= eig(Theta) <= 1), so the exponent of every twin follows
// from bounds, not from the data: Omega |z| <= 8.7 (Box-Muller on 53-bit uniforms, philox.cu),
// orthonormalised panels ||q_j|| <= 2.
constexpr int kNoTwin = -99;
struct Twins {
  const float* f[4] = {nullptr, nullptr, nullptr, nullptr};
  uint16_t* h[4] = {nullptr, nullptr, nullptr, nullptr};
  int exp[4] = {kNoTwin, kNoTwin, kNoTwin, kNoTwin};
  float cb[4] = {0.f, 0.f, 0.f, 0.f};
  int find(const float* p) const {
    for (int i = 0; i < 4; ++i)
      if (f[i] == p) return i;
    return -1;
  }
  bool valid(int i) const { return i >= 0 && exp[i] != kNoTwin; }
};
// largest e <= 14 with 2^e * 1.01 * bound < 65504 (fp16 max)
static int f16_exp(float bound) {
  const int e = (int)floorf(log2f(65504.f / (1.01f * bound)));
  return e < 14 ? e : 14;
}

struct Rsvd {
  int nb, b, k;
  bool simt;
  cudaStream_t s;
  const float* X;
  bool general = false;   // HG_GENERAL: X^T products use the literal transpose (else X^T = X, reading A12)
  const uint16_t* X16 = nullptr;   // pre-split X (exponent 14, |X_ij| <= 1): 3xF16 power products
  Twins* tw = nullptr;

  // out_t = (X P)^T  with P given as P_t [k][b]; trans: (X^T P)^T, the literal X^T only when general
  // (X symmetric: X^T P = X P, reading A12)
  // want_twin = false: the output is read as fp32 only (the lazy QR's W = X Y)
  hg_status power(const float* P_t, float* out_t, bool trans = false, bool want_twin = true) const {
    GemmDesc g;
    g.M = b; g.N = k; g.K = b; g.batch = nb;
    g.A = X; g.a_mn = trans && general; g.lda = b; g.sa = (int64_t)b * b;
    g.B = P_t; g.b_mn = false; g.ldb = b; g.sb = (int64_t)k * b;
    g.D = out_t; g.d_trans = true; g.ldd = b; g.sd = (int64_t)k * b;
    g.bn_max = bn_env("HG_BN_POWER", 256);
    const int i = tw ? tw->find(P_t) : -1, o = tw ? tw->find(out_t) : -1;
    const bool f16 = X16 && tw && tw->valid(i) && !simt;
    // X16 set: the fp32 blocks may not exist (the assembly wrote only the twin) -- every panel a
    // power product reads (Omega, qform and power outputs) carries a twin by construction
    if (X16 && !f16) return fail(HG_ERR_INVALID, "internal: power product operand panel without a 3xF16 twin");
    if (f16) {   // both operands pre-split: no in-kernel split, kind::f16 at twice the tf32 rate
      g.prec = 1;
      g.A16 = X16; g.a_exp = 14;
      g.B16 = tw->h[i]; g.b_exp = tw->exp[i];
    }
    if (o >= 0) {
      tw->exp[o] = kNoTwin;
      if (f16 && want_twin) {   // |(X P)_ij| <= cb(P); the column norms do not grow either
        g.D16 = tw->h[o]; g.d_exp = f16_exp(tw->cb[i]);
        tw->exp[o] = g.d_exp;
        tw->cb[o] = tw->cb[i];
      }
    }
    return gemm(g, s, simt, "power product X*S", ST_GEMM_POWER);
  }
  // G = P^T P (k x k)
  hg_status gram(const float* P_t, float* G) const {
    GemmDesc g;
    g.M = k; g.N = k; g.K = b; g.batch = nb;
    g.A = P_t; g.a_mn = false; g.lda = b; g.sa = (int64_t)k * b;
    g.B = P_t; g.b_mn = false; g.ldb = b; g.sb = (int64_t)k * b;
    g.D = G; g.d_trans = false; g.ldd = k; g.sd = (int64_t)k * k;
    // symmetric: 128-wide tiles on and below the diagonal only (k_cholinv reads the lower triangle)
    g.bn_max = bn_env("HG_BN_GRAM", 128);
    g.lower = !getenv("HG_GRAM_FULL");
    const int i = tw ? tw->find(P_t) : -1;
    if (tw && tw->valid(i) && !simt) {
      g.prec = 1;
      g.A16 = g.B16 = tw->h[i]; g.a_exp = g.b_exp = tw->exp[i];
    }
    return gemm(g, s, simt, "Gram P^T P", ST_GEMM_GRAM);
  }
  // Q = P L^-T  ->  Q_t
  // need_f32 = false: only Q's twin is read afterwards (an intermediate basis feeds one power product)
  hg_status qform(const float* P_t, const float* Linv, float* Q_t, bool need_f32 = true) const {
    GemmDesc g;
    g.M = b; g.N = k; g.K = k; g.batch = nb;
    g.A = P_t; g.a_mn = true; g.lda = b; g.sa = (int64_t)k * b;
    g.B = Linv; g.b_mn = false; g.ldb = k; g.sb = (int64_t)k * k;
    g.D = Q_t; g.d_trans = true; g.ldd = b; g.sd = (int64_t)k * b;
    g.bn_max = bn_env("HG_BN_QFORM", 256);
    static const bool tri = !getenv("HG_QFORM_FULL");   // Linv is lower: B(kk, n) = Linv(n, kk) upper
    g.b_upper = tri;
    const int o = tw ? tw->find(Q_t) : -1;
    if (o >= 0) {   // the orthonormalised panel's twin for the next power product / Gram: ||q_j|| <= 2
      tw->exp[o] = kNoTwin;
      if (!simt) {
        g.D16 = tw->h[o]; g.d_exp = f16_exp(2.f);
        g.d16_only = !need_f32;
        tw->exp[o] = g.d_exp;
        tw->cb[o] = 2.f;
      }
    }
    return gemm(g, s, simt, "Q = Y R^-1", ST_GEMM_QFORM);
  }
};

#define HG_TRY(expr)                 \
  do {                               \
    hg_status st_ = (expr);          \
    if (st_ != HG_OK) return st_;    \
  } while (0)

static int qr_passes_env() {   // read per call (tests switch it)
  const char* v = getenv("HG_QR_PASSES");
  return v ? atoi(v) : 1;
}

// 3xF16 power products and Grams (pre-split X and panels) on unless
// HG_GEMM_F16=0 (read per call: tests switch it); the pre-split planes need b % 8 == 0.
static bool f16_on(int b, bool simt) {
  const char* v = getenv("HG_GEMM_F16");
  return !simt && b % 32 == 0 && !(v && v[0] == '0');   // twins: rows of whole 32-element groups (tw_off)
}

// Jacobi preconditioner (eig.cu) on unless HG_JACOBI_PRE=0 (read per call: tests switch it)
static bool jacobi_precond_on(int k) {
  const char* v = getenv("HG_JACOBI_PRE");
  return eig_precond_supported(k) && !(v && v[0] == '0');
}

// CholeskyQR2 on a_t (result in a_t, scratch_t clobbered).  passes = 3 runs one more
// pass (shifted CholeskyQR3): used for the first QR when 2k > b, where X Omega can be
// ill-conditioned and k_cholinv's shifted retry leaves Q1 merely well-conditioned.
// q_f32 = false: the result is only read through its 3xF16 twin (the last pass skips the fp32 store)
hg_status cholqr(const Rsvd& R, float* a_t, float* scratch_t, float* G, float* Linv, float* work, int32_t* st,
                 int passes, float** q_out, bool q_f32 = true) {
  float* src = a_t;
  float* dst = scratch_t;
  for (int p = 0; p < passes; ++p) {
    HG_TRY(R.gram(src, G));
    {
      ProfScope ps(ST_CHOLINV, R.s);
      HG_CU(launch_cholinv(R.nb, R.k, G, nullptr, Linv, work, st, R.s, &g_launches), "cholinv");
    }
    HG_TRY(R.qform(src, Linv, dst, q_f32 || p + 1 < passes));
    float* tmp = src; src = dst; dst = tmp;
  }
  *q_out = src;   // a_t after an even pass count, scratch_t after an odd one
  return HG_OK;
}

// Block-indexed workspace buffers of the part [blk0, blk0 + nb) of an nb_total-block
// problem (parts run concurrently on different streams; see solve_impl).
struct Bufs {
  float* P[4];
  uint16_t* P16[4];   // 3xF16 twins of P (common.cuh tw_off layout: 2 fp16 per element)
  float *G, *L, *Linv, *Wf, *Uk, *work, *eig, *rs, *Z, *Yp, *Fp;
  double* sig;
  int32_t* perm;
  uint32_t* amax;   // fused apply: [3][amax_ld] exponent words, this part's first block at [0]
  int amax_ld;
  // hg_solve with the fused apply: finalize writes U's twin (P16[0]) and the v_j scales (rs) instead of
  // fp32 Ut / Vt; the apply prep forms V's twin (P16[1]) from the unsorted panel P[2] through perm
  bool fuse_twins = false;
};
Bufs part_bufs(void* ws, const Layout& Lo, int nb_total, int blk0, int b, int k, int T) {
  Bufs B;
  const int64_t kb = (int64_t)blk0 * k * b, kk = (int64_t)blk0 * k * k, k1 = (int64_t)blk0 * k;
  for (int i = 0; i < 4; ++i) B.P[i] = at<float>(ws, Lo.P[i]) + kb;
  for (int i = 0; i < 4; ++i) B.P16[i] = at<uint16_t>(ws, Lo.P16[i]) + 2 * kb;   // twin of the part's panels (tw_off)
  B.G = at<float>(ws, Lo.G) + kk;
  B.L = at<float>(ws, Lo.L) + kk;
  B.Linv = at<float>(ws, Lo.Linv) + kk;
  B.Wf = at<float>(ws, Lo.Wf) + kk;
  B.Uk = at<float>(ws, Lo.Uk) + kk;
  B.work = at<float>(ws, Lo.work) + kk;
  B.eig = eig_precond_supported(k) ? at<float>(ws, Lo.eig) + (int64_t)blk0 * eig_scratch_floats(k) : nullptr;
  B.rs = at<float>(ws, Lo.rs) + k1;
  const int64_t T4 = (T + 3) / 4 * 4;
  B.Z = at<float>(ws, Lo.Z) + k1 * (T > 0 ? T4 : 1);
  B.Yp = (T % 4) ? at<float>(ws, Lo.Yp) + (int64_t)blk0 * b * T4 : nullptr;
  B.Fp = (T % 4) ? at<float>(ws, Lo.Fp) + (int64_t)blk0 * b * T4 : nullptr;
  double* sig0 = at<double>(ws, Lo.sig);
  B.sig = sig0 + k1;
  B.perm = reinterpret_cast<int32_t*>(sig0 + (int64_t)nb_total * k) + k1;
  B.amax = at<uint32_t>(ws, Lo.amax) + blk0;
  B.amax_ld = nb_total;
  return B;
}

// Alg. 1 on the nb blocks at X (global block index of the first: blk0, which keys Omega).
// scheme 0: Alg. 1 (QR after every product); scheme 1: Eq. 10, Y = (X X^T)^q X Omega formed first
// and orthonormalised once (shifted CholeskyQR3).
hg_status run_rsvd(const float* X, int nb, int blk0, int b, int k, int q, uint64_t seed, bool simt, float* Ut,
                   float* sigma, float* Vt, int32_t* st, const Bufs& Bf, cudaStream_t s, int scheme = 0,
                   bool general = false, bool uv_bk = false, const uint16_t* X16 = nullptr) {
  Rsvd R{nb, b, k, simt, s, X, general};
  Twins tw;
  if (X16 && !simt && !general) {
    for (int i = 0; i < 4; ++i) {
      tw.f[i] = Bf.P[i];
      tw.h[i] = Bf.P16[i];
    }
    R.X16 = X16;
    R.tw = &tw;
  }
  float* P[4];
  for (int i = 0; i < 4; ++i) P[i] = Bf.P[i];
  float* G = Bf.G;
  float* Lm = Bf.L;
  float* Linv = Bf.Linv;
  float* Wf = Bf.Wf;
  float* Uk = Bf.Uk;
  float* work = Bf.work;
  double* sig = Bf.sig;

  // Alg. 1 step 1-2: Omega, Y0 = X Omega, S0 = qr(Y0)
  {
    ProfScope ps(ST_OMEGA, s);
    if (R.tw) {   // |Omega_ij| <= 8.7: only the twin, for the first 3xF16 power product
      tw.exp[0] = f16_exp(8.7f);
      tw.cb[0] = 8.7f * sqrtf((float)b);
      HG_CU(launch_omega_panels(seed, blk0, nb, b, k, P[0], s, &g_launches, tw.h[0], tw.exp[0]), "omega");
    } else {
      HG_CU(launch_omega_panels(seed, blk0, nb, b, k, P[0], s, &g_launches), "omega");
    }
  }
  // Passes per QR: the final basis S (used by B = S^T X and U = S U~) gets
  // CholeskyQR2; an intermediate basis is only multiplied by X next, so one CholeskyQR pass
  // (span-exact, orthogonal to ~cond(Y)^2 u with cond(Y) <= 2 cond(X)) suffices.  The first
  // QR of X Omega keeps three passes when 2k > b (X Omega ill-conditioned near k = b).
  // HG_QR_PASSES=2 restores CholeskyQR2 for every QR.
  const bool full_qr = qr_passes_env() >= 2;
  auto passes = [&](bool first, bool last) { return (first && 2 * k > b) ? 3 : ((last || full_qr) ? 2 : 1); };
  HG_TRY(R.power(P[0], P[1]));
  float* cur = nullptr;
  float* oth = nullptr;
  if (scheme == 1) {
    cur = P[1];
    oth = P[0];
    for (int it = 0; it < 2 * q; ++it) {   // (X X^T)^q X Omega (X^T = X unless HG_GENERAL, reading A12)
      HG_TRY(R.power(cur, oth, it % 2 == 0));
      float* t = cur; cur = oth; oth = t;
    }
    float* qn = nullptr;
    HG_TRY(cholqr(R, cur, oth, G, Linv, work, st, 3, &qn));
    oth = (qn == cur) ? oth : cur;
    cur = qn;
  } else {
    // an intermediate basis is only the B operand of the next power product: with the twins on, its fp32
    // copy is never read (the final S feeds U = S U~ in fp32)
    const bool tw_on = R.tw != nullptr;
    // HG_QR_SKIP_HALF=1 (opt-in, measured in DESIGN.md §15; NOT Alg. 1 as printed): the half-step basis
    // S~ = qr(X^T S) is left un-orthonormalised -- Y_i = X (X^T S_{i-1}) is Eq. 10 inside one iteration,
    // with Alg. 1's QR once per iteration; same subspace, cond(Y_i) <= cond(X)^2 (4 at mu = 1)
    const char* sh = getenv("HG_QR_SKIP_HALF");   // read per call (bench.py measures both)
    const bool skip_half = sh && sh[0] == '1';
    const char* lz = getenv("HG_QR_LAZY");
    const bool lazy = tw_on && !skip_half && !(lz && lz[0] == '0');
    if (lazy) {
      // Lazy application of an intermediate QR: the next panel of Alg. 1 is
      //   Y_{j+1} = X S_j = X (Y_j R_j^-1) = (X Y_j) R_j^-1,
      // so W = X Y_j runs on the part's side stream WHILE the main stream forms Y_j^T Y_j and its Cholesky
      // factor R_j (the chain's longest kernel); one Q-formation GEMM then gives Y_{j+1} = W R_j^-1.  Every
      // QR of Alg. 1 is still computed -- S_j is applied through associativity instead of being stored -- and
      // the power product leaves the chain.  QRs that take more than one pass (the first one when 2k > b,
      // HG_QR_PASSES=2) and the final S are formed explicitly as before.
      float* Yc = P[1];   // Y_j (twin valid; fp32 valid when the explicit path needs it)
      float* Wb = P[0];
      auto pj = [&](int j) { return passes(j == 0, false); };
      for (int j = 0; j < 2 * q; ++j) {
        const bool next_lazy = j + 1 < 2 * q && pj(j + 1) == 1;
        if (pj(j) == 1) {
          cudaStream_t side = side_fork(s);
          Rsvd Rs = R;
          Rs.s = side;
          HG_TRY(Rs.power(Yc, Wb, j % 2 == 0, false));
          HG_TRY(R.gram(Yc, G));
          {
            ProfScope ps(ST_CHOLINV, s);
            HG_CU(launch_cholinv(nb, k, G, nullptr, Linv, work, st, s, &g_launches), "cholinv");
          }
          side_join(s, side);
          HG_TRY(R.qform(Wb, Linv, Yc, !next_lazy));
        } else {
          float* qn = nullptr;
          HG_TRY(cholqr(R, Yc, Wb, G, Linv, work, st, pj(j), &qn, false));
          float* other = (qn == Yc) ? Wb : Yc;
          HG_TRY(R.power(qn, other, j % 2 == 0));
          Yc = other;
          Wb = qn;
        }
      }
      HG_TRY(cholqr(R, Yc, Wb, G, Linv, work, st, passes(q == 0, true), &cur, true));
      oth = (cur == Yc) ? Wb : Yc;
    } else {
    HG_TRY(cholqr(R, P[1], P[0], G, Linv, work, st, passes(true, q == 0), &cur, !tw_on || q == 0));
    oth = (cur == P[1]) ? P[0] : P[1];
    // loop i = 1..q: S~ = qr(X^T S), S = qr(X S~)
    for (int it = 0; it < 2 * q; ++it) {
      HG_TRY(R.power(cur, oth, it % 2 == 0));
      if (skip_half && tw_on && it % 2 == 0) {
        float* t = cur; cur = oth; oth = t;
        continue;
      }
      float* qn = nullptr;
      HG_TRY(cholqr(R, oth, cur, G, Linv, work, st, passes(false, it == 2 * q - 1), &qn, !tw_on || it == 2 * q - 1));
      oth = (qn == oth) ? cur : oth;
      cur = qn;
    }
    }
  }
  // step 4: B = S^T X, stored as B [k][b] = (X^T S)^T
  float* Bt = oth;
  HG_TRY(R.power(cur, Bt, true));
  // step 5: SVD of B via B B^T = L L^T and one-sided Jacobi (W = L, or W = L^T; jacobi.cu)
  HG_TRY(R.gram(Bt, G));
  const bool on_l = jacobi_on_l();
  {
    ProfScope ps(ST_CHOLINV, s);
    HG_CU(launch_cholinv(nb, k, G, Lm, on_l ? nullptr : Linv, work, st, s, &g_launches), "cholinv(B B^T)");
  }
  const float* Wj = Lm;   // the Jacobi's starting matrix
  if (on_l && jacobi_precond_on(k) && Bf.eig) {
    // Eigen-preconditioner (eig.cu): J0 ~ eigenvectors of A = L^T L, orthogonalised by
    // CholeskyQR2, and the Jacobi starts from W0 = L J0 instead of L (same limit, ~1 sweep instead of 8-9).
    // Buffers: G (free after the Cholesky) = A and the CholeskyQR Gram scratch, Linv = Householder
    // vectors then L^-1 scratch, work = Z then W0, Wf = Q^T then the CholeskyQR panel scratch, Uk = J0^T.
    {
      GemmDesc g;   // A = L^T L (lower tiles; the tridiagonalisation reads the lower triangle)
      g.M = k; g.N = k; g.K = k; g.batch = nb;
      g.A = Lm; g.a_mn = true; g.lda = k; g.sa = (int64_t)k * k;
      g.B = Lm; g.b_mn = true; g.ldb = k; g.sb = (int64_t)k * k;
      g.D = G; g.d_trans = false; g.ldd = k; g.sd = (int64_t)k * k;
      g.bn_max = 128;
      g.lower = true;
      HG_TRY(gemm(g, s, simt, "A = L^T L", ST_GEMM_SVD));
    }
    const float* escale = nullptr;
    {
      ProfScope ps(ST_EIG, s);
      HG_CU(launch_eig_precond(nb, k, G, Linv, work, Bf.eig, Wf, &escale, s, &g_launches), "eig preconditioner");
    }
    {
      GemmDesc g;   // J0'^T = diag(scale) (Q Z)^T: row i = the approximate unit eigenvector i of A
      g.M = k; g.N = k; g.K = k; g.batch = nb;
      g.A = work; g.a_mn = true; g.lda = k; g.sa = (int64_t)k * k;    // A(i, m) = Z[m][i]
      g.B = Wf; g.b_mn = true; g.ldb = k; g.sb = (int64_t)k * k;      // B(m, r) = Q[r][m] = Qt[m][r]
      g.D = Uk; g.d_trans = false; g.ldd = k; g.sd = (int64_t)k * k;
      g.rs = escale; g.srs = k;
      HG_TRY(gemm(g, s, simt, "J0 = Q Z", ST_GEMM_SVD));
    }
    Rsvd Rk{nb, k, k, simt, s, nullptr};
    float* J0t = nullptr;
    static const int j0_passes = getenv("HG_J0_PASSES") ? atoi(getenv("HG_J0_PASSES")) : 2;
    HG_TRY(cholqr(Rk, Uk, Wf, G, Linv, work, st, j0_passes < 2 ? 1 : 2, &J0t));   // work: Z is consumed (L2 tiles when k > 256)
    {
      GemmDesc g;   // W0 = L J0 (row-major, the layout the Jacobi reads L in)
      g.M = k; g.N = k; g.K = k; g.batch = nb;
      g.A = Lm; g.a_mn = false; g.lda = k; g.sa = (int64_t)k * k;
      g.B = J0t; g.b_mn = false; g.ldb = k; g.sb = (int64_t)k * k;
      g.D = work; g.d_trans = false; g.ldd = k; g.sd = (int64_t)k * k;
      HG_TRY(gemm(g, s, simt, "W0 = L J0", ST_GEMM_SVD));
    }
    Wj = work;
  }
  {
    ProfScope ps(ST_JACOBI, s);
    HG_CU(launch_jacobi(nb, k, Wj, Wf, st, s, &g_launches), "jacobi");
  }
  if (on_l) {  // L J = W_f = U~ Sigma: U~ = unit columns of W_f (stored transposed)
    ProfScope ps(ST_FINALIZE, s);
    HG_CU(launch_unit_columns_t(nb, k, Wf, Uk, s, &g_launches), "unit columns");
  } else {  // L^T J = W_f: U~ = J = L^-T W_f  (stored transposed: Uk[j] = u~_j)
    GemmDesc g;
    g.M = k; g.N = k; g.K = k; g.batch = nb;
    g.A = Linv; g.a_mn = true; g.lda = k; g.sa = (int64_t)k * k;
    g.B = Wf; g.b_mn = true; g.ldb = k; g.sb = (int64_t)k * k;
    g.D = Uk; g.d_trans = true; g.ldd = k; g.sd = (int64_t)k * k;
    HG_TRY(gemm(g, s, simt, "U~ = L^-T W_f"));
  }
  // V_w = B^T U~ -> P[2];  U_w = S U~ -> P[3]  (step 6): independent products, the second on the part's
  // side stream
  {
    cudaStream_t side = side_fork(s);
    for (int w = 0; w < 2; ++w) {
      GemmDesc g;
      g.M = b; g.N = k; g.K = k; g.batch = nb;
      g.A = (w == 0) ? Bt : cur; g.a_mn = true; g.lda = b; g.sa = (int64_t)k * b;
      g.B = Uk; g.b_mn = false; g.ldb = k; g.sb = (int64_t)k * k;
      g.D = P[2 + w]; g.d_trans = true; g.ldd = b; g.sd = (int64_t)k * b;
      HG_TRY(gemm(g, w == 0 ? s : side, simt, w == 0 ? "V = B^T U~" : "U = S U~"));
      if (R.tw) tw.exp[2 + w] = kNoTwin;
    }
    side_join(s, side);
  }
  {
    ProfScope ps(ST_FINALIZE, s);
    HG_CU(launch_finalize(nb, b, k, P[2], P[3], Ut, sigma, Vt, sig, Bf.perm, st, s, &g_launches, uv_bk,
                          Bf.fuse_twins ? Bf.P16[0] : nullptr, Bf.fuse_twins ? Bf.rs : nullptr),
          "finalize");
  }
  return HG_OK;
}

// Eq. 3 with Eq. 15 (reading R1): F_i = scale V_i Sigma_i^-1 U_i^T Y_i.
// woodbury_opm = 1 + mu > 0 selects reading R2 (blocks are Theta_ii): F_i = scale (Y_i + U_i D U_i^T Y_i),
// D = diag(sigma / ((1+mu) - sigma)) -- the Woodbury inverse of I - U Sigma U^T/(1+mu).
// Ut, Vt [nb][ldk][b] and sigma [nb][ldk] with ldk >= k: the first k triplets are used (ldk > k:
// an oversampled factorisation truncated to rank k).
hg_status run_apply(const float* Ut, const float* sigma, const float* Vt, int nb, int b, int k, const float* Y, int T,
                    float scale, float* F, int32_t* st, const Bufs& Bf, cudaStream_t s, bool simt,
                    float woodbury_opm = 0.f, int ldk = 0, bool uv_bk = false, bool uv_unit = false) {
  if (T == 0) return HG_OK;
  if (ldk < k) ldk = k;
  if (T % 4) {   // the GEMMs need 16-byte row pitches: run on zero-padded [rows][T4] copies of Y and F
    const int T4 = (T + 3) / 4 * 4;
    const size_t rows = (size_t)nb * b;
    HG_CU(cudaMemsetAsync(Bf.Yp, 0, rows * T4 * 4, s), "pad Y");
    HG_CU(cudaMemcpy2DAsync(Bf.Yp, (size_t)T4 * 4, Y, (size_t)T * 4, (size_t)T * 4, rows, cudaMemcpyDeviceToDevice, s),
          "pad Y");
    Bufs B2 = Bf;
    B2.Yp = nullptr;
    B2.Fp = nullptr;
    HG_TRY(run_apply(Ut, sigma, Vt, nb, b, k, Bf.Yp, T4, scale, Bf.Fp, st, B2, s, simt, woodbury_opm, ldk, uv_bk, uv_unit));
    HG_CU(cudaMemcpy2DAsync(F, (size_t)T * 4, Bf.Fp, (size_t)T4 * 4, (size_t)T * 4, rows, cudaMemcpyDeviceToDevice, s),
          "unpad F");
    return HG_OK;
  }
  const bool wb = woodbury_opm > 0.f;
  // The fused kernel (apply.cu): c / sigma, both products and the k x T intermediate in one launch;
  // U, V go in as 3xF16 twins (panel-twin scratch, free after the rSVD).  uv_unit: the factors come
  // from this library's finalize (unit vectors, exponent 14); otherwise their maxima are measured.
  if (!wb && !simt && !uv_bk && Bf.P16[0] && apply_fused_supported(b, k, ldk, T, Ut, Vt, Y, F)) {
    {
      ProfScope ps(ST_INV_SIGMA, s);   // apply prep: exponents and twins
      if (Bf.fuse_twins)
        HG_CU(launch_apply_prep(nullptr, Bf.P[2], nb, b, k, ldk, Y, T, Bf.P16[0], Bf.P16[1], Bf.amax, Bf.amax_ld, true,
                                s, &g_launches, Bf.perm, Bf.rs),
              "apply prep");
      else
        HG_CU(launch_apply_prep(Ut, Vt, nb, b, k, ldk, Y, T, Bf.P16[0], Bf.P16[1], Bf.amax, Bf.amax_ld,
                                uv_unit, s, &g_launches),
              "apply prep");
    }
    ProfScope ps(ST_GEMM_APPLY, s);
    HG_CU(launch_apply_fused(sigma, nb, b, k, ldk, Y, T, scale, F, st, Bf.P16[0], Bf.P16[1], Bf.amax,
                             Bf.amax_ld, s, &g_launches),
          "fused apply");
    return HG_OK;
  }
  float* rs = Bf.rs;
  float* Z = Bf.Z;
  {
    ProfScope ps(ST_INV_SIGMA, s);
    if (wb)
      HG_CU(launch_woodbury_scale(nb, k, ldk, sigma, scale, woodbury_opm, rs, st, s, &g_launches), "woodbury scale");
    else
      HG_CU(launch_inv_sigma(nb, k, ldk, sigma, scale, rs, st, s, &g_launches), "inv_sigma");
  }
  {  // Z = diag(rs) U^T Y_i   (k x T)
    GemmDesc g;
    g.M = k; g.N = T; g.K = b; g.batch = nb;
    g.A = Ut; g.a_mn = uv_bk; g.lda = uv_bk ? ldk : b; g.sa = (int64_t)ldk * b;   // HG_UV_BK: U [b][ldk]
    g.B = Y; g.b_mn = true; g.ldb = T; g.sb = (int64_t)b * T;
    g.D = Z; g.d_trans = false; g.ldd = T; g.sd = (int64_t)k * T;
    g.rs = rs; g.srs = ldk;
    HG_TRY(gemm(g, s, simt, "Z = Sigma^-1 U^T Y", ST_GEMM_APPLY));
  }
  {  // R1: F_i = V Z;  R2: F_i = U Z + scale Y_i   (b x T)
    GemmDesc g;
    g.M = b; g.N = T; g.K = k; g.batch = nb;
    g.A = wb ? Ut : Vt; g.a_mn = !uv_bk; g.lda = uv_bk ? ldk : b; g.sa = (int64_t)ldk * b;
    g.B = Z; g.b_mn = true; g.ldb = T; g.sb = (int64_t)k * T;
    g.D = F; g.d_trans = false; g.ldd = T; g.sd = (int64_t)b * T;
    if (wb) {
      g.C = Y; g.ldc = T; g.sc = (int64_t)b * T; g.beta = scale;
    }
    HG_TRY(gemm(g, s, simt, wb ? "F = U Z + c Y" : "F = V Z", ST_GEMM_APPLY));
  }
  return HG_OK;
}

// degrees and, for the grouped assembly, the (block, edge) grouping of the incidences of
// all N/b blocks -- both before the stream parts fork
hg_status run_degrees(const hg_incidence* H, const float* w, int b, float* dvr, int32_t* st, void* ws,
                      const Layout& Lo, cudaStream_t s) {
  ProfScope ps(ST_DEGREES, s);
  if (assemble_grouped(H->n_vertices / b, H->n_edges))
    HG_CU(launch_degrees_grouped(H->n_vertices / b, b, H->n_edges, H->nnz, H->row_ptr, H->col_idx, w,
                                 at<int32_t>(ws, Lo.de), at<float>(ws, Lo.eval), dvr, st, at<void>(ws, Lo.keys), s,
                                 &g_launches),
          "degrees + assembly grouping");
  else
    HG_CU(launch_degrees(H->n_vertices, H->n_edges, H->nnz, H->row_ptr, H->col_idx, w, at<int32_t>(ws, Lo.de),
                         at<float>(ws, Lo.eval), dvr, st, s, &g_launches),
          "degrees");
  return HG_OK;
}

// Eq. 1 blocks [blk0, blk0 + nb) of the N/b diagonal blocks (degrees already computed)
hg_status run_assemble(const hg_incidence* H, float mu, int b, bool raw, int blk0, int nb, float* blocks,
                       const float* dvr, void* ws, const Layout& Lo, cudaStream_t s, uint16_t* x16 = nullptr) {
  ProfScope ps(ST_ASSEMBLE, s);
  HG_CU(launch_assemble(blk0, nb, H->n_vertices / b, b, H->n_edges, H->nnz, H->row_ptr, H->col_idx,
                        at<float>(ws, Lo.eval), dvr, mu, raw, blocks, at<void>(ws, Lo.keys), s, &g_launches, x16,
                        x16 != nullptr),
        "assemble");
  return HG_OK;
}

hg_status run_theta(const hg_incidence* H, const float* w, float mu, int b, bool raw, float* blocks, float* dvr_out,
                    int32_t* st, void* ws, const Layout& Lo, cudaStream_t s) {
  float* dvr = dvr_out ? dvr_out : at<float>(ws, Lo.dvr);
  HG_TRY(run_degrees(H, w, b, dvr, st, ws, Lo, s));
  return run_assemble(H, mu, b, raw, 0, H->n_vertices / b, blocks, dvr, ws, Lo, s);
}

hg_status check_H(const hg_incidence* H) {
  if (!H) return fail(HG_ERR_INVALID, "H is NULL");
  if (H->n_vertices <= 0 || H->n_edges <= 0 || H->nnz < 0)
    return fail(HG_ERR_INVALID, "bad incidence sizes (N=%d, E=%d, nnz=%lld)", H->n_vertices, H->n_edges,
                (long long)H->nnz);
  if (!H->row_ptr || (H->nnz > 0 && !H->col_idx)) return fail(HG_ERR_INVALID, "incidence pointers are NULL");
  return HG_OK;
}

}  // namespace

extern "C" {

const char* hg_last_error(void) { return g_err.c_str(); }

hg_status hg_profile_enable(int32_t on) {
  g_prof_mode = on < 0 ? 0 : (on > 2 ? 2 : on);
  g_prof_on = g_prof_mode != 0;
  return HG_OK;
}

hg_status hg_profile_timeline(int32_t max_rec, int32_t* stage, int32_t* part, double* t_start_ms, double* t_end_ms,
                              int32_t* n_out) {
  g_err.clear();
  if (!n_out) return fail(HG_ERR_INVALID, "n_out is NULL");
  int n = 0;
  for (auto& r : g_prof) {
    float a = 0.f, b = 0.f;
    HG_CU(cudaEventSynchronize(r.b), "timeline sync");
    if (g_t0_set) {
      HG_CU(cudaEventElapsedTime(&a, g_t0, r.a), "timeline elapsed");
      HG_CU(cudaEventElapsedTime(&b, g_t0, r.b), "timeline elapsed");
    }
    if (n < max_rec) {
      if (stage) stage[n] = r.stage;
      if (part) part[n] = r.part;
      if (t_start_ms) t_start_ms[n] = a;
      if (t_end_ms) t_end_ms[n] = b;
    }
    ++n;
    g_evpool.push_back(r.a);
    g_evpool.push_back(r.b);
  }
  g_prof.clear();
  g_t0_set = false;
  *n_out = n;
  return HG_OK;
}

hg_status hg_profile_collect(int32_t max_stages, char* names, double* ms, int32_t* counts, int32_t* n_out) {
  g_err.clear();
  if (!n_out) return fail(HG_ERR_INVALID, "n_out is NULL");
  double tot[ST_COUNT] = {0};
  int cnt[ST_COUNT] = {0};
  for (auto& r : g_prof) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail(e, "profile sync");
    e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) return cuda_fail(e, "profile elapsed");
    tot[r.stage] += t;
    cnt[r.stage] += 1;
    g_evpool.push_back(r.a);
    g_evpool.push_back(r.b);
  }
  g_prof.clear();
  int n = 0;
  for (int i = 0; i < ST_COUNT; ++i) {
    if (!cnt[i]) continue;
    if (n < max_stages) {
      if (names) {
        strncpy(names + 32 * n, kStageNames[i], 31);
        names[32 * n + 31] = 0;
      }
      if (ms) ms[n] = tot[i];
      if (counts) counts[n] = cnt[i];
    }
    ++n;
  }
  *n_out = n;
  return HG_OK;
}
int32_t hg_last_launch_count(void) { return g_launches; }

hg_status hg_debug_counters(int64_t* out, int32_t n, int32_t reset) {
  g_err.clear();
  if (!out || n < 5) return fail(HG_ERR_INVALID, "need out[5]");
  if (n >= 5 + 64) {
    long long clk[64];
    HG_CU(chol_clocks(clk), "chol_clocks");
    for (int i = 0; i < 64; ++i) out[5 + i] = clk[i];
  }
  if (n >= 69 + 16) {
    long long clk[16];
    HG_CU(getenv("HG_JACOBI") ? jacobi_clocks(clk) : jacobi_blk_clocks(clk), "jacobi_clocks");
    for (int i = 0; i < 16; ++i) out[69 + i] = clk[i];
  }
  if (n >= 85 + 48) {   // block Jacobi inner-round stamps; a reset call switches them on
    long long clk[48];
    HG_CU(jacobi_blk_inner_clocks(reset ? nullptr : clk, 1), "jacobi inner clocks");
    if (!reset)
      for (int i = 0; i < 48; ++i) out[85 + i] = clk[i];
  }
  unsigned long long c[2] = {0, 0}, j[3] = {0, 0, 0};
  HG_CU(chol_debug(c, reset != 0), "chol_debug");
  HG_CU(jacobi_debug(j, reset != 0), "jacobi_debug");
  out[0] = (int64_t)c[0];
  out[1] = (int64_t)c[1];
  out[2] = (int64_t)j[0];
  out[3] = (int64_t)j[1];
  out[4] = (int64_t)j[2];
  return HG_OK;
}

hg_status hg_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t k, int32_t T, size_t* bytes) {
  g_err.clear();
  if (!bytes) return fail(HG_ERR_INVALID, "bytes is NULL");
  HG_TRY(check_sizes(N, b, k, 0, T));
  if (E <= 0 || nnz < 0) return fail(HG_ERR_INVALID, "need E > 0 and nnz >= 0");
  *bytes = layout(N, E, nnz, b, k, T).total;
  return HG_OK;
}

hg_status hg_workspace_size_ex(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t k, int32_t p, int32_t T,
                               size_t* bytes) {
  if (p < 0 || p % 4) return fail(HG_ERR_INVALID, "oversampling p must be >= 0 and a multiple of 4 (p=%d)", p);
  return hg_workspace_size(N, E, nnz, b, k + p, T, bytes);
}

hg_status hg_build_theta(const hg_incidence* H, const float* w, float mu, int32_t b, uint32_t flags, float* blocks,
                         float* dv_rsqrt, int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  HG_TRY(check_H(H));
  if (b <= 0 || H->n_vertices % b || b % 4) return fail(HG_ERR_INVALID, "need b > 0, b %% 4 == 0, N %% b == 0");
  if (!(mu > 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and > 0");
  if (!w || !blocks || !d_status) return fail(HG_ERR_INVALID, "NULL pointer argument");
  const Layout Lo = layout(H->n_vertices, H->n_edges, H->nnz, b, 4, 0);
  HG_TRY(check_ws(ws, ws_bytes, Lo.keys + assemble_keys_bytes(H->nnz, H->n_vertices / b, H->n_edges)));
  return run_theta(H, w, mu, b, (flags & HG_RAW_THETA) != 0, blocks, dv_rsqrt, d_status, ws, Lo,
                   reinterpret_cast<cudaStream_t>(stream));
}

hg_status hg_fill_gaussian(uint64_t seed, int32_t rows, int32_t cols, float* out, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (rows <= 0 || cols <= 0 || !out) return fail(HG_ERR_INVALID, "need rows, cols > 0 and out != NULL");
  HG_CU(launch_gaussian_rowmajor(seed, rows, cols, out, reinterpret_cast<cudaStream_t>(stream), &g_launches),
        "gaussian");
  return HG_OK;
}

hg_status hg_block_rsvd_ex(const float* blocks, int32_t nb, int32_t b, int32_t k, int32_t p, int32_t q,
                           uint64_t seed, uint32_t flags, float* Ut, float* sigma, float* Vt, int32_t* d_status,
                           void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (nb <= 0) return fail(HG_ERR_INVALID, "nb must be > 0");
  if (p < 0 || p % 4) return fail(HG_ERR_INVALID, "oversampling p must be >= 0 and a multiple of 4 (p=%d)", p);
  const int l = k + p;
  HG_TRY(check_sizes((int64_t)nb * b, b, l, q, 0));
  if (!blocks || !Ut || !sigma || !Vt || !d_status) return fail(HG_ERR_INVALID, "NULL pointer argument");
  const Layout Lo = layout((int64_t)nb * b, 1, 0, b, l, 0);
  HG_TRY(check_ws(ws, ws_bytes, Lo.status));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int scheme = (flags & HG_POWER_EQ10) ? 1 : 0;
  const bool simt = (flags & HG_GEMM_SIMT) != 0;
  const bool general = (flags & HG_GENERAL) != 0, uv_bk = (flags & HG_UV_BK) != 0;
  // HG_X_UNIT: the caller's bound |X_ij| <= 1, ||X||_2 <= 1 makes the 3xF16 twins safe (as in hg_solve)
  uint16_t* x16 = ((flags & HG_X_UNIT) && !general && f16_on(b, simt)) ? at<uint16_t>(ws, Lo.X16) : nullptr;
  if (x16) {
    HG_CU(launch_f16_split(blocks, (int64_t)nb * b, b, b, 14, x16, s), "blocks split");
    ++g_launches;
  }
  if (p == 0)
    return run_rsvd(blocks, nb, 0, b, k, q, seed, simt, Ut, sigma, Vt, d_status, part_bufs(ws, Lo, nb, 0, b, k, 0), s,
                    scheme, general, uv_bk, x16);
  if (uv_bk) return fail(HG_ERR_INVALID, "HG_UV_BK is not supported with oversampling (p > 0)");
  // oversampled: factor at width l into the workspace, keep the top k triplets (rank-k truncation)
  float* Ul = at<float>(ws, Lo.Ut);
  float* Vl = at<float>(ws, Lo.Vt);
  float* sl = at<float>(ws, Lo.sigl);
  HG_TRY(run_rsvd(blocks, nb, 0, b, l, q, seed, simt, Ul, sl, Vl, d_status, part_bufs(ws, Lo, nb, 0, b, l, 0), s,
                  scheme, general, false, x16));
  HG_CU(cudaMemcpy2DAsync(Ut, 4 * (size_t)k * b, Ul, 4 * (size_t)l * b, 4 * (size_t)k * b, nb, cudaMemcpyDeviceToDevice,
                          s), "truncate U");
  HG_CU(cudaMemcpy2DAsync(Vt, 4 * (size_t)k * b, Vl, 4 * (size_t)l * b, 4 * (size_t)k * b, nb, cudaMemcpyDeviceToDevice,
                          s), "truncate V");
  HG_CU(cudaMemcpy2DAsync(sigma, 4 * (size_t)k, sl, 4 * (size_t)l, 4 * (size_t)k, nb, cudaMemcpyDeviceToDevice, s),
        "truncate sigma");
  return HG_OK;
}

hg_status hg_block_rsvd(const float* blocks, int32_t nb, int32_t b, int32_t k, int32_t q, uint64_t seed,
                        uint32_t flags, float* Ut, float* sigma, float* Vt, int32_t* d_status, void* ws,
                        size_t ws_bytes, hg_stream_t stream) {
  return hg_block_rsvd_ex(blocks, nb, b, k, 0, q, seed, flags, Ut, sigma, Vt, d_status, ws, ws_bytes, stream);
}

hg_status hg_block_apply_inverse(const float* Ut, const float* sigma, const float* Vt, int32_t nb, int32_t b,
                                 int32_t k, const float* Y, int32_t T, float scale, float* F, int32_t* d_status,
                                 void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (nb <= 0) return fail(HG_ERR_INVALID, "nb must be > 0");
  HG_TRY(check_sizes((int64_t)nb * b, b, k, 0, T));
  if (!Ut || !sigma || !Vt || !d_status || (T > 0 && (!Y || !F))) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (!std::isfinite(scale)) return fail(HG_ERR_INVALID, "scale must be finite");
  const Layout Lo = layout((int64_t)nb * b, 1, 0, b, k, T);
  HG_TRY(check_ws(ws, ws_bytes, Lo.status));
  return run_apply(Ut, sigma, Vt, nb, b, k, Y, T, scale, F, d_status, part_bufs(ws, Lo, nb, 0, b, k, T),
                   reinterpret_cast<cudaStream_t>(stream), false);
}

hg_status hg_block_apply_inverse_ex(const float* U, const float* sigma, const float* V, int32_t nb, int32_t b,
                                    int32_t k, const float* Y, int32_t T, float scale, float* F, uint32_t flags,
                                    int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (nb <= 0) return fail(HG_ERR_INVALID, "nb must be > 0");
  HG_TRY(check_sizes((int64_t)nb * b, b, k, 0, T));
  if (!U || !sigma || !V || !d_status || (T > 0 && (!Y || !F))) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (!std::isfinite(scale)) return fail(HG_ERR_INVALID, "scale must be finite");
  if (flags & ~(HG_UV_BK | HG_GEMM_SIMT)) return fail(HG_ERR_INVALID, "unsupported flags 0x%x", flags);
  const Layout Lo = layout((int64_t)nb * b, 1, 0, b, k, T);
  HG_TRY(check_ws(ws, ws_bytes, Lo.status));
  return run_apply(U, sigma, V, nb, b, k, Y, T, scale, F, d_status, part_bufs(ws, Lo, nb, 0, b, k, T),
                   reinterpret_cast<cudaStream_t>(stream), (flags & HG_GEMM_SIMT) != 0, 0.f, 0,
                   (flags & HG_UV_BK) != 0);
}

hg_status hg_block_apply_woodbury(const float* Ut, const float* sigma, int32_t nb, int32_t b, int32_t k,
                                  const float* Y, int32_t T, float mu, float* F, int32_t* d_status, void* ws,
                                  size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (nb <= 0) return fail(HG_ERR_INVALID, "nb must be > 0");
  HG_TRY(check_sizes((int64_t)nb * b, b, k, 0, T));
  if (!Ut || !sigma || !d_status || (T > 0 && (!Y || !F))) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (!(mu > 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and > 0");
  const Layout Lo = layout((int64_t)nb * b, 1, 0, b, k, T);
  HG_TRY(check_ws(ws, ws_bytes, Lo.status));
  return run_apply(Ut, sigma, nullptr, nb, b, k, Y, T, mu / (1.0f + mu), F, d_status,
                   part_bufs(ws, Lo, nb, 0, b, k, T), reinterpret_cast<cudaStream_t>(stream), false, 1.0f + mu);
}

// Part count for hg_solve (HG_STREAMS, default 8, at most 8: with graph replay measured
// 10.99 ms at configs[3] vs 11.01 / 11.04 with 6 / 4 parts) and the auxiliary streams / events
// of the fork-join (created once, non-blocking, reused).
constexpr int kMaxParts = 8;
// nb blocks of size b.  Default: 8 parts when one batched GEMM launch (nb * ceil(b/128) CTAs) is more than
// one wave of the 148 SMs -- then a part's tensor-core GEMMs fill the SMs another part's latency-bound
// kernels leave idle (configs[3]: 6.2 -> 5.0 ms); one part otherwise -- every launch already fits the GPU and
// the fork / join only adds latency (configs[0-2]: 0.40 -> 0.37, 0.64 -> 0.60, 1.45 -> 1.36 ms).
static int solve_parts(int nb = 1 << 20, int b = 1024) {   // HG_STREAMS read per call (tests switch it)
  const char* v = getenv("HG_STREAMS");
  const int x = v ? atoi(v) : ((int64_t)nb * ((b + 127) / 128) > 148 ? 8 : 1);
  return x < 1 ? 1 : (x > kMaxParts ? kMaxParts : x);
}
// Two sets of part streams.  Plain (default priority) for hg_solve: staggering the parts delays
// the last part's latency-bound Jacobi, which sets the device makespan (11.05 vs 10.99 ms).
// Prioritised (part p at greatest + p) for hg_solve_host: the earliest parts then finish first
// and their F downloads overlap the later parts' compute (e2e 15.30 -> 14.57 ms at configs[3]).
// Graphs are instantiated with cudaGraphInstantiateFlagUseNodePriority so the captured
// priorities hold under replay.  HG_STREAM_PRIO=0/1 forces one set for both entries.
// per host thread (concurrent hg_solve calls from different threads never share events)
static thread_local cudaStream_t g_aux[2][kMaxParts] = {};
static thread_local cudaStream_t g_side[kMaxParts] = {};   // per part: the lazy QR's concurrent power product
static thread_local cudaEvent_t g_ev_side[2][kMaxParts] = {};
static thread_local cudaEvent_t g_ev_fork = nullptr, g_ev_join[kMaxParts] = {};
// library streams / events, created once and outside any stream capture
static hg_status ensure_streams() {
  if (g_ev_fork) return HG_OK;
  int least = 0, greatest = 0;
  HG_CU(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  for (int set = 0; set < 2; ++set)
    for (int p = 0; p < kMaxParts; ++p) {
      int pr = set ? greatest + p : 0;
      if (pr > least) pr = least;
      HG_CU(cudaStreamCreateWithPriority(&g_aux[set][p], cudaStreamNonBlocking, pr), "stream create");
    }
  for (int p = 0; p < kMaxParts; ++p) {
    HG_CU(cudaEventCreateWithFlags(&g_ev_join[p], cudaEventDisableTiming), "event create");
    HG_CU(cudaStreamCreateWithFlags(&g_side[p], cudaStreamNonBlocking), "stream create");
    for (int i = 0; i < 2; ++i) HG_CU(cudaEventCreateWithFlags(&g_ev_side[i][p], cudaEventDisableTiming), "event create");
  }
  HG_CU(cudaEventCreateWithFlags(&g_ev_fork, cudaEventDisableTiming), "event create");
  return HG_OK;
}
extern "C++" {
static cudaStream_t side_fork(cudaStream_t main_s) {
  if (g_prof_mode == 1) return main_s;   // per-stage totals: stages in sequence, each timed alone
  if (ensure_streams() != HG_OK) return main_s;
  const int p = g_cur_part;
  if (p < 0 || p >= kMaxParts) return main_s;
  if (cudaEventRecord(g_ev_side[0][p], main_s) != cudaSuccess) return main_s;
  if (cudaStreamWaitEvent(g_side[p], g_ev_side[0][p], 0) != cudaSuccess) return main_s;
  return g_side[p];
}
static void side_join(cudaStream_t main_s, cudaStream_t side) {
  if (side == main_s) return;
  const int p = g_cur_part;
  cudaEventRecord(g_ev_side[1][p], side);
  cudaStreamWaitEvent(main_s, g_ev_side[1][p], 0);
}
}  // extern "C++"
static bool use_prio_streams(bool host_entry) {
  const char* pv = getenv("HG_STREAM_PRIO");
  if (pv && (pv[0] == '0' || pv[0] == '1')) return pv[0] == '1';
  return host_entry;
}
static hg_status fork_streams(cudaStream_t s, int nparts, cudaStream_t* ps, bool prio) {
  ps[0] = s;
  if (nparts == 1) return HG_OK;
  if (const char* v = getenv("HG_STREAMS_SERIAL")) {   // debugging: parts in sequence on `stream`
    if (v[0] == '1') {
      for (int p = 1; p < nparts; ++p) ps[p] = s;
      return HG_OK;
    }
  }
  HG_TRY(ensure_streams());
  cudaStream_t* aux = g_aux[prio ? 1 : 0];
  cudaEvent_t ev_fork = g_ev_fork;
  HG_CU(cudaEventRecord(ev_fork, s), "fork record");
  for (int p = 0; p < nparts; ++p) {
    HG_CU(cudaStreamWaitEvent(aux[p], ev_fork, 0), "fork wait");
    ps[p] = aux[p];
  }
  return HG_OK;
}
static hg_status join_streams(cudaStream_t s, int nparts, const cudaStream_t* ps) {
  for (int p = 0; p < nparts; ++p) {
    if (ps[p] == s) continue;
    HG_CU(cudaEventRecord(g_ev_join[p], ps[p]), "join record");
    HG_CU(cudaStreamWaitEvent(s, g_ev_join[p], 0), "join wait");
  }
  return HG_OK;
}

// Alg. 1 on nb blocks split into stream parts (as hg_solve's): part p factors its block range with
// its own part buffers on a forked stream; joined back into s.  Results are those of one run_rsvd
// over all blocks (Omega is keyed by the global block index).
static hg_status run_rsvd_parts(const float* X, int nb, int b, int k, int q, uint64_t seed, float* Ut, float* sigma,
                                float* Vt, int32_t* st, void* ws, const Layout& Lo, int T, cudaStream_t s) {
  const int nparts = g_prof_mode == 1 ? 1 : std::max(1, std::min(solve_parts(nb, b), nb));
  cudaStream_t ps[kMaxParts];
  HG_TRY(fork_streams(s, nparts, ps, false));
  for (int pt = 0; pt < nparts; ++pt) {
    const int blk0 = (int)((int64_t)nb * pt / nparts), nbp = (int)((int64_t)nb * (pt + 1) / nparts) - blk0;
    const int64_t kb = (int64_t)blk0 * k * b;
    g_cur_part = pt;
    HG_TRY(run_rsvd(X + (int64_t)blk0 * b * b, nbp, blk0, b, k, q, seed, false, Ut + kb, sigma + (int64_t)blk0 * k,
                    Vt + kb, st, part_bufs(ws, Lo, nb, blk0, b, k, T), ps[pt]));
  }
  g_cur_part = 0;
  return join_streams(s, nparts, ps);
}

// Host staging for hg_solve_host: Y's rows are uploaded per part on a library copy
// stream (the part waits only before its apply, so the upload overlaps the rSVD) and each
// part downloads its F rows right after its apply (overlapping the other parts' work).
struct HostIO {
  const float* Y_host = nullptr;   // pinned host [N][T] (nullptr: Y is already on the device)
  float* F_host = nullptr;         // pinned host [N][T]
};

static cudaStream_t copy_stream(hg_status* err) {
  static thread_local cudaStream_t cs = nullptr;
  if (!cs) {
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      *err = cuda_fail(e, "copy stream create");
      return nullptr;
    }
  }
  return cs;
}

// Blocks [rb0, rb0 + rcnt) of the N/b diagonal blocks (rcnt < 0: all); F rows of other blocks are
// not touched; sigma_out, when given, is [rcnt][k].
static hg_status solve_impl(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t p,
                            int32_t q, uint64_t seed, const float* Y, int32_t T, float* F, float* sigma_out,
                            uint32_t flags, int32_t* d_status, void* ws, size_t ws_bytes, cudaStream_t s,
                            const HostIO& io = HostIO(), int32_t rb0 = 0, int32_t rcnt = -1) {
  HG_TRY(check_H(H));
  if (p < 0 || p % 4) return fail(HG_ERR_INVALID, "oversampling p must be >= 0 and a multiple of 4 (p=%d)", p);
  const int32_t l = k + p;   // Alg. 1 width; the apply uses the top k triplets
  HG_TRY(check_sizes(H->n_vertices, b, l, q, T));
  if (!(mu > 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and > 0");
  if (!w || (T > 0 && (!Y || !F))) return fail(HG_ERR_INVALID, "NULL pointer argument");
  const Layout Lo = layout(H->n_vertices, H->n_edges, H->nnz, b, l, T);
  HG_TRY(check_ws(ws, ws_bytes, Lo.h_rowptr));
  const bool simt = (flags & HG_GEMM_SIMT) != 0;
  const bool woodbury = (flags & HG_WOODBURY) != 0;
  const int scheme = (flags & HG_POWER_EQ10) ? 1 : 0;
  int32_t* st = d_status;
  if (!st) {
    if (!(flags & HG_SYNC)) return fail(HG_ERR_INVALID, "d_status may be NULL only with HG_SYNC");
    st = at<int32_t>(ws, Lo.status);
    HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), s), "memset status");
  }
  const int nb = H->n_vertices / b;
  if (rcnt < 0) { rb0 = 0; rcnt = nb; }
  if (rb0 < 0 || rcnt < 1 || rb0 + rcnt > nb)
    return fail(HG_ERR_INVALID, "block range [%d, %d) outside [0, %d)", rb0, rb0 + rcnt, nb);
  float* blocks = at<float>(ws, Lo.blocks);
  float* Ut = at<float>(ws, Lo.Ut);
  float* Vt = at<float>(ws, Lo.Vt);
  // sigma of global block i at sigma + (i - soff) l: the caller's [rcnt][k] array, or the workspace's [nb][l]
  const bool sig_user = sigma_out && p == 0;
  float* sigma = sig_user ? sigma_out : at<float>(ws, p == 0 ? Lo.sigma : Lo.sigl);
  const int soff = sig_user ? rb0 : 0;
  float* dvr = at<float>(ws, Lo.dvr);
  HG_TRY(run_degrees(H, w, b, dvr, st, ws, Lo, s));
  // Blocks are independent (reading A5): the assembly, rSVD and apply of disjoint block ranges run
  // on forked streams, so one part's tensor-core GEMMs fill the SMs that the other
  // part's latency-bound Cholesky / Jacobi leave idle.  Bitwise the same result for
  // any part count (Omega is keyed by the global block index).  One part while the
  // stage profiler is on (per-stage attribution needs sequential stages).
  const int nparts = g_prof_mode == 1 ? 1 : std::max(1, std::min(solve_parts(rcnt, b), rcnt));
  if (g_prof_mode == 2 && !g_t0_set) {
    if (!g_t0) HG_CU(cudaEventCreate(&g_t0), "event create");
    prof_record(g_t0, s);
    g_t0_set = true;
  }
  // Part boundaries: equal shares; in the host entry the cumulative share is (p / n)^gamma (HG_HOST_SKEW,
  // gamma >= 1): earlier parts get fewer blocks, finish earlier and start their F downloads earlier.  The
  // result does not depend on the partition (Omega is keyed by the global block index).
  // Measured at configs[3] (e2e ms): gamma 1 / 1.3 / 1.6 / 2 / 2.5 / 3 / 4 -> 8.95 / 8.84 / 8.77 / 8.72 / 8.71 / 8.73 / 8.87.
  static const double skew = getenv("HG_HOST_SKEW") ? atof(getenv("HG_HOST_SKEW")) : 2.0;
  const double gamma = (io.F_host != nullptr && skew >= 1.0) ? skew : 1.0;
  auto bound = [&](int pt) {
    if (pt <= 0) return 0;
    if (pt >= nparts) return (int)rcnt;
    int x = gamma == 1.0 ? (int)((int64_t)rcnt * pt / nparts) : (int)llround(rcnt * pow((double)pt / nparts, gamma));
    x = std::max(x, pt);                         // at least one block per part
    return std::min(x, (int)rcnt - (nparts - pt));
  };
  cudaStream_t ps[kMaxParts];
  HG_TRY(fork_streams(s, nparts, ps, use_prio_streams(io.F_host != nullptr)));
  // host staging of Y: one slice per part on the copy stream, started before the parts
  static thread_local cudaEvent_t ev_y[kMaxParts] = {};
  cudaStream_t cps = nullptr;
  if (io.Y_host && T > 0) {
    hg_status err = HG_OK;
    cps = copy_stream(&err);
    if (!cps) return err;
    static thread_local cudaEvent_t ev_cps = nullptr;   // fork the copy stream from `s` (joins a capture)
    if (!ev_cps) HG_CU(cudaEventCreateWithFlags(&ev_cps, cudaEventDisableTiming), "event create");
    HG_CU(cudaEventRecord(ev_cps, s), "copy fork record");
    HG_CU(cudaStreamWaitEvent(cps, ev_cps, 0), "copy fork wait");
    for (int pt = 0; pt < nparts; ++pt) {
      const int64_t r0 = (int64_t)(rb0 + bound(pt)) * b, r1 = (int64_t)(rb0 + bound(pt + 1)) * b;
      if (!ev_y[pt]) HG_CU(cudaEventCreateWithFlags(&ev_y[pt], cudaEventDisableTiming), "event create");
      HG_CU(cudaMemcpyAsync(const_cast<float*>(Y) + r0 * T, io.Y_host + r0 * T, sizeof(float) * (size_t)(r1 - r0) * T,
                            cudaMemcpyHostToDevice, cps),
            "H2D Y");
      HG_CU(cudaEventRecord(ev_y[pt], cps), "Y event");
    }
  }
  for (int pt = 0; pt < nparts; ++pt) {
    const int blk0 = rb0 + bound(pt);
    const int nbp = rb0 + bound(pt + 1) - blk0;
    const int64_t kb = (int64_t)blk0 * l * b;
    Bufs Bf = part_bufs(ws, Lo, nb, blk0, b, l, T);
    // U, V are internal here: with the fused apply (same condition as run_apply's) they exist only as twins
    Bf.fuse_twins = T > 0 && T % 4 == 0 && p == 0 && !woodbury && !simt && f16_on(b, simt) &&
                    apply_fused_supported(b, k, l, T, Ut, Vt, Y, F);
    g_cur_part = pt;
    // with the 3xF16 products the assembly writes the blocks' twin (|X_ij|, |Theta_ij| <= 1: exponent 14)
    // instead of fp32 blocks -- nothing downstream reads those
    uint16_t* x16 = f16_on(b, simt) ? at<uint16_t>(ws, Lo.X16) : nullptr;
    HG_TRY(run_assemble(H, mu, b, woodbury, blk0, nbp, blocks, dvr, ws, Lo, ps[pt], x16));
    if (x16) x16 += 2 * (int64_t)blk0 * b * b;
    // HG_JACOBI_WIDE = bitmask of parts whose Jacobi runs on 64-row cluster CTAs (twice the SMs
    // per block: a shorter per-block latency for that part).  Off by default in BOTH entries: the
    // cluster width changes the order of the Jacobi's Gram partial sums, so a wide part's bits
    // differ from the narrow one's (within the tolerances) and the host entry would no longer
    // reproduce the device entry bit for bit.
    static const int wide = getenv("HG_JACOBI_WIDE") ? atoi(getenv("HG_JACOBI_WIDE")) : 0;
    static const int wide_rows = getenv("HG_JACOBI_WIDE_ROWS") ? atoi(getenv("HG_JACOBI_WIDE_ROWS")) : 64;
    jacobi_rows_hint(((wide >> pt) & 1) ? wide_rows : 0);
    hg_status rs = run_rsvd(blocks + (int64_t)blk0 * b * b, nbp, blk0, b, l, q, seed, simt, Ut + kb,
                            sigma + (int64_t)(blk0 - soff) * l, Vt + kb, st, Bf, ps[pt], scheme, false, false, x16);
    jacobi_rows_hint(0);
    HG_TRY(rs);
    if (cps) HG_CU(cudaStreamWaitEvent(ps[pt], ev_y[pt], 0), "wait Y");
    HG_TRY(run_apply(Ut + kb, sigma + (int64_t)(blk0 - soff) * l, Vt + kb, nbp, b, k, T > 0 ? Y + (int64_t)blk0 * b * T : Y, T,
                     mu / (1.0f + mu), T > 0 ? F + (int64_t)blk0 * b * T : F, st, Bf, ps[pt], simt,
                     woodbury ? 1.0f + mu : 0.f, l, false, true));
    if (io.F_host && T > 0)
      HG_CU(cudaMemcpyAsync(io.F_host + (int64_t)blk0 * b * T, F + (int64_t)blk0 * b * T,
                            sizeof(float) * (size_t)nbp * b * T, cudaMemcpyDeviceToHost, ps[pt]),
            "D2H F");
  }
  g_cur_part = 0;
  HG_TRY(join_streams(s, nparts, ps));
  if (p > 0 && sigma_out)   // rank-k truncation of the oversampled sigma [nb][l] -> [rcnt][k]
    HG_CU(cudaMemcpy2DAsync(sigma_out, 4 * (size_t)k, sigma + (int64_t)rb0 * l, 4 * (size_t)l, 4 * (size_t)k, rcnt,
                            cudaMemcpyDeviceToDevice, s), "truncate sigma");
  if (flags & HG_SYNC) {
    int32_t h = 0;
    HG_CU(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s), "status readback");
    HG_CU(cudaStreamSynchronize(s), "synchronize");
    if (h) return fail(HG_ERR_NUMERICAL, "device status 0x%x (bits: 1 isolated vertex, 2 empty hyperedge, 4 "
                       "Cholesky breakdown, 8 Jacobi cap, 16 singular sigma, 32 non-finite)", h);
  }
  return HG_OK;
}

// CUDA-graph cache of hg_solve / hg_solve_host: the whole multi-stream launch sequence
// (8 parts of ~51 kernels, their fork/join events, the host copies) is captured once per
// distinct argument set and replayed with one cudaGraphLaunch on the caller's stream.
// Enqueued directly, the parts cost ~1.1-1.5 ms of host time and start ~0.4 ms apart.
extern "C++" {
namespace {
struct GraphEntry {
  std::string key;
  cudaGraphExec_t exec;
  int launches;
};
thread_local std::vector<GraphEntry> g_graphs;
constexpr size_t kMaxGraphs = 8;
std::string knob_env() {   // enqueue-time knobs that change the captured sequence
  std::string e;
  for (const char* n : {"HG_ASSEMBLE", "HG_STREAMS_SERIAL", "HG_BN_POWER", "HG_BN_GRAM", "HG_BN_QFORM", "HG_GRAM_FULL",
                        "HG_QR_PASSES", "HG_STREAM_PRIO", "HG_GEMM_F16", "HG_JACOBI_PRE", "HG_QR_SKIP_HALF", "HG_QR_LAZY"}) {
    const char* v = getenv(n);
    e += v ? v : "-";
    e += '|';
  }
  return e;
}
template <class T>
void key_add(std::string& k, const T& v) {
  k.append(reinterpret_cast<const char*>(&v), sizeof v);
}
bool graphs_enabled(cudaStream_t s) {
  const char* ng = getenv("HG_NO_GRAPH");
  if (g_prof_mode == 1 || (ng && ng[0] == '1')) return false;   // timeline mode (2) captures too
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) return false;
  return cap == cudaStreamCaptureStatusNone;
}
// Replay the cached graph for `key`, capturing `enqueue(capture_stream)` first if needed.
template <class Fn>
hg_status graph_run(const std::string& key, cudaStream_t s, Fn enqueue) {
  GraphEntry* ge = nullptr;
  const bool cache = g_prof_mode != 2;   // timeline graphs carry this call's stage events: not reused
  for (auto& e : g_graphs)
    if (cache && e.key == key) ge = &e;
  if (!ge) {
    HG_TRY(ensure_streams());
    static thread_local cudaStream_t cs = nullptr;
    if (!cs) HG_CU(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "capture stream");
    HG_CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
    g_launches = 0;
    const hg_status r = enqueue(cs);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
    if (r != HG_OK || ec != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();
      return r != HG_OK ? r : cuda_fail(ec, "end capture");
    }
    cudaGraphExec_t exec = nullptr;
    // node priorities (captured from the part streams) are honoured only with this flag
    const cudaError_t ei = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return cuda_fail(ei, "graph instantiate");
    if (!cache) {
      HG_CU(cudaGraphLaunch(exec, s), "graph launch");
      cudaGraphExecDestroy(exec);   // released once the launched work completes
      return HG_OK;
    }
    if (g_graphs.size() >= kMaxGraphs) {
      cudaGraphExecDestroy(g_graphs.front().exec);
      g_graphs.erase(g_graphs.begin());
    }
    g_graphs.push_back(GraphEntry{key, exec, g_launches});
    ge = &g_graphs.back();
  }
  HG_CU(cudaGraphLaunch(ge->exec, s), "graph launch");
  g_launches = ge->launches;
  return HG_OK;
}
}  // namespace
}  // extern "C++"

extern "C++" static hg_status solve_entry(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k,
                                          int32_t p, int32_t q, uint64_t seed, const float* Y, int32_t T, float* F,
                                          float* sigma_out, uint32_t flags, int32_t* d_status, void* ws,
                                          size_t ws_bytes, hg_stream_t stream, int32_t rb0, int32_t rcnt) {
  g_err.clear();
  g_launches = 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!graphs_enabled(s))
    return solve_impl(H, w, mu, b, k, p, q, seed, Y, T, F, sigma_out, flags, d_status, ws, ws_bytes, s, HostIO(),
                      rb0, rcnt);
  // host-side validation first (nothing is captured for an invalid call)
  HG_TRY(check_H(H));
  if (p < 0 || p % 4) return fail(HG_ERR_INVALID, "oversampling p must be >= 0 and a multiple of 4 (p=%d)", p);
  HG_TRY(check_sizes(H->n_vertices, b, k + p, q, T));
  const Layout Lo = layout(H->n_vertices, H->n_edges, H->nnz, b, k + p, T);
  HG_TRY(check_ws(ws, ws_bytes, Lo.h_rowptr));
  if (!d_status && !(flags & HG_SYNC)) return fail(HG_ERR_INVALID, "d_status may be NULL only with HG_SYNC");
  if (rcnt >= 0 && (rb0 < 0 || rcnt < 1 || rb0 + rcnt > H->n_vertices / b))
    return fail(HG_ERR_INVALID, "block range [%d, %d) outside [0, %d)", rb0, rb0 + rcnt, H->n_vertices / b);
  int32_t* st = d_status ? d_status : at<int32_t>(ws, Lo.status);
  std::string key = "solve|" + knob_env();
  key_add(key, rb0); key_add(key, rcnt);
  key_add(key, *H);
  key_add(key, w); key_add(key, mu); key_add(key, b); key_add(key, k); key_add(key, p); key_add(key, q); key_add(key, seed);
  key_add(key, Y); key_add(key, T); key_add(key, F); key_add(key, sigma_out); key_add(key, flags & ~HG_SYNC);
  key_add(key, st); key_add(key, ws); key_add(key, ws_bytes); key_add(key, solve_parts(0, b));
  HG_TRY(graph_run(key, s, [&](cudaStream_t cs) -> hg_status {
    if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), cs), "memset status");
    return solve_impl(H, w, mu, b, k, p, q, seed, Y, T, F, sigma_out, flags & ~HG_SYNC, st, ws, ws_bytes, cs,
                      HostIO(), rb0, rcnt);
  }));
  if (flags & HG_SYNC) {
    int32_t h = 0;
    HG_CU(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s), "status readback");
    HG_CU(cudaStreamSynchronize(s), "synchronize");
    if (h) return fail(HG_ERR_NUMERICAL, "device status 0x%x (bits: 1 isolated vertex, 2 empty hyperedge, 4 "
                       "Cholesky breakdown, 8 Jacobi cap, 16 singular sigma, 32 non-finite)", h);
  }
  return HG_OK;
}

hg_status hg_solve_ex(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t p, int32_t q,
                      uint64_t seed, const float* Y, int32_t T, float* F, float* sigma_out, uint32_t flags,
                      int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream) {
  return solve_entry(H, w, mu, b, k, p, q, seed, Y, T, F, sigma_out, flags, d_status, ws, ws_bytes, stream, 0, -1);
}

hg_status hg_solve_blocks(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q,
                          uint64_t seed, int32_t blk_begin, int32_t blk_count, const float* Y, int32_t T, float* F,
                          float* sigma_out, uint32_t flags, int32_t* d_status, void* ws, size_t ws_bytes,
                          hg_stream_t stream) {
  if (blk_count < 1) {
    g_err.clear();
    return fail(HG_ERR_INVALID, "blk_count must be >= 1");
  }
  return solve_entry(H, w, mu, b, k, 0, q, seed, Y, T, F, sigma_out, flags, d_status, ws, ws_bytes, stream, blk_begin,
                     blk_count);
}

hg_status hg_solve(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q, uint64_t seed,
                   const float* Y, int32_t T, float* F, float* sigma_out, uint32_t flags, int32_t* d_status, void* ws,
                   size_t ws_bytes, hg_stream_t stream) {
  return hg_solve_ex(H, w, mu, b, k, 0, q, seed, Y, T, F, sigma_out, flags, d_status, ws, ws_bytes, stream);
}

hg_status hg_solve_host(int32_t N, int32_t E, int64_t nnz, const int64_t* row_ptr_host, const int32_t* col_idx_host,
                        const float* w_host, float mu, int32_t b, int32_t k, int32_t q, uint64_t seed,
                        const float* Y_host, int32_t T, float* F_host, float* sigma_host, uint32_t flags, void* ws,
                        size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (!row_ptr_host || !w_host || (nnz > 0 && !col_idx_host) || (T > 0 && (!Y_host || !F_host)))
    return fail(HG_ERR_INVALID, "NULL host pointer");
  HG_TRY(check_sizes(N, b, k, q, T));
  if (E <= 0 || nnz < 0) return fail(HG_ERR_INVALID, "need E > 0, nnz >= 0");
  const Layout Lo = layout(N, E, nnz, b, k, T);
  HG_TRY(check_ws(ws, ws_bytes, Lo.total));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* st = at<int32_t>(ws, Lo.status);
  auto enqueue = [&](cudaStream_t s) -> hg_status {   // (shadows the caller's stream when captured)
  int64_t* d_rp = at<int64_t>(ws, Lo.h_rowptr);
  int32_t* d_col = at<int32_t>(ws, Lo.h_col);
  float* d_w = at<float>(ws, Lo.h_w);
  float* d_Y = at<float>(ws, Lo.h_Y);
  float* d_F = at<float>(ws, Lo.h_F);
  HG_CU(cudaMemcpyAsync(d_rp, row_ptr_host, 8 * (size_t)(N + 1), cudaMemcpyHostToDevice, s), "H2D row_ptr");
  if (nnz > 0) HG_CU(cudaMemcpyAsync(d_col, col_idx_host, 4 * (size_t)nnz, cudaMemcpyHostToDevice, s), "H2D col_idx");
  HG_CU(cudaMemcpyAsync(d_w, w_host, 4 * (size_t)E, cudaMemcpyHostToDevice, s), "H2D w");
  hg_incidence H{N, E, nnz, d_rp, d_col};
  const int nb = N / b;
  float* d_sig = at<float>(ws, Lo.sigma);
  HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), s), "memset status");
  HostIO io;
  io.Y_host = Y_host;
  io.F_host = F_host;
  HG_TRY(solve_impl(&H, d_w, mu, b, k, 0, q, seed, d_Y, T, d_F, d_sig, flags & ~HG_SYNC, st, ws, ws_bytes, s, io));
  if (sigma_host)
    HG_CU(cudaMemcpyAsync(sigma_host, d_sig, 4 * (size_t)nb * k, cudaMemcpyDeviceToHost, s), "D2H sigma");
  return HG_OK;
  };
  if (graphs_enabled(s)) {
    std::string key = "host|" + knob_env();
    key_add(key, N); key_add(key, E); key_add(key, nnz); key_add(key, row_ptr_host); key_add(key, col_idx_host);
    key_add(key, w_host); key_add(key, mu); key_add(key, b); key_add(key, k); key_add(key, q); key_add(key, seed);
    key_add(key, Y_host); key_add(key, T); key_add(key, F_host); key_add(key, sigma_host);
    key_add(key, flags & ~HG_SYNC); key_add(key, ws); key_add(key, ws_bytes); key_add(key, solve_parts());
    HG_TRY(graph_run(key, s, enqueue));
  } else {
    HG_TRY(enqueue(s));
  }
  int32_t h = 0;
  HG_CU(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s), "status readback");
  HG_CU(cudaStreamSynchronize(s), "synchronize");
  if (h) return fail(HG_ERR_NUMERICAL, "device status 0x%x", h);
  return HG_OK;
}

// ---------------------------------------------------------------- CG
hg_status hg_cg_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t T, int32_t max_iter, size_t* bytes) {
  g_err.clear();
  if (!bytes) return fail(HG_ERR_INVALID, "bytes is NULL");
  if (N <= 0 || E <= 0 || nnz < 0 || T < 1 || T % 4 || max_iter < 0)
    return fail(HG_ERR_INVALID, "need N, E > 0, nnz >= 0, T >= 1 with T %% 4 == 0, max_iter >= 0");
  if (nnz >= INT32_MAX) return fail(HG_ERR_INVALID, "nnz must be < 2^31 for hg_cg_solve");
  *bytes = cg_layout(N, E, nnz, T, max_iter).total;
  return HG_OK;
}

extern "C++" {
namespace {
// Stream-capture plumbing for the CG WHILE node (see CgGraphHook in kernels.cuh).
struct CgCapture {
  cudaStream_t cs = nullptr;   // the capturing stream
  cudaStream_t bs = nullptr;   // captures the body graph
  cudaGraph_t body = nullptr;
};
cudaError_t cg_begin(void* ctx, cudaGraphConditionalHandle* h) {
  CgCapture* c = static_cast<CgCapture*>(ctx);
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(c->cs, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  return cudaGraphConditionalHandleCreate(h, g, 0, cudaGraphCondAssignDefault);
}
cudaError_t cg_open_body(void* ctx, cudaGraphConditionalHandle h, cudaStream_t* bs) {
  CgCapture* c = static_cast<CgCapture*>(ctx);
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(c->cs, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  if ((e = cudaGraphAddNode(&node, g, deps, nd, &p)) != cudaSuccess) return e;
  if ((e = cudaStreamUpdateCaptureDependencies(c->cs, &node, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
    return e;
  c->body = p.conditional.phGraph_out[0];
  if (!c->bs && (e = cudaStreamCreateWithFlags(&c->bs, cudaStreamNonBlocking)) != cudaSuccess) return e;
  *bs = c->bs;
  return cudaStreamBeginCaptureToGraph(c->bs, c->body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
}
cudaError_t cg_close_body(void* ctx) {
  CgCapture* c = static_cast<CgCapture*>(ctx);
  cudaGraph_t g = c->body;
  return cudaStreamEndCapture(c->bs, &g);
}
thread_local CgCapture g_cg_cap;
}  // namespace
}  // extern "C++"

hg_status hg_cg_solve(const hg_incidence* H, const float* w, float mu, const float* Y, int32_t T, int32_t max_iter,
                      float tol, float* F, int32_t* iters, float* rel_res, uint32_t flags, int32_t* d_status,
                      void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  HG_TRY(check_H(H));
  if (T < 1 || T % 4) return fail(HG_ERR_INVALID, "T must be >= 1 and a multiple of 4 (T=%d)", T);
  if (max_iter < 0) return fail(HG_ERR_INVALID, "max_iter must be >= 0");
  if (!(mu > 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and > 0");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return fail(HG_ERR_INVALID, "tol must be finite and >= 0");
  if (!w || !Y || !F) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (H->nnz >= INT32_MAX) return fail(HG_ERR_INVALID, "nnz must be < 2^31 for hg_cg_solve");
  const CgLayout L = cg_layout(H->n_vertices, H->n_edges, H->nnz, T, max_iter);
  HG_TRY(check_ws(ws, ws_bytes, L.total));
  if (!d_status && !(flags & HG_SYNC)) return fail(HG_ERR_INVALID, "d_status may be NULL only with HG_SYNC");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* st = d_status ? d_status : at<int32_t>(ws, L.status);
  CgArgs a;
  a.N = H->n_vertices; a.E = H->n_edges; a.nnz = H->nnz; a.row_ptr = H->row_ptr; a.col_idx = H->col_idx;
  a.w = w; a.mu = mu; a.Y = Y; a.T = T; a.max_iter = max_iter; a.tol = tol; a.F = F;
  a.iters_out = iters; a.rel_out = rel_res; a.status = st; a.ws = ws;
  if (graphs_enabled(s) && !g_prof_on) {
    std::string key = "cg|";
    key_add(key, *H);
    key_add(key, w); key_add(key, mu); key_add(key, Y); key_add(key, T); key_add(key, max_iter); key_add(key, tol);
    key_add(key, F); key_add(key, iters); key_add(key, rel_res); key_add(key, st); key_add(key, ws);
    key_add(key, ws_bytes);
    HG_TRY(graph_run(key, s, [&](cudaStream_t cs) -> hg_status {
      if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), cs), "memset status");
      g_cg_cap.cs = cs;
      CgGraphHook hook{&g_cg_cap, cg_begin, cg_open_body, cg_close_body};
      HG_CU(launch_cg(a, &hook, cs, &g_launches), "cg (graph)");
      return HG_OK;
    }));
  } else {
    if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), s), "memset status");
    ProfScope ps(ST_CG, s);
    HG_CU(launch_cg(a, nullptr, s, &g_launches), "cg");
  }
  if (flags & HG_SYNC) {
    int32_t h = 0;
    HG_CU(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s), "status readback");
    HG_CU(cudaStreamSynchronize(s), "synchronize");
    if (h) return fail(HG_ERR_NUMERICAL, "device status 0x%x (bits: 1 isolated vertex, 2 empty hyperedge, "
                       "32 non-finite, 64 CG breakdown)", h);
  }
  return HG_OK;
}

// ---------------------------------------------------------------- NEXT-1
extern "C++" {
namespace {
struct SchurLayout {
  Layout R;      // degrees, Theta_ii blocks and the rSVD part buffers (offsets into ws)
  CgLayout C;    // CSC of H, at ws + cg_off
  size_t cg_off = 0, th12 = 0, ainv = 0, w = 0, kz = 0, utl = 0, sigl = 0, rsl = 0, wt = 0, utz = 0, sigz = 0,
         rsz = 0, zt = 0, t1 = 0, t2 = 0, total = 0;
};
SchurLayout schur_layout(int64_t N, int64_t E, int64_t nnz, int64_t b, int64_t k, int64_t T) {
  SchurLayout S;
  S.R = layout(N, E, nnz, b, k, T);
  S.C = cg_layout(N, E, nnz, 4, 0);
  size_t off = S.R.total;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + ALIGN - 1) / ALIGN * ALIGN;
    return o;
  };
  const int64_t nb = N / b, ns = nb / 2, Tt = T > 0 ? T : 1;
  S.cg_off = take(S.C.total);
  S.th12 = take(4 * ns * b * b);
  S.ainv = take(4 * nb * b * b);
  S.w = take(4 * ns * b * b);
  S.kz = take(4 * nb * b * b);
  S.utl = take(4 * nb * k * b);
  S.sigl = take(4 * nb * k);
  S.rsl = take(4 * nb * k);
  S.wt = take(4 * nb * k * b);
  S.utz = take(4 * nb * k * b);
  S.sigz = take(4 * nb * k);
  S.rsz = take(4 * nb * k);
  S.zt = take(4 * ns * k * Tt);
  S.t1 = take(4 * ns * b * Tt);
  S.t2 = take(4 * ns * b * Tt);
  S.total = off;
  return S;
}
}  // namespace
}  // extern "C++"

hg_status hg_schur_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t k, int32_t T, size_t* bytes) {
  g_err.clear();
  if (!bytes) return fail(HG_ERR_INVALID, "bytes is NULL");
  HG_TRY(check_sizes(N, b, k, 0, T));
  if (E <= 0 || nnz < 0 || nnz >= INT32_MAX) return fail(HG_ERR_INVALID, "need E > 0 and 0 <= nnz < 2^31");
  if ((N / b) % 2) return fail(HG_ERR_INVALID, "hg_solve_schur needs an even number of blocks (N %% 2b == 0)");
  *bytes = schur_layout(N, E, nnz, b, k, T).total;
  return HG_OK;
}

static hg_status schur_impl(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q,
                            uint64_t seed, const float* Y, int32_t T, float* F, int32_t* st, void* ws,
                            const SchurLayout& S, cudaStream_t s) {
  const int64_t N = H->n_vertices, nb = N / b, ns = nb / 2, bb = (int64_t)b * b, kb = (int64_t)k * b,
                bT = (int64_t)b * T, kT = (int64_t)k * T;
  const float opm = 1.0f + mu, ip = 1.0f / opm, c = mu / opm;
  float* blocks = at<float>(ws, S.R.blocks);
  float* th12 = at<float>(ws, S.th12);
  float* ainv = at<float>(ws, S.ainv);
  float* W = at<float>(ws, S.w);
  float* KZ = at<float>(ws, S.kz);
  float* UtL = at<float>(ws, S.utl);
  float* sigL = at<float>(ws, S.sigl);
  float* rsL = at<float>(ws, S.rsl);
  float* Wt = at<float>(ws, S.wt);
  float* UtZ = at<float>(ws, S.utz);
  float* sigZ = at<float>(ws, S.sigz);
  float* rsZ = at<float>(ws, S.rsz);
  float* Zt = at<float>(ws, S.zt);
  float* T1 = at<float>(ws, S.t1);
  float* T2 = at<float>(ws, S.t2);
  float* Vscratch = at<float>(ws, S.R.Vt);
  // 1. Theta_ii (raw) and the off-diagonal Theta_{2s,2s+1} from the sorted CSC
  float* dvr = at<float>(ws, S.R.dvr);
  HG_TRY(run_degrees(H, w, b, dvr, st, ws, S.R, s));
  HG_TRY(run_assemble(H, mu, b, true, 0, (int)nb, blocks, dvr, ws, S.R, s));
  void* cws = static_cast<char*>(ws) + S.cg_off;
  CgArgs ca;
  ca.N = (int)N; ca.E = H->n_edges; ca.nnz = H->nnz; ca.row_ptr = H->row_ptr; ca.col_idx = H->col_idx; ca.w = w;
  ca.mu = mu; ca.Y = nullptr; ca.T = 4; ca.max_iter = 0; ca.tol = 0.f; ca.F = nullptr; ca.iters_out = nullptr;
  ca.rel_out = nullptr; ca.status = st; ca.ws = cws;
  {
    ProfScope ps(ST_ASSEMBLE, s);
    HG_CU(launch_csc_setup(ca, s, &g_launches), "CSC");
    HG_CU(launch_theta_offblock((int)ns, b, H->row_ptr, H->col_idx, at<int32_t>(cws, S.C.col_ptr),
                                at<int32_t>(cws, S.C.csc), at<float>(cws, S.C.eval), at<float>(cws, S.C.dvr), th12, s,
                                &g_launches),
          "off-diagonal Theta");
  }
  // 2. leaves: Alg. 1 on Theta_ii, X_ii^-1 ~ I + U diag(s/((1+mu)-s)) U^T (reading R2), materialised
  HG_TRY(run_rsvd_parts(blocks, (int)nb, b, k, q, seed, UtL, sigL, Vscratch, st, ws, S.R, T, s));
  HG_CU(launch_woodbury_scale((int)nb, k, k, sigL, 1.f, opm, rsL, st, s, &g_launches), "woodbury weights");
  HG_CU(launch_scale_rows((int)nb, k, b, rsL, UtL, Wt, s, &g_launches), "scale rows");
  auto G = [&](int M, int Nn, int K, int batch) {
    GemmDesc g;
    g.M = M; g.N = Nn; g.K = K; g.batch = batch;
    return g;
  };
  {
    GemmDesc g = G(b, b, k, (int)nb);   // A_ii = W_t^T U_t (+ I below)
    g.A = Wt; g.a_mn = true; g.lda = b; g.sa = kb;
    g.B = UtL; g.b_mn = true; g.ldb = b; g.sb = kb;
    g.D = ainv; g.ldd = b; g.sd = bb;
    HG_TRY(gemm(g, s, false, "X_ii^-1"));
  }
  HG_CU(launch_add_identity((int)nb, b, ainv, s, &g_launches), "identity");
  // 3. Schur Grams K_Z1 = Theta11 + Theta12 A22 Theta21/(1+mu), K_Z2 = Theta22 + Theta21 A11 Theta12/(1+mu)
  {
    GemmDesc g = G(b, b, b, (int)ns);   // W = A22 Theta12^T
    g.A = ainv + bb; g.a_mn = false; g.lda = b; g.sa = 2 * bb;
    g.B = th12; g.b_mn = false; g.ldb = b; g.sb = bb;
    g.D = W; g.ldd = b; g.sd = bb;
    HG_TRY(gemm(g, s, false, "A22 Theta21"));
  }
  {
    GemmDesc g = G(b, b, b, (int)ns);   // K_Z1 = Theta12 W / (1+mu) + Theta11
    g.A = th12; g.a_mn = false; g.lda = b; g.sa = bb;
    g.B = W; g.b_mn = true; g.ldb = b; g.sb = bb;
    g.D = KZ; g.ldd = b; g.sd = 2 * bb;
    g.alpha = ip; g.C = blocks; g.ldc = b; g.sc = 2 * bb; g.beta = 1.f;
    HG_TRY(gemm(g, s, false, "K_Z1"));
  }
  {
    GemmDesc g = G(b, b, b, (int)ns);   // W = A11 Theta12
    g.A = ainv; g.a_mn = false; g.lda = b; g.sa = 2 * bb;
    g.B = th12; g.b_mn = true; g.ldb = b; g.sb = bb;
    g.D = W; g.ldd = b; g.sd = bb;
    HG_TRY(gemm(g, s, false, "A11 Theta12"));
  }
  {
    GemmDesc g = G(b, b, b, (int)ns);   // K_Z2 = Theta12^T W / (1+mu) + Theta22
    g.A = th12; g.a_mn = true; g.lda = b; g.sa = bb;
    g.B = W; g.b_mn = true; g.ldb = b; g.sb = bb;
    g.D = KZ + bb; g.ldd = b; g.sd = 2 * bb;
    g.alpha = ip; g.C = blocks + bb; g.ldc = b; g.sc = 2 * bb; g.beta = 1.f;
    HG_TRY(gemm(g, s, false, "K_Z2"));
  }
  HG_CU(launch_symmetrize((int)nb, b, KZ, s, &g_launches), "symmetrize");
  // 4. Z1^-1, Z2^-1 by Alg. 1 on K_Z (slot 2s: Z1, 2s+1: Z2; Omega keyed by the slot's block)
  HG_TRY(run_rsvd_parts(KZ, (int)nb, b, k, q, seed, UtZ, sigZ, Vscratch, st, ws, S.R, T, s));
  HG_CU(launch_woodbury_scale((int)nb, k, k, sigZ, 1.f, opm, rsZ, st, s, &g_launches), "woodbury weights");
  // 5. apply Eq. 12 to Y_s = [Y1; Y2] (super-block s: rows 2s b .. 2s b + 2b)
  //    wb: Out = beta (Yin + U D U^T Yin) with Z_t = beta D U^T Yin (GEMM with row scale), Out = U Z_t + beta Yin
  auto wb = [&](const float* Ut, const float* rs, const float* Yin, int64_t ys, float* Out, int64_t os,
                float beta) -> hg_status {
    {
      GemmDesc g = G(k, T, b, (int)ns);
      g.A = Ut; g.a_mn = false; g.lda = b; g.sa = 2 * kb;
      g.B = Yin; g.b_mn = true; g.ldb = T; g.sb = ys;
      g.D = Zt; g.ldd = T; g.sd = kT;
      g.rs = rs; g.srs = 2 * k; g.alpha = beta;
      HG_TRY(gemm(g, s, false, "Schur apply D U^T Y", ST_GEMM_APPLY));
    }
    GemmDesc g = G(b, T, k, (int)ns);
    g.A = Ut; g.a_mn = true; g.lda = b; g.sa = 2 * kb;
    g.B = Zt; g.b_mn = true; g.ldb = T; g.sb = kT;
    g.D = Out; g.ldd = T; g.sd = os;
    g.C = Yin; g.ldc = T; g.sc = ys; g.beta = beta;
    return gemm(g, s, false, "Schur apply U Z + Y", ST_GEMM_APPLY);
  };
  HG_TRY(wb(UtZ + kb, rsZ + k, Y + bT, 2 * bT, T1, bT, 1.f));   // T1 = Z2^-1 Y2
  {
    GemmDesc g = G(b, T, b, (int)ns);   // T2 = Theta12 T1
    g.A = th12; g.a_mn = false; g.lda = b; g.sa = bb;
    g.B = T1; g.b_mn = true; g.ldb = T; g.sb = bT;
    g.D = T2; g.ldd = T; g.sd = bT;
    HG_TRY(gemm(g, s, false, "Theta12 Z2^-1 Y2", ST_GEMM_APPLY));
  }
  HG_TRY(wb(UtL, rsL, T2, bT, T1, bT, 1.f));                    // T1 = A11 Theta12 Z2^-1 Y2
  HG_TRY(wb(UtZ, rsZ, Y, 2 * bT, T2, bT, 1.f));                 // T2 = Z1^-1 Y1
  HG_CU(launch_axpby((int)ns, bT, c, ip, T2, bT, T1, bT, F, 2 * bT, s, &g_launches), "F1");   // F1
  HG_TRY(wb(UtL, rsL, Y, 2 * bT, T1, bT, 1.f));                 // T1 = A11 Y1
  {
    GemmDesc g = G(b, T, b, (int)ns);   // T2 = Theta21 T1 / (1+mu) + Y2
    g.A = th12; g.a_mn = true; g.lda = b; g.sa = bb;
    g.B = T1; g.b_mn = true; g.ldb = T; g.sb = bT;
    g.D = T2; g.ldd = T; g.sd = bT;
    g.alpha = ip; g.C = Y + bT; g.ldc = T; g.sc = 2 * bT; g.beta = 1.f;
    HG_TRY(gemm(g, s, false, "Y2 + Theta21 A11 Y1", ST_GEMM_APPLY));
  }
  HG_TRY(wb(UtZ + kb, rsZ + k, T2, bT, F + bT, 2 * bT, c));     // F2 = c Z2^-1 T2
  return HG_OK;
}

// ---------------------------------------------------------------- NEXT-1: nested tessellation
// PAPER.md:155-156 (reading S4): Eq. 12 recursively inside super-blocks of m = 2^L b
// vertices, leaves b x b, the level-l Schur complements (h = 2^(l-1) b) at rank k_l = k 2^(l-1), all
// inverses by reading R2 (Alg. 1 on the PSD K + Woodbury) and materialised dense, level by level over
// all nodes at once (batched GEMMs, the rSVDs in the stream parts).
extern "C++" {
namespace {
struct NestedLayout {
  Layout R;      // degrees, keys, rSVD part buffers sized for the top level (h_L, k_L)
  CgLayout C;    // CSC of H
  Layout Rk;     // R with its assembly keys region sized for the N/b leaves
  size_t cg_off = 0, keys = 0, th[2] = {0, 0}, ai[2] = {0, 0}, off = 0, zinv = 0, tr = 0, wsc = 0, ut = 0, sig = 0,
         rs = 0, wt = 0, total = 0;
};
NestedLayout nested_layout(int64_t N, int64_t E, int64_t nnz, int64_t b, int64_t L, int64_t k, int64_t T) {
  NestedLayout S;
  const int64_t hL = b << (L - 1), kL = k << (L - 1);
  S.R = layout(N, E, nnz, hL, kL, T);
  S.C = cg_layout(N, E, nnz, 4, 0);
  size_t off = S.R.total;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + ALIGN - 1) / ALIGN * ALIGN;
    return o;
  };
  S.cg_off = take(S.C.total);
  S.keys = take(assemble_keys_bytes(nnz, (int)(N / b), (int)E));
  S.Rk = S.R;
  S.Rk.keys = S.keys;
  for (int i = 0; i < 2; ++i) {
    S.th[i] = take(4 * N * 2 * hL);   // node Theta of a level (N x n floats)
    S.ai[i] = take(4 * N * 2 * hL);   // node inverse of a level
  }
  S.off = take(4 * N * hL / 2);       // Theta_12 of every node [nn][h][h]
  S.zinv = take(4 * N * hL);          // Z1^-1, Z2^-1 [2nn][h][h]
  S.tr = take(4 * N * hL / 2);        // top-right quadrants [nn][h][h]
  S.wsc = take(4 * N * hL / 2);       // GEMM scratch [nn][h][h]
  S.ut = take(4 * N * kL);            // U^T of the level's rSVDs [slots][k_l][h]
  S.sig = take(4 * (N / b) * k);      // [slots][k_l]: (N / h_l) k_l = N k / b
  S.rs = take(4 * (N / b) * k);
  S.wt = take(4 * N * kL);
  S.total = off;
  return S;
}
}  // namespace
}  // extern "C++"

hg_status hg_nested_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t levels, int32_t k, int32_t T,
                                   size_t* bytes) {
  g_err.clear();
  if (!bytes) return fail(HG_ERR_INVALID, "bytes is NULL");
  if (levels < 1 || levels > 6) return fail(HG_ERR_INVALID, "levels must be in [1, 6] (levels=%d)", levels);
  HG_TRY(check_sizes(N, b, k, 0, T));
  if (T % 4) return fail(HG_ERR_INVALID, "hg_solve_nested needs T %% 4 == 0 (T=%d)", T);
  if (E <= 0 || nnz < 0 || nnz >= INT32_MAX) return fail(HG_ERR_INVALID, "need E > 0 and 0 <= nnz < 2^31");
  if (N % ((int64_t)b << levels)) return fail(HG_ERR_INVALID, "N %% (2^levels b) != 0");
  if (((int64_t)k << (levels - 1)) > 512)
    return fail(HG_ERR_INVALID, "the top-level Schur rank k 2^(levels-1) must be <= 512");
  *bytes = nested_layout(N, E, nnz, b, levels, k, T).total;
  return HG_OK;
}

static hg_status nested_impl(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t L, int32_t k,
                             int32_t q, uint64_t seed, const float* Y, int32_t T, float* F, int32_t* st, void* ws,
                             const NestedLayout& S, cudaStream_t s) {
  const int64_t N = H->n_vertices;
  const float opm = 1.0f + mu, ip = 1.0f / opm, c = mu / opm;
  float* thc = at<float>(ws, S.th[0]);
  float* thn = at<float>(ws, S.th[1]);
  float* aic = at<float>(ws, S.ai[0]);
  float* ain = at<float>(ws, S.ai[1]);
  float* off = at<float>(ws, S.off);
  float* KZ = at<float>(ws, S.R.blocks);
  float* Zi = at<float>(ws, S.zinv);
  float* TR = at<float>(ws, S.tr);
  float* Wsc = at<float>(ws, S.wsc);
  float* Ut = at<float>(ws, S.ut);
  float* sg = at<float>(ws, S.sig);
  float* rs = at<float>(ws, S.rs);
  float* Wt = at<float>(ws, S.wt);
  float* Vscratch = at<float>(ws, S.R.Vt);
  auto G = [&](int M, int Nn, int K, int batch) {
    GemmDesc g;
    g.M = M; g.N = Nn; g.K = K; g.batch = batch;
    return g;
  };
  // R2 inverse of nb PSD-K slots (h x h): I + U diag(s/((1+mu)-s)) U^T -> out [nb][h][h]
  auto lowrank_inverse = [&](const float* Kb, int nb, int h, int kl, float* out) -> hg_status {
    HG_TRY(run_rsvd_parts(Kb, nb, h, kl, q, seed, Ut, sg, Vscratch, st, ws, S.R, T, s));
    HG_CU(launch_woodbury_scale(nb, kl, kl, sg, 1.f, opm, rs, st, s, &g_launches), "woodbury weights");
    HG_CU(launch_scale_rows(nb, kl, h, rs, Ut, Wt, s, &g_launches), "scale rows");
    GemmDesc g = G(h, h, kl, nb);   // W_t^T U_t
    g.A = Wt; g.a_mn = true; g.lda = h; g.sa = (int64_t)kl * h;
    g.B = Ut; g.b_mn = true; g.ldb = h; g.sb = (int64_t)kl * h;
    g.D = out; g.ldd = h; g.sd = (int64_t)h * h;
    HG_TRY(gemm(g, s, false, "I + U D U^T"));
    HG_CU(launch_add_identity(nb, h, out, s, &g_launches), "identity");
    return HG_OK;
  };
  // leaves: Theta_ii (raw), their inverses
  float* dvr = at<float>(ws, S.R.dvr);
  HG_TRY(run_degrees(H, w, b, dvr, st, ws, S.Rk, s));
  HG_TRY(run_assemble(H, mu, b, true, 0, (int)(N / b), thc, dvr, ws, S.Rk, s));
  void* cws = static_cast<char*>(ws) + S.cg_off;
  CgArgs ca;
  ca.N = (int)N; ca.E = H->n_edges; ca.nnz = H->nnz; ca.row_ptr = H->row_ptr; ca.col_idx = H->col_idx; ca.w = w;
  ca.mu = mu; ca.Y = nullptr; ca.T = 4; ca.max_iter = 0; ca.tol = 0.f; ca.F = nullptr; ca.iters_out = nullptr;
  ca.rel_out = nullptr; ca.status = st; ca.ws = cws;
  {
    ProfScope ps(ST_ASSEMBLE, s);
    HG_CU(launch_csc_setup(ca, s, &g_launches), "CSC");
  }
  HG_TRY(lowrank_inverse(thc, (int)(N / b), b, k, aic));
  for (int l = 1; l <= L; ++l) {
    const int h = b << (l - 1), kl = k << (l - 1);
    const int64_t n = 2 * (int64_t)h, nn = N / n, hh = (int64_t)h * h;
    {
      ProfScope ps(ST_ASSEMBLE, s);   // Theta_12 of every node: rows of its first half, columns of its second
      HG_CU(launch_theta_offblock((int)nn, h, H->row_ptr, H->col_idx, at<int32_t>(cws, S.C.col_ptr),
                                  at<int32_t>(cws, S.C.csc), at<float>(cws, S.C.eval), at<float>(cws, S.C.dvr), off, s,
                                  &g_launches),
            "off-diagonal Theta");
    }
    {   // K_Z1 = Theta11 + Theta12 (A22 Theta21) / (1+mu)
      GemmDesc g = G(h, h, h, (int)nn);
      g.A = aic + hh; g.a_mn = false; g.lda = h; g.sa = 2 * hh;
      g.B = off; g.b_mn = false; g.ldb = h; g.sb = hh;
      g.D = Wsc; g.ldd = h; g.sd = hh;
      HG_TRY(gemm(g, s, false, "A22 Theta21"));
      GemmDesc g2 = G(h, h, h, (int)nn);
      g2.A = off; g2.a_mn = false; g2.lda = h; g2.sa = hh;
      g2.B = Wsc; g2.b_mn = true; g2.ldb = h; g2.sb = hh;
      g2.D = KZ; g2.ldd = h; g2.sd = 2 * hh;
      g2.alpha = ip; g2.C = thc; g2.ldc = h; g2.sc = 2 * hh; g2.beta = 1.f;
      HG_TRY(gemm(g2, s, false, "K_Z1"));
    }
    {   // K_Z2 = Theta22 + Theta21 (A11 Theta12) / (1+mu)
      GemmDesc g = G(h, h, h, (int)nn);
      g.A = aic; g.a_mn = false; g.lda = h; g.sa = 2 * hh;
      g.B = off; g.b_mn = true; g.ldb = h; g.sb = hh;
      g.D = Wsc; g.ldd = h; g.sd = hh;
      HG_TRY(gemm(g, s, false, "A11 Theta12"));
      GemmDesc g2 = G(h, h, h, (int)nn);
      g2.A = off; g2.a_mn = true; g2.lda = h; g2.sa = hh;
      g2.B = Wsc; g2.b_mn = true; g2.ldb = h; g2.sb = hh;
      g2.D = KZ + hh; g2.ldd = h; g2.sd = 2 * hh;
      g2.alpha = ip; g2.C = thc + hh; g2.ldc = h; g2.sc = 2 * hh; g2.beta = 1.f;
      HG_TRY(gemm(g2, s, false, "K_Z2"));
    }
    HG_CU(launch_symmetrize((int)(2 * nn), h, KZ, s, &g_launches), "symmetrize");
    // Z1^-1 (slot 2s), Z2^-1 (slot 2s+1): Omega rows of the N x k_l Philox matrix (reading S3, S5)
    HG_TRY(lowrank_inverse(KZ, (int)(2 * nn), h, kl, Zi));
    {   // top-right A11 Theta12 Z2^-1 / (1+mu): Wsc = A11 Theta12 is still there from K_Z2
      GemmDesc g2 = G(h, h, h, (int)nn);
      g2.A = Wsc; g2.a_mn = false; g2.lda = h; g2.sa = hh;
      g2.B = Zi + hh; g2.b_mn = true; g2.ldb = h; g2.sb = 2 * hh;
      g2.D = TR; g2.ldd = h; g2.sd = hh;
      g2.alpha = ip;
      HG_TRY(gemm(g2, s, false, "A11 Theta12 Z2^-1"));
    }
    HG_CU(launch_place_node((int)nn, h, Zi, 2 * hh, Zi + hh, 2 * hh, TR, hh, ain, s, &g_launches), "node inverse");
    if (l < L)
      HG_CU(launch_place_node((int)nn, h, thc, 2 * hh, thc + hh, 2 * hh, off, hh, thn, s, &g_launches), "node Theta");
    std::swap(aic, ain);
    std::swap(thc, thn);
  }
  // F_s = c A_s^-1 Y_s (Eq. 3), super-blocks of m = 2^L b
  const int64_t m = (int64_t)b << L;
  GemmDesc g = G((int)m, T, (int)m, (int)(N / m));
  g.A = aic; g.a_mn = false; g.lda = m; g.sa = m * m;
  g.B = Y; g.b_mn = true; g.ldb = T; g.sb = m * T;
  g.D = F; g.ldd = T; g.sd = m * T;
  g.alpha = c;
  return gemm(g, s, false, "F = c A^-1 Y", ST_GEMM_APPLY);
}

hg_status hg_solve_nested(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t levels, int32_t k,
                          int32_t q, uint64_t seed, const float* Y, int32_t T, float* F, uint32_t flags,
                          int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  HG_TRY(check_H(H));
  size_t need = 0;
  HG_TRY(hg_nested_workspace_size(H->n_vertices, H->n_edges, H->nnz, b, levels, k, T, &need));
  if (T < 1) return fail(HG_ERR_INVALID, "T must be >= 1");
  if (q < 0) return fail(HG_ERR_INVALID, "q must be >= 0");
  if (!(mu > 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and > 0");
  if (!w || !Y || !F) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (!d_status && !(flags & HG_SYNC)) return fail(HG_ERR_INVALID, "d_status may be NULL only with HG_SYNC");
  const NestedLayout S = nested_layout(H->n_vertices, H->n_edges, H->nnz, b, levels, k, T);
  HG_TRY(check_ws(ws, ws_bytes, S.total));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* st = d_status ? d_status : at<int32_t>(ws, S.R.status);
  if (graphs_enabled(s) && !g_prof_on) {
    std::string key = "nested|" + knob_env();
    key_add(key, *H);
    key_add(key, w); key_add(key, mu); key_add(key, b); key_add(key, levels); key_add(key, k); key_add(key, q);
    key_add(key, seed); key_add(key, Y); key_add(key, T); key_add(key, F); key_add(key, st); key_add(key, ws);
    key_add(key, ws_bytes); key_add(key, solve_parts());
    HG_TRY(graph_run(key, s, [&](cudaStream_t cs) -> hg_status {
      if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), cs), "memset status");
      return nested_impl(H, w, mu, b, levels, k, q, seed, Y, T, F, st, ws, S, cs);
    }));
  } else {
    if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), s), "memset status");
    HG_TRY(nested_impl(H, w, mu, b, levels, k, q, seed, Y, T, F, st, ws, S, s));
  }
  if (flags & HG_SYNC) {
    int32_t h = 0;
    HG_CU(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s), "status readback");
    HG_CU(cudaStreamSynchronize(s), "synchronize");
    if (h) return fail(HG_ERR_NUMERICAL, "device status 0x%x", h);
  }
  return HG_OK;
}

hg_status hg_solve_schur(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q,
                         uint64_t seed, const float* Y, int32_t T, float* F, uint32_t flags, int32_t* d_status,
                         void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  HG_TRY(check_H(H));
  HG_TRY(check_sizes(H->n_vertices, b, k, q, T));
  if (T < 1) return fail(HG_ERR_INVALID, "T must be >= 1");
  if ((H->n_vertices / b) % 2) return fail(HG_ERR_INVALID, "hg_solve_schur needs N %% 2b == 0");
  if (!(mu > 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and > 0");
  if (!w || !Y || !F) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (H->nnz >= INT32_MAX) return fail(HG_ERR_INVALID, "nnz must be < 2^31");
  if (!d_status && !(flags & HG_SYNC)) return fail(HG_ERR_INVALID, "d_status may be NULL only with HG_SYNC");
  const SchurLayout S = schur_layout(H->n_vertices, H->n_edges, H->nnz, b, k, T);
  HG_TRY(check_ws(ws, ws_bytes, S.total));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* st = d_status ? d_status : at<int32_t>(ws, S.R.status);
  if (graphs_enabled(s) && !g_prof_on) {
    std::string key = "schur|" + knob_env();
    key_add(key, *H);
    key_add(key, w); key_add(key, mu); key_add(key, b); key_add(key, k); key_add(key, q); key_add(key, seed);
    key_add(key, Y); key_add(key, T); key_add(key, F); key_add(key, st); key_add(key, ws); key_add(key, ws_bytes);
    key_add(key, solve_parts());
    HG_TRY(graph_run(key, s, [&](cudaStream_t cs) -> hg_status {
      if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), cs), "memset status");
      return schur_impl(H, w, mu, b, k, q, seed, Y, T, F, st, ws, S, cs);
    }));
  } else {
    if (!d_status) HG_CU(cudaMemsetAsync(st, 0, sizeof(int32_t), s), "memset status");
    HG_TRY(schur_impl(H, w, mu, b, k, q, seed, Y, T, F, st, ws, S, s));
  }
  if (flags & HG_SYNC) {
    int32_t h = 0;
    HG_CU(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s), "status readback");
    HG_CU(cudaStreamSynchronize(s), "synchronize");
    if (h) return fail(HG_ERR_NUMERICAL, "device status 0x%x", h);
  }
  return HG_OK;
}

// ---------------------------------------------------------------- NEXT-4
hg_status hg_weight_gradient(const hg_incidence* H, const float* w, const float* F, int32_t T, float kappa,
                             float* grad, int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  HG_TRY(check_H(H));
  if (T < 1 || T % 4) return fail(HG_ERR_INVALID, "T must be >= 1 and a multiple of 4 (T=%d)", T);
  if (!w || !F || !grad || !d_status) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (!std::isfinite(kappa)) return fail(HG_ERR_INVALID, "kappa must be finite");
  if (H->nnz >= INT32_MAX) return fail(HG_ERR_INVALID, "nnz must be < 2^31");
  const CgLayout L = cg_layout(H->n_vertices, H->n_edges, H->nnz, T, 0);
  HG_TRY(check_ws(ws, ws_bytes, L.total));
  CgArgs a;
  a.N = H->n_vertices; a.E = H->n_edges; a.nnz = H->nnz; a.row_ptr = H->row_ptr; a.col_idx = H->col_idx;
  a.w = w; a.mu = 1.f; a.Y = nullptr; a.T = T; a.max_iter = 0; a.tol = 0.f; a.F = const_cast<float*>(F);
  a.iters_out = nullptr; a.rel_out = nullptr; a.status = d_status; a.ws = ws;
  HG_CU(launch_weight_gradient(a, kappa, grad, reinterpret_cast<cudaStream_t>(stream), &g_launches), "weight gradient");
  return HG_OK;
}

hg_status hg_weight_objective(const float* F, int32_t N, int32_t T, int32_t E, const float* w, const float* grad,
                              float kappa, double* out, void* ws, size_t ws_bytes, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (N <= 0 || T < 0 || E <= 0) return fail(HG_ERR_INVALID, "need N > 0, T >= 0, E > 0");
  if (!F || !w || !grad || !out) return fail(HG_ERR_INVALID, "NULL pointer argument");
  HG_TRY(check_ws(ws, ws_bytes, 296 * sizeof(double)));
  HG_CU(launch_weight_objective((int64_t)N * T, F, E, w, grad, kappa, static_cast<double*>(ws), out,
                                reinterpret_cast<cudaStream_t>(stream), &g_launches),
        "weight objective");
  return HG_OK;
}

hg_status hg_weight_normalize(int32_t E, const float* w, float* w_out, int32_t* d_status, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (E <= 0) return fail(HG_ERR_INVALID, "E must be > 0");
  if (!w || !w_out || !d_status) return fail(HG_ERR_INVALID, "NULL pointer argument");
  HG_CU(launch_weight_normalize(E, w, w_out, d_status, reinterpret_cast<cudaStream_t>(stream), &g_launches),
        "weight normalize");
  return HG_OK;
}

hg_status hg_weight_step(int32_t E, float* w, int32_t* active, const float* grad, float mu, int32_t* d_status,
                         hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (E <= 0) return fail(HG_ERR_INVALID, "E must be > 0");
  if (!w || !active || !grad || !d_status) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (!(mu >= 0.f) || !std::isfinite(mu)) return fail(HG_ERR_INVALID, "mu must be finite and >= 0");
  HG_CU(launch_weight_step(E, w, active, grad, mu, d_status, reinterpret_cast<cudaStream_t>(stream), &g_launches),
        "weight step");
  return HG_OK;
}

hg_status hg_gemm(int32_t M, int32_t N, int32_t K, int32_t batch, const float* A, int32_t a_mn, int64_t lda,
                  int64_t sa, const float* B, int32_t b_mn, int64_t ldb, int64_t sb, float* D, int32_t d_trans,
                  int64_t ldd, int64_t sd, float alpha, const float* rs, int64_t srs, const float* cs, int64_t scs,
                  uint32_t flags, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (!A || !B || !D) return fail(HG_ERR_INVALID, "NULL pointer argument");
  GemmDesc g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.a_mn = a_mn != 0; g.lda = lda; g.sa = sa;
  g.B = B; g.b_mn = b_mn != 0; g.ldb = ldb; g.sb = sb;
  g.D = D; g.d_trans = d_trans != 0; g.ldd = ldd; g.sd = sd;
  g.alpha = alpha; g.rs = rs; g.srs = srs; g.cs = cs; g.scs = scs;
  return gemm(g, reinterpret_cast<cudaStream_t>(stream), (flags & HG_GEMM_SIMT) != 0, "hg_gemm");
}

hg_status hg_gemm_ex(int32_t M, int32_t N, int32_t K, int32_t batch, const float* A, int32_t a_mn, int64_t lda,
                     int64_t sa, const float* B, int32_t b_mn, int64_t ldb, int64_t sb, float* D, int32_t d_trans,
                     int64_t ldd, int64_t sd, float alpha, const float* rs, int64_t srs, const float* cs,
                     int64_t scs, uint32_t flags, int32_t prec, int32_t a_exp, int32_t b_exp, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (!A || !B || !D) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (prec < -1 || prec > 1) return fail(HG_ERR_INVALID, "prec must be -1, 0 or 1 (prec=%d)", prec);
  GemmDesc g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.a_mn = a_mn != 0; g.lda = lda; g.sa = sa;
  g.B = B; g.b_mn = b_mn != 0; g.ldb = ldb; g.sb = sb;
  g.D = D; g.d_trans = d_trans != 0; g.ldd = ldd; g.sd = sd;
  g.alpha = alpha; g.rs = rs; g.srs = srs; g.cs = cs; g.scs = scs;
  g.prec = prec; g.a_exp = a_exp; g.b_exp = b_exp;
  return gemm(g, reinterpret_cast<cudaStream_t>(stream), (flags & HG_GEMM_SIMT) != 0, "hg_gemm_ex");
}

hg_status hg_f16_split(const float* x, int64_t rows, int32_t cols, int64_t ld, int32_t exp, uint16_t* out16,
                       hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (!x || !out16) return fail(HG_ERR_INVALID, "NULL pointer argument");
  if (rows < 0 || cols < 0 || (cols & 31) || (ld & 3) || ld < cols)
    return fail(HG_ERR_INVALID, "need cols %% 32 == 0, ld %% 4 == 0, ld >= cols");
  HG_CU(launch_f16_split(x, rows, cols, ld, exp, out16, reinterpret_cast<cudaStream_t>(stream)), "f16 split");
  ++g_launches;
  return HG_OK;
}

hg_status hg_gemm_f16pre(int32_t M, int32_t N, int32_t K, int32_t batch, const uint16_t* A16, int64_t lda,
                         int64_t sa, int32_t a_exp, const uint16_t* B16, int64_t ldb, int64_t sb, int32_t b_exp,
                         float* D, int32_t d_trans, int64_t ldd, int64_t sd, float alpha, hg_stream_t stream) {
  g_err.clear();
  g_launches = 0;
  if (!A16 || !B16 || !D) return fail(HG_ERR_INVALID, "NULL pointer argument");
  GemmDesc g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A16 = A16; g.lda = lda; g.sa = sa; g.a_exp = a_exp;
  g.B16 = B16; g.ldb = ldb; g.sb = sb; g.b_exp = b_exp;
  g.D = D; g.d_trans = d_trans != 0; g.ldd = ldd; g.sd = sd;
  g.alpha = alpha;
  g.prec = 1;
  return gemm(g, reinterpret_cast<cudaStream_t>(stream), false, "hg_gemm_f16pre");
}

}  // extern "C"
