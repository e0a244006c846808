/*
 * hg.h -- C ABI of libhgrsvd: the block randomized SVD hot path of
 * arXiv:1908.08281 on NVIDIA B200 (sm_100a).
 *
 * The path (section 3, Alg. 1 and Eqs. 1, 3, 11, 15):
 *   1. hg_build_theta          diagonal b x b blocks X_ii of X = I - Theta/(1+mu),
 *                              Theta = Dv^-1/2 H W De^-1 H^T Dv^-1/2      (Eq. 1)
 *   2. hg_block_rsvd           per block, Alg. 1 with l = k, pi = q
 *   3. hg_block_apply_inverse  F_i = scale * V_i Sigma_i^-1 U_i^T Y_i      (Eq. 3,
 *                                                                           PAPER.md:160-163 Eq. 15)
 *   hg_solve = 1 -> 2 -> 3 from the CSR incidence to F (hg_solve_host: from host buffers;
 *   hg_solve_blocks: one block range, a rank's share of a sharded problem).
 *
 * Beyond the hot path (each against the same FP64 oracle):
 *   hg_solve_ex / hg_block_rsvd_ex  oversampling l = k + p, Eq. 10 scheme
 *   HG_WOODBURY, hg_block_apply_woodbury  reading R2: Alg. 1 on Theta_ii
 *   hg_solve_schur                  one 2x2 Schur level, Eqs. 11-14
 *   hg_cg_solve                     CG on Eq. 5, Eqs. 16-20
 *   hg_weight_gradient / _step / _objective  the hyperedge-weight update
 *
 * Conventions for every entry point:
 *   - Pointers are DEVICE pointers owned by the caller unless a name says
 *     "host"; nothing is retained after return.  Matrices are dense row-major
 *     fp32 unless noted.  "[a][b][c]" gives the dimensions, last contiguous.
 *   - Work is enqueued on `stream` and is asynchronous unless stated.  The
 *     library never allocates device memory on these calls: scratch comes
 *     from the caller's workspace `ws` (size from hg_workspace_size, 256-byte
 *     aligned; CG / Schur entries have their own size queries).  Distinct
 *     workspaces make concurrent calls thread-safe (the library's part
 *     streams and events are per host thread).
 *   - Host-side validation failures return HG_ERR_INVALID synchronously and
 *     enqueue nothing.  Data-dependent failures found on the device are OR-ed
 *     as bit flags into the caller's device word *d_status (0 = ok; the
 *     caller zeroes it); hg_solve with HG_SYNC and hg_solve_host read it back
 *     and return HG_ERR_NUMERICAL.  CUDA launch/runtime errors return
 *     HG_ERR_CUDA.  hg_last_error() describes the last failure on the calling
 *     host thread.
 *   - Singular vectors are returned TRANSPOSED: Ut[i] = U_i^T (k x b) and
 *     Vt[i] = V_i^T (k x b), i.e. each singular vector is one contiguous row.
 *     Singular values are non-increasing; the sign of each pair (u_j, v_j) is
 *     fixed so that the largest-|.| entry of u_j is positive.
 */
#ifndef HG_H_
#define HG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hg_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  HG_OK = 0,
  HG_ERR_INVALID = 2,   /* bad argument / workspace too small (host-side, synchronous) */
  HG_ERR_NUMERICAL = 3, /* device status word non-zero (see hg_status_flags)            */
  HG_ERR_CUDA = 4       /* CUDA runtime / launch error                                   */
} hg_status;

/* Device status word bits (OR-ed into *d_status). */
enum hg_status_flags {
  HG_ST_ISOLATED_VERTEX = 1 << 0, /* delta(v) = 0                 */
  HG_ST_EMPTY_EDGE = 1 << 1,      /* delta(e) = 0                                            */
  HG_ST_CHOL_BREAKDOWN = 1 << 2,  /* CholeskyQR pivot <= 0: Y_i rank-deficient to fp32        */
  HG_ST_JACOBI_CAP = 1 << 3,      /* one-sided Jacobi did not converge in the sweep cap      */
  HG_ST_SINGULAR_SIGMA = 1 << 4,  /* sigma_j <= 1e-6 sigma_1 at apply      */
  HG_ST_NONFINITE = 1 << 5,       /* NaN/Inf met                                             */
  HG_ST_CG_BREAKDOWN = 1 << 6,    /* hg_cg_solve: p^T X p <= 0 (X is SPD: corrupt input only)  */
  HG_ST_SIMPLEX_DEGENERATE = 1 << 7 /* hg_weight_step: every hyperedge weight clamped to 0     */
};

/* flags */
#define HG_RAW_THETA (1u << 0)  /* hg_build_theta: write Theta_ii instead of X_ii          */
#define HG_SYNC (1u << 1)       /* hg_solve: synchronise `stream`, map *d_status to status  */
#define HG_WOODBURY (1u << 2)   /* hg_solve(_host): reading R2, see  */
                                /* hg_block_apply_woodbury                                     */
#define HG_POWER_EQ10 (1u << 3) /* hg_block_rsvd(_ex) / hg_solve(_ex): the Eq. 10 scheme     */
                                /* Y = (X X^T)^q X Omega, one QR at the end  */
#define HG_GENERAL (1u << 4)    /* hg_block_rsvd(_ex): blocks need not be symmetric -- the X^T   */
                                /* products of Alg. 1 use the literal transpose   */
#define HG_UV_BK (1u << 5)      /* hg_block_rsvd / hg_block_apply_inverse_ex: U, V [nb][b][k]    */
                                /* (column j = u_j) instead of the transposed Ut, Vt [nb][k][b]  */
#define HG_X_UNIT (1u << 6)     /* hg_block_rsvd(_ex): the caller guarantees |X_ij| <= 1 and     */
                                /* ||X_ii||_2 <= 1 (true of hg_build_theta's X_ii and Theta_ii):  */
                                /* enables the 3xF16 power products and Grams the solve entries  */
                                /* use (off: 3xTF32).  Needs b % 8 == 0 */
                                /* and no HG_GENERAL; ignored otherwise.                          */
#define HG_GEMM_SIMT (1u << 8)  /* verification only: CUDA-core fp32 GEMMs, not tcgen05    */

/* Hypergraph incidence H (H(v,e) = 1 iff v in e) in CSR over
 * vertices; values are implicitly 1.  Device pointers. */
typedef struct {
  int32_t n_vertices;     /* N = |V| (m in the paper)                        */
  int32_t n_edges;        /* E = |E| (n in the paper)                        */
  int64_t nnz;            /* number of incidences                            */
  const int64_t* row_ptr; /* [N+1], row_ptr[0] = 0, row_ptr[N] = nnz         */
  const int32_t* col_idx; /* [nnz] hyperedge ids in [0,E), strictly increasing per row */
} hg_incidence;

/* Bytes of workspace needed by any call below for these sizes (T may be 0
 * when no apply is made).  Returns HG_ERR_INVALID on bad sizes. */
hg_status hg_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t k, int32_t T,
                            size_t* bytes);

/* Eq. 1 diagonal blocks.  For block i (vertices [ib,(i+1)b)):
 *   X_ii[u][v] = delta_uv - r_u r_v sum_{e ni u,v} w_e/delta(e) / (1+mu),  r = delta(v)^-1/2,
 * with delta(v) = sum_e w_e H(v,e), delta(e) = sum_v H(v,e).
 *   w        [E] hyperedge weights (> 0 expected; not normalised, reading A9)
 *   mu       the regulariser theta > 0 (configs' "mu")
 *   b        block size, N % b == 0
 *   flags    HG_RAW_THETA writes Theta_ii instead of X_ii
 *   blocks   out [N/b][b][b]; bitwise symmetric
 *   dv_rsqrt out [N] r_v, may be NULL
 * Device errors: HG_ST_ISOLATED_VERTEX, HG_ST_EMPTY_EDGE. */
hg_status hg_build_theta(const hg_incidence* H, const float* w, float mu, int32_t b, uint32_t flags,
                         float* blocks, float* dv_rsqrt, int32_t* d_status, void* ws, size_t ws_bytes,
                         hg_stream_t stream);

/* Alg. 1 step 1 test matrix (reading A6):
 *   out[r][c] (rows x cols) = normal number r*cols + c of the Philox4x64-10
 *   stream keyed by (seed, 0): raw block j = Philox(ctr=(j+1,0,0,0)) gives
 *   normals 4j..4j+3 by Box-Muller in fp64, rounded to fp32.
 * Exported so the stream can be pinned; hg_block_rsvd draws the same numbers
 * internally (block i uses rows [ib,(i+1)b) of the N x k matrix). */
hg_status hg_fill_gaussian(uint64_t seed, int32_t rows, int32_t cols, float* out, hg_stream_t stream);

/* Alg. 1 on each of nb blocks, rank l = k (no oversampling,
 * reading A3), q subspace-iteration passes:
 *   Y0 = X Omega, S0 = qr(Y0); for i = 1..q: S~ = qr(X^T S), S = qr(X S~);
 *   B = S^T X; B = U~ Sigma V^T; U = S U~.
 * X_ii^T = X_ii is assumed (hg_build_theta writes bitwise-symmetric blocks;
 * reading A12) unless flags has HG_GENERAL, which multiplies by the literal X^T in
 * the S~ = qr(X^T S) and B = S^T X steps.  QR is CholeskyQR2; the SVD is one-sided
 * Jacobi started from an eigen-preconditioner for k <= 256.
 *   blocks [nb][b][b]   input blocks (symmetric unless HG_GENERAL)
 *   1 <= k <= min(b, 512); b % 4 == 0 and k % 4 == 0 (16-byte TMA row strides)
 *   Ut, Vt [nb][k][b]   out, U_i^T and V_i^T (HG_UV_BK: U, V [nb][b][k]);
 *   sigma [nb][k] out, non-increasing
 * Device errors: HG_ST_CHOL_BREAKDOWN, HG_ST_JACOBI_CAP, HG_ST_NONFINITE. */
hg_status hg_block_rsvd(const float* blocks, int32_t nb, int32_t b, int32_t k, int32_t q, uint64_t seed,
                        uint32_t flags, float* Ut, float* sigma, float* Vt, int32_t* d_status, void* ws,
                        size_t ws_bytes, hg_stream_t stream);

/* Alg. 1 with oversampling ("l = k + pi"): the
 * factorisation runs at width l = k + p (Omega is the N x l Philox matrix) and the top k
 * singular triplets are returned (rank-k truncation).  p >= 0, p % 4 == 0, l <= min(b, 512);
 * p = 0 is hg_block_rsvd.  Workspace: hg_workspace_size_ex (= hg_workspace_size at k + p).
 * flags: HG_POWER_EQ10 selects the Eq. 10 scheme (only for well-conditioned blocks such as
 * X_ii, cond <= 2: for Theta_ii its (X X^T)^q X Omega exceeds fp32 range of accuracy, as the
 * paper warns, "more sensitive to round-off errors"). */
hg_status hg_block_rsvd_ex(const float* blocks, int32_t nb, int32_t b, int32_t k, int32_t p, int32_t q,
                           uint64_t seed, uint32_t flags, float* Ut, float* sigma, float* Vt, int32_t* d_status,
                           void* ws, size_t ws_bytes, hg_stream_t stream);
hg_status hg_workspace_size_ex(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t k, int32_t p, int32_t T,
                               size_t* bytes);
/* Eq. 3 with Eq. 15 per block:
 *   F_i = scale * V_i diag(1/sigma_i) U_i^T Y_i,   Y_i = rows [ib,(i+1)b) of Y.
 *   Y, F [nb*b][T];  scale = mu/(1+mu) for Eq. 3.
 *   T >= 0 arbitrary (T % 4 != 0: Y and F pass through 16-byte-pitched workspace copies).
 * One fused kernel (c / sigma, both products, the k x T intermediate on chip; 3xF16 with the operand
 * exponents taken from per-block maxima of Y, Ut, Vt) when k <= 256, k % 32 == 0 and b % 32 == 0;
 * otherwise a scale kernel and two 3xTF32 GEMMs.  Either way F matches the FP64 definition to ~2e-6.
 * Device errors: HG_ST_SINGULAR_SIGMA (sigma_j <= 1e-6 sigma_1; reading A14: that triplet is dropped). */
hg_status hg_block_apply_inverse(const float* Ut, const float* sigma, const float* Vt, int32_t nb, int32_t b,
                                 int32_t k, const float* Y, int32_t T, float scale, float* F,
                                 int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream);
/* hg_block_apply_inverse with flags: HG_UV_BK takes U, V [nb][b][k] (hg_block_rsvd with HG_UV_BK);
 * HG_GEMM_SIMT as for hg_gemm. */
hg_status hg_block_apply_inverse_ex(const float* U, const float* sigma, const float* V, int32_t nb, int32_t b,
                                    int32_t k, const float* Y, int32_t T, float scale, float* F, uint32_t flags,
                                    int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream);

/* Reading R2 (the paper calls the X blocks "low-rank", PAPER.md:102,
 * 138, yet X = I - Theta/(1+mu) is full-rank, its low-rank part being Theta): given the
 * rank-k rSVD U Sigma V^T of Theta_ii (hg_build_theta with HG_RAW_THETA, then
 * hg_block_rsvd), the Woodbury identity on X_ii = I - U Sigma U^T/(1+mu) gives
 *   F_i = c (Y_i + U_i diag(sigma_j / ((1+mu) - sigma_j)) U_i^T Y_i),  c = mu/(1+mu)  (Eq. 3).
 *   Ut [nb][k][b] (U_i^T), sigma [nb][k]; Y, F [nb*b][T];  mu > 0.
 * Device errors: HG_ST_SINGULAR_SIGMA if some sigma_j >= 1+mu (impossible for Theta, pin P2). */
hg_status hg_block_apply_woodbury(const float* Ut, const float* sigma, int32_t nb, int32_t b, int32_t k,
                                  const float* Y, int32_t T, float mu, float* F, int32_t* d_status, void* ws,
                                  size_t ws_bytes, hg_stream_t stream);
/* The whole hot path: hg_build_theta -> hg_block_rsvd -> hg_block_apply_inverse
 * with scale = mu/(1+mu); with flags HG_WOODBURY reading R2 instead: Theta_ii blocks ->
 * hg_block_rsvd -> hg_block_apply_woodbury (sigma_out then holds Theta_ii's singular values).
 * sigma_out [N/b][k] may be NULL.  Asynchronous
 * unless flags has HG_SYNC (then the stream is synchronised and a non-zero
 * *d_status returns HG_ERR_NUMERICAL).  d_status may be NULL only with HG_SYNC
 * (a word inside ws is used).
 * Concurrency: after the degrees, disjoint block ranges (HG_STREAMS parts,
 * default 8, at most 8) run their assembly, rSVD and apply on library-owned non-blocking
 * streams forked from and joined back into `stream` with events, so all work
 * is still ordered after prior work on `stream` and before later work (also
 * under stream capture).  The result is bitwise independent of the part count.
 * The whole sequence is captured once per distinct argument set into a CUDA graph
 * (a per-thread cache of 8) and replayed with one cudaGraphLaunch on `stream`; when
 * `stream` is itself capturing, or profiling is on, or HG_NO_GRAPH=1, the kernels
 * are enqueued directly. */
hg_status hg_solve(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q,
                   uint64_t seed, const float* Y, int32_t T, float* F, float* sigma_out, uint32_t flags,
                   int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream);
/* hg_solve with oversampling p (see hg_block_rsvd_ex; the apply uses the top k triplets,
 * sigma_out [N/b][k]); flags may add HG_POWER_EQ10 and HG_WOODBURY.  hg_solve = p = 0. */
hg_status hg_solve_ex(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t p, int32_t q,
                      uint64_t seed, const float* Y, int32_t T, float* F, float* sigma_out, uint32_t flags,
                      int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream);

/* hg_solve restricted to the diagonal blocks [blk_begin, blk_begin + blk_count) -- one rank's
 * share of a problem sharded over GPUs (blocks are independent, so ranks
 * need no collective; the optional exchange is an all-gather of F).  Y and F are the full
 * [N][T] arrays: only the range's rows are read / written.  sigma_out [blk_count][k] or NULL.
 * Results are bitwise those of hg_solve for the same blocks (Omega is keyed by the global
 * block index). */
hg_status hg_solve_blocks(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q,
                          uint64_t seed, int32_t blk_begin, int32_t blk_count, const float* Y, int32_t T, float* F,
                          float* sigma_out, uint32_t flags, int32_t* d_status, void* ws, size_t ws_bytes,
                          hg_stream_t stream);
/* hg_solve from HOST buffers (end-to-end entry): copies row_ptr, col_idx, w, Y
 * host->device, solves, copies F (and sigma_host if non-NULL) device->host,
 * synchronises.  ws (device) is caller-provided as above; host buffers should
 * be pinned for full copy bandwidth.  H and w are uploaded first on `stream`;
 * Y's rows are uploaded per part on a library copy stream and each part waits
 * for its slice only before its apply (the upload overlaps the rSVD); each part
 * downloads its F rows right after its apply.  Returns the device status. */
hg_status hg_solve_host(int32_t N, int32_t E, int64_t nnz, const int64_t* row_ptr_host,
                        const int32_t* col_idx_host, const float* w_host, float mu, int32_t b, int32_t k,
                        int32_t q, uint64_t seed, const float* Y_host, int32_t T, float* F_host,
                        float* sigma_host, uint32_t flags, void* ws, size_t ws_bytes, hg_stream_t stream);

/* ---- The paper's second approach: conjugate gradient on Eq. 5,
 *   X f = theta/(1+theta) y,   X = I - Theta/(1+theta)         (Eq. 1 for Theta)
 * with the iteration of PAPER.md:165-178 (Eqs. 16-20), run independently for each of the T
 * columns of Y:  f_0 = 0, r_0 = p_0 = c y;  alpha_i = r^T r / p^T X p;  f += alpha p;
 * r -= alpha X p;  beta_i = r_i^T r_i / r_{i-1}^T r_{i-1};  p = r + beta p.
 * X is applied matrix-free through H every iteration (never assembled).  Stopping (DESIGN.md
 * reading C2): column t stops once ||r_i|| <= tol ||r_0|| or after max_iter iterations; a zero
 * column takes no iteration (f = 0).  fp32 vectors, fp64 scalars.
 *   Y, F      [N][T] fp32 (device); T % 4 == 0, T >= 1
 *   max_iter  >= 0;  tol >= 0 (0 = run exactly max_iter iterations)
 *   iters     [T] int32 iterations taken per column, may be NULL
 *   rel_res   [T] fp32 ||r||/||r_0|| of the recurrence residual at exit, may be NULL
 *   flags     HG_SYNC as for hg_solve (d_status may then be NULL)
 * Scratch: hg_cg_workspace_size (about 4 vectors of N x T, one of E x T, plus the CSC of H).
 * Graph mode (stream not capturing, HG_NO_GRAPH unset): the whole solve is one cached CUDA
 * graph whose iteration body is a device-driven WHILE node (no host round trip per
 * iteration); otherwise max_iter bodies are enqueued and return at once after convergence.
 * Device errors: HG_ST_ISOLATED_VERTEX, HG_ST_EMPTY_EDGE, HG_ST_CG_BREAKDOWN, HG_ST_NONFINITE. */
hg_status hg_cg_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t T, int32_t max_iter, size_t* bytes);
hg_status hg_cg_solve(const hg_incidence* H, const float* w, float mu, const float* Y, int32_t T, int32_t max_iter,
                      float tol, float* F, int32_t* iters, float* rel_res, uint32_t flags, int32_t* d_status,
                      void* ws, size_t ws_bytes, hg_stream_t stream);
/* ---- NEXT-1: one level of the 2x2 Schur-complement inverse (PAPER.md:127-154,
 * Eqs. 11-14) over super-blocks of two adjacent diagonal blocks (2s, 2s+1), reading S1:
 *   X_s = [[X11, X12], [X21, X22]],  Z1 = X11 - X12 X22^-1 X21,  Z2 = X22 - X21 X11^-1 X12,
 *   X_s^-1 = [[Z1^-1, -X11^-1 X12 Z2^-1], [-Z2^-1 X21 X11^-1, Z2^-1]],   F_s = c X_s^-1 Y_s,
 * with X11^-1, X22^-1, Z1^-1, Z2^-1 "by randomized SVD" in reading R2: each is
 * I - K/(1+mu) with K PSD (K = Theta_ii; K_Z1 = Theta11 + Theta12 X22^-1 Theta21/(1+mu), ...),
 * factored by Alg. 1 (rank k, q passes) and inverted by Woodbury.  Omega for X11 and Z1 is block
 * 2s's rows of the N x k Philox matrix, for X22 and Z2 block 2s+1's (reading S3).
 *   N % 2b == 0; other sizes as hg_solve; Y, F [N][T]; flags HG_SYNC.
 * Workspace: hg_schur_workspace_size.  Device errors as hg_solve. */
hg_status hg_schur_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t k, int32_t T,
                                  size_t* bytes);
hg_status hg_solve_schur(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t k, int32_t q,
                         uint64_t seed, const float* Y, int32_t T, float* F, uint32_t flags, int32_t* d_status,
                         void* ws, size_t ws_bytes, hg_stream_t stream);
/* ---- NEXT-1: the nested tessellation ("nested tessellations of
 * submatrices created along the main diagonal"), reading S4: Eq. 12 applied recursively inside super-
 * blocks of m = 2^levels b vertices down to b x b leaves.  A node of n = 2^l b vertices (l >= 1) takes
 * its halves' inverses A11, A22 from the level below, Theta12 between its halves, the Schur complements
 *   K_Z1 = Theta11 + Theta12 A22 Theta21/(1+mu),  K_Z2 = Theta22 + Theta21 A11 Theta12/(1+mu)
 * (Eqs. 13-14, X = I - Theta/(1+mu)), inverts Z1 = I - K_Z1/(1+mu), Z2 likewise by Alg. 1 at rank
 * k_l = k 2^(l-1) + Woodbury (reading R2; Omega = the halves' rows of the N x k_l Philox matrix), and
 * materialises its inverse [[Z1^-1, A11 Theta12 Z2^-1/(1+mu)], [(.)^T, Z2^-1]] (Eq. 12); leaves by
 * Alg. 1 on Theta_ii at rank k.  F_s = mu/(1+mu) A_s^-1 Y_s (Eq. 3).  levels = 1 is hg_solve_schur's
 * one-level scheme; k = b makes every inverse exact (the super-block solve).
 *   1 <= levels <= 6, N % (2^levels b) == 0, 1 <= k <= b, k 2^(levels-1) <= 512, T % 4 == 0.
 *   Workspace: hg_nested_workspace_size (dense node matrices: ~4 N 2^levels b floats).  flags: HG_SYNC. */
hg_status hg_nested_workspace_size(int32_t N, int32_t E, int64_t nnz, int32_t b, int32_t levels, int32_t k, int32_t T,
                                   size_t* bytes);
hg_status hg_solve_nested(const hg_incidence* H, const float* w, float mu, int32_t b, int32_t levels, int32_t k,
                          int32_t q, uint64_t seed, const float* Y, int32_t T, float* F, uint32_t flags,
                          int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream);
/* ---- NEXT-4: the hyperedge-weight update with f fixed.
 * P(w) = sum_t f_t^T L f_t + kappa ||w||^2, L = I - Theta(w) (reading N1: the T columns of F are
 * summed).  hg_weight_gradient: the frozen-degree gradient (D_v, D_e held at the current w)
 *   grad_e = -(1/delta(e)) sum_t (sum_{v in e} f_t[v] / sqrt(delta(v)))^2 + 2 kappa w_e
 *   H, w as for hg_solve; F [N][T] (T % 4 == 0); grad [E] out.
 *   Workspace: hg_cg_workspace_size(N, E, nnz, T, 0) (the CSC of H is rebuilt per call).
 * hg_weight_step: one steepest-descent step w <- w - mu g on the simplex 1^T w = 1, w >= 0
 * (reading N2): g made mean-free over the free coordinates and zero on clamped ones
 * (active[e] = 1), then negative free coordinates are clamped to 0 (joining the active set)
 * and the excess mass removed evenly from the remaining free ones, until none is negative.
 *   w [E] fp32 in/out, active [E] int32 in/out, grad [E].  One CTA; fp64 reductions.
 * Device errors: HG_ST_SIMPLEX_DEGENERATE (every coordinate clamped). */
hg_status hg_weight_gradient(const hg_incidence* H, const float* w, const float* F, int32_t T, float kappa,
                             float* grad, int32_t* d_status, void* ws, size_t ws_bytes, hg_stream_t stream);
hg_status hg_weight_step(int32_t E, float* w, int32_t* active, const float* grad, float mu, int32_t* d_status,
                         hg_stream_t stream);
/* Projection of a starting weight vector onto the simplex's affine hull, w_out = w / (1^T w), the start
 * of the constrained iteration of PAPER.md:50-52 (1^T w = 1, w >= 0).  w, w_out [E] (may alias).  One
 * CTA, fixed-order fp64 sum.  Device errors: HG_ST_SIMPLEX_DEGENERATE (a negative or non-finite w_e, or
 * 1^T w <= 0; w_out = w then). */
hg_status hg_weight_normalize(int32_t E, const float* w, float* w_out, int32_t* d_status, hg_stream_t stream);
/* The objective P(w) = sum_t f_t^T L f_t + kappa ||w||^2 at the w the gradient was taken at (degrees
 * from w): since P is linear in w at fixed degrees apart from the penalty,
 *   P(w) = ||F||^2 + w^T grad(w) - kappa ||w||^2   (grad from hg_weight_gradient at the same w).
 *   F [N][T]; out: one fp64 (device); ws: >= 296 doubles of device scratch.  Fixed-order sums. */
hg_status hg_weight_objective(const float* F, int32_t N, int32_t T, int32_t E, const float* w, const float* grad,
                              float kappa, double* out, void* ws, size_t ws_bytes, hg_stream_t stream);
/* Verification export of the batched GEMM the path runs on (3xTF32 on
 * tcgen05, or fp32 CUDA cores with HG_GEMM_SIMT):
 *   for g < batch: D_g(m,n) = alpha * rs_g[m] * cs_g[n] * sum_kk A_g(m,kk) B_g(kk,n)
 *   A_g(m,kk) = A[g*sa + (a_mn ? kk*lda + m : m*lda + kk)]
 *   B_g(kk,n) = B[g*sb + (b_mn ? kk*ldb + n : n*ldb + kk)]
 *   d_trans ? D[g*sd + n*ldd + m] : D[g*sd + m*ldd + n]
 *   rs/cs may be NULL (= 1), with batch strides srs/scs. */
hg_status hg_gemm(int32_t M, int32_t N, int32_t K, int32_t batch, const float* A, int32_t a_mn, int64_t lda,
                  int64_t sa, const float* B, int32_t b_mn, int64_t ldb, int64_t sb, float* D, int32_t d_trans,
                  int64_t ldd, int64_t sd, float alpha, const float* rs, int64_t srs, const float* cs,
                  int64_t scs, uint32_t flags, hg_stream_t stream);
/* hg_gemm with an explicit precision: prec -1 = the process default (HG_GEMM_PREC env, 3xTF32
 * unless "f16"), 0 = 3xTF32, 1 = 3xF16 -- each operand x is split as hi = fp16_rn(2^e x),
 * lo = fp16_rn(2^e x - hi) with e = a_exp for A, b_exp for B (the result is rescaled by
 * 2^-(a_exp + b_exp)); the caller picks e so that 2^e max|x| < 65504 (|e| <= 40), else
 * the fp16 hi part overflows to inf.  Same layouts and flags as hg_gemm. */
hg_status hg_gemm_ex(int32_t M, int32_t N, int32_t K, int32_t batch, const float* A, int32_t a_mn, int64_t lda,
                     int64_t sa, const float* B, int32_t b_mn, int64_t ldb, int64_t sb, float* D, int32_t d_trans,
                     int64_t ldd, int64_t sd, float alpha, const float* rs, int64_t srs, const float* cs,
                     int64_t scs, uint32_t flags, int32_t prec, int32_t a_exp, int32_t b_exp, hg_stream_t stream);

/* Verification exports of the 3xF16 twin-operand path.  hg_f16_split: out16 = the twin of the dense
 * rows x cols fp32 matrix x (row pitch ld; cols % 32 == 0): element o = r*cols + c has its hi half
 * fp16_rn(2^exp x) at out16[2 o - (o % 32)] and its lo half fp16_rn(2^exp x - hi) 32 entries further
 * (fp16 bit patterns; out16 holds 2 rows cols entries) -- per 32 elements the 32 hi then the 32 lo, so a
 * 64 x R TMA box lands as the tensor core's 128-byte operand rows.
 * hg_gemm_f16pre: D = alpha 2^-(a_exp + b_exp) A B with both operands given as twins of the K-major
 * arrays A[g*sa + m*lda + kk], B[g*sb + n*ldb + kk]; lda, ldb, sa, sb multiples of 32. */
hg_status hg_f16_split(const float* x, int64_t rows, int32_t cols, int64_t ld, int32_t exp, uint16_t* out16,
                       hg_stream_t stream);
hg_status hg_gemm_f16pre(int32_t M, int32_t N, int32_t K, int32_t batch, const uint16_t* A16, int64_t lda,
                         int64_t sa, int32_t a_exp, const uint16_t* B16, int64_t ldb, int64_t sb, int32_t b_exp,
                         float* D, int32_t d_trans, int64_t ldd, int64_t sd, float alpha, hg_stream_t stream);

/* Stage profiler (tracing).  hg_profile_enable(1) makes the calls on this host
 * thread bracket each stage launch with CUDA events on its stream (off by
 * default).  hg_profile_collect synchronises those events, writes per-stage
 * totals -- names[i] (32-byte NUL-terminated slots), ms[i] summed elapsed time,
 * counts[i] launches -- for up to max_stages stages, sets *n_out to the number
 * of stages seen, and clears the record.  Stages: degrees, assemble, omega,
 * gemm_power, gemm_gram, gemm_qform, gemm_svd, gemm_apply, cholinv, jacobi,
 * finalize, inv_sigma.  Host pointers. */
hg_status hg_profile_enable(int32_t on);
hg_status hg_profile_collect(int32_t max_stages, char* names, double* ms, int32_t* counts, int32_t* n_out);

/* Timeline mode: hg_profile_enable(2) keeps hg_solve's stream parts concurrent
 * (mode 1 runs them in sequence so per-stage totals do not overlap) and
 * records, per stage launch group, its part and start / end in ms from the
 * start of the first hg_solve since the last collect.  hg_profile_timeline
 * writes up to max_rec records (stage ids in the order listed above), sets
 * *n_out to the number recorded and clears the record.  Host pointers. */
hg_status hg_profile_timeline(int32_t max_rec, int32_t* stage, int32_t* part, double* t_start_ms, double* t_end_ms,
                              int32_t* n_out);

/* Diagnostics (device-wide counters since the last reset; synchronous):
 * out[0] near-identity CholeskyQR factorizations, out[1] full ones,
 * out[2] max Jacobi sweeps of any block, out[3] total sweeps, out[4] blocks;
 * with n >= 69, out[5..68] are clock64 phase stamps of the last full Cholesky;
 * with n >= 85, out[69..84] block-Jacobi outer-round stamps; with n >= 133,
 * out[85..132] block-Jacobi inner-round stamps (a reset call enables them). */
hg_status hg_debug_counters(int64_t* out, int32_t n, int32_t reset);

/* Debug, only meaningful in a build with -DHG_JB_SWEEPMAX (else the values stay 0):
 * out == NULL clears the per-sweep maxima and switches recording on (on != 0) or off;
 * else copies them out: out[64 * 40] floats, slot (blk, sweep) = largest
 * a_pq^2 / (a_pp a_qq) that block slot blk (blockIdx within a launch) saw in that
 * sweep of the block Jacobi (stopping rule).  Returns a cudaError_t value. */
int hg_debug_jacobi_sweepmax(float* out, int on);

/* Number of kernels the last hg_* call on this host thread enqueued. */
int32_t hg_last_launch_count(void);

/* Message for the last failing call on this host thread ("" if none). */
const char* hg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HG_H_ */
