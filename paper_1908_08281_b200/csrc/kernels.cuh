// kernels.cuh -- launchers for the non-GEMM kernels of the path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// theta.cu -- PAPER.md:30-40 (degrees, Eq. 1, X = I - Theta/(1+mu))
cudaError_t launch_degrees(int N, int E, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                           int32_t* de_cnt, float* edge_val, float* dv_rsqrt, int32_t* status,
                           cudaStream_t s, int* launches);
cudaError_t launch_assemble(int blk0, int nb, int nb_total, int b, int E, int64_t nnz, const int64_t* row_ptr,
                            const int32_t* col_idx, const float* edge_val, const float* dv_rsqrt, float mu,
                            bool raw_theta, float* blocks, void* keys_ws, cudaStream_t s, int* launches,
                            uint16_t* x16 = nullptr, bool skip_f32 = false);
// (x16: also write the 3xF16 twin of the blocks, 2^14 X in the tw_off layout of common.cuh;
//  skip_f32: the fp32 blocks are not needed (written anyway on the fallback paths))
size_t assemble_keys_bytes(int64_t nnz, int nb, int E);
// grouped assembly (default when nb * E is small enough): degrees and the (block, edge) grouping of the
// incidences of all nb_total blocks once per solve (instead of launch_degrees), before launch_assemble
bool assemble_grouped(int nb, int E);
cudaError_t launch_degrees_grouped(int nb_total, int b, int E, int64_t nnz, const int64_t* row_ptr,
                                   const int32_t* col_idx, const float* w, int32_t* de_cnt, float* edge_val,
                                   float* dv_rsqrt, int32_t* status, void* keys_ws, cudaStream_t s, int* launches);

// philox.cu -- Alg. 1 step 1, reading A6
// panel: out[i][c][m] = Omega[i*b + m][c] (Omega is N x k, normal index r*k + c)
cudaError_t launch_omega_panels(uint64_t seed, int blk0, int nb, int b, int k, float* out, cudaStream_t s,
                                int* launches,
                                uint16_t* out16 = nullptr, int exp = 0);
// (out16: write only the 3xF16 twin of 2^exp Omega (common.cuh tw_off layout) -- not out)
// row-major rows x cols: out[r][c] = normal r*cols + c
cudaError_t launch_gaussian_rowmajor(uint64_t seed, int rows, int cols, float* out, cudaStream_t s,
                                     int* launches);

// chol.cu -- CholeskyQR: G = L L^T (lower L), Linv = L^-1 (skipped when Linv is null);
// near-identity first-order path
cudaError_t launch_cholinv(int nb, int k, const float* G, float* L, float* Linv, float* work,
                           int32_t* status, cudaStream_t s, int* launches);

// jacobi.cu -- one-sided Jacobi on W = L (or L^T, see jacobi_on_l): W_f = W J with orthogonal columns
cudaError_t launch_jacobi(int nb, int k, const float* L, float* Wf, int32_t* status, cudaStream_t s,
                          int* launches);

// finalize.cu -- sigma_j = ||V_w column j|| (fp64), sort, normalise, sign rule
cudaError_t launch_finalize(int nb, int b, int k, const float* Vw_t, const float* Uw_t, float* Ut, float* sigma,
                            float* Vt, double* sig_raw, int32_t* perm, int32_t* status, cudaStream_t s,
                            int* launches, bool uv_bk = false, uint16_t* u16 = nullptr, float* vs_out = nullptr);
// (u16: instead of Ut / Vt write U's 3xF16 twin (exponent 14, b % 32 == 0) and vs_out[i][j] = sign_j / sigma_j,
//  the scale of v_j = vs B^T u~_j -- the fused apply's inputs, launch_apply_prep with perm / vs)
// apply prep: rs[i][j] = scale / sigma[i][j]; flags singular sigma
// (sigma, rs are [nb][ld]; the first k per block are used, the rest of rs is zeroed)
cudaError_t launch_inv_sigma(int nb, int k, int ld, const float* sigma, float scale, float* rs, int32_t* status,
                             cudaStream_t s, int* launches);

// apply.cu -- the fused Eq. 15 apply: prep (exponent words, U / V twins) + one kernel
bool apply_fused_supported(int b, int k, int ldk, int T, const void* Ut, const void* Vt, const void* Y, const void* F);
size_t apply_fused_amax_bytes(int nb);
cudaError_t launch_apply_prep(const float* Ut, const float* Vt, int nb, int b, int k, int ldk, const float* Y, int T,
                              uint16_t* u16, uint16_t* v16, uint32_t* amax, int amax_ld, bool uv_unit,
                              cudaStream_t s, int* launches, const int32_t* perm = nullptr, const float* vs = nullptr);
// (perm / vs given: u16 is already written (launch_finalize), Ut is unused and Vt is the unsorted,
//  unnormalised Vw_t [nb][k][b]: V's twin takes row perm[j] scaled by vs[j])
cudaError_t launch_apply_fused(const float* sigma, int nb, int b, int k, int ldk, const float* Y, int T, float scale,
                               float* F, int32_t* status, const uint16_t* u16, const uint16_t* v16,
                               const uint32_t* amax, int amax_ld, cudaStream_t s, int* launches);

// reading R2: rs[i][j] = c sigma_ij / ((1+mu) - sigma_ij)  (Woodbury weights)
cudaError_t launch_woodbury_scale(int nb, int k, int ld, const float* sigma, float c, float one_plus_mu, float* rs,
                                  int32_t* status, cudaStream_t s, int* launches);

// debug counters (device globals): chol {near-identity, full}; jacobi {max sweeps, total sweeps, blocks}
cudaError_t chol_debug(unsigned long long* out, bool reset);
cudaError_t jacobi_debug(unsigned long long* out, bool reset);
cudaError_t chol_clocks(long long* out);
cudaError_t jacobi_clocks(long long* out);
cudaError_t launch_jacobi_blk(int nb, int k, const float* L, float* Wf, int32_t* status, cudaStream_t s,
                              int* launches);
cudaError_t jacobi_blk_debug(unsigned long long* out, bool reset);
// rows per cluster CTA for the next block-Jacobi launches of this thread (0: default)
void jacobi_rows_hint(int rows);
cudaError_t jacobi_blk_clocks(long long* out);

// true when launch_jacobi orthogonalises the columns of L (then U~ = unit columns of W_f)
bool jacobi_on_l();
// Uk[blk][j][r] = W_f[blk][r][j] / ||W_f[blk][:, j]||  (fp64 norms; zero columns stay zero)
cudaError_t launch_unit_columns_t(int nb, int k, const float* Wf, float* Uk, cudaStream_t s, int* launches);
// debug: inner-round clock stamps of the block Jacobi (enable != 0 switches them on; out may be NULL)
cudaError_t jacobi_blk_inner_clocks(long long* out, int enable);


// cg.cu -- the second approach: CG on Eq. 5, matrix-free through H
struct CgArgs {
  int N, E;
  int64_t nnz;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const float* w;
  float mu;
  const float* Y;      // [N][T]
  int T;
  int max_iter;
  float tol;
  float* F;            // [N][T]
  int32_t* iters_out;  // [T] or null
  float* rel_out;      // [T] or null
  int32_t* status;
  void* ws;
};
struct CgLayout {
  int TS, ns, nparts;
  int64_t max_items, max_big;
  size_t de, eval, dvr, col_ptr, item_ptr, slot_ptr, big_ptr, cursor, totals, csc_tmp, csc, items, bigs;
  size_t P, R, F, XP, sqpart, Q, part, red, rr, rr0, alpha, beta, active, iters, ctl, status, total;
};
// Graph mode: begin() creates the WHILE node's handle in the graph being captured; open_body()
// adds the conditional node after the captured work so far and returns a stream capturing into
// its body graph; close_body() ends that capture.
struct CgGraphHook {
  void* ctx;
  cudaError_t (*begin)(void* ctx, cudaGraphConditionalHandle* h);
  cudaError_t (*open_body)(void* ctx, cudaGraphConditionalHandle h, cudaStream_t* body_stream);
  cudaError_t (*close_body)(void* ctx);
};
int cg_lanes(int T);
CgLayout cg_layout(int64_t N, int64_t E, int64_t nnz, int64_t T, int64_t max_iter);
cudaError_t launch_cg(const CgArgs& a, const CgGraphHook* hook, cudaStream_t s, int* launches);
// NEXT-4: frozen-degree gradient (a.F = F [N][T] read-only, a.ws a CG
// workspace of hg_cg_workspace_size(N, E, nnz, T, 0)) and one simplex step
cudaError_t launch_weight_gradient(const CgArgs& a, float kappa, float* grad, cudaStream_t s, int* launches);
cudaError_t launch_weight_step(int E, float* w, int32_t* active, const float* grad, float mu, int32_t* status,
                               cudaStream_t s, int* launches);
cudaError_t launch_weight_normalize(int E, const float* w, float* wo, int32_t* status, cudaStream_t s,
                                    int* launches);

// schur.cu -- NEXT-1: the non-GEMM pieces of one Eq. 12 level
cudaError_t launch_theta_offblock(int ns, int b, const int64_t* row_ptr, const int32_t* col, const int32_t* col_ptr,
                                  const int32_t* csc, const float* eval, const float* dvr, float* out, cudaStream_t s,
                                  int* launches);
cudaError_t launch_scale_rows(int nb, int k, int b, const float* d, const float* Ut, float* Wt, cudaStream_t s,
                              int* launches);
cudaError_t launch_add_identity(int nb, int b, float* A, cudaStream_t s, int* launches);
cudaError_t launch_symmetrize(int nb, int b, float* K, cudaStream_t s, int* launches);
// nested tessellation: out[s] (2h x 2h) = [[TL[s], TR[s]], [TR[s]^T, BR[s]]] (batch strides sTL, sBR, sTR)
cudaError_t launch_place_node(int nn, int h, const float* TL, int64_t sTL, const float* BR, int64_t sBR, const float* TR,
                              int64_t sTR, float* out, cudaStream_t s, int* launches);
cudaError_t launch_axpby(int ns, int64_t len, float c, float g, const float* P, int64_t pp, const float* Q, int64_t pq,
                         float* F, int64_t pf, cudaStream_t s, int* launches);
// cg.cu: degrees + the sorted CSC of H (for the off-diagonal assembly); a.ws is a CG workspace
cudaError_t launch_csc_setup(const CgArgs& a, cudaStream_t s, int* launches);
cudaError_t launch_weight_objective(int64_t nF, const float* F, int E, const float* w, const float* grad, float kappa,
                                    double* part, double* out, cudaStream_t s, int* launches);

// eig.cu -- eigen-preconditioner of the Jacobi (k <= 512): from A = L^T L [nb][k][k] (lower triangle
// read): Q^T A Q = T tridiagonal (Hv: Householder vectors, [nb][k][k]), Z [nb][k][k] column i = the
// (unnormalised) eigenvector of T for its i-th smallest eigenvalue, *scale -> [nb][k] its 1/norm, and
// Qt [nb][k][k] = Q^T.  The approximate eigenvectors of A are the columns of Q Z diag(scale).
// scratch: eig_scratch_floats(k) floats per block (16-byte aligned).
bool eig_precond_supported(int k);
size_t eig_scratch_floats(int k);
cudaError_t launch_eig_precond(int nb, int k, const float* A, float* Hv, float* Z, float* scratch, float* Qt,
                               const float** scale, cudaStream_t s, int* launches);
