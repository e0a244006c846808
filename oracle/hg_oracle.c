/*
 * hg_oracle.c -- plain, slow, FP64 CPU oracle for the block randomized SVD hot
 * path of arXiv:1908.08281 ("Block randomized SVD and conjugate gradient for
 * adaptive hypergraph learning").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_1908_08281_b200/csrc); neither side includes the other.
 *
 * Every function follows the paper's definitions in the paper's order, in
 * double precision, with plain loops (no blocking, no fusion):
 *   or_degrees          PAPER.md:30      delta(v) = sum_e w(e) H(v,e), delta(e) = sum_v H(v,e)
 *   or_theta_block      PAPER.md:32-34   Eq. 1, Theta = Dv^-1/2 H W De^-1 H^T Dv^-1/2 (diagonal block)
 *                       PAPER.md:40      X = I - Theta/(1+theta)
 *   or_philox4x64_10 /  PAPER.md:111-113 Alg. 1 step 1, iid N(0,1) Omega; reading A6
 *   or_gaussian_f32                      (Philox4x64-10 + Box-Muller, rounded to fp32)
 *   or_qr_householder   PAPER.md:114-117 "compute its QR factorization" (Householder, diag(R) >= 0)
 *   or_svd_gkr          PAPER.md:122     Alg. 1 step 5, SVD of B (Golub-Kahan-Reinsch)
 *   or_rsvd_block       PAPER.md:108-124 Alg. 1 (literal X^T in the loop), Eq. 7 residual
 *   or_apply_block      PAPER.md:43-45,160-163  Eq. 3 with Eq. 15: f = c V Sigma^-1 U^T y
 *   or_apply_woodbury   SURVEY.md §8(f) NEXT-3 reading R2: X_ii^-1 ~ I + U diag(s/((1+theta)-s)) U^T from
 *                       the rank-k rSVD U S V^T of Theta_ii (Woodbury identity on X = I - Theta/(1+theta),
 *                       PAPER.md:40; Alg. 1 applied to the PSD low-rank part)
 *   or_solve            the whole path over a chosen subset of diagonal blocks (mode 0: reading R1,
 *                       Alg. 1 on X_ii + Eq. 15; mode 1: reading R2, Alg. 1 on Theta_ii + Woodbury)
 *   or_theta_offblock   PAPER.md:32-34   Eq. 1 off-diagonal block Theta_ij (rows of block i, columns of block j)
 *   or_lowrank_inverse  NEXT-3 reading R2: (I - K/(1+theta))^-1 ~ I + U diag(s/((1+theta)-s)) U^T, Alg. 1 on K
 *   or_solve_schur      PAPER.md:127-154 Eqs. 11-14 (NEXT-1): one 2x2 Schur level over pairs of adjacent
 *                       diagonal blocks, X11^-1, X22^-1, Z1^-1, Z2^-1 by rSVD (reading R2)
 *   or_solve_nested     PAPER.md:155-156 (NEXT-1): the nested tessellation, Eq. 12 recursively inside
 *                       super-blocks of 2^L b vertices, leaves and Schur complements by reading R2
 *   or_weight_objective PAPER.md:46-52   P(w) = sum_t f_t^T L f_t + kappa ||w||^2, L = I - Theta(w) (NEXT-4)
 *   or_weight_gradient  PAPER.md:56-58   frozen-degree gradient of P (SPEC.md gradient_frozen)
 *   or_weight_step      PAPER.md:54-58   w <- w - mu grad on the simplex, clamped coordinates stay 0
 *   or_apply_X          PAPER.md:30-40   X p = p - (1/(1+theta)) Dv^-1/2 H W De^-1 H^T Dv^-1/2 p (matrix-free)
 *   or_cg_solve         PAPER.md:165-178 the paper's second approach: CG on Eq. 5, X f = theta/(1+theta) y
 *                                        (Eqs. 16-20), one independent CG per right-hand-side column
 *
 * Pinned by tests/test_oracle_*.py against closed forms, library routines,
 * brute force and invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_INVALID 2
#define OR_ERR_NUMERICAL 3

static void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    strncpy(err, msg, (size_t)errlen - 1);
    err[errlen - 1] = '\0';
  }
}

/* ------------------------------------------------------------------------ */
/* Philox4x64-10 (Salmon, Moraes, Dror, Shaw, SC'11), counter-based RNG.      */
/* ------------------------------------------------------------------------ */
static void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

void or_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
  uint64_t x0 = ctr_in[0], x1 = ctr_in[1], x2 = ctr_in[2], x3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(M0, x0, &hi0, &lo0);
    mulhilo64(M1, x2, &hi1, &lo1);
    uint64_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* Raw block j (0-based) = Philox(counter = (j+1, 0, 0, 0), key = (seed, 0)). */
void or_philox_raw(uint64_t seed, int64_t first_block, int64_t n_blocks, uint64_t* out) {
  uint64_t key[2] = {seed, 0};
  for (int64_t j = 0; j < n_blocks; ++j) {
    uint64_t ctr[4] = {(uint64_t)(first_block + j + 1), 0, 0, 0};
    or_philox4x64_10(ctr, key, out + 4 * j);
  }
}

/* Normals with global index [start, start+n): block j = idx/4 yields 4 normals via
 * Box-Muller on (x0,x1) and (x2,x3): u = ((x >> 11) + 0.5) * 2^-53,
 * z_{2i} = sqrt(-2 ln u_{2i}) cos(2 pi u_{2i+1}), z_{2i+1} = sqrt(-2 ln u_{2i}) sin(2 pi u_{2i+1});
 * computed in fp64 and rounded to fp32. */
void or_gaussian_f32(uint64_t seed, int64_t start, int64_t n, float* out) {
  const double two_pi = 6.283185307179586476925286766559;
  const double inv53 = 1.0 / 9007199254740992.0; /* 2^-53 */
  uint64_t key[2] = {seed, 0};
  int64_t cached = -1;
  double z[4] = {0, 0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    int64_t idx = start + i;
    int64_t blk = idx / 4;
    if (blk != cached) {
      uint64_t ctr[4] = {(uint64_t)(blk + 1), 0, 0, 0}, x[4];
      or_philox4x64_10(ctr, key, x);
      for (int p = 0; p < 2; ++p) {
        double u0 = ((double)(x[2 * p] >> 11) + 0.5) * inv53;
        double u1 = ((double)(x[2 * p + 1] >> 11) + 0.5) * inv53;
        double r = sqrt(-2.0 * log(u0));
        z[2 * p] = r * cos(two_pi * u1);
        z[2 * p + 1] = r * sin(two_pi * u1);
      }
      cached = blk;
    }
    out[i] = (float)z[idx % 4];
  }
}

/* ------------------------------------------------------------------------ */
/* Eq. 1 and X                                              */
/* ------------------------------------------------------------------------ */
/* delta(e) = sum_v H(v,e);  delta(v) = sum_e w(e) H(v,e).
 * Returns OR_ERR_NUMERICAL on an empty hyperedge or an isolated vertex. */
int or_degrees(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx,
               const float* w, double* dv, double* de, char* err, int errlen) {
  for (int32_t e = 0; e < E; ++e) de[e] = 0.0;
  for (int32_t v = 0; v < N; ++v) {
    double s = 0.0;
    for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
      int32_t e = col_idx[p];
      if (e < 0 || e >= E) { set_err(err, errlen, "hyperedge index out of range"); return OR_ERR_INVALID; }
      de[e] += 1.0;
      s += (double)w[e];
    }
    dv[v] = s;
  }
  for (int32_t e = 0; e < E; ++e)
    if (de[e] == 0.0) {
      char m[96]; snprintf(m, sizeof m, "empty hyperedge %d (delta(e)=0)", e);
      set_err(err, errlen, m); return OR_ERR_NUMERICAL;
    }
  for (int32_t v = 0; v < N; ++v)
    if (!(dv[v] > 0.0)) {
      char m[96]; snprintf(m, sizeof m, "isolated vertex %d (delta(v)=0)", v);
      set_err(err, errlen, m); return OR_ERR_NUMERICAL;
    }
  return OR_OK;
}

/* Theta_ii[u][v] = dv_u^-1/2 dv_v^-1/2 sum_e H(u,e) w(e)/delta(e) H(v,e), u,v in block i.
 * If mu > 0 the block of X = I - Theta/(1+mu) is written instead. */
void or_theta_block(int32_t b, int32_t blk, const int64_t* row_ptr, const int32_t* col_idx,
                    const float* w, const double* dv, const double* de, double mu, double* out) {
  int64_t base = (int64_t)blk * b;
  for (int32_t u = 0; u < b; ++u) {
    for (int32_t v = 0; v < b; ++v) {
      int64_t pu = row_ptr[base + u], eu = row_ptr[base + u + 1];
      int64_t pv = row_ptr[base + v], ev = row_ptr[base + v + 1];
      double s = 0.0;
      while (pu < eu && pv < ev) { /* common hyperedges of u and v (sorted rows) */
        if (col_idx[pu] < col_idx[pv]) ++pu;
        else if (col_idx[pu] > col_idx[pv]) ++pv;
        else { int32_t e = col_idx[pu]; s += (double)w[e] / de[e]; ++pu; ++pv; }
      }
      double th = s / sqrt(dv[base + u]) / sqrt(dv[base + v]);
      out[(int64_t)u * b + v] = (mu > 0.0) ? ((u == v ? 1.0 : 0.0) - th / (1.0 + mu)) : th;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Dense helpers (row-major)                                                  */
/* ------------------------------------------------------------------------ */
/* C (m x n) = A (m x p) * B (p x n) */
static void mm(int m, int p, int n, const double* A, const double* B, double* C) {
  for (int i = 0; i < m; ++i) {
    double* c = C + (int64_t)i * n;
    for (int j = 0; j < n; ++j) c[j] = 0.0;
    for (int t = 0; t < p; ++t) {
      double a = A[(int64_t)i * p + t];
      const double* bb = B + (int64_t)t * n;
      for (int j = 0; j < n; ++j) c[j] += a * bb[j];
    }
  }
}
/* C (m x n) = A^T * B, A (p x m), B (p x n) */
static void mtm(int m, int p, int n, const double* A, const double* B, double* C) {
  for (int i = 0; i < m * n; ++i) C[i] = 0.0;
  for (int t = 0; t < p; ++t) {
    const double* a = A + (int64_t)t * m;
    const double* bb = B + (int64_t)t * n;
    for (int i = 0; i < m; ++i) {
      double ai = a[i];
      double* c = C + (int64_t)i * n;
      for (int j = 0; j < n; ++j) c[j] += ai * bb[j];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Householder thin QR (Golub & Van Loan, Alg. 5.2.1), m >= n.                */
/* A = Q R, Q m x n orthonormal columns, R n x n upper triangular, diag >= 0. */
/* ------------------------------------------------------------------------ */
void or_qr_householder(int32_t m, int32_t n, const double* A, double* Q, double* R) {
  double* W = (double*)malloc(sizeof(double) * (size_t)m * n);   /* working copy */
  double* V = (double*)malloc(sizeof(double) * (size_t)m * n);   /* Householder vectors, column j */
  double* beta = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(W, A, sizeof(double) * (size_t)m * n);
  for (int j = 0; j < n; ++j) {
    /* v = house(W[j:m, j]) : x - alpha e1 with alpha = -sign(x0) ||x|| */
    double nrm = 0.0;
    for (int i = j; i < m; ++i) nrm += W[(int64_t)i * n + j] * W[(int64_t)i * n + j];
    nrm = sqrt(nrm);
    double x0 = W[(int64_t)j * n + j];
    double alpha = (x0 >= 0.0) ? -nrm : nrm;
    for (int i = 0; i < m; ++i) V[(int64_t)i * n + j] = 0.0;
    if (nrm == 0.0) { beta[j] = 0.0; continue; }
    V[(int64_t)j * n + j] = x0 - alpha;
    for (int i = j + 1; i < m; ++i) V[(int64_t)i * n + j] = W[(int64_t)i * n + j];
    double vtv = 0.0;
    for (int i = j; i < m; ++i) vtv += V[(int64_t)i * n + j] * V[(int64_t)i * n + j];
    beta[j] = (vtv > 0.0) ? 2.0 / vtv : 0.0;
    /* W[j:m, j:n] -= beta v (v^T W[j:m, j:n]) */
    for (int c = j; c < n; ++c) {
      double s = 0.0;
      for (int i = j; i < m; ++i) s += V[(int64_t)i * n + j] * W[(int64_t)i * n + c];
      s *= beta[j];
      for (int i = j; i < m; ++i) W[(int64_t)i * n + c] -= s * V[(int64_t)i * n + j];
    }
    W[(int64_t)j * n + j] = alpha;
    for (int i = j + 1; i < m; ++i) W[(int64_t)i * n + j] = 0.0;
  }
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < n; ++c) R[(int64_t)i * n + c] = (c >= i) ? W[(int64_t)i * n + c] : 0.0;
  /* Q = H_0 H_1 ... H_{n-1} [I_n; 0], accumulated backward */
  for (int i = 0; i < m; ++i)
    for (int c = 0; c < n; ++c) Q[(int64_t)i * n + c] = (i == c) ? 1.0 : 0.0;
  for (int j = n - 1; j >= 0; --j) {
    if (beta[j] == 0.0) continue;
    for (int c = 0; c < n; ++c) {
      double s = 0.0;
      for (int i = j; i < m; ++i) s += V[(int64_t)i * n + j] * Q[(int64_t)i * n + c];
      s *= beta[j];
      for (int i = j; i < m; ++i) Q[(int64_t)i * n + c] -= s * V[(int64_t)i * n + j];
    }
  }
  /* sign convention: diag(R) >= 0 (flip row of R and column of Q) */
  for (int j = 0; j < n; ++j)
    if (R[(int64_t)j * n + j] < 0.0) {
      for (int c = 0; c < n; ++c) R[(int64_t)j * n + c] = -R[(int64_t)j * n + c];
      for (int i = 0; i < m; ++i) Q[(int64_t)i * n + j] = -Q[(int64_t)i * n + j];
    }
  free(W); free(V); free(beta);
}

/* ------------------------------------------------------------------------ */
/* Golub-Kahan-Reinsch SVD of a square n x n matrix (Golub & Van Loan,        */
/* Alg. 8.6.1 / 8.6.2): Householder bidiagonalisation, then implicit-shift    */
/* QR sweeps on the bidiagonal with zero-diagonal chasing.                    */
/* A = U diag(s) V^T, s >= 0 non-increasing.  Returns 0 or OR_ERR_NUMERICAL.  */
/* ------------------------------------------------------------------------ */
/* R(p,q,c,s): identity with [p][p]=c [p][q]=s [q][p]=-s [q][q]=c */
static void rot_cols(double* M, int rows, int ld, int p, int q, double c, double s) {
  for (int i = 0; i < rows; ++i) {               /* M <- M R */
    double a = M[(int64_t)i * ld + p], b = M[(int64_t)i * ld + q];
    M[(int64_t)i * ld + p] = c * a - s * b;
    M[(int64_t)i * ld + q] = s * a + c * b;
  }
}
static void rot_rows(double* M, int cols, int ld, int p, int q, double c, double s) {
  double* rp = M + (int64_t)p * ld;                /* M <- R^T M */
  double* rq = M + (int64_t)q * ld;
  for (int j = 0; j < cols; ++j) {
    double a = rp[j], b = rq[j];
    rp[j] = c * a - s * b;
    rq[j] = s * a + c * b;
  }
}

int or_svd_gkr(int32_t n, const double* A, double* U, double* s_out, double* V) {
  double* W = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(W, A, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n * n; ++i) { U[i] = 0.0; V[i] = 0.0; }
  for (int i = 0; i < n; ++i) { U[(int64_t)i * n + i] = 1.0; V[(int64_t)i * n + i] = 1.0; }
  /* invariant: A = U W V^T */
  /* 1. bidiagonalisation */
  for (int j = 0; j < n; ++j) {
    /* left reflector: zero W[j+1:n, j] ; W <- H W, U <- U H */
    double nrm = 0.0;
    for (int i = j; i < n; ++i) nrm += W[(int64_t)i * n + j] * W[(int64_t)i * n + j];
    nrm = sqrt(nrm);
    if (nrm > 0.0) {
      double x0 = W[(int64_t)j * n + j], alpha = (x0 >= 0.0) ? -nrm : nrm;
      for (int i = 0; i < n; ++i) v[i] = 0.0;
      v[j] = x0 - alpha;
      for (int i = j + 1; i < n; ++i) v[i] = W[(int64_t)i * n + j];
      double vtv = 0.0;
      for (int i = j; i < n; ++i) vtv += v[i] * v[i];
      if (vtv > 0.0) {
        double beta = 2.0 / vtv;
        for (int c = 0; c < n; ++c) {
          double t = 0.0;
          for (int i = j; i < n; ++i) t += v[i] * W[(int64_t)i * n + c];
          t *= beta;
          for (int i = j; i < n; ++i) W[(int64_t)i * n + c] -= t * v[i];
        }
        for (int r = 0; r < n; ++r) {
          double t = 0.0;
          for (int i = j; i < n; ++i) t += U[(int64_t)r * n + i] * v[i];
          t *= beta;
          for (int i = j; i < n; ++i) U[(int64_t)r * n + i] -= t * v[i];
        }
        for (int i = j + 1; i < n; ++i) W[(int64_t)i * n + j] = 0.0;
      }
    }
    /* right reflector: zero W[j, j+2:n] ; W <- W H, V <- V H */
    if (j + 2 <= n - 1) {
      nrm = 0.0;
      for (int c = j + 1; c < n; ++c) nrm += W[(int64_t)j * n + c] * W[(int64_t)j * n + c];
      nrm = sqrt(nrm);
      if (nrm > 0.0) {
        double x0 = W[(int64_t)j * n + j + 1], alpha = (x0 >= 0.0) ? -nrm : nrm;
        for (int i = 0; i < n; ++i) v[i] = 0.0;
        v[j + 1] = x0 - alpha;
        for (int c = j + 2; c < n; ++c) v[c] = W[(int64_t)j * n + c];
        double vtv = 0.0;
        for (int c = j + 1; c < n; ++c) vtv += v[c] * v[c];
        if (vtv > 0.0) {
          double beta = 2.0 / vtv;
          for (int r = 0; r < n; ++r) {
            double t = 0.0;
            for (int c = j + 1; c < n; ++c) t += W[(int64_t)r * n + c] * v[c];
            t *= beta;
            for (int c = j + 1; c < n; ++c) W[(int64_t)r * n + c] -= t * v[c];
          }
          for (int r = 0; r < n; ++r) {
            double t = 0.0;
            for (int c = j + 1; c < n; ++c) t += V[(int64_t)r * n + c] * v[c];
            t *= beta;
            for (int c = j + 1; c < n; ++c) V[(int64_t)r * n + c] -= t * v[c];
          }
          for (int c = j + 2; c < n; ++c) W[(int64_t)j * n + c] = 0.0;
        }
      }
    }
  }
  /* 2. implicit-shift QR on the bidiagonal */
  const double eps = 2.220446049250313e-16;
  double bnorm = 0.0;
  for (int i = 0; i < n; ++i) {
    double t = fabs(W[(int64_t)i * n + i]) + (i + 1 < n ? fabs(W[(int64_t)i * n + i + 1]) : 0.0);
    if (t > bnorm) bnorm = t;
  }
  int status = OR_OK;
  long max_steps = 75L * (n > 1 ? n : 1) + 100;
  long steps = 0;
  for (;;) {
    for (int i = 0; i + 1 < n; ++i) {
      double f = W[(int64_t)i * n + i + 1];
      if (fabs(f) <= eps * (fabs(W[(int64_t)i * n + i]) + fabs(W[(int64_t)(i + 1) * n + i + 1])))
        W[(int64_t)i * n + i + 1] = 0.0;
    }
    for (int i = 0; i < n; ++i)
      if (fabs(W[(int64_t)i * n + i]) <= eps * bnorm) W[(int64_t)i * n + i] = 0.0;
    int hi = n - 1;
    while (hi > 0 && W[(int64_t)(hi - 1) * n + hi] == 0.0) --hi;
    if (hi == 0) break;                                  /* diagonal: converged */
    int lo = hi - 1;
    while (lo > 0 && W[(int64_t)(lo - 1) * n + lo] != 0.0) --lo;
    if (++steps > max_steps) { status = OR_ERR_NUMERICAL; break; }
    /* zero diagonal inside the block: chase the row's superdiagonal out */
    int zi = -1;
    for (int i = lo; i < hi; ++i) if (W[(int64_t)i * n + i] == 0.0) { zi = i; break; }
    if (zi >= 0) {
      for (int j = zi + 1; j <= hi; ++j) {
        double y = W[(int64_t)j * n + j], z = W[(int64_t)zi * n + j];
        double r = hypot(y, z);
        if (r == 0.0) continue;
        double c = y / r, s = z / r;
        rot_rows(W, n, n, j, zi, c, -s);   /* row_j' = c row_j + s row_zi ; row_zi' = -s row_j + c row_zi */
        rot_cols(U, n, n, j, zi, c, -s);
        W[(int64_t)zi * n + j] = 0.0;
      }
      continue;
    }
    if (W[(int64_t)hi * n + hi] == 0.0) {               /* zero last diagonal: chase column upward */
      for (int j = hi - 1; j >= lo; --j) {
        double y = W[(int64_t)j * n + j], z = W[(int64_t)j * n + hi];
        double r = hypot(y, z);
        if (r == 0.0) continue;
        double c = y / r, s = z / r;
        rot_cols(W, n, n, j, hi, c, -s);
        rot_cols(V, n, n, j, hi, c, -s);
        W[(int64_t)j * n + hi] = 0.0;
      }
      continue;
    }
    /* Golub-Kahan SVD step (Alg. 8.6.1) on rows/cols lo..hi */
    double dm = W[(int64_t)(hi - 1) * n + hi - 1];
    double fm = (hi - 1 > lo) ? W[(int64_t)(hi - 2) * n + hi - 1] : 0.0;
    double dn = W[(int64_t)hi * n + hi], fn = W[(int64_t)(hi - 1) * n + hi];
    double t11 = dm * dm + fm * fm, t12 = dm * fn, t22 = dn * dn + fn * fn;
    double dd = 0.5 * (t11 - t22);
    double sg = (dd >= 0.0) ? 1.0 : -1.0;
    double den = dd + sg * sqrt(dd * dd + t12 * t12);
    double mu = (den != 0.0) ? t22 - t12 * t12 / den : t22;
    double y = W[(int64_t)lo * n + lo] * W[(int64_t)lo * n + lo] - mu;
    double z = W[(int64_t)lo * n + lo] * W[(int64_t)lo * n + lo + 1];
    for (int k = lo; k < hi; ++k) {
      double r = hypot(y, z), c = 1.0, s = 0.0;
      if (r != 0.0) { c = y / r; s = -z / r; }
      rot_cols(W, n, n, k, k + 1, c, s);               /* [y z] R = [r 0] */
      rot_cols(V, n, n, k, k + 1, c, s);
      if (k > lo) W[(int64_t)(k - 1) * n + k + 1] = 0.0;
      y = W[(int64_t)k * n + k];
      z = W[(int64_t)(k + 1) * n + k];
      r = hypot(y, z); c = 1.0; s = 0.0;
      if (r != 0.0) { c = y / r; s = -z / r; }
      rot_rows(W, n, n, k, k + 1, c, s);               /* R^T [y; z] = [r; 0] */
      rot_cols(U, n, n, k, k + 1, c, s);
      W[(int64_t)(k + 1) * n + k] = 0.0;
      if (k < hi - 1) {
        y = W[(int64_t)k * n + k + 1];
        z = W[(int64_t)k * n + k + 2];
      }
    }
  }
  /* 3. non-negative singular values, sorted non-increasing */
  for (int i = 0; i < n; ++i) {
    double d = W[(int64_t)i * n + i];
    if (d < 0.0) {
      d = -d;
      for (int r = 0; r < n; ++r) V[(int64_t)r * n + i] = -V[(int64_t)r * n + i];
    }
    s_out[i] = d;
  }
  for (int i = 0; i < n; ++i) {                        /* selection sort, stable in index */
    int best = i;
    for (int j = i + 1; j < n; ++j) if (s_out[j] > s_out[best]) best = j;
    if (best != i) {
      double t = s_out[i]; s_out[i] = s_out[best]; s_out[best] = t;
      for (int r = 0; r < n; ++r) {
        t = U[(int64_t)r * n + i]; U[(int64_t)r * n + i] = U[(int64_t)r * n + best]; U[(int64_t)r * n + best] = t;
        t = V[(int64_t)r * n + i]; V[(int64_t)r * n + i] = V[(int64_t)r * n + best]; V[(int64_t)r * n + best] = t;
      }
    }
  }
  free(W); free(v);
  return status;
}

/* SVD of a k x m matrix B with k <= m: B = Ut diag(s) Vb^T, Ut k x k, Vb m x k.
 * Via A = B^T (m x k) = Q R (Householder), R = Ur diag(s) Vr^T (GKR), so
 * B = Vr diag(s) (Q Ur)^T. */
int or_svd_wide(int32_t k, int32_t m, const double* B, double* Ut, double* s, double* Vb) {
  double* A = (double*)malloc(sizeof(double) * (size_t)m * k);
  double* Q = (double*)malloc(sizeof(double) * (size_t)m * k);
  double* R = (double*)malloc(sizeof(double) * (size_t)k * k);
  double* Ur = (double*)malloc(sizeof(double) * (size_t)k * k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < m; ++j) A[(int64_t)j * k + i] = B[(int64_t)i * m + j];
  or_qr_householder(m, k, A, Q, R);
  int st = or_svd_gkr(k, R, Ur, s, Ut);
  mm(m, k, k, Q, Ur, Vb);
  free(A); free(Q); free(R); free(Ur);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Alg. 1 on one m x m block X, rank l = k (no oversampling), */
/* pi = q loop passes, Omega given (m x k).                                    */
/* Outputs U, V (m x k), sigma (k), and resid = ||X - S S^T X||_F (Eq. 7).     */
/* Sign rule: the largest-|.| entry of each U column is >= 0 (V flips too).    */
/* ------------------------------------------------------------------------ */
int or_rsvd_block_ex(int32_t m, int32_t k, int32_t q, int32_t scheme, const double* X, const double* Omega,
                     double* U, double* sigma, double* V, double* resid, double* S_out);

int or_rsvd_block(int32_t m, int32_t k, int32_t q, const double* X, const double* Omega,
                  double* U, double* sigma, double* V, double* resid, double* S_out) {
  return or_rsvd_block_ex(m, k, q, 0, X, Omega, U, sigma, V, resid, S_out);
}

/* scheme 0: Alg. 1 steps 2-3 (QR after every product).
 * scheme 1: Eq. 10, Y = (X X^T)^pi X Omega formed first, then ONE QR
 *           ("more sensitive to round-off errors").  Steps 4-6 are the same. */
int or_rsvd_block_ex(int32_t m, int32_t k, int32_t q, int32_t scheme, const double* X, const double* Omega,
                     double* U, double* sigma, double* V, double* resid, double* S_out) {
  size_t mk = (size_t)m * k, kk = (size_t)k * k, mm2 = (size_t)m * m;
  double* Y = (double*)malloc(sizeof(double) * mk);
  double* S = (double*)malloc(sizeof(double) * mk);
  double* St = (double*)malloc(sizeof(double) * mk);
  double* R = (double*)malloc(sizeof(double) * kk);
  double* B = (double*)malloc(sizeof(double) * mk);
  double* Ut = (double*)malloc(sizeof(double) * kk);
  if (scheme == 1) {
    /* Eq. 10: Y = (X X^T)^pi X Omega, then S = qr(Y) */
    mm(m, m, k, X, Omega, Y);
    for (int it = 0; it < q; ++it) {
      mtm(m, m, k, X, Y, St);                   /* X^T Y */
      mm(m, m, k, X, St, Y);                    /* X X^T Y */
    }
    or_qr_householder(m, k, Y, S, R);
  } else {
  /* step 2: Y0 = X Omega, Y0 = S0 R0 */
  mm(m, m, k, X, Omega, Y);
  or_qr_householder(m, k, Y, S, R);
  /* loop i = 1..pi: Ytil = X^T S_{i-1} = Stil Rtil ; Y = X Stil = S R */
  for (int it = 0; it < q; ++it) {
    mtm(m, m, k, X, S, Y);                      /* X^T S (literal transpose) */
    or_qr_householder(m, k, Y, St, R);
    mm(m, m, k, X, St, Y);
    or_qr_householder(m, k, Y, S, R);
  }
  }
  /* step 4: B = S^T X (k x m) */
  mtm(k, m, m, S, X, B);
  /* step 5: B = Ut Sigma V^T */
  int st = or_svd_wide(k, m, B, Ut, sigma, V);
  /* step 6: U = S Ut */
  mm(m, k, k, S, Ut, U);
  for (int j = 0; j < k; ++j) {
    int arg = 0; double best = -1.0;
    for (int i = 0; i < m; ++i) { double a = fabs(U[(int64_t)i * k + j]); if (a > best) { best = a; arg = i; } }
    if (U[(int64_t)arg * k + j] < 0.0) {
      for (int i = 0; i < m; ++i) { U[(int64_t)i * k + j] = -U[(int64_t)i * k + j]; V[(int64_t)i * k + j] = -V[(int64_t)i * k + j]; }
    }
  }
  if (resid) {                                   /* Eq. 7: ||X - S S^T X||_F = ||X - S B||_F */
    double* SB = (double*)malloc(sizeof(double) * mm2);
    mm(m, k, m, S, B, SB);
    double acc = 0.0;
    for (size_t i = 0; i < mm2; ++i) { double d = X[i] - SB[i]; acc += d * d; }
    *resid = sqrt(acc);
    free(SB);
  }
  if (S_out) memcpy(S_out, S, sizeof(double) * mk);
  free(Y); free(S); free(St); free(R); free(B); free(Ut);
  return st;
}

/* Eq. 3 with Eq. 15 on one block: F = scale * V Sigma^-1 (U^T Y), Y m x T. */
void or_apply_block(int32_t m, int32_t k, int32_t T, const double* U, const double* sigma,
                    const double* V, const double* Y, double scale, double* F) {
  double* Z = (double*)malloc(sizeof(double) * (size_t)k * T);
  mtm(k, m, T, U, Y, Z);                          /* U^T Y */
  for (int j = 0; j < k; ++j)
    for (int t = 0; t < T; ++t) Z[(int64_t)j * T + t] *= scale / sigma[j];
  mm(m, k, T, V, Z, F);
  free(Z);
}

/* Reading R2 on one block: with Theta_ii ~ U diag(s) U^T (rank k),
 *   X_ii = I - Theta_ii/(1+mu)  =>  X_ii^-1 ~ I + U diag(s_j / ((1+mu) - s_j)) U^T   (Woodbury)
 * and F = c X_ii^-1 Y = c (Y + U diag(s_j/((1+mu) - s_j)) U^T Y), c = mu/(1+mu) (Eq. 3). */
void or_apply_woodbury(int32_t m, int32_t k, int32_t T, const double* U, const double* sigma, const double* Y,
                       double mu, double* F) {
  double c = mu / (1.0 + mu);
  double* Z = (double*)malloc(sizeof(double) * (size_t)k * (T > 0 ? T : 1));
  mtm(k, m, T, U, Y, Z);                          /* U^T Y */
  for (int j = 0; j < k; ++j) {
    double d = sigma[j] / ((1.0 + mu) - sigma[j]);
    for (int t = 0; t < T; ++t) Z[(int64_t)j * T + t] *= d;
  }
  mm(m, k, T, U, Z, F);                           /* U D U^T Y */
  for (int64_t i = 0; i < (int64_t)m * T; ++i) F[i] = c * (Y[i] + F[i]);
  free(Z);
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: the 2x2 Schur-complement inverse (Eqs. 11-14)   */
/* ------------------------------------------------------------------------ */
/* Theta_ij[u][v] = dv_u^-1/2 dv_v^-1/2 sum_e H(u,e) w(e)/delta(e) H(v,e), u in block bi, v in block bj. */
void or_theta_offblock(int32_t b, int32_t bi, int32_t bj, const int64_t* row_ptr, const int32_t* col_idx,
                       const float* w, const double* dv, const double* de, double* out) {
  int64_t bu = (int64_t)bi * b, bv = (int64_t)bj * b;
  for (int32_t u = 0; u < b; ++u)
    for (int32_t v = 0; v < b; ++v) {
      int64_t pu = row_ptr[bu + u], eu = row_ptr[bu + u + 1];
      int64_t pv = row_ptr[bv + v], ev = row_ptr[bv + v + 1];
      double acc = 0.0;
      while (pu < eu && pv < ev) {
        if (col_idx[pu] < col_idx[pv]) ++pu;
        else if (col_idx[pu] > col_idx[pv]) ++pv;
        else { int32_t e = col_idx[pu]; acc += (double)w[e] / de[e]; ++pu; ++pv; }
      }
      out[(int64_t)u * b + v] = acc / sqrt(dv[bu + u]) / sqrt(dv[bv + v]);
    }
}

/* Reading R2 on a general block: for S = I - K/(1+mu) with K symmetric PSD (m x m), Alg. 1 on K
 * (rank k, q passes, Omega given) gives K ~ U diag(s) U^T and, by Woodbury,
 *   S^-1 ~ Ainv = I + U diag(s_j / ((1+mu) - s_j)) U^T   (dense m x m out). */
int or_lowrank_inverse(int32_t m, int32_t k, int32_t q, const double* K, const double* Omega, double mu,
                       double* Ainv) {
  double* U = (double*)malloc(sizeof(double) * (size_t)m * k);
  double* V = (double*)malloc(sizeof(double) * (size_t)m * k);
  double* sg = (double*)malloc(sizeof(double) * (size_t)k);
  int st = or_rsvd_block(m, k, q, K, Omega, U, sg, V, NULL, NULL);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double a = (i == j) ? 1.0 : 0.0;
      for (int t = 0; t < k; ++t) a += U[(int64_t)i * k + t] * (sg[t] / ((1.0 + mu) - sg[t])) * U[(int64_t)j * k + t];
      Ainv[(int64_t)i * m + j] = a;
    }
  free(U); free(V); free(sg);
  return st;
}

/* One level of Eq. 12 on the super-block of diagonal blocks (2s, 2s+1) (reading S1):
 *   X_s = [[X11, X12], [X21, X22]],  X_ij = delta_ij I - Theta_ij/(1+mu)
 *   Z1 = X11 - X12 X22^-1 X21,  Z2 = X22 - X21 X11^-1 X12               (Eqs. 13-14)
 *   X_s^-1 = [[Z1^-1, -X11^-1 X12 Z2^-1], [-Z2^-1 X21 X11^-1, Z2^-1]]   (Eq. 12)
 * with X11^-1, X22^-1, Z1^-1, Z2^-1 "by randomized SVD", reading R2: each
 * is I - K/(1+mu) with K PSD -- K11 = Theta11, K_Z1 = Theta11 + Theta12 X22^-1 Theta21/(1+mu)
 * (since X12 = -Theta12/(1+mu)) -- inverted by or_lowrank_inverse; Omega for X11 and Z1 is
 * block 2s's rows of the N x k Philox matrix, for X22 and Z2 block 2s+1's (reading S3).
 * F_s = c X_s^-1 Y_s, c = mu/(1+mu) (Eq. 3).  sel[n_sel] are super-block indices; F is
 * [n_sel * 2b][T] in sel order. */
int or_solve_schur(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                   double mu, int32_t b, int32_t k, int32_t q, uint64_t seed, const float* Y, int32_t T,
                   int32_t n_sel, const int32_t* sel, double* F, char* err, int errlen) {
  if (N <= 0 || E <= 0 || b <= 0 || N % (2 * b) != 0 || k < 1 || k > b || q < 0 || !(mu > 0.0) || T < 0) {
    set_err(err, errlen, "invalid arguments (need N % 2b == 0, 1 <= k <= b, q >= 0, mu > 0)");
    return OR_ERR_INVALID;
  }
  for (int i = 0; i < n_sel; ++i)
    if (sel[i] < 0 || sel[i] >= N / (2 * b)) { set_err(err, errlen, "super-block out of range"); return OR_ERR_INVALID; }
  double* dv = (double*)malloc(sizeof(double) * (size_t)N);
  double* de = (double*)malloc(sizeof(double) * (size_t)E);
  int st = or_degrees(N, E, row_ptr, col_idx, w, dv, de, err, errlen);
  if (st != OR_OK) { free(dv); free(de); return st; }
  const double c = mu / (1.0 + mu), ip = 1.0 / (1.0 + mu);
  int fail = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < n_sel; ++s) {
    const int i1 = 2 * sel[s], i2 = i1 + 1;
    size_t bb = (size_t)b * b, bk = (size_t)b * k, bt = (size_t)b * (T > 0 ? T : 1);
    double *T11 = malloc(sizeof(double) * bb), *T22 = malloc(sizeof(double) * bb), *T12 = malloc(sizeof(double) * bb);
    double *T21 = malloc(sizeof(double) * bb), *A11 = malloc(sizeof(double) * bb), *A22 = malloc(sizeof(double) * bb);
    double *Z1i = malloc(sizeof(double) * bb), *Z2i = malloc(sizeof(double) * bb), *W1 = malloc(sizeof(double) * bb);
    double *K1 = malloc(sizeof(double) * bb), *K2 = malloc(sizeof(double) * bb);
    double *O1 = malloc(sizeof(double) * bk), *O2 = malloc(sizeof(double) * bk);
    float* Of = malloc(sizeof(float) * bk);
    double *Y1 = malloc(sizeof(double) * bt), *Y2 = malloc(sizeof(double) * bt), *G = malloc(sizeof(double) * bt);
    double *H = malloc(sizeof(double) * bt), *P = malloc(sizeof(double) * bt);
    or_theta_block(b, i1, row_ptr, col_idx, w, dv, de, 0.0, T11);
    or_theta_block(b, i2, row_ptr, col_idx, w, dv, de, 0.0, T22);
    or_theta_offblock(b, i1, i2, row_ptr, col_idx, w, dv, de, T12);
    or_theta_offblock(b, i2, i1, row_ptr, col_idx, w, dv, de, T21);   /* = T12^T, computed literally */
    or_gaussian_f32(seed, (int64_t)i1 * b * k, (int64_t)bk, Of);
    for (size_t i = 0; i < bk; ++i) O1[i] = (double)Of[i];
    or_gaussian_f32(seed, (int64_t)i2 * b * k, (int64_t)bk, Of);
    for (size_t i = 0; i < bk; ++i) O2[i] = (double)Of[i];
    int r = 0;
    r |= or_lowrank_inverse(b, k, q, T11, O1, mu, A11);                /* X11^-1 */
    r |= or_lowrank_inverse(b, k, q, T22, O2, mu, A22);                /* X22^-1 */
    /* K_Z1 = Theta11 + Theta12 X22^-1 Theta21 / (1+mu);  K_Z2 = Theta22 + Theta21 X11^-1 Theta12 / (1+mu) */
    mm(b, b, b, A22, T21, W1);
    mm(b, b, b, T12, W1, K1);
    for (size_t i = 0; i < bb; ++i) K1[i] = T11[i] + ip * K1[i];
    mm(b, b, b, A11, T12, W1);
    mm(b, b, b, T21, W1, K2);
    for (size_t i = 0; i < bb; ++i) K2[i] = T22[i] + ip * K2[i];
    r |= or_lowrank_inverse(b, k, q, K1, O1, mu, Z1i);                 /* Z1^-1 */
    r |= or_lowrank_inverse(b, k, q, K2, O2, mu, Z2i);                 /* Z2^-1 */
    if (r) {
#pragma omp atomic write
      fail = OR_ERR_NUMERICAL;
    }
    for (int i = 0; i < b; ++i)
      for (int t = 0; t < T; ++t) {
        Y1[(int64_t)i * T + t] = (double)Y[((int64_t)i1 * b + i) * T + t];
        Y2[(int64_t)i * T + t] = (double)Y[((int64_t)i2 * b + i) * T + t];
      }
    double* F1 = F + (size_t)s * 2 * b * T;
    double* F2 = F1 + (size_t)b * T;
    if (T > 0) {
      /* top: Z1^-1 Y1 - X11^-1 X12 Z2^-1 Y2 = Z1^-1 Y1 + X11^-1 Theta12 Z2^-1 Y2 / (1+mu) */
      mm(b, b, T, Z2i, Y2, G);
      mm(b, b, T, T12, G, H);
      mm(b, b, T, A11, H, P);
      mm(b, b, T, Z1i, Y1, G);
      for (size_t i = 0; i < (size_t)b * T; ++i) F1[i] = c * (G[i] + ip * P[i]);
      /* bottom: -Z2^-1 X21 X11^-1 Y1 + Z2^-1 Y2 = Z2^-1 (Y2 + Theta21 X11^-1 Y1 / (1+mu)) */
      mm(b, b, T, A11, Y1, G);
      mm(b, b, T, T21, G, H);
      for (size_t i = 0; i < (size_t)b * T; ++i) H[i] = Y2[i] + ip * H[i];
      mm(b, b, T, Z2i, H, P);
      for (size_t i = 0; i < (size_t)b * T; ++i) F2[i] = c * P[i];
    }
    free(T11); free(T22); free(T12); free(T21); free(A11); free(A22); free(Z1i); free(Z2i); free(W1);
    free(K1); free(K2); free(O1); free(O2); free(Of); free(Y1); free(Y2); free(G); free(H); free(P);
  }
  free(dv); free(de);
  if (fail) { set_err(err, errlen, "numerical failure in a randomized SVD"); return fail; }
  return OR_OK;
}

/* Nested tessellation ("nested tessellations of submatrices created along the main
 * diagonal"; reading S4 in DESIGN.md): the inverse of a super-block of m = 2^L b vertices by Eq. 12
 * applied recursively to its diagonal halves down to b x b leaves.  A node of n = 2^l b vertices
 * starting at vertex r0 (l >= 1, halves of h = n/2):
 *   A11 = inverse of the first half, A22 = of the second (the recursion; leaves by reading R2 with
 *   rank k and Omega = rows [r0, r0+b) of the N x k Philox matrix);
 *   Theta11, Theta22 = the halves' Theta blocks, Theta12 = Theta[first half, second half], Theta21
 *   literally (or_theta_offblock with block size h);
 *   K_Z1 = Theta11 + Theta12 A22 Theta21/(1+mu), K_Z2 = Theta22 + Theta21 A11 Theta12/(1+mu)
 *   (Eqs. 13-14 with X12 = -Theta12/(1+mu), reading S2); Z1^-1, Z2^-1 by or_lowrank_inverse at rank
 *   k_l = k 2^(l-1) (the same rank-to-dimension ratio k/b at every level, reading S5) with Omega =
 *   rows [r0, r0+h) resp. [r0+h, r0+n) of the N x k_l Philox matrix (reading S3 generalised);
 *   node inverse (Eq. 12, X12 = -Theta12/(1+mu), X21 = -Theta21/(1+mu)):
 *     [[Z1^-1, A11 Theta12 Z2^-1/(1+mu)], [Z2^-1 Theta21 A11/(1+mu), Z2^-1]].
 * Writes the node's inverse Ainv and Theta block (both n x n, dense). */
static int nested_node(int32_t N, int32_t l, int64_t r0, int32_t b, int32_t k, int32_t q, uint64_t seed, double mu,
                       const int64_t* row_ptr, const int32_t* col_idx, const float* w, const double* dv,
                       const double* de, double* Ainv, double* Th) {
  const int64_t n = (int64_t)b << l;
  if (l == 0) {
    double* Om = (double*)malloc(sizeof(double) * (size_t)b * k);
    float* Of = (float*)malloc(sizeof(float) * (size_t)b * k);
    or_theta_block(b, (int32_t)(r0 / b), row_ptr, col_idx, w, dv, de, 0.0, Th);
    or_gaussian_f32(seed, r0 * k, (int64_t)b * k, Of);
    for (int64_t i = 0; i < (int64_t)b * k; ++i) Om[i] = (double)Of[i];
    int st = or_lowrank_inverse(b, k, q, Th, Om, mu, Ainv);
    free(Om); free(Of);
    return st;
  }
  const int64_t h = n / 2, hh = h * h;
  const int32_t kl = k << (l - 1);
  const double ip = 1.0 / (1.0 + mu);
  double *A11 = malloc(sizeof(double) * hh), *A22 = malloc(sizeof(double) * hh);
  double *T11 = malloc(sizeof(double) * hh), *T22 = malloc(sizeof(double) * hh);
  double *T12 = malloc(sizeof(double) * hh), *T21 = malloc(sizeof(double) * hh);
  double *W1 = malloc(sizeof(double) * hh), *K1 = malloc(sizeof(double) * hh), *K2 = malloc(sizeof(double) * hh);
  double *Z1i = malloc(sizeof(double) * hh), *Z2i = malloc(sizeof(double) * hh);
  double *O1 = malloc(sizeof(double) * h * kl), *O2 = malloc(sizeof(double) * h * kl);
  float* Of = malloc(sizeof(float) * h * kl);
  int st = nested_node(N, l - 1, r0, b, k, q, seed, mu, row_ptr, col_idx, w, dv, de, A11, T11);
  st |= nested_node(N, l - 1, r0 + h, b, k, q, seed, mu, row_ptr, col_idx, w, dv, de, A22, T22);
  or_theta_offblock((int32_t)h, (int32_t)(r0 / h), (int32_t)(r0 / h + 1), row_ptr, col_idx, w, dv, de, T12);
  or_theta_offblock((int32_t)h, (int32_t)(r0 / h + 1), (int32_t)(r0 / h), row_ptr, col_idx, w, dv, de, T21);
  mm((int)h, (int)h, (int)h, A22, T21, W1);
  mm((int)h, (int)h, (int)h, T12, W1, K1);
  for (int64_t i = 0; i < hh; ++i) K1[i] = T11[i] + ip * K1[i];
  mm((int)h, (int)h, (int)h, A11, T12, W1);
  mm((int)h, (int)h, (int)h, T21, W1, K2);
  for (int64_t i = 0; i < hh; ++i) K2[i] = T22[i] + ip * K2[i];
  or_gaussian_f32(seed, r0 * kl, h * kl, Of);
  for (int64_t i = 0; i < h * kl; ++i) O1[i] = (double)Of[i];
  or_gaussian_f32(seed, (r0 + h) * kl, h * kl, Of);
  for (int64_t i = 0; i < h * kl; ++i) O2[i] = (double)Of[i];
  st |= or_lowrank_inverse((int32_t)h, kl, q, K1, O1, mu, Z1i);
  st |= or_lowrank_inverse((int32_t)h, kl, q, K2, O2, mu, Z2i);
  /* top-right A11 Theta12 Z2^-1 / (1+mu) -> K1 (scratch); bottom-left Z2^-1 Theta21 A11 / (1+mu) -> K2 */
  mm((int)h, (int)h, (int)h, A11, T12, W1);
  mm((int)h, (int)h, (int)h, W1, Z2i, K1);
  mm((int)h, (int)h, (int)h, Z2i, T21, W1);
  mm((int)h, (int)h, (int)h, W1, A11, K2);
  for (int64_t i = 0; i < h; ++i)
    for (int64_t j = 0; j < h; ++j) {
      Ainv[i * n + j] = Z1i[i * h + j];
      Ainv[i * n + h + j] = ip * K1[i * h + j];
      Ainv[(h + i) * n + j] = ip * K2[i * h + j];
      Ainv[(h + i) * n + h + j] = Z2i[i * h + j];
      Th[i * n + j] = T11[i * h + j];
      Th[i * n + h + j] = T12[i * h + j];
      Th[(h + i) * n + j] = T21[i * h + j];
      Th[(h + i) * n + h + j] = T22[i * h + j];
    }
  free(A11); free(A22); free(T11); free(T22); free(T12); free(T21); free(W1); free(K1); free(K2); free(Z1i);
  free(Z2i); free(O1); free(O2); free(Of);
  return st;
}

/* F_s = c A_s^-1 Y_s (Eq. 3) for the selected super-blocks s of m = 2^L b vertices (nested_node at
 * level L); F is [n_sel * m][T] in sel order.  Constraints: L >= 1, N % m == 0, 1 <= k <= b. */
int or_solve_nested(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                    double mu, int32_t b, int32_t L, int32_t k, int32_t q, uint64_t seed, const float* Y, int32_t T,
                    int32_t n_sel, const int32_t* sel, double* F, char* err, int errlen) {
  const int64_t m = (int64_t)b << (L > 0 ? L : 0);
  if (N <= 0 || E <= 0 || b <= 0 || L < 1 || L > 8 || N % m != 0 || k < 1 || k > b || q < 0 || !(mu > 0.0) ||
      T < 0) {
    set_err(err, errlen, "invalid arguments (need L >= 1, N % (2^L b) == 0, 1 <= k <= b, q >= 0, mu > 0)");
    return OR_ERR_INVALID;
  }
  for (int i = 0; i < n_sel; ++i)
    if (sel[i] < 0 || sel[i] >= N / m) { set_err(err, errlen, "super-block out of range"); return OR_ERR_INVALID; }
  double* dv = (double*)malloc(sizeof(double) * (size_t)N);
  double* de = (double*)malloc(sizeof(double) * (size_t)E);
  int st = or_degrees(N, E, row_ptr, col_idx, w, dv, de, err, errlen);
  if (st != OR_OK) { free(dv); free(de); return st; }
  const double c = mu / (1.0 + mu);
  int fail = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < n_sel; ++s) {
    double* Ainv = (double*)malloc(sizeof(double) * (size_t)(m * m));
    double* Th = (double*)malloc(sizeof(double) * (size_t)(m * m));
    const int64_t r0 = (int64_t)sel[s] * m;
    int r = nested_node(N, L, r0, b, k, q, seed, mu, row_ptr, col_idx, w, dv, de, Ainv, Th);
    if (r) {
#pragma omp atomic write
      fail = OR_ERR_NUMERICAL;
    }
    double* Fs = F + (size_t)s * m * T;
    for (int64_t i = 0; i < m; ++i)
      for (int t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int64_t j = 0; j < m; ++j) acc += Ainv[i * m + j] * (double)Y[(r0 + j) * T + t];
        Fs[i * T + t] = c * acc;
      }
    free(Ainv); free(Th);
  }
  free(dv); free(de);
  if (fail) { set_err(err, errlen, "numerical failure in a randomized SVD"); return fail; }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Whole path over a subset of diagonal blocks.                              */
/* sel[n_sel] are block indices; outputs are packed in `sel` order:          */
/*   F [n_sel*b][T], sigma [n_sel][k], U/V [n_sel][b][k] (optional),          */
/*   resid [n_sel] (optional), X_out [n_sel][b][b] (optional, the X blocks).  */
/* ------------------------------------------------------------------------ */
int or_solve_mode(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                  double mu, int32_t b, int32_t k, int32_t q, uint64_t seed, const float* Y, int32_t T,
                  int32_t n_sel, const int32_t* sel, double* F, double* sigma, double* U_out, double* V_out,
                  double* resid, double* X_out, int32_t mode, int32_t p, int32_t scheme, char* err, int errlen);

int or_solve(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
             double mu, int32_t b, int32_t k, int32_t q, uint64_t seed, const float* Y, int32_t T,
             int32_t n_sel, const int32_t* sel, double* F, double* sigma, double* U_out, double* V_out,
             double* resid, double* X_out, char* err, int errlen) {
  return or_solve_mode(N, E, row_ptr, col_idx, w, mu, b, k, q, seed, Y, T, n_sel, sel, F, sigma, U_out, V_out,
                       resid, X_out, 0, 0, 0, err, errlen);
}

/* mode 0: reading R1 (Alg. 1 on X_ii, Eq. 15 apply); mode 1: reading R2 (Alg. 1 on Theta_ii,
 * Woodbury apply; X_out then holds the Theta_ii blocks the rSVD factored).
 * p: oversampling (l = k + pi): Alg. 1 runs with l = k + p columns (Omega is the
 * global N x l Philox matrix), the rank-k truncation (top k singular triplets) is applied.
 * scheme: 0 = Alg. 1, 1 = Eq. 10 (see or_rsvd_block_ex). */
int or_solve_mode(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                  double mu, int32_t b, int32_t k, int32_t q, uint64_t seed, const float* Y, int32_t T,
                  int32_t n_sel, const int32_t* sel, double* F, double* sigma, double* U_out, double* V_out,
                  double* resid, double* X_out, int32_t mode, int32_t p, int32_t scheme, char* err, int errlen) {
  if (mode != 0 && mode != 1) { set_err(err, errlen, "mode must be 0 (R1) or 1 (R2)"); return OR_ERR_INVALID; }
  if (p < 0 || k + p > b || (scheme != 0 && scheme != 1)) {
    set_err(err, errlen, "need p >= 0, k + p <= b, scheme 0 or 1"); return OR_ERR_INVALID;
  }
  const int32_t l = k + p;
  if (N <= 0 || E <= 0 || b <= 0 || N % b != 0 || k < 1 || k > b || q < 0 || !(mu > 0.0) || T < 0) {
    set_err(err, errlen, "invalid arguments (need N % b == 0, 1 <= k <= b, q >= 0, mu > 0)");
    return OR_ERR_INVALID;
  }
  for (int i = 0; i < n_sel; ++i)
    if (sel[i] < 0 || sel[i] >= N / b) { set_err(err, errlen, "selected block out of range"); return OR_ERR_INVALID; }
  double* dv = (double*)malloc(sizeof(double) * (size_t)N);
  double* de = (double*)malloc(sizeof(double) * (size_t)E);
  int st = or_degrees(N, E, row_ptr, col_idx, w, dv, de, err, errlen);
  if (st != OR_OK) { free(dv); free(de); return st; }
  double c = mu / (1.0 + mu);
  int fail = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < n_sel; ++s) {
    int blk = sel[s];
    size_t bb = (size_t)b * b, bk = (size_t)b * k, bl = (size_t)b * l;
    double* X = (double*)malloc(sizeof(double) * bb);
    double* Om = (double*)malloc(sizeof(double) * bl);
    float* Omf = (float*)malloc(sizeof(float) * bl);
    double* Ul = (double*)malloc(sizeof(double) * bl);
    double* Vl = (double*)malloc(sizeof(double) * bl);
    double* sl = (double*)malloc(sizeof(double) * l);
    double* U = (double*)malloc(sizeof(double) * bk);
    double* V = (double*)malloc(sizeof(double) * bk);
    double* Yi = (double*)malloc(sizeof(double) * (size_t)b * (T > 0 ? T : 1));
    or_theta_block(b, blk, row_ptr, col_idx, w, dv, de, mode == 1 ? 0.0 : mu, X);
    or_gaussian_f32(seed, (int64_t)blk * b * l, (int64_t)bl, Omf);
    for (size_t i = 0; i < bl; ++i) Om[i] = (double)Omf[i];
    int r = or_rsvd_block_ex(b, l, q, scheme, X, Om, Ul, sl, Vl, resid ? resid + s : NULL, NULL);
    /* rank-k truncation: the top k singular triplets (sigma is non-increasing) */
    for (int i = 0; i < b; ++i)
      for (int j = 0; j < k; ++j) { U[(int64_t)i * k + j] = Ul[(int64_t)i * l + j]; V[(int64_t)i * k + j] = Vl[(int64_t)i * l + j]; }
    for (int j = 0; j < k; ++j) sigma[(size_t)s * k + j] = sl[j];
    if (r != OR_OK) {
#pragma omp atomic write
      fail = r;
    }
    for (int j = 0; j < k && mode == 0; ++j)
      if (!(sigma[(size_t)s * k + j] > 1e-12 * sigma[(size_t)s * k])) {
#pragma omp atomic write
        fail = OR_ERR_NUMERICAL;
      }
    for (int i = 0; i < b; ++i)
      for (int t = 0; t < T; ++t) Yi[(int64_t)i * T + t] = (double)Y[((int64_t)blk * b + i) * T + t];
    if (T > 0 && mode == 0) or_apply_block(b, k, T, U, sigma + (size_t)s * k, V, Yi, c, F + (size_t)s * b * T);
    if (T > 0 && mode == 1) or_apply_woodbury(b, k, T, U, sigma + (size_t)s * k, Yi, mu, F + (size_t)s * b * T);
    if (U_out) memcpy(U_out + (size_t)s * bk, U, sizeof(double) * bk);
    if (V_out) memcpy(V_out + (size_t)s * bk, V, sizeof(double) * bk);
    if (X_out) memcpy(X_out + (size_t)s * bb, X, sizeof(double) * bb);
    free(X); free(Om); free(Omf); free(U); free(V); free(Yi); free(Ul); free(Vl); free(sl);
  }
  free(dv); free(de);
  if (fail) { set_err(err, errlen, "numerical failure (SVD non-convergence or singular sigma)"); return fail; }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: the hyperedge-weight update, f fixed             */
/* ------------------------------------------------------------------------ */
/* s[e][t] = h_e^T Dv^-1/2 f_t = sum_{v in e} f_t[v] / sqrt(delta(v)), delta(v) from w. */
static void edge_projections(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx,
                             const double* dv, const double* F, int32_t T, double* S) {
  for (int64_t i = 0; i < (int64_t)E * T; ++i) S[i] = 0.0;
  for (int32_t v = 0; v < N; ++v) {
    double r = 1.0 / sqrt(dv[v]);
    for (int64_t q = row_ptr[v]; q < row_ptr[v + 1]; ++q) {
      int32_t e = col_idx[q];
      for (int32_t t = 0; t < T; ++t) S[(int64_t)e * T + t] += r * F[(int64_t)v * T + t];
    }
  }
}

/* P(w) = sum_t f_t^T L(w) f_t + kappa ||w||^2 with L = I - A(w) (Eq. 1 with w, degrees re-derived)
 * (reading N1: the T columns of F are summed). */
int or_weight_objective(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                        const double* F, int32_t T, double kappa, double* out, char* err, int errlen) {
  double* dv = (double*)malloc(sizeof(double) * (size_t)N);
  double* de = (double*)malloc(sizeof(double) * (size_t)E);
  int st = or_degrees(N, E, row_ptr, col_idx, w, dv, de, err, errlen);
  if (st != OR_OK) { free(dv); free(de); return st; }
  double* S = (double*)malloc(sizeof(double) * (size_t)E * (T > 0 ? T : 1));
  edge_projections(N, E, row_ptr, col_idx, dv, F, T, S);
  double ff = 0.0, fAf = 0.0, ww = 0.0;
  for (int64_t i = 0; i < (int64_t)N * T; ++i) ff += F[i] * F[i];
  for (int32_t e = 0; e < E; ++e) {
    double se = 0.0;
    for (int32_t t = 0; t < T; ++t) se += S[(int64_t)e * T + t] * S[(int64_t)e * T + t];
    fAf += (double)w[e] / de[e] * se;           /* f^T Dv^-1/2 H W De^-1 H^T Dv^-1/2 f */
    ww += (double)w[e] * (double)w[e];
  }
  *out = ff - fAf + kappa * ww;
  free(dv); free(de); free(S);
  return OR_OK;
}

/* Frozen-degree gradient (SPEC.md gradient_frozen; PAPER.md:56-58 steepest descent on P):
 * D_v, D_e held at the current w, so only the explicit W of Eq. 1 differentiates:
 *   grad_e = -(1/delta(e)) sum_t (h_e^T Dv^-1/2 f_t)^2 + 2 kappa w_e. */
int or_weight_gradient(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                       const double* F, int32_t T, double kappa, double* grad, char* err, int errlen) {
  double* dv = (double*)malloc(sizeof(double) * (size_t)N);
  double* de = (double*)malloc(sizeof(double) * (size_t)E);
  int st = or_degrees(N, E, row_ptr, col_idx, w, dv, de, err, errlen);
  if (st != OR_OK) { free(dv); free(de); return st; }
  double* S = (double*)malloc(sizeof(double) * (size_t)E * (T > 0 ? T : 1));
  edge_projections(N, E, row_ptr, col_idx, dv, F, T, S);
  for (int32_t e = 0; e < E; ++e) {
    double se = 0.0;
    for (int32_t t = 0; t < T; ++t) se += S[(int64_t)e * T + t] * S[(int64_t)e * T + t];
    grad[e] = -se / de[e] + 2.0 * kappa * (double)w[e];
  }
  free(dv); free(de); free(S);
  return OR_OK;
}

/* One steepest-descent step on the simplex (Eq. 5's active constraints;
 * SPEC.md steepest_descent_step), reading N2:
 *   1. g_e -= mean of g over the free (non-clamped) coordinates   (G_1: 1^T w = 1 stays active)
 *   2. g_e  = 0 on clamped coordinates                             (G_j, j > 1: w_e = 0 stays)
 *   3. w   -= mu g
 *   4. while a free coordinate is < 0: clamp every such one to 0 (it joins the active set) and
 *      subtract the excess (sum w - 1) evenly from the remaining free coordinates.
 * active[e] = 1 marks clamped coordinates (in/out).  Error if every coordinate is clamped. */
int or_weight_step(int32_t E, double* w, int32_t* active, const double* grad, double mu, char* err, int errlen) {
  int32_t nfree = 0;
  double gm = 0.0;
  for (int32_t e = 0; e < E; ++e) if (!active[e]) { gm += grad[e]; ++nfree; }
  if (nfree == 0) { set_err(err, errlen, "every hyperedge weight is clamped (degenerate simplex)"); return OR_ERR_NUMERICAL; }
  gm /= nfree;
  for (int32_t e = 0; e < E; ++e) if (!active[e]) w[e] -= mu * (grad[e] - gm);
  for (;;) {
    int clamped = 0;
    for (int32_t e = 0; e < E; ++e)
      if (!active[e] && w[e] < 0.0) { w[e] = 0.0; active[e] = 1; ++clamped; }
    if (!clamped) break;
    double sum = 0.0;
    nfree = 0;
    for (int32_t e = 0; e < E; ++e) { sum += w[e]; if (!active[e]) ++nfree; }
    if (nfree == 0) { set_err(err, errlen, "every hyperedge weight is clamped (degenerate simplex)"); return OR_ERR_NUMERICAL; }
    double ex = (sum - 1.0) / nfree;
    for (int32_t e = 0; e < E; ++e) if (!active[e]) w[e] -= ex;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Second approach: conjugate gradient on Eq. 5          */
/* ------------------------------------------------------------------------ */
/* out = X p for one vector p of length N, X = I - A/(1+mu), A = Eq. 1 applied
 * right to left: s = Dv^-1/2 p;  t = H^T s;  t = W De^-1 t;  u = H t;
 * A p = Dv^-1/2 u.  t is scratch of length E. */
void or_apply_X(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                const double* dv, const double* de, double mu, const double* p, double* t, double* out) {
  for (int32_t e = 0; e < E; ++e) t[e] = 0.0;
  for (int32_t v = 0; v < N; ++v) {                    /* t = H^T Dv^-1/2 p */
    double sv = p[v] / sqrt(dv[v]);
    for (int64_t q = row_ptr[v]; q < row_ptr[v + 1]; ++q) t[col_idx[q]] += sv;
  }
  for (int32_t e = 0; e < E; ++e) t[e] *= (double)w[e] / de[e];   /* W De^-1 */
  for (int32_t v = 0; v < N; ++v) {                    /* A p = Dv^-1/2 H t */
    double u = 0.0;
    for (int64_t q = row_ptr[v]; q < row_ptr[v + 1]; ++q) u += t[col_idx[q]];
    out[v] = p[v] - (u / sqrt(dv[v])) / (1.0 + mu);
  }
}

static double dot(int32_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int32_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* CG (Eqs. 16-20) on X f = c y, c = theta/(1+theta) (Eq. 5),
 * independently for every column t of Y (N x T, row-major fp32):
 *   f_0 = 0 (reading C1), r_0 = c y - X f_0, p_0 = r_0;
 *   for i >= 1:  alpha_i = r_{i-1}^T r_{i-1} / p_{i-1}^T X p_{i-1}      (Eq. 19)
 *                f_i = f_{i-1} + alpha_i p_{i-1}                         (Eq. 16)
 *                r_i = r_{i-1} - alpha_i X p_{i-1}                       (Eq. 17)
 *                beta_i = r_i^T r_i / r_{i-1}^T r_{i-1}                  (Eq. 20)
 *                p_i = r_i + beta_i p_{i-1}                              (Eq. 18)
 * Stopping (reading C2): before iteration i, stop when ||r_{i-1}|| <= tol ||r_0||
 * or i > max_iter.  A zero column (r_0 = 0) takes no iteration and f = 0.
 * Outputs: F (N x T fp64), iters[T] (iterations taken), rel_res[T] = ||r||/||r_0||
 * of the recurrence residual at exit (0 for a zero column). */
int or_cg_solve(int32_t N, int32_t E, const int64_t* row_ptr, const int32_t* col_idx, const float* w,
                double mu, const float* Y, int32_t T, int32_t max_iter, double tol, double* F,
                int32_t* iters, double* rel_res, char* err, int errlen) {
  if (N <= 0 || E <= 0 || T < 0 || max_iter < 0 || !(mu > 0.0) || !(tol >= 0.0)) {
    set_err(err, errlen, "invalid arguments (need N, E > 0, T >= 0, max_iter >= 0, mu > 0, tol >= 0)");
    return OR_ERR_INVALID;
  }
  double* dv = (double*)malloc(sizeof(double) * (size_t)N);
  double* de = (double*)malloc(sizeof(double) * (size_t)E);
  int st = or_degrees(N, E, row_ptr, col_idx, w, dv, de, err, errlen);
  if (st != OR_OK) { free(dv); free(de); return st; }
  double c = mu / (1.0 + mu);
  int fail = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t col = 0; col < T; ++col) {
    double* f = (double*)malloc(sizeof(double) * (size_t)N);
    double* r = (double*)malloc(sizeof(double) * (size_t)N);
    double* p = (double*)malloc(sizeof(double) * (size_t)N);
    double* Xp = (double*)malloc(sizeof(double) * (size_t)N);
    double* t = (double*)malloc(sizeof(double) * (size_t)E);
    for (int32_t v = 0; v < N; ++v) f[v] = 0.0;
    or_apply_X(N, E, row_ptr, col_idx, w, dv, de, mu, f, t, Xp);
    for (int32_t v = 0; v < N; ++v) {
      r[v] = c * (double)Y[(int64_t)v * T + col] - Xp[v];
      p[v] = r[v];
    }
    double rr = dot(N, r, r), rr0 = rr;
    int32_t i = 0;
    if (rr0 > 0.0) {
      while (i < max_iter && !(sqrt(rr) <= tol * sqrt(rr0))) {
        or_apply_X(N, E, row_ptr, col_idx, w, dv, de, mu, p, t, Xp);
        double pXp = dot(N, p, Xp);
        if (!(pXp > 0.0)) {
#pragma omp atomic write
          fail = OR_ERR_NUMERICAL;
          break;
        }
        double alpha = rr / pXp;
        for (int32_t v = 0; v < N; ++v) f[v] += alpha * p[v];
        for (int32_t v = 0; v < N; ++v) r[v] -= alpha * Xp[v];
        double rr_new = dot(N, r, r);
        double beta = rr_new / rr;
        for (int32_t v = 0; v < N; ++v) p[v] = r[v] + beta * p[v];
        rr = rr_new;
        ++i;
      }
    }
    for (int32_t v = 0; v < N; ++v) F[(int64_t)v * T + col] = f[v];
    iters[col] = i;
    rel_res[col] = rr0 > 0.0 ? sqrt(rr / rr0) : 0.0;
    free(f); free(r); free(p); free(Xp); free(t);
  }
  free(dv); free(de);
  if (fail) { set_err(err, errlen, "CG breakdown (p^T X p <= 0)"); return fail; }
  return OR_OK;
}

/* Threading only (test infrastructure): results are bit-identical at any thread count. */
void or_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
