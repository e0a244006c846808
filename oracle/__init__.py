"""FP64 CPU oracle for the block randomized SVD hot path (ctypes binding).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs.  The product package
(paper_1908_08281_b200) never imports this module, and this module never
imports the product.  The C source (hg_oracle.c) cites the PAPER.md passage
each function follows.

Arrays: row-major numpy float64 unless noted.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hg_oracle.c")
_LIB = os.path.join(_HERE, "libhg_oracle.so")

OK, ERR_INVALID, ERR_NUMERICAL = 0, 2, 3


def build(force: bool = False) -> str:
    """Compile hg_oracle.c with gcc (OpenMP over blocks only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u64, dbl, cp, ci = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_double, ctypes.c_char_p, ctypes.c_int)
        L.or_philox4x64_10.argtypes = [P, P, P]
        L.or_philox_raw.argtypes = [u64, i64, i64, P]
        L.or_gaussian_f32.argtypes = [u64, i64, i64, P]
        L.or_degrees.argtypes = [i32, i32, P, P, P, P, P, cp, ci]
        L.or_degrees.restype = ci
        L.or_theta_block.argtypes = [i32, i32, P, P, P, P, P, dbl, P]
        L.or_qr_householder.argtypes = [i32, i32, P, P, P]
        L.or_svd_gkr.argtypes = [i32, P, P, P, P]
        L.or_svd_gkr.restype = ci
        L.or_svd_wide.argtypes = [i32, i32, P, P, P, P]
        L.or_svd_wide.restype = ci
        L.or_rsvd_block.argtypes = [i32, i32, i32, P, P, P, P, P, P, P]
        L.or_rsvd_block.restype = ci
        L.or_apply_block.argtypes = [i32, i32, i32, P, P, P, P, dbl, P]
        L.or_solve.argtypes = [i32, i32, P, P, P, dbl, i32, i32, i32, u64, P, i32, i32, P,
                               P, P, P, P, P, P, cp, ci]
        L.or_solve.restype = ci
        L.or_solve_mode.argtypes = [i32, i32, P, P, P, dbl, i32, i32, i32, u64, P, i32, i32, P,
                                    P, P, P, P, P, P, i32, i32, i32, cp, ci]
        L.or_rsvd_block_ex.argtypes = [i32, i32, i32, i32, P, P, P, P, P, P, P]
        L.or_rsvd_block_ex.restype = ci
        L.or_solve_mode.restype = ci
        L.or_apply_woodbury.argtypes = [i32, i32, i32, P, P, P, dbl, P]
        L.or_apply_woodbury.restype = None
        L.or_theta_offblock.argtypes = [i32, i32, i32, P, P, P, P, P, P]
        L.or_theta_offblock.restype = None
        L.or_lowrank_inverse.argtypes = [i32, i32, i32, P, P, dbl, P]
        L.or_lowrank_inverse.restype = ci
        L.or_solve_schur.argtypes = [i32, i32, P, P, P, dbl, i32, i32, i32, u64, P, i32, i32, P, P, cp, ci]
        L.or_solve_nested.argtypes = [i32, i32, P, P, P, dbl, i32, i32, i32, i32, u64, P, i32, i32, P, P, cp, ci]
        L.or_solve_nested.restype = ci
        L.or_solve_schur.restype = ci
        L.or_weight_objective.argtypes = [i32, i32, P, P, P, P, i32, dbl, P, cp, ci]
        L.or_weight_objective.restype = ci
        L.or_weight_gradient.argtypes = [i32, i32, P, P, P, P, i32, dbl, P, cp, ci]
        L.or_weight_gradient.restype = ci
        L.or_weight_step.argtypes = [i32, P, P, P, dbl, cp, ci]
        L.or_weight_step.restype = ci
        L.or_apply_X.argtypes = [i32, i32, P, P, P, P, P, dbl, P, P, P]
        L.or_apply_X.restype = None
        L.or_cg_solve.argtypes = [i32, i32, P, P, P, dbl, P, i32, i32, dbl, P, P, P, cp, ci]
        L.or_cg_solve.restype = ci
        L.or_num_threads.restype = ci
        L.or_set_num_threads.argtypes = [ci]
        L.or_set_num_threads.restype = None
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


# ---------------------------------------------------------------- primitives
def philox4x64_10(ctr: Sequence[int], key: Sequence[int]) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint64)
    k = np.asarray(key, dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().or_philox4x64_10(_p(c), _p(k), _p(out))
    return out


def philox_raw(seed: int, n_blocks: int, first_block: int = 0) -> np.ndarray:
    out = np.zeros(4 * n_blocks, dtype=np.uint64)
    lib().or_philox_raw(seed, first_block, n_blocks, _p(out))
    return out


def gaussian_f32(seed: int, n: int, start: int = 0) -> np.ndarray:
    out = np.zeros(n, dtype=np.float32)
    lib().or_gaussian_f32(seed, start, n, _p(out))
    return out


def omega(seed: int, N: int, k: int) -> np.ndarray:
    """The global N x k Omega (fp32): entry (r, c) is normal index r*k + c."""
    return gaussian_f32(seed, N * k).reshape(N, k)


def degrees(row_ptr, col_idx, w):
    N, E = len(row_ptr) - 1, len(w)
    dv, de = np.zeros(N), np.zeros(E)
    err = ctypes.create_string_buffer(256)
    st = lib().or_degrees(N, E, _p(row_ptr), _p(col_idx), _p(w), _p(dv), _p(de), err, 256)
    if st != OK:
        raise OracleError(st, err.value.decode())
    return dv, de


def theta_block(row_ptr, col_idx, w, b: int, blk: int, mu: float = 0.0) -> np.ndarray:
    """Theta_ii (mu == 0) or X_ii = I - Theta_ii/(1+mu) (mu > 0), fp64 b x b."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    w = np.ascontiguousarray(w, np.float32)
    dv, de = degrees(row_ptr, col_idx, w)
    out = np.zeros((b, b))
    lib().or_theta_block(b, blk, _p(row_ptr), _p(col_idx), _p(w), _p(dv), _p(de), mu, _p(out))
    return out


def qr_householder(A: np.ndarray):
    A = np.ascontiguousarray(A, np.float64)
    m, n = A.shape
    Q, R = np.zeros((m, n)), np.zeros((n, n))
    lib().or_qr_householder(m, n, _p(A), _p(Q), _p(R))
    return Q, R


def svd_square(A: np.ndarray):
    A = np.ascontiguousarray(A, np.float64)
    n = A.shape[0]
    U, s, V = np.zeros((n, n)), np.zeros(n), np.zeros((n, n))
    st = lib().or_svd_gkr(n, _p(A), _p(U), _p(s), _p(V))
    if st != OK:
        raise OracleError(st, "SVD did not converge")
    return U, s, V


def svd_wide(B: np.ndarray):
    """B (k x m, k <= m) = Ut diag(s) Vb^T."""
    B = np.ascontiguousarray(B, np.float64)
    k, m = B.shape
    Ut, s, Vb = np.zeros((k, k)), np.zeros(k), np.zeros((m, k))
    st = lib().or_svd_wide(k, m, _p(B), _p(Ut), _p(s), _p(Vb))
    if st != OK:
        raise OracleError(st, "SVD did not converge")
    return Ut, s, Vb


def rsvd_block(X: np.ndarray, Omega: np.ndarray, q: int, want_S: bool = False, eq10: bool = False):
    """Alg. 1 on one block (l = k; eq10: the Eq. 10 scheme).  Returns U, sigma, V, resid[, S]."""
    X = np.ascontiguousarray(X, np.float64)
    Om = np.ascontiguousarray(Omega, np.float64)
    m, k = Om.shape
    U, V, s = np.zeros((m, k)), np.zeros((m, k)), np.zeros(k)
    resid = np.zeros(1)
    S = np.zeros((m, k)) if want_S else None
    st = lib().or_rsvd_block_ex(m, k, q, 1 if eq10 else 0, _p(X), _p(Om), _p(U), _p(s), _p(V), _p(resid), _p(S))
    if st != OK:
        raise OracleError(st, "SVD did not converge")
    if want_S:
        return U, s, V, float(resid[0]), S
    return U, s, V, float(resid[0])


def apply_block(U, sigma, V, Y, scale: float) -> np.ndarray:
    U = np.ascontiguousarray(U, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    s = np.ascontiguousarray(sigma, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    m, k = U.shape
    T = Y.shape[1]
    F = np.zeros((m, T))
    lib().or_apply_block(m, k, T, _p(U), _p(s), _p(V), _p(Y), scale, _p(F))
    return F


class SolveResult:
    def __init__(self, blocks, F, sigma, U, V, resid, X, seconds, threads):
        self.blocks, self.F, self.sigma, self.U, self.V = blocks, F, sigma, U, V
        self.resid, self.X, self.seconds, self.threads = resid, X, seconds, threads


def set_num_threads(n: int) -> None:
    """OpenMP threads of the oracle (results are bit-identical at any count)."""
    lib().or_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().or_num_threads())


def apply_woodbury(U, sigma, Y, mu: float) -> np.ndarray:
    """Reading R2: F = c (Y + U diag(s/((1+mu) - s)) U^T Y), c = mu/(1+mu)."""
    U = np.ascontiguousarray(U, np.float64)
    s = np.ascontiguousarray(sigma, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    m, k = U.shape
    T = Y.shape[1]
    F = np.zeros((m, T))
    lib().or_apply_woodbury(m, k, T, _p(U), _p(s), _p(Y), mu, _p(F))
    return F


def solve(row_ptr, col_idx, w, Y, *, mu: float, b: int, k: int, q: int, seed: int,
          blocks: Optional[Sequence[int]] = None, want_UV: bool = False,
          want_X: bool = False, woodbury: bool = False, p: int = 0, eq10: bool = False) -> SolveResult:
    """The whole path (degrees -> X_ii -> Alg. 1 -> Eq. 3/15 apply) on `blocks`.

    woodbury=True: reading R2 (Alg. 1 on Theta_ii, Woodbury apply).
    p: oversampling, Alg. 1 at l = k + p columns then rank-k truncation.
    eq10=True: the Eq. 10 power scheme instead of Alg. 1's per-step QR.
    F rows for block i are F[s*b:(s+1)*b] where s is i's position in `blocks`.
    """
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    w = np.ascontiguousarray(w, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    N, E = len(row_ptr) - 1, len(w)
    T = Y.shape[1] if Y.ndim == 2 else 0
    nb = N // b if b > 0 else 0
    sel = np.asarray(range(nb) if blocks is None else blocks, dtype=np.int32)
    ns = len(sel)
    F = np.zeros((ns * b, T))
    sigma = np.zeros((ns, k))
    resid = np.zeros(ns)
    U = np.zeros((ns, b, k)) if want_UV else None
    V = np.zeros((ns, b, k)) if want_UV else None
    X = np.zeros((ns, b, b)) if want_X else None
    err = ctypes.create_string_buffer(256)
    t0 = time.perf_counter()
    st = lib().or_solve_mode(N, E, _p(row_ptr), _p(col_idx), _p(w), mu, b, k, q, seed, _p(Y), T, ns,
                             _p(sel), _p(F), _p(sigma), _p(U), _p(V), _p(resid), _p(X), 1 if woodbury else 0,
                             int(p), 1 if eq10 else 0, err, 256)
    dt = time.perf_counter() - t0
    if st != OK:
        raise OracleError(st, err.value.decode())
    return SolveResult(list(map(int, sel)), F, sigma, U, V, resid, X, dt, lib().or_num_threads())


# ------------------------------------------------- second approach: CG
def _csr(row_ptr, col_idx, w):
    return (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
            np.ascontiguousarray(w, np.float32))


def apply_X(row_ptr, col_idx, w, p, *, mu: float) -> np.ndarray:
    """X p for one length-N vector, matrix-free through H."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    N, E = len(row_ptr) - 1, len(w)
    dv, de = degrees(row_ptr, col_idx, w)
    p = np.ascontiguousarray(p, np.float64)
    out, t = np.zeros(N), np.zeros(E)
    lib().or_apply_X(N, E, _p(row_ptr), _p(col_idx), _p(w), _p(dv), _p(de), mu, _p(p), _p(t), _p(out))
    return out


class CGResult:
    def __init__(self, F, iters, rel_res, seconds, threads):
        self.F, self.iters, self.rel_res, self.seconds, self.threads = F, iters, rel_res, seconds, threads


def cg_solve(row_ptr, col_idx, w, Y, *, mu: float, max_iter: int, tol: float) -> CGResult:
    """CG on X F = theta/(1+theta) Y (Eqs. 5, 16-20), one independent CG per column of Y."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    Y = np.ascontiguousarray(Y, np.float32)
    N, E = len(row_ptr) - 1, len(w)
    T = Y.shape[1]
    F = np.zeros((N, T))
    iters = np.zeros(T, np.int32)
    rel = np.zeros(T)
    err = ctypes.create_string_buffer(256)
    t0 = time.perf_counter()
    st = lib().or_cg_solve(N, E, _p(row_ptr), _p(col_idx), _p(w), mu, _p(Y), T, max_iter, tol,
                           _p(F), _p(iters), _p(rel), err, 256)
    dt = time.perf_counter() - t0
    if st != OK:
        raise OracleError(st, err.value.decode())
    return CGResult(F, iters, rel, dt, lib().or_num_threads())


# ------------------------------------------ NEXT-4: hyperedge-weight update
def _F2(F):
    F = np.ascontiguousarray(F, np.float64)
    return F[:, None] if F.ndim == 1 else F


def weight_objective(row_ptr, col_idx, w, F, *, kappa: float) -> float:
    """P(w) = sum_t f_t^T L(w) f_t + kappa ||w||^2 (degrees re-derived from w)."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    F = _F2(F)
    out = np.zeros(1)
    err = ctypes.create_string_buffer(256)
    st = lib().or_weight_objective(len(row_ptr) - 1, len(w), _p(row_ptr), _p(col_idx), _p(w), _p(F), F.shape[1],
                                   kappa, _p(out), err, 256)
    if st != OK:
        raise OracleError(st, err.value.decode())
    return float(out[0])


def weight_gradient(row_ptr, col_idx, w, F, *, kappa: float) -> np.ndarray:
    """Frozen-degree gradient -(1/delta(e)) sum_t (h_e^T Dv^-1/2 f_t)^2 + 2 kappa w_e."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    F = _F2(F)
    g = np.zeros(len(w))
    err = ctypes.create_string_buffer(256)
    st = lib().or_weight_gradient(len(row_ptr) - 1, len(w), _p(row_ptr), _p(col_idx), _p(w), _p(F), F.shape[1],
                                  kappa, _p(g), err, 256)
    if st != OK:
        raise OracleError(st, err.value.decode())
    return g


def weight_step(w, active, grad, mu: float):
    """One simplex-constrained steepest-descent step; returns (w, active) copies."""
    w = np.array(w, np.float64)
    active = np.array(active, np.int32)
    grad = np.ascontiguousarray(grad, np.float64)
    err = ctypes.create_string_buffer(256)
    st = lib().or_weight_step(len(w), _p(w), _p(active), _p(grad), mu, err, 256)
    if st != OK:
        raise OracleError(st, err.value.decode())
    return w, active


# ------------------------------------------ NEXT-1: 2x2 Schur-complement inverse
def theta_offblock(row_ptr, col_idx, w, b: int, bi: int, bj: int) -> np.ndarray:
    """Theta restricted to rows of block bi and columns of block bj (Eq. 1), fp64 b x b."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    dv, de = degrees(row_ptr, col_idx, w)
    out = np.zeros((b, b))
    lib().or_theta_offblock(b, bi, bj, _p(row_ptr), _p(col_idx), _p(w), _p(dv), _p(de), _p(out))
    return out


def lowrank_inverse(K, Omega, q: int, mu: float) -> np.ndarray:
    """(I - K/(1+mu))^-1 ~ I + U diag(s/((1+mu)-s)) U^T from Alg. 1 on PSD K (reading R2)."""
    K = np.ascontiguousarray(K, np.float64)
    Om = np.ascontiguousarray(Omega, np.float64)
    m, k = Om.shape
    out = np.zeros((m, m))
    st = lib().or_lowrank_inverse(m, k, q, _p(K), _p(Om), mu, _p(out))
    if st != OK:
        raise OracleError(st, "SVD did not converge")
    return out


def solve_nested(row_ptr, col_idx, w, Y, *, mu: float, b: int, levels: int, k: int, q: int, seed: int,
                 superblocks: Optional[Sequence[int]] = None):
    """Nested tessellation: Eq. 12 recursively inside super-blocks of m = 2^levels b, leaves
    b x b, level-l Schur complements at rank k 2^(l-1); returns (F [n*m][T], superblocks, seconds)."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    Y = np.ascontiguousarray(Y, np.float32)
    N, E = len(row_ptr) - 1, len(w)
    T = Y.shape[1]
    m = b << levels
    ns = N // m if m > 0 else 0
    sel = np.asarray(range(ns) if superblocks is None else superblocks, dtype=np.int32)
    F = np.zeros((len(sel) * m, T))
    err = ctypes.create_string_buffer(256)
    t0 = time.perf_counter()
    st = lib().or_solve_nested(N, E, _p(row_ptr), _p(col_idx), _p(w), mu, b, levels, k, q, seed, _p(Y), T,
                               len(sel), _p(sel), _p(F), err, 256)
    dt = time.perf_counter() - t0
    if st != OK:
        raise OracleError(st, err.value.decode())
    return F, list(map(int, sel)), dt


def solve_schur(row_ptr, col_idx, w, Y, *, mu: float, b: int, k: int, q: int, seed: int,
                superblocks: Optional[Sequence[int]] = None):
    """One Eq. 12 level over super-blocks of 2b (blocks 2s, 2s+1); returns (F [n*2b][T], superblocks, seconds)."""
    row_ptr, col_idx, w = _csr(row_ptr, col_idx, w)
    Y = np.ascontiguousarray(Y, np.float32)
    N, E = len(row_ptr) - 1, len(w)
    T = Y.shape[1]
    ns = N // (2 * b) if b > 0 else 0
    sel = np.asarray(range(ns) if superblocks is None else superblocks, dtype=np.int32)
    F = np.zeros((len(sel) * 2 * b, T))
    err = ctypes.create_string_buffer(256)
    t0 = time.perf_counter()
    st = lib().or_solve_schur(N, E, _p(row_ptr), _p(col_idx), _p(w), mu, b, k, q, seed, _p(Y), T, len(sel),
                              _p(sel), _p(F), err, 256)
    dt = time.perf_counter() - t0
    if st != OK:
        raise OracleError(st, err.value.decode())
    return F, list(map(int, sel)), dt
