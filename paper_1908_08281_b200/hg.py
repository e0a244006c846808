"""Thin ctypes binding of libhgrsvd (include/hg.h) -- argument marshalling only.

Every step of the path runs in the library's CUDA kernels; PyTorch is used
only to own device memory and to name the current stream.  There is no CPU
path: importing this module raises if libhgrsvd.so is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Tuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# HG_LIB=check loads the bounds-checked build (libhgrsvd_check.so: device traps on index violations,
# the substitute for compute-sanitizer, which is closed on this pool)
LIB_PATH = os.path.join(_HERE, "libhgrsvd_check.so" if os.environ.get("HG_LIB") == "check" else "libhgrsvd.so")

HG_OK, HG_ERR_INVALID, HG_ERR_NUMERICAL, HG_ERR_CUDA = 0, 2, 3, 4
HG_RAW_THETA, HG_SYNC, HG_WOODBURY, HG_POWER_EQ10, HG_GEMM_SIMT = 1 << 0, 1 << 1, 1 << 2, 1 << 3, 1 << 8
HG_GENERAL, HG_UV_BK, HG_X_UNIT = 1 << 4, 1 << 5, 1 << 6
ST_FLAGS = {1: "isolated vertex", 2: "empty hyperedge", 4: "Cholesky breakdown", 8: "Jacobi sweep cap",
            16: "singular sigma", 32: "non-finite value", 64: "CG breakdown", 128: "degenerate simplex"}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1908_08281_b200.build` "
                      "(there is no fallback path)")

_lib = ctypes.CDLL(LIB_PATH)
_P, _i32, _i64, _u32, _u64, _f32, _sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                          ctypes.c_uint64, ctypes.c_float, ctypes.c_size_t)


class _Incidence(ctypes.Structure):
    _fields_ = [("n_vertices", _i32), ("n_edges", _i32), ("nnz", _i64), ("row_ptr", _P), ("col_idx", _P)]


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_workspace_size = _sig("hg_workspace_size", ctypes.c_int, _i32, _i32, _i64, _i32, _i32, _i32,
                       ctypes.POINTER(_sz))
_build_theta = _sig("hg_build_theta", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _i32, _u32, _P, _P, _P,
                    _P, _sz, _P)
_fill_gaussian = _sig("hg_fill_gaussian", ctypes.c_int, _u64, _i32, _i32, _P, _P)
_block_rsvd = _sig("hg_block_rsvd", ctypes.c_int, _P, _i32, _i32, _i32, _i32, _u64, _u32, _P, _P, _P, _P, _P, _sz,
                   _P)
_block_apply = _sig("hg_block_apply_inverse", ctypes.c_int, _P, _P, _P, _i32, _i32, _i32, _P, _i32, _f32, _P, _P, _P,
                    _sz, _P)
_workspace_size_ex = _sig("hg_workspace_size_ex", ctypes.c_int, _i32, _i32, _i64, _i32, _i32, _i32, _i32,
                          ctypes.POINTER(_sz))
_block_rsvd_ex = _sig("hg_block_rsvd_ex", ctypes.c_int, _P, _i32, _i32, _i32, _i32, _i32, _u64, _u32, _P, _P, _P, _P,
                      _P, _sz, _P)
_solve_ex = _sig("hg_solve_ex", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _i32, _i32, _i32, _i32, _u64, _P,
                 _i32, _P, _P, _u32, _P, _P, _sz, _P)
_solve_blocks = _sig("hg_solve_blocks", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _i32, _i32, _i32, _u64,
                     _i32, _i32, _P, _i32, _P, _P, _u32, _P, _P, _sz, _P)
_block_woodbury = _sig("hg_block_apply_woodbury", ctypes.c_int, _P, _P, _i32, _i32, _i32, _P, _i32, _f32, _P, _P,
                       _P, _sz, _P)
_solve = _sig("hg_solve", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _i32, _i32, _i32, _u64, _P, _i32, _P,
              _P, _u32, _P, _P, _sz, _P)
_solve_host = _sig("hg_solve_host", ctypes.c_int, _i32, _i32, _i64, _P, _P, _P, _f32, _i32, _i32, _i32, _u64, _P,
                   _i32, _P, _P, _u32, _P, _sz, _P)
_gemm = _sig("hg_gemm", ctypes.c_int, _i32, _i32, _i32, _i32, _P, _i32, _i64, _i64, _P, _i32, _i64, _i64, _P, _i32,
             _i64, _i64, _f32, _P, _i64, _P, _i64, _u32, _P)
_f16_split = _sig("hg_f16_split", ctypes.c_int, _P, _i64, _i32, _i64, _i32, _P, _P)
_gemm_f16pre = _sig("hg_gemm_f16pre", ctypes.c_int, _i32, _i32, _i32, _i32, _P, _i64, _i64, _i32, _P, _i64, _i64,
                    _i32, _P, _i32, _i64, _i64, _f32, _P)
_gemm_ex = _sig("hg_gemm_ex", ctypes.c_int, _i32, _i32, _i32, _i32, _P, _i32, _i64, _i64, _P, _i32, _i64, _i64, _P,
                _i32, _i64, _i64, _f32, _P, _i64, _P, _i64, _u32, _i32, _i32, _i32, _P)
_cg_workspace_size = _sig("hg_cg_workspace_size", ctypes.c_int, _i32, _i32, _i64, _i32, _i32, ctypes.POINTER(_sz))
_cg_solve = _sig("hg_cg_solve", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _P, _i32, _i32, _f32, _P, _P, _P,
                 _u32, _P, _P, _sz, _P)
_weight_gradient = _sig("hg_weight_gradient", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _P, _i32, _f32, _P, _P,
                        _P, _sz, _P)
_weight_objective = _sig("hg_weight_objective", ctypes.c_int, _P, _i32, _i32, _i32, _P, _P, _f32, _P, _P, _sz, _P)
_weight_step = _sig("hg_weight_step", ctypes.c_int, _i32, _P, _P, _P, _f32, _P, _P)
_weight_normalize = _sig("hg_weight_normalize", ctypes.c_int, _i32, _P, _P, _P, _P)
_nested_ws = _sig("hg_nested_workspace_size", ctypes.c_int, _i32, _i32, _i64, _i32, _i32, _i32, _i32, ctypes.POINTER(_sz))
_solve_nested = _sig("hg_solve_nested", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _i32, _i32, _i32, _i32, _u64,
                     _P, _i32, _P, _u32, _P, _P, _sz, _P)
_block_apply_ex = _sig("hg_block_apply_inverse_ex", ctypes.c_int, _P, _P, _P, _i32, _i32, _i32, _P, _i32, _f32, _P,
                       _u32, _P, _P, _sz, _P)
_schur_ws = _sig("hg_schur_workspace_size", ctypes.c_int, _i32, _i32, _i64, _i32, _i32, _i32, ctypes.POINTER(_sz))
_solve_schur = _sig("hg_solve_schur", ctypes.c_int, ctypes.POINTER(_Incidence), _P, _f32, _i32, _i32, _i32, _u64, _P,
                    _i32, _P, _u32, _P, _P, _sz, _P)
_last_error = _sig("hg_last_error", ctypes.c_char_p)
_prof_enable = _sig("hg_profile_enable", ctypes.c_int, _i32)
_prof_collect = _sig("hg_profile_collect", ctypes.c_int, _i32, _P, _P, _P, ctypes.POINTER(_i32))
_prof_timeline = _sig("hg_profile_timeline", ctypes.c_int, _i32, _P, _P, _P, _P, ctypes.POINTER(_i32))
_last_launches = _sig("hg_last_launch_count", ctypes.c_int32)
_debug_counters = _sig("hg_debug_counters", ctypes.c_int, _P, _i32, _i32)

EXPORTS = ("hg_workspace_size", "hg_build_theta", "hg_fill_gaussian", "hg_block_rsvd", "hg_block_apply_inverse",
           "hg_solve", "hg_solve_host", "hg_gemm", "hg_gemm_ex", "hg_f16_split", "hg_gemm_f16pre", "hg_last_error", "hg_last_launch_count", "hg_profile_enable",
           "hg_profile_collect", "hg_profile_timeline", "hg_debug_counters", "hg_cg_workspace_size", "hg_cg_solve",
           "hg_block_apply_woodbury", "hg_workspace_size_ex", "hg_block_rsvd_ex", "hg_solve_ex",
           "hg_weight_gradient", "hg_weight_step", "hg_schur_workspace_size",
           "hg_solve_schur", "hg_solve_blocks", "hg_weight_objective", "hg_debug_jacobi_sweepmax",
           "hg_block_apply_inverse_ex", "hg_weight_normalize", "hg_nested_workspace_size", "hg_solve_nested")


class HGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hg status {status}: {msg}")
        self.status = status


def _check(st: int):
    if st != HG_OK:
        raise HGError(st, _last_error().decode())


def last_launch_count() -> int:
    return int(_last_launches())


def debug_counters(reset: bool = False) -> dict:
    import numpy as np
    out = np.zeros(133, dtype=np.int64)
    _check(_debug_counters(out.ctypes.data_as(_P), 133, int(reset)))
    return {"chol_near_identity": int(out[0]), "chol_full": int(out[1]), "jacobi_max_sweeps": int(out[2]),
            "jacobi_total_sweeps": int(out[3]), "jacobi_blocks": int(out[4]), "chol_clk": out[5:69].tolist(),
            "jac_clk": out[69:85].tolist(), "jac_inner_clk": out[85:133].tolist()}


def debug_jacobi_sweepmax(on=None):
    """Per-sweep maximum block-Jacobi rotation measure (only in a -DHG_JB_SWEEPMAX build).
    on=True/False: clear and switch recording on/off; on=None: return float32 [64, 40] of
    |a_pq| / sqrt(a_pp a_qq) (block slot, sweep)."""
    import numpy as np
    fn = _lib.hg_debug_jacobi_sweepmax
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    fn.restype = ctypes.c_int
    if on is not None:
        if fn(None, int(bool(on))) != 0:
            raise HGError(HG_ERR_CUDA, "hg_debug_jacobi_sweepmax")
        return None
    out = np.zeros(64 * 40, dtype=np.float32)
    if fn(out.ctypes.data, 0) != 0:
        raise HGError(HG_ERR_CUDA, "hg_debug_jacobi_sweepmax")
    return np.sqrt(out.reshape(64, 40))


STAGES = ("degrees", "assemble", "omega", "gemm_power", "gemm_gram", "gemm_qform", "gemm_svd", "gemm_apply",
          "cholinv", "jacobi", "finalize", "inv_sigma", "cg", "eig_precond")


def profile_enable(on=True):
    """on: False/0 off, True/1 per-stage totals (stream parts in sequence), 2 timeline."""
    _check(_prof_enable(int(on)))


def profile_timeline(max_rec: int = 4096):
    """[(stage, part, start_ms, end_ms)] since the first hg_solve after the last collect."""
    import numpy as np
    st = np.zeros(max_rec, np.int32)
    pa = np.zeros(max_rec, np.int32)
    t0 = np.zeros(max_rec, np.float64)
    t1 = np.zeros(max_rec, np.float64)
    n = _i32(0)
    _check(_prof_timeline(max_rec, st.ctypes.data_as(_P), pa.ctypes.data_as(_P), t0.ctypes.data_as(_P),
                          t1.ctypes.data_as(_P), ctypes.byref(n)))
    m = min(n.value, max_rec)
    return [(STAGES[st[i]], int(pa[i]), float(t0[i]), float(t1[i])) for i in range(m)]


def profile_collect() -> dict:
    """{stage: (total_ms, launches)} recorded since the last collect (synchronises)."""
    import numpy as np
    names = ctypes.create_string_buffer(32 * 32)
    ms = np.zeros(32)
    cnt = np.zeros(32, dtype=np.int32)
    n = _i32(0)
    _check(_prof_collect(32, names, ms.ctypes.data_as(_P), cnt.ctypes.data_as(_P), ctypes.byref(n)))
    out = {}
    for i in range(min(n.value, 32)):
        nm = names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor, dtype) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"expected a contiguous {dtype} tensor, got {t.dtype}")
    return t


def workspace_size(N: int, E: int, nnz: int, b: int, k: int, T: int, p: int = 0) -> int:
    out = _sz(0)
    if p:
        _check(_workspace_size_ex(N, E, nnz, b, k, p, T, ctypes.byref(out)))
    else:
        _check(_workspace_size(N, E, nnz, b, k, T, ctypes.byref(out)))
    return int(out.value)


class Workspace:
    """Device scratch for the library (256-byte aligned torch allocation)."""

    def __init__(self, nbytes: int, device=None):
        self.buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device or "cuda")
        off = (-self.buf.data_ptr()) % 256
        self.ptr = ctypes.c_void_p(self.buf.data_ptr() + off)
        self.nbytes = nbytes

    @classmethod
    def for_sizes(cls, N, E, nnz, b, k, T, device=None, p: int = 0):
        return cls(workspace_size(N, E, nnz, b, k, T, p), device)


@dataclass
class Incidence:
    row_ptr: torch.Tensor   # int64 [N+1] cuda
    col_idx: torch.Tensor   # int32 [nnz] cuda
    n_edges: int

    @property
    def N(self):
        return self.row_ptr.numel() - 1

    @property
    def nnz(self):
        return self.col_idx.numel()

    def c(self) -> _Incidence:
        _dev(self.row_ptr, torch.int64)
        _dev(self.col_idx, torch.int32)
        return _Incidence(self.N, self.n_edges, self.nnz, self.row_ptr.data_ptr(), self.col_idx.data_ptr())


def build_theta(H: Incidence, w: torch.Tensor, mu: float, b: int, *, raw: bool = False,
                ws: Optional[Workspace] = None, status: Optional[torch.Tensor] = None, stream=None):
    """Diagonal blocks X_ii (or Theta_ii with raw=True) [N/b][b][b] and r = delta(v)^-1/2 [N]."""
    _dev(w, torch.float32)
    N = H.N
    ws = ws or Workspace.for_sizes(N, H.n_edges, H.nnz, b, 4, 0)
    blocks = torch.empty((N // b, b, b), dtype=torch.float32, device=w.device)
    dvr = torch.empty(N, dtype=torch.float32, device=w.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=w.device)
    inc = H.c()
    _check(_build_theta(ctypes.byref(inc), _ptr(w), mu, b, HG_RAW_THETA if raw else 0, _ptr(blocks), _ptr(dvr),
                        _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return blocks, dvr, st


def fill_gaussian(seed: int, rows: int, cols: int, device="cuda", stream=None) -> torch.Tensor:
    out = torch.empty((rows, cols), dtype=torch.float32, device=device)
    _check(_fill_gaussian(seed, rows, cols, _ptr(out), _stream(stream)))
    return out


def block_rsvd(blocks: torch.Tensor, k: int, q: int, seed: int, *, simt: bool = False, p: int = 0,
               eq10: bool = False, general: bool = False, uv_bk: bool = False, x_unit: bool = False,
               ws: Optional[Workspace] = None, status: Optional[torch.Tensor] = None, stream=None):
    """Alg. 1 on each block (oversampling p, Eq. 10 scheme with eq10; general: literal X^T products for
    non-symmetric blocks): Ut [nb][k][b], sigma [nb][k], Vt [nb][k][b], status -- with uv_bk the first and
    third are U, V [nb][b][k].  x_unit: the caller guarantees |X_ij| <= 1 and ||X_ii||_2 <= 1 (blocks from
    build_theta): the 3xF16 power products of the solve entries (HG_X_UNIT)."""
    _dev(blocks, torch.float32)
    nb, b, _ = blocks.shape
    ws = ws or Workspace.for_sizes(nb * b, 1, 0, b, k, 0, p=p)
    shape = (nb, b, k) if uv_bk else (nb, k, b)
    Ut = torch.empty(shape, dtype=torch.float32, device=blocks.device)
    Vt = torch.empty_like(Ut)
    sigma = torch.empty((nb, k), dtype=torch.float32, device=blocks.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=blocks.device)
    flags = (HG_GEMM_SIMT if simt else 0) | (HG_POWER_EQ10 if eq10 else 0) | (HG_GENERAL if general else 0) | \
        (HG_UV_BK if uv_bk else 0) | (HG_X_UNIT if x_unit else 0)
    _check(_block_rsvd_ex(_ptr(blocks), nb, b, k, p, q, seed, flags, _ptr(Ut), _ptr(sigma), _ptr(Vt),
                          _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return Ut, sigma, Vt, st


def block_apply_inverse(Ut: torch.Tensor, sigma: torch.Tensor, Vt: torch.Tensor, Y: torch.Tensor, scale: float, *,
                        ws: Optional[Workspace] = None, status: Optional[torch.Tensor] = None, stream=None):
    """F_i = scale * V_i Sigma_i^-1 U_i^T Y_i; returns F [N][T], status."""
    for t in (Ut, sigma, Vt, Y):
        _dev(t, torch.float32)
    nb, k, b = Ut.shape
    T = Y.shape[1]
    ws = ws or Workspace.for_sizes(nb * b, 1, 0, b, k, T)
    F = torch.empty((nb * b, T), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    _check(_block_apply(_ptr(Ut), _ptr(sigma), _ptr(Vt), nb, b, k, _ptr(Y), T, scale, _ptr(F), _ptr(st), ws.ptr,
                        ws.nbytes, _stream(stream)))
    return F, st


def block_apply_inverse_ex(U: torch.Tensor, sigma: torch.Tensor, V: torch.Tensor, Y: torch.Tensor, scale: float, *,
                           uv_bk: bool = False, ws: Optional[Workspace] = None,
                           status: Optional[torch.Tensor] = None, stream=None):
    """block_apply_inverse with U, V in either layout: uv_bk -> [nb][b][k], else [nb][k][b]."""
    for t in (U, sigma, V, Y):
        _dev(t, torch.float32)
    nb = U.shape[0]
    b, k = (U.shape[1], U.shape[2]) if uv_bk else (U.shape[2], U.shape[1])
    T = Y.shape[1]
    ws = ws or Workspace.for_sizes(nb * b, 1, 0, b, k, T)
    F = torch.empty((nb * b, T), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    _check(_block_apply_ex(_ptr(U), _ptr(sigma), _ptr(V), nb, b, k, _ptr(Y), T, scale, _ptr(F),
                           HG_UV_BK if uv_bk else 0, _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return F, st


def block_apply_woodbury(Ut: torch.Tensor, sigma: torch.Tensor, Y: torch.Tensor, mu: float, *,
                         ws: Optional[Workspace] = None, status: Optional[torch.Tensor] = None, stream=None):
    """Reading R2: F_i = c (Y_i + U_i diag(s/((1+mu)-s)) U_i^T Y_i) from the rSVD of Theta_ii."""
    for t in (Ut, sigma, Y):
        _dev(t, torch.float32)
    nb, k, b = Ut.shape
    T = Y.shape[1]
    ws = ws or Workspace.for_sizes(nb * b, 1, 0, b, k, T)
    F = torch.empty((nb * b, T), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    _check(_block_woodbury(_ptr(Ut), _ptr(sigma), nb, b, k, _ptr(Y), T, mu, _ptr(F), _ptr(st), ws.ptr, ws.nbytes,
                           _stream(stream)))
    return F, st


def solve(H: Incidence, w: torch.Tensor, Y: torch.Tensor, *, mu: float, b: int, k: int, q: int, seed: int,
          sync: bool = True, simt: bool = False, woodbury: bool = False, p: int = 0, eq10: bool = False,
          ws: Optional[Workspace] = None,
          F: Optional[torch.Tensor] = None, sigma: Optional[torch.Tensor] = None,
          status: Optional[torch.Tensor] = None, stream=None) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """The whole path from CSR H to F [N][T] (and sigma [N/b][k])."""
    _dev(w, torch.float32)
    _dev(Y, torch.float32)
    N, T = H.N, Y.shape[1]
    ws = ws or Workspace.for_sizes(N, H.n_edges, H.nnz, b, k, T, p=p)
    F = F if F is not None else torch.empty((N, T), dtype=torch.float32, device=Y.device)
    sigma = sigma if sigma is not None else torch.empty((N // b, k), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    flags = ((HG_SYNC if sync else 0) | (HG_GEMM_SIMT if simt else 0) | (HG_WOODBURY if woodbury else 0) |
             (HG_POWER_EQ10 if eq10 else 0))
    inc = H.c()
    if p:
        _check(_solve_ex(ctypes.byref(inc), _ptr(w), mu, b, k, p, q, seed, _ptr(Y), T, _ptr(F), _ptr(sigma), flags,
                         _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    else:
        _check(_solve(ctypes.byref(inc), _ptr(w), mu, b, k, q, seed, _ptr(Y), T, _ptr(F), _ptr(sigma), flags,
                      _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return F, sigma, st


def solve_blocks(H: Incidence, w: torch.Tensor, Y: torch.Tensor, *, mu: float, b: int, k: int, q: int, seed: int,
                 blk_begin: int, blk_count: int, sync: bool = True, ws: Optional[Workspace] = None,
                 F: Optional[torch.Tensor] = None, sigma: Optional[torch.Tensor] = None,
                 status: Optional[torch.Tensor] = None, stream=None):
    """hg_solve on blocks [blk_begin, blk_begin + blk_count) (one rank's share); F is the full [N][T]."""
    _dev(w, torch.float32)
    _dev(Y, torch.float32)
    N, T = H.N, Y.shape[1]
    ws = ws or Workspace.for_sizes(N, H.n_edges, H.nnz, b, k, T)
    F = F if F is not None else torch.zeros((N, T), dtype=torch.float32, device=Y.device)
    sigma = sigma if sigma is not None else torch.empty((blk_count, k), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    inc = H.c()
    _check(_solve_blocks(ctypes.byref(inc), _ptr(w), mu, b, k, q, seed, blk_begin, blk_count, _ptr(Y), T, _ptr(F),
                         _ptr(sigma), HG_SYNC if sync else 0, _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return F, sigma, st


def solve_host(row_ptr, col_idx, w, Y, *, mu: float, b: int, k: int, q: int, seed: int, F=None, sigma=None,
               woodbury: bool = False, ws: Optional[Workspace] = None, stream=None):
    """End-to-end entry from HOST tensors (pinned for full copy bandwidth): returns F, sigma on the host."""
    N, T, E, nnz = row_ptr.numel() - 1, Y.shape[1], w.numel(), col_idx.numel()
    ws = ws or Workspace.for_sizes(N, E, nnz, b, k, T)
    F = F if F is not None else torch.empty((N, T), dtype=torch.float32, pin_memory=True)
    sigma = sigma if sigma is not None else torch.empty((N // b, k), dtype=torch.float32, pin_memory=True)
    for t, dt in ((row_ptr, torch.int64), (col_idx, torch.int32), (w, torch.float32), (Y, torch.float32),
                  (F, torch.float32), (sigma, torch.float32)):
        if t.is_cuda or t.dtype != dt or not t.is_contiguous():
            raise ValueError("solve_host expects contiguous host tensors")
    _check(_solve_host(N, E, nnz, _ptr(row_ptr), _ptr(col_idx), _ptr(w), mu, b, k, q, seed, _ptr(Y), T, _ptr(F),
                       _ptr(sigma), HG_WOODBURY if woodbury else 0, ws.ptr, ws.nbytes, _stream(stream)))
    return F, sigma


def gemm(A: torch.Tensor, B: torch.Tensor, *, M: int, N: int, K: int, batch: int = 1, a_mn: bool = False, lda: int,
         sa: int = 0, b_mn: bool = False, ldb: int, sb: int = 0, D: torch.Tensor, d_trans: bool = False, ldd: int,
         sd: int = 0, alpha: float = 1.0, rs: Optional[torch.Tensor] = None, srs: int = 0,
         cs: Optional[torch.Tensor] = None, scs: int = 0, simt: bool = False, prec: Optional[int] = None,
         a_exp: int = 0, b_exp: int = 0, stream=None):
    """Verification export of the batched GEMM (see hg.h): 3xTF32, or 3xF16 with prec=1 (operands
    prescaled by 2^a_exp / 2^b_exp before the fp16 split)."""
    if prec is None:
        _check(_gemm(M, N, K, batch, _ptr(A), int(a_mn), lda, sa, _ptr(B), int(b_mn), ldb, sb, _ptr(D), int(d_trans),
                     ldd, sd, alpha, _ptr(rs), srs, _ptr(cs), scs, HG_GEMM_SIMT if simt else 0, _stream(stream)))
    else:
        _check(_gemm_ex(M, N, K, batch, _ptr(A), int(a_mn), lda, sa, _ptr(B), int(b_mn), ldb, sb, _ptr(D),
                        int(d_trans), ldd, sd, alpha, _ptr(rs), srs, _ptr(cs), scs, HG_GEMM_SIMT if simt else 0,
                        prec, a_exp, b_exp, _stream(stream)))
    return D


def f16_split(x: torch.Tensor, exp: int, stream=None):
    """Verification export: the 3xF16 twin of a 2D/3D fp32 tensor (last dim % 32 == 0): an int16 tensor of
    twice the elements holding, per 32 consecutive elements, the 32 fp16 bit patterns of hi = fp16(2^exp x)
    and then the 32 of lo = fp16(2^exp x - hi)."""
    _dev(x, torch.float32)
    cols = x.shape[-1]
    rows = x.numel() // cols
    out = torch.empty(x.shape[:-1] + (2 * cols,), dtype=torch.int16, device=x.device)
    _check(_f16_split(_ptr(x), rows, cols, cols, exp, _ptr(out), _stream(stream)))
    return out


def gemm_f16pre(A16: torch.Tensor, B16: torch.Tensor, *, M: int, N: int, K: int, batch: int,
                lda: int, sa: int, a_exp: int, ldb: int, sb: int, b_exp: int, D: torch.Tensor, d_trans: bool = False,
                ldd: int, sd: int = 0, alpha: float = 1.0, stream=None):
    """Verification export: 3xF16 GEMM on twin K-major operands (f16_split outputs; lda, sa, ldb, sb in
    elements of the fp32 arrays)."""
    _check(_gemm_f16pre(M, N, K, batch, _ptr(A16), lda, sa, a_exp, _ptr(B16), ldb, sb, b_exp, _ptr(D),
                        int(d_trans), ldd, sd, alpha, _stream(stream)))
    return D


def cg_workspace_size(N: int, E: int, nnz: int, T: int, max_iter: int) -> int:
    out = _sz(0)
    _check(_cg_workspace_size(N, E, nnz, T, max_iter, ctypes.byref(out)))
    return int(out.value)


def cg_solve(H: Incidence, w: torch.Tensor, Y: torch.Tensor, *, mu: float, max_iter: int, tol: float,
             sync: bool = True, ws: Optional[Workspace] = None, F: Optional[torch.Tensor] = None,
             iters: Optional[torch.Tensor] = None, rel_res: Optional[torch.Tensor] = None,
             status: Optional[torch.Tensor] = None, stream=None):
    """CG on X F = theta/(1+theta) Y, one CG per column: returns F, iters, rel_res, status."""
    _dev(w, torch.float32)
    _dev(Y, torch.float32)
    N, T = H.N, Y.shape[1]
    ws = ws or Workspace(cg_workspace_size(N, H.n_edges, H.nnz, T, max_iter), Y.device)
    F = F if F is not None else torch.empty((N, T), dtype=torch.float32, device=Y.device)
    iters = iters if iters is not None else torch.empty(T, dtype=torch.int32, device=Y.device)
    rel_res = rel_res if rel_res is not None else torch.empty(T, dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    inc = H.c()
    _check(_cg_solve(ctypes.byref(inc), _ptr(w), mu, _ptr(Y), T, max_iter, tol, _ptr(F), _ptr(iters), _ptr(rel_res),
                     HG_SYNC if sync else 0, _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return F, iters, rel_res, st


def weight_gradient(H: Incidence, w: torch.Tensor, F: torch.Tensor, *, kappa: float, ws: Optional[Workspace] = None,
                    grad: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None, stream=None):
    """NEXT-4 frozen-degree gradient of P(w): returns grad [E], status."""
    _dev(w, torch.float32)
    _dev(F, torch.float32)
    N, T = F.shape
    ws = ws or Workspace(cg_workspace_size(N, H.n_edges, H.nnz, T, 0), F.device)
    grad = grad if grad is not None else torch.empty(H.n_edges, dtype=torch.float32, device=F.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=F.device)
    inc = H.c()
    _check(_weight_gradient(ctypes.byref(inc), _ptr(w), _ptr(F), T, kappa, _ptr(grad), _ptr(st), ws.ptr, ws.nbytes,
                            _stream(stream)))
    return grad, st


def weight_step(w: torch.Tensor, active: torch.Tensor, grad: torch.Tensor, mu: float, *,
                status: Optional[torch.Tensor] = None, stream=None):
    """One simplex-constrained steepest-descent step, in place on w and active; returns status."""
    _dev(w, torch.float32)
    _dev(active, torch.int32)
    _dev(grad, torch.float32)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=w.device)
    _check(_weight_step(w.numel(), _ptr(w), _ptr(active), _ptr(grad), mu, _ptr(st), _stream(stream)))
    return st


def weight_normalize(w: torch.Tensor, *, status: Optional[torch.Tensor] = None, stream=None):
    """w / (1^T w) on the device (the start of the simplex iteration); returns (w_out, status)."""
    _dev(w, torch.float32)
    wo = torch.empty_like(w)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=w.device)
    _check(_weight_normalize(w.numel(), _ptr(w), _ptr(wo), _ptr(st), _stream(stream)))
    return wo, st


def schur_workspace_size(N: int, E: int, nnz: int, b: int, k: int, T: int) -> int:
    out = _sz(0)
    _check(_schur_ws(N, E, nnz, b, k, T, ctypes.byref(out)))
    return int(out.value)


def solve_schur(H: Incidence, w: torch.Tensor, Y: torch.Tensor, *, mu: float, b: int, k: int, q: int, seed: int,
                sync: bool = True, ws: Optional[Workspace] = None, F: Optional[torch.Tensor] = None,
                status: Optional[torch.Tensor] = None, stream=None):
    """NEXT-1: one Eq. 12 level over pairs of adjacent blocks (reading R2 inverses): returns F, status."""
    _dev(w, torch.float32)
    _dev(Y, torch.float32)
    N, T = H.N, Y.shape[1]
    ws = ws or Workspace(schur_workspace_size(N, H.n_edges, H.nnz, b, k, T), Y.device)
    F = F if F is not None else torch.empty((N, T), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    inc = H.c()
    _check(_solve_schur(ctypes.byref(inc), _ptr(w), mu, b, k, q, seed, _ptr(Y), T, _ptr(F), HG_SYNC if sync else 0,
                        _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return F, st


def nested_workspace_size(N: int, E: int, nnz: int, b: int, levels: int, k: int, T: int) -> int:
    n = _sz(0)
    _check(_nested_ws(N, E, nnz, b, levels, k, T, ctypes.byref(n)))
    return n.value


def solve_nested(H: Incidence, w: torch.Tensor, Y: torch.Tensor, *, mu: float, b: int, levels: int, k: int, q: int,
                 seed: int, sync: bool = True, ws: Optional[Workspace] = None, F: Optional[torch.Tensor] = None,
                 status: Optional[torch.Tensor] = None, stream=None):
    """NEXT-1: the nested tessellation (Eq. 12 recursively inside super-blocks of b * 2^levels): returns F, status."""
    _dev(w, torch.float32)
    _dev(Y, torch.float32)
    N, T = Y.shape
    ws = ws or Workspace(nested_workspace_size(N, H.n_edges, H.nnz, b, levels, k, T), Y.device)
    F = F if F is not None else torch.empty((N, T), dtype=torch.float32, device=Y.device)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=Y.device)
    inc = H.c()
    _check(_solve_nested(ctypes.byref(inc), _ptr(w), mu, b, levels, k, q, seed, _ptr(Y), T, _ptr(F),
                         HG_SYNC if sync else 0, _ptr(st), ws.ptr, ws.nbytes, _stream(stream)))
    return F, st


def tessellate(super_block: int, threshold: int):
    """SPEC.md tessellate on a super-block of `super_block` vertices: midpoint splits until the leaf
    dimension is <= threshold (reading S6 of the 50 -> 500 schedule); returns (b, levels)."""
    levels = 0
    while (super_block >> levels) > threshold and (super_block >> levels) % 2 == 0:
        levels += 1
    return super_block >> levels, levels


def weight_objective(F: torch.Tensor, w: torch.Tensor, grad: torch.Tensor, *, kappa: float, stream=None) -> float:
    """P(w) = ||F||^2 + w^T grad - kappa ||w||^2 (grad from weight_gradient at this w), computed on the device."""
    for t in (F, w, grad):
        _dev(t, torch.float32)
    out = torch.zeros(1, dtype=torch.float64, device=F.device)
    scratch = torch.empty(296, dtype=torch.float64, device=F.device)
    _check(_weight_objective(_ptr(F), F.shape[0], F.shape[1], w.numel(), _ptr(w), _ptr(grad), kappa, _ptr(out),
                             _ptr(scratch), scratch.numel() * 8, _stream(stream)))
    return float(out.item())


def learn_weights(H: Incidence, w0: torch.Tensor, F: torch.Tensor, *, kappa: float, mu: float, steps: int,
                  ws: Optional[Workspace] = None):
    """NEXT-4 driver (SPEC.md learn_weights): with F fixed, `steps` accepted simplex steps of steepest descent
    on P(w); a step that increases P is rejected and mu halved.  Every step runs in the library's kernels
    (gradient, step, objective); this loop only decides accept / reject.  Returns (w, active, trace of P, mu)."""
    N, T = F.shape
    ws = ws or Workspace(cg_workspace_size(N, H.n_edges, H.nnz, T, 0), F.device)
    w, st0 = weight_normalize(w0.contiguous())
    if int(st0.item()) != 0:
        raise HGError(HG_ERR_NUMERICAL, "w0 is not a valid start for the simplex (negative, non-finite or zero sum)")
    active = torch.zeros(H.n_edges, dtype=torch.int32, device=F.device)
    g, st = weight_gradient(H, w, F, kappa=kappa, ws=ws)
    P = weight_objective(F, w, g, kappa=kappa)
    trace = [P]
    done, tries = 0, 0
    while done < steps and tries < 8 * steps:
        tries += 1
        w_try, a_try = w.clone(), active.clone()
        st = weight_step(w_try, a_try, g, mu)
        g_try, st2 = weight_gradient(H, w_try, F, kappa=kappa, ws=ws)
        P_try = weight_objective(F, w_try, g_try, kappa=kappa)
        if int(st.item()) != 0 or int(st2.item()) != 0 or not (P_try <= P):
            mu *= 0.5
            continue
        w, active, g, P = w_try, a_try, g_try, P_try
        trace.append(P)
        done += 1
    return w, active, trace, mu


def adaptive_learning(H: Incidence, w0: torch.Tensor, Y: torch.Tensor, *, mu: float, kappa: float, outer: int = 2,
                      weight_steps: int = 5, step: float = 1e-4, solver: str = "cg", b: int = 0, k: int = 0,
                      q: int = 0, seed: int = 0, cg_tol: float = 1e-6, cg_max_iter: int = 100,
                      super_block: int = 1024, thresholds=(50, 500), rank_ratio: float = 0.25):
    """The paper's alternation (Table 2): solve Eq. 3 for F with the current w (the CG of
    PAPER.md:165-178, the block rSVD path with solver="rsvd", or the nested tessellation with
    solver="nested": super-blocks of `super_block` vertices tessellated down to leaves <= thresholds[i] in
    outer pass i -- the paper's 50 -> 500 schedule, reading S6 -- leaf rank rank_ratio * b),
    then update w with F fixed (learn_weights), `outer` times.  Returns (F, w, history) with history[i] =
    (P before, P after) of outer pass i.  Composition of library calls only."""
    w, st0 = weight_normalize(w0.contiguous())
    if int(st0.item()) != 0:
        raise HGError(HG_ERR_NUMERICAL, "w0 is not a valid start for the simplex (negative, non-finite or zero sum)")
    hist = []
    F = None
    for _ in range(outer):
        if solver == "cg":
            F, _, _, _ = cg_solve(H, w, Y, mu=mu, max_iter=cg_max_iter, tol=cg_tol)
        elif solver == "nested":
            bl, lv = tessellate(super_block, thresholds[min(len(hist), len(thresholds) - 1)])
            lv = min(max(lv, 1), 6)
            bl = super_block >> lv
            kl = max(4, int(round(bl * rank_ratio / 4)) * 4)
            F, _ = solve_nested(H, w, Y, mu=mu, b=bl, levels=lv, k=min(kl, bl), q=q, seed=seed)
        else:
            F, _, _ = solve(H, w, Y, mu=mu, b=b, k=k, q=q, seed=seed)
        w_new, _, trace, step = learn_weights(H, w, F, kappa=kappa, mu=step, steps=weight_steps)
        hist.append((trace[0], trace[-1]))
        w = w_new
    return F, w, hist


def incidence_to_device(row_ptr, col_idx, n_edges: int, device="cuda") -> Incidence:
    return Incidence(torch.as_tensor(row_ptr, dtype=torch.int64).to(device).contiguous(),
                     torch.as_tensor(col_idx, dtype=torch.int32).to(device).contiguous(), int(n_edges))
