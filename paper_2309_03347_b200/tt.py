"""Thin Python binding over libtt (include/tt.h): device containers on torch
tensors and functions with the C-ABI names.  Argument marshalling only —
every step of the hot path runs in the CUDA kernels of libtt.so.

TT-vector cores are column-major [r_k, n_k, r_{k+1}] stored compactly at the
start of rank-capacity slots; ranks are device int32 (include/tt.h)."""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import TTError, check, lib

F64 = torch.float64


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


class _Workspace:
    """Grow-only device scratch buffer (uint8 tensor) shared by calls."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return self.buf


_WS = _Workspace()


def workspace(nbytes: int, device="cuda") -> torch.Tensor:
    return _WS.get(nbytes, torch.device(device))


class TTVec:
    """TT-vector in device memory with rank-capacity slots."""

    def __init__(self, n: Sequence[int], rcap: Sequence[int], device="cuda"):
        self.d = len(n)
        self.n = [int(v) for v in n]
        self.rcap = [int(v) for v in rcap]
        assert len(self.rcap) == self.d + 1 and self.rcap[0] == 1 and self.rcap[-1] == 1
        sizes = [self.rcap[k] * self.n[k] * self.rcap[k + 1] for k in range(self.d)]
        self.off = [int(v) for v in np.concatenate([[0], np.cumsum(sizes)[:-1]])]
        self.device = torch.device(device)
        self.data = torch.zeros(int(sum(sizes)), dtype=F64, device=self.device)
        self.r_dev = torch.ones(self.d + 1, dtype=torch.int32, device=self.device)
        self._n = (C.c_int32 * self.d)(*self.n)
        self._rcap = (C.c_int32 * (self.d + 1))(*self.rcap)
        self._off = (C.c_int64 * self.d)(*self.off)
        self._c = _lib.tt_vec(self.d, self._n, self.r_dev.data_ptr(), self._rcap, self.data.data_ptr(), self._off)

    @property
    def c(self):
        return C.byref(self._c)

    @classmethod
    def from_cores(cls, cores: List[np.ndarray], rcap: Optional[Sequence[int]] = None, device="cuda"):
        n = [c.shape[1] for c in cores]
        r = [c.shape[0] for c in cores] + [cores[-1].shape[2]]
        if rcap is None:
            rcap = r
        rcap = [max(int(a), int(b)) for a, b in zip(rcap, r)]
        v = cls(n, rcap, device)
        v.set_cores(cores)
        return v

    def set_cores(self, cores: List[np.ndarray]):
        r = [c.shape[0] for c in cores] + [cores[-1].shape[2]]
        host = torch.zeros(self.data.numel(), dtype=F64)
        for k, c in enumerate(cores):
            assert c.shape[1] == self.n[k] and c.shape[0] <= self.rcap[k] and c.shape[2] <= self.rcap[k + 1]
            flat = torch.from_numpy(np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1, order="F")))
            host[self.off[k]:self.off[k] + flat.numel()] = flat
        self.data.copy_(host)
        self.r_dev.copy_(torch.tensor(r, dtype=torch.int32))

    def ranks(self) -> List[int]:
        return [int(v) for v in self.r_dev.cpu()]

    def cores(self) -> List[np.ndarray]:
        r = self.ranks()
        host = self.data.cpu().numpy()
        out = []
        for k in range(self.d):
            size = r[k] * self.n[k] * r[k + 1]
            out.append(host[self.off[k]:self.off[k] + size].reshape(r[k], self.n[k], r[k + 1], order="F").copy())
        return out


class TTMat:
    """TT-matrix in device memory; cores [R_k, m_k, n_k, R_{k+1}] column-major."""

    def __init__(self, m: Sequence[int], n: Sequence[int], Rcap: Sequence[int], device="cuda"):
        self.d = len(m)
        self.m = [int(v) for v in m]
        self.n = [int(v) for v in n]
        self.Rcap = [int(v) for v in Rcap]
        sizes = [self.Rcap[k] * self.m[k] * self.n[k] * self.Rcap[k + 1] for k in range(self.d)]
        self.off = [int(v) for v in np.concatenate([[0], np.cumsum(sizes)[:-1]])]
        self.device = torch.device(device)
        self.data = torch.zeros(int(sum(sizes)), dtype=F64, device=self.device)
        self.R_dev = torch.ones(self.d + 1, dtype=torch.int32, device=self.device)
        self._m = (C.c_int32 * self.d)(*self.m)
        self._n = (C.c_int32 * self.d)(*self.n)
        self._Rcap = (C.c_int32 * (self.d + 1))(*self.Rcap)
        self._off = (C.c_int64 * self.d)(*self.off)
        self._c = _lib.tt_mat(self.d, self._m, self._n, self.R_dev.data_ptr(), self._Rcap,
                              self.data.data_ptr(), self._off)
        # the same storage viewed as a TT-vector with mode m_k n_k (row index fastest)
        self._mn = (C.c_int32 * self.d)(*[a * b for a, b in zip(self.m, self.n)])
        self._vc = _lib.tt_vec(self.d, self._mn, self.R_dev.data_ptr(), self._Rcap, self.data.data_ptr(), self._off)

    @property
    def c(self):
        return C.byref(self._c)

    @property
    def as_vec_c(self):
        return C.byref(self._vc)

    @classmethod
    def from_cores(cls, cores: List[np.ndarray], Rcap=None, device="cuda"):
        m = [c.shape[1] for c in cores]
        n = [c.shape[2] for c in cores]
        R = [c.shape[0] for c in cores] + [cores[-1].shape[3]]
        Rcap = R if Rcap is None else [max(int(a), int(b)) for a, b in zip(Rcap, R)]
        A = cls(m, n, Rcap, device)
        A.set_cores(cores)
        return A

    def set_cores(self, cores):
        R = [c.shape[0] for c in cores] + [cores[-1].shape[3]]
        host = torch.zeros(self.data.numel(), dtype=F64)
        for k, c in enumerate(cores):
            flat = torch.from_numpy(np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1, order="F")))
            host[self.off[k]:self.off[k] + flat.numel()] = flat
        self.data.copy_(host)
        self.R_dev.copy_(torch.tensor(R, dtype=torch.int32))

    def ranks(self):
        return [int(v) for v in self.R_dev.cpu()]

    def cores(self):
        R = self.ranks()
        host = self.data.cpu().numpy()
        out = []
        for k in range(self.d):
            size = R[k] * self.m[k] * self.n[k] * R[k + 1]
            out.append(host[self.off[k]:self.off[k] + size].reshape(R[k], self.m[k], self.n[k], R[k + 1],
                                                                     order="F").copy())
        return out


# ------------------------------------------------------------ operations ---

def tt_matvec(A: TTMat, x: TTVec, y: TTVec, stream=None):
    check(lib().tt_matvec(A.c, x.c, y.c, C.c_void_p(_stream(stream))))
    return y


class MatvecBatch:
    """Marshalled arguments of one batched product (the ctypes descriptor arrays
    and the workspace are built once; each call is one ABI call)."""

    def __init__(self, As, xs, ys):
        self.B = len(As)
        self.keep = (As, xs, ys)
        self.Ac = (_lib.tt_mat * self.B)(*[a._c for a in As])
        self.xc = (_lib.tt_vec * self.B)(*[v._c for v in xs])
        self.yc = (_lib.tt_vec * self.B)(*[v._c for v in ys])
        nb = lib().tt_matvec_batched_workspace(self.B, self.Ac)
        self.ws = torch.empty(max(int(nb), 256), dtype=torch.uint8, device=xs[0].device)

    def __call__(self, stream=None):
        check(lib().tt_matvec_batched(self.B, self.Ac, self.xc, self.yc, _ptr(self.ws), self.ws.numel(),
                                      C.c_void_p(_stream(stream))))
        return self.keep[2]


def tt_matvec_batched(As, xs, ys, stream=None):
    """B independent products in one launch (C ABI tt_matvec_batched)."""
    return MatvecBatch(As, xs, ys)(stream)


def matvec_out(A: TTMat, x: TTVec) -> TTVec:
    """Allocate y with capacities R*r and compute y = A x."""
    y = TTVec(A.m, [a * b for a, b in zip(A.Rcap, x.rcap)], A.device)
    return tt_matvec(A, x, y)


def tt_add(x: TTVec, y: TTVec, z: TTVec, alpha: Optional[torch.Tensor] = None,
           beta: Optional[torch.Tensor] = None, stream=None):
    check(lib().tt_add(x.c, _ptr(alpha), y.c, _ptr(beta), z.c, C.c_void_p(_stream(stream))))
    return z


def tt_scale(x: TTVec, alpha: torch.Tensor, stream=None):
    check(lib().tt_scale(x.c, _ptr(alpha), C.c_void_p(_stream(stream))))
    return x


def tt_copy(x: TTVec, y: TTVec, stream=None):
    check(lib().tt_copy(x.c, y.c, C.c_void_p(_stream(stream))))
    return y


def tt_dot(x: TTVec, y: TTVec, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    if out is None:
        out = torch.zeros(1, dtype=F64, device=x.device)
    nb = lib().tt_dot_workspace(x.c, y.c)
    ws = workspace(nb, x.device)
    check(lib().tt_dot(x.c, y.c, _ptr(out), _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    return out


def tt_orthogonalize(x: TTVec, direction: int = -1, norm: Optional[torch.Tensor] = None, stream=None):
    if norm is None:
        norm = torch.zeros(1, dtype=F64, device=x.device)
    nb = lib().tt_orthogonalize_workspace(x.c)
    ws = workspace(nb, x.device)
    check(lib().tt_orthogonalize(x.c, int(direction), _ptr(norm), _ptr(ws), ws.numel(),
                                 C.c_void_p(_stream(stream))))
    return norm


def tt_round(x: TTVec, eps: float, rmax: int = 1 << 30, want_info: bool = False, stream=None):
    disc = sv = None
    stride = 0
    if want_info:
        disc = torch.zeros(max(x.d - 1, 1), dtype=F64, device=x.device)
        stride = max(x.rcap)
        sv = torch.zeros(max(x.d - 1, 1) * stride, dtype=F64, device=x.device)
    nb = lib().tt_round_workspace(x.c)
    ws = workspace(nb, x.device)
    check(lib().tt_round(x.c, float(eps), int(min(rmax, 2**31 - 1)), _ptr(disc), _ptr(sv), int(stride),
                         _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    if want_info:
        return x, disc, sv.view(max(x.d - 1, 1), stride)
    return x


def tt_normalize(x: TTVec, norm: Optional[torch.Tensor] = None, stream=None):
    """x <- x / ||x||_F on the device; returns the norm (device tensor)."""
    if norm is None:
        norm = torch.zeros(1, dtype=F64, device=x.device)
    nb = lib().tt_orthogonalize_workspace(x.c)
    ws = workspace(nb, x.device)
    check(lib().tt_normalize(x.c, _ptr(norm), _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    return norm


class RoundBatch:
    """Marshalled arguments of one batched rounding (tt_round_batched): the ctypes
    descriptor array and the workspace are built once; each call is one ABI call."""

    def __init__(self, xs):
        self.B = len(xs)
        self.keep = xs
        self.xc = (_lib.tt_vec * self.B)(*[v._c for v in xs])
        nb = lib().tt_round_batched_workspace(self.B, self.xc)
        if nb == 0:
            raise TTError(1, "tt_round_batched: workspace query rejected the instances")
        self.ws = torch.empty(int(nb), dtype=torch.uint8, device=xs[0].device)
        self.disc = torch.zeros(self.B * max(xs[0].d - 1, 1), dtype=F64, device=xs[0].device)

    def __call__(self, eps: float, rmax: int = 1 << 30, stream=None):
        check(lib().tt_round_batched(self.B, self.xc, float(eps), int(min(rmax, 2**31 - 1)), _ptr(self.disc),
                                     _ptr(self.ws), self.ws.numel(), C.c_void_p(_stream(stream))))
        return self.disc.view(self.B, -1)


def tt_round_batched(xs, eps: float, rmax: int = 1 << 30, stream=None):
    """tt_round of B independent TT-vectors in place, one launch per step for all."""
    return RoundBatch(xs)(eps, rmax, stream)


def als_local_apply(dims, Phi, Ak, Psi, x, y, stream=None, ws=None):
    """dims = (rA, R, rB, m, n, rAp, Rp, rBp); arrays are flat device tensors.
    ws: dedicated uint8 workspace (>= als_workspace bytes) for concurrent calls."""
    nb = lib().als_workspace(*dims)
    if ws is None:
        ws = workspace(nb, x.device)
    check(lib().als_local_apply(*[int(v) for v in dims], _ptr(Phi), _ptr(Ak), _ptr(Psi), _ptr(x), _ptr(y),
                                _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    return y


def als_update_interfaces(direction, dims, Iprev, Yk, Ak, Xk, Inext, stream=None, ws=None):
    """dims = (rY, R, rX, m, n, rYp, Rp, rXp); Ak = None for the vector interface."""
    nb = lib().als_workspace(*dims)
    if ws is None:
        ws = workspace(nb, Yk.device)
    check(lib().als_update_interfaces(int(direction), *[int(v) for v in dims], _ptr(Iprev), _ptr(Yk), _ptr(Ak),
                                      _ptr(Xk), _ptr(Inext), _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    return Inext


CORE_DENSE, CORE_DIAG = 0, 1


def core_kinds(A: "TTMat", stream=None):
    """Device-detected structure of every operator core (tt_core_kinds):
    returns (kinds, off-diagonal ratios) as host lists."""
    kinds = (C.c_int32 * A.d)()
    ratio = (C.c_double * A.d)()
    ws = workspace(768, A.data.device)
    check(lib().tt_core_kinds(A.c, C.cast(kinds, C.c_void_p), C.cast(ratio, C.c_void_p), _ptr(ws), ws.numel(),
                              C.c_void_p(_stream(stream))))
    return list(kinds), list(ratio)


def als_local_apply_structured(kind, absorb, dims, Phi, Ak, Psi, x, y, stream=None):
    """als_local_apply for a core of the given kind (CORE_DENSE / CORE_DIAG);
    absorb = 1 folds the left operator rank into the left interface first."""
    nb = lib().als_workspace_structured(int(kind), int(absorb), *dims)
    ws = workspace(nb, x.device)
    check(lib().als_local_apply_structured(int(kind), int(absorb), *[int(v) for v in dims], _ptr(Phi), _ptr(Ak),
                                           _ptr(Psi), _ptr(x), _ptr(y), _ptr(ws), ws.numel(),
                                           C.c_void_p(_stream(stream))))
    return y


def als_update_interfaces_structured(kind, absorb, direction, dims, Iprev, Yk, Ak, Xk, Inext, stream=None):
    nb = lib().als_workspace_structured(int(kind), int(absorb), *dims)
    ws = workspace(nb, Yk.device)
    check(lib().als_update_interfaces_structured(int(kind), int(absorb), int(direction), *[int(v) for v in dims],
                                                 _ptr(Iprev), _ptr(Yk), _ptr(Ak), _ptr(Xk), _ptr(Inext), _ptr(ws),
                                                 ws.numel(), C.c_void_p(_stream(stream))))
    return Inext


# ------------------------------------------------------------------ a7 ---

def amen_solve(A: TTMat, b: TTVec, x: TTVec, z: TTVec, eps: float, rmax: int = 1 << 20, max_sweeps: int = 20,
               restart: int = 40, max_restarts: int = 50, local_tol: float = 0.0, local_dense_max: int = 0,
               stream=None):
    """x <- AMEn solution of A x = b (x: initial guess in, solution out; z: residual TT).
    local_dense_max > 0: local systems of that size or smaller are solved densely."""
    o = _lib.amen_opts(float(eps), float(local_tol), int(max_sweeps), int(min(rmax, 2**30)), int(restart),
                       int(max_restarts), int(local_dense_max))
    nb = lib().amen_workspace(A.c, b.c, x.c, z.c, C.byref(o))
    if nb == 0:
        check(lib().amen_solve(A.c, b.c, x.c, z.c, C.byref(o), None, None, None, 0, C.c_void_p(_stream(stream))))
    ws = workspace(nb, x.device)
    sweeps = torch.zeros(1, dtype=torch.int32, device=x.device)
    res = torch.zeros(1, dtype=torch.float64, device=x.device)
    check(lib().amen_solve(A.c, b.c, x.c, z.c, C.byref(o), _ptr(sweeps), _ptr(res), _ptr(ws), ws.numel(),
                           C.c_void_p(_stream(stream))))
    return x, sweeps, res


def amen_mv(A: TTMat, b: TTVec, y: TTVec, z: TTVec, eps: float, rmax: int = 1 << 20, max_sweeps: int = 20,
            stream=None):
    """y <- A b by the fit-based sweeps (NEXT-1; y: initial guess in, product out; z: residual TT)."""
    nb = lib().amen_mv_workspace(A.c, b.c, y.c, z.c)
    if nb == 0:
        check(lib().amen_mv(A.c, b.c, y.c, z.c, float(eps), int(max_sweeps), int(min(rmax, 2**30)), None, None, 0,
                            C.c_void_p(_stream(stream))))
    ws = workspace(nb, y.device)
    sweeps = torch.zeros(1, dtype=torch.int32, device=y.device)
    check(lib().amen_mv(A.c, b.c, y.c, z.c, float(eps), int(max_sweeps), int(min(rmax, 2**30)), _ptr(sweeps),
                        _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    return y, sweeps


# ------------------------------------------------------------------ a9 ---

_MV = {"exact": 0, "amen_mv": 1}


class KeffResult:
    def __init__(self, k, iters, k_hist, sweeps_hist, status, res_hist=None, inner_hist=None, res=None):
        self.k, self.iters, self.k_hist, self.sweeps_hist, self.status = k, iters, k_hist, sweeps_hist, status
        self.res_hist, self.inner_hist, self.res = res_hist, inner_hist, res


def _keff_opts(tol_k, tol_res, eps_round, eps_solve, max_outer, rmax, max_sweeps, restart, max_restarts, matvec,
               mv_max_sweeps, warm=False, local_dense_max=0):
    return _lib.keff_opts(float(tol_k), float(tol_res), float(eps_round), float(eps_solve), int(max_outer),
                          int(min(rmax, 2**30)), int(max_sweeps), 0, int(restart), int(max_restarts),
                          int(local_dense_max), _MV[matvec], int(mv_max_sweeps), int(bool(warm)))


def keff_fixed_point(H: TTMat, S: TTMat, F: TTMat, psi: TTVec, z: TTVec, k0: float = 1.0, tol_k: float = 1e-10,
                     eps_round: float = 1e-12, eps_solve: float = 1e-11, max_outer: int = 200, rmax: int = 1 << 20,
                     max_sweeps: int = 20, restart: int = 40, max_restarts: int = 50, hist_cap: int = 256,
                     matvec: str = "exact", mv_max_sweeps: int = 10, tol_res: float = -1.0, warm: bool = False,
                     ws: Optional[torch.Tensor] = None, local_dense_max: int = 0, stream=None) -> KeffResult:
    """matvec: "exact" (exact products + rounding) or "amen_mv" (fit-based product, NEXT-1).
    tol_res > 0: fixed-point residual every iteration, required for convergence;
    0: evaluated once at the end; < 0: not evaluated.  warm: continue the previous
    call with the same operators and options (keff_opts.warm, include/tt.h); a warm
    call needs the workspace of that call: pass a dedicated uint8 tensor `ws`
    (keff_workspace_bytes) to both."""
    o = _keff_opts(tol_k, tol_res, eps_round, eps_solve, max_outer, rmax, max_sweeps, restart, max_restarts, matvec,
                   mv_max_sweeps, warm, local_dense_max)
    dev = psi.device
    k = torch.zeros(1, dtype=torch.float64, device=dev)
    iters = torch.zeros(1, dtype=torch.int32, device=dev)
    kh = torch.zeros(hist_cap, dtype=torch.float64, device=dev)
    rh = torch.zeros(hist_cap, dtype=torch.float64, device=dev)
    sh = torch.zeros(hist_cap, dtype=torch.int32, device=dev)
    ih = torch.zeros(hist_cap, dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    res = torch.zeros(1, dtype=torch.float64, device=dev)
    rep = _lib.keff_report(k.data_ptr(), iters.data_ptr(), kh.data_ptr(), rh.data_ptr(), int(hist_cap), st.data_ptr(),
                           sh.data_ptr(), ih.data_ptr(), res.data_ptr())
    nb = lib().keff_workspace(H.c, S.c, F.c, psi.c, z.c, C.byref(o))
    if nb == 0:
        check(lib().keff_fixed_point(H.c, S.c, F.c, psi.c, z.c, float(k0), C.byref(o), C.byref(rep), None, 0,
                                     C.c_void_p(_stream(stream))))
    if ws is None:
        ws = workspace(nb, dev)
    elif ws.numel() < nb:
        raise ValueError(f"keff_fixed_point: workspace of {ws.numel()} bytes, {nb} needed")
    check(lib().keff_fixed_point(H.c, S.c, F.c, psi.c, z.c, float(k0), C.byref(o), C.byref(rep), _ptr(ws),
                                 ws.numel(), C.c_void_p(_stream(stream))))
    return KeffResult(k, iters, kh, sh, st, rh, ih, res)


def keff_workspace_bytes(H: TTMat, S: TTMat, F: TTMat, psi: TTVec, z: TTVec, tol_res: float = -1.0,
                         rmax: int = 1 << 20, matvec: str = "exact", restart: int = 40, local_dense_max: int = 0) -> int:
    o = _keff_opts(1e-10, tol_res, 1e-12, 1e-11, 1, rmax, 1, restart, 1, matvec, 1, False, local_dense_max)
    return int(lib().keff_workspace(H.c, S.c, F.c, psi.c, z.c, C.byref(o)))


# -------------------------------------------------------------- NEXT-2 ---

class AlphaResult:
    def __init__(self, alpha, k, iters, alpha_hist, k_hist, keff_iters_hist, status):
        self.alpha, self.k, self.iters = alpha, k, iters
        self.alpha_hist, self.k_hist, self.keff_iters_hist, self.status = alpha_hist, k_hist, keff_iters_hist, status


def alpha_secant(H: TTMat, V: TTMat, S: TTMat, F: TTMat, psi: TTVec, z: TTVec, alpha0: float = 0.0,
                 alpha1: float = 0.01, tol: float = 1e-9, eps_op: float = 1e-13, max_alpha: int = 50,
                 tol_k: float = 1e-10, eps_round: float = 1e-12, eps_solve: float = 1e-11, max_outer: int = 200,
                 rmax: int = 1 << 20, max_sweeps: int = 20, restart: int = 40, max_restarts: int = 50,
                 hist_cap: int = 64, matvec: str = "exact", mv_max_sweeps: int = 10, stream=None) -> AlphaResult:
    """alpha eigenvalue by the secant loop around the device k-eff solve (NEXT-2)."""
    ko = _keff_opts(tol_k, -1.0, eps_round, eps_solve, max_outer, rmax, max_sweeps, restart, max_restarts, matvec,
                    mv_max_sweeps)
    o = _lib.alpha_opts(float(alpha0), float(alpha1), float(tol), float(eps_op), int(max_alpha), ko)
    dev = psi.device
    a = torch.zeros(1, dtype=torch.float64, device=dev)
    k = torch.zeros(1, dtype=torch.float64, device=dev)
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    ah = torch.zeros(hist_cap, dtype=torch.float64, device=dev)
    kh = torch.zeros(hist_cap, dtype=torch.float64, device=dev)
    ih = torch.zeros(hist_cap, dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    rep = _lib.alpha_report(a.data_ptr(), k.data_ptr(), it.data_ptr(), ah.data_ptr(), kh.data_ptr(), ih.data_ptr(),
                            int(hist_cap), st.data_ptr())
    nb = lib().alpha_workspace(H.c, V.c, S.c, F.c, psi.c, z.c, C.byref(o))
    if nb == 0:
        check(lib().alpha_secant(H.c, V.c, S.c, F.c, psi.c, z.c, C.byref(o), C.byref(rep), None, 0,
                                 C.c_void_p(_stream(stream))))
    ws = workspace(nb, dev)
    check(lib().alpha_secant(H.c, V.c, S.c, F.c, psi.c, z.c, C.byref(o), C.byref(rep), _ptr(ws), ws.numel(),
                             C.c_void_p(_stream(stream))))
    return AlphaResult(a, k, it, ah, kh, ih, st)


# ------------------------------------------------------------ K11 graphs ---

def set_graph_mode(mode: int):
    """Driver execution mode of the calling thread (include/tt.h tt_set_graph_mode):
    2 device-resident loops (default), 1 replayed sequences + host-polled loops,
    0 no graphs, -1 the environment default."""
    lib().tt_set_graph_mode(int(mode))


def graph_mode() -> int:
    return int(lib().tt_graph_mode())


def graph_stats():
    """(captures, replays, cached graphs) of the calling thread so far."""
    c, r, n = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    lib().tt_graph_stats(C.byref(c), C.byref(r), C.byref(n))
    return c.value, r.value, n.value
