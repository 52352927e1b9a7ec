"""Transport operators H, S, F on the device (§3.2-3.3).

The per-octant rank-1 factor matrices come from libtt's host-side C++
constructor (tt_transport_terms); power-of-two spatial factors are converted to
QTT on the GPU by Algorithm 1 (tt_qtt_matrix_dev: TT-SVD by
rounding the exact index-forwarding TT) when the problem asks for QTT; the sum
over octants / parts (ranks add) and the rank
reduction run on the GPU with tt_add and tt_round.  One-off setup, not
a hot-path step."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .tt import TTMat, TTVec, tt_add, tt_round

OPS = {"H": 0, "S": 1, "F": 2}


def _dp(a):
    return a.ctypes.data_as(C.c_void_p)


def factor_terms_1d(prob, op: str):
    q = prob["quad"]
    nv, G = int(prob["nv"]), int(prob["G"])
    L = len(q["w"])
    m = prob["materials"][0]
    arr = [np.ascontiguousarray(a, dtype=np.float64) for a in
           (q["mu"], q["w"], m["sigma_t"], m["sigma_s"].reshape(-1, order="F"), m["nu_sigma_f"], prob["chi"])]
    args = [OPS[op], nv, float(prob["extent"]), G, L, *[_dp(a) for a in arr]]
    lib = _lib.lib()
    nt = lib.tt_transport_terms_1d(*args, None)
    if nt < 0:
        raise _lib.TTError(1, lib.tt_last_error().decode())
    per = nv * nv + L * L + G * G
    out = np.zeros(nt * per, dtype=np.float64)
    lib.tt_transport_terms_1d(*args, _dp(out))
    terms = []
    for t in range(nt):
        p = out[t * per:(t + 1) * per]
        o, fac = 0, []
        for n in (nv, L, G):
            fac.append(p[o:o + n * n].reshape(n, n, order="F"))
            o += n * n
        terms.append(fac)
    return terms


def _unpack(out, nt, sizes):
    per = sum(n * n for n in sizes)
    terms = []
    for t in range(nt):
        p = out[t * per:(t + 1) * per]
        o, fac = 0, []
        for n in sizes:
            fac.append(p[o:o + n * n].reshape(n, n, order="F"))
            o += n * n
        terms.append(fac)
    return terms


def velocity_terms(prob):
    """Rank-1 terms of V^{-1} from libtt's host constructor."""
    q = prob["quad"]
    dim = int(prob.get("dim", 3))
    nv, G = int(prob["nv"]), int(prob["G"])
    L = len(q["w"])
    inv_v = np.ascontiguousarray(prob["inv_v"], dtype=np.float64)
    arr = [np.ascontiguousarray(q[k], dtype=np.float64) if k in q else None for k in ("mu", "eta", "xi")]
    refl = 1 if prob.get("boundary", "vacuum") == "reflective" else 0
    args = [dim, nv, G, L, *[(_dp(a) if a is not None else None) for a in arr], _dp(inv_v), refl]
    lib = _lib.lib()
    nt = lib.tt_velocity_terms(*args, None)
    if nt < 0:
        raise _lib.TTError(1, lib.tt_last_error().decode())
    sizes = (nv, L, G) if dim == 1 else (nv, nv, nv, L, G)
    out = np.zeros(nt * sum(n * n for n in sizes), dtype=np.float64)
    lib.tt_velocity_terms(*args, _dp(out))
    return _unpack(out, nt, sizes)


def factor_terms(prob, op: str):
    if op == "V":
        return velocity_terms(prob)
    if prob.get("dim", 3) == 1:
        return factor_terms_1d(prob, op)
    q = prob["quad"]
    nv, G = int(prob["nv"]), int(prob["G"])
    L = len(q["w"])
    mats = prob["materials"]
    st = np.ascontiguousarray(np.concatenate([m["sigma_t"] for m in mats]), dtype=np.float64)
    ss = np.ascontiguousarray(np.concatenate([m["sigma_s"].reshape(-1, order="F") for m in mats]), dtype=np.float64)
    nf = np.ascontiguousarray(np.concatenate([m["nu_sigma_f"] for m in mats]), dtype=np.float64)
    chi = np.ascontiguousarray(prob["chi"], dtype=np.float64)
    boxes = prob["boxes"]
    lo = np.ascontiguousarray(np.array([b[0] for b in boxes], dtype=np.int32).reshape(-1))
    hi = np.ascontiguousarray(np.array([b[1] for b in boxes], dtype=np.int32).reshape(-1))
    bm = np.ascontiguousarray(np.array([b[2] for b in boxes], dtype=np.int32))
    arr = [np.ascontiguousarray(q[k], dtype=np.float64) for k in ("mu", "eta", "xi", "w")]
    args = [OPS[op], nv, float(prob["extent"]), G, L, *[_dp(a) for a in arr], len(mats), _dp(st), _dp(ss),
            _dp(nf), _dp(chi), len(boxes), _dp(lo), _dp(hi), _dp(bm)]
    lib = _lib.lib()
    fn = lib.tt_transport_terms_reflective if prob.get("boundary", "vacuum") == "reflective" else lib.tt_transport_terms
    nt = fn(*args, None)
    if nt < 0:
        raise _lib.TTError(1, lib.tt_last_error().decode())
    per = 3 * nv * nv + L * L + G * G
    out = np.zeros(nt * per, dtype=np.float64)
    fn(*args, _dp(out))
    terms = []
    for t in range(nt):
        p = out[t * per:(t + 1) * per]
        o = 0
        fac = []
        for n in (nv, nv, nv, L, G):
            fac.append(p[o:o + n * n].reshape(n, n, order="F"))
            o += n * n
        terms.append(fac)
    return terms


class _QttCache:
    """Device QTT conversion of the factors: one TT-vector slot and workspace per
    matrix size, identical factors (the same D / Ip matrix in several octant
    terms) converted once."""

    def __init__(self):
        self.slots, self.done = {}, {}

    def get(self, M: np.ndarray, eps: float, device):
        key = (M.shape[0], eps, M.tobytes())
        hit = self.done.get(key)
        if hit is not None:
            return hit
        import torch
        from .tt import workspace
        n = M.shape[0]
        l = int(round(np.log2(n)))
        if (1 << l) != n or l < 1:
            raise _lib.TTError(1, "qtt_matrix: n must be a power of two >= 2")
        if n not in self.slots:
            rc = [1 << (2 * min(t, l - t)) for t in range(l + 1)]
            self.slots[n] = TTVec([4] * l, rc, device)
        q = self.slots[n]
        Md = torch.from_numpy(np.ascontiguousarray(M.reshape(-1, order="F"), dtype=np.float64)).to(q.device)
        lib = _lib.lib()
        ws = workspace(lib.tt_qtt_matrix_dev_workspace(q.c), q.device)
        _lib.check(lib.tt_qtt_matrix_dev(n, C.c_void_p(Md.data_ptr()), float(eps), q.c, C.c_void_p(ws.data_ptr()),
                                         ws.numel(), C.c_void_p(torch.cuda.current_stream(q.device).cuda_stream)))
        cores = [c.reshape(c.shape[0], 2, 2, c.shape[2], order="F") for c in q.cores()]
        self.done[key] = cores
        return cores


_QTT = _QttCache()


def qtt_matrix(M: np.ndarray, eps: float = 1e-14, device="cuda"):
    """QTT cores [r, 2, 2, r'] of a 2^l x 2^l matrix by libtt's device Alg. 1."""
    return _QTT.get(np.asarray(M, dtype=np.float64), eps, device)


def term_cores(fac, qtt: bool, device="cuda"):
    """Cores of one rank-1 term in core order (x, y, z, angle, group)."""
    if not qtt:
        return [f.reshape(1, f.shape[0], f.shape[1], 1, order="F") for f in fac]
    cores = []
    for f in fac[:-2]:
        cores += qtt_matrix(f, device=device)
    for f in fac[-2:]:
        cores.append(f.reshape(1, f.shape[0], f.shape[1], 1, order="F"))
    return cores


def _sum_round(term_list, eps, device) -> TTMat:
    rows = [c.shape[1] for c in term_list[0]]
    d = len(rows)
    acc = None
    for cores in term_list:
        r = [c.shape[0] for c in cores] + [1]
        term = TTVec([m * m for m in rows], r, device)
        term.set_cores([c.reshape(c.shape[0], -1, c.shape[3], order="F") for c in cores])
        if acc is None:
            acc = term
            continue
        cap = [1] + [a + b for a, b in zip(acc.rcap[1:-1], term.rcap[1:-1])] + [1]
        nxt = TTVec(acc.n, cap, device)
        tt_add(acc, term, nxt)
        acc = nxt
    tt_round(acc, eps)
    R = acc.ranks()
    A = TTMat(rows, rows, R, device)
    A.set_cores([c.reshape(c.shape[0], m, m, c.shape[2], order="F") for c, m in zip(acc.cores(), rows)])
    return A


def operator(prob, op: str, eps: float = 1e-13, device="cuda", qtt=None) -> TTMat:
    """Sum of the rank-1 terms (device tt_add), then device tt_round."""
    if qtt is None:
        qtt = bool(prob.get("qtt", False))
    terms = factor_terms(prob, op)
    return _sum_round([term_cores(f, qtt, device) for f in terms], eps, device)


def operators(prob, eps: float = 1e-13, device="cuda", qtt=None, velocity=False):
    """H, S, F (and V^{-1} with velocity=True, for the alpha problem)."""
    keys = ("H", "S", "F", "V") if velocity else ("H", "S", "F")
    return {k: operator(prob, k, eps, device, qtt) for k in keys}


def modes(prob, qtt=None):
    if qtt is None:
        qtt = bool(prob.get("qtt", False))
    nv, L, G = int(prob["nv"]), len(prob["quad"]["w"]), int(prob["G"])
    dim = int(prob.get("dim", 3))
    if not qtt:
        return [nv] * dim + [L, G]
    l = int(round(np.log2(nv)))
    return [2] * (dim * l) + [L, G]
