"""Transport operators H, S, F on the device (§3.2-3.3).

The per-octant rank-1 factor matrices come from libtt's host-side C++
constructor (tt_transport_terms); the sum over octants / parts (ranks add,
P:1290-1293) and the rank reduction run on the GPU with
tt_add and tt_round.  One-off setup, not a hot-path step."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .tt import TTMat, TTVec, tt_add, tt_round

OPS = {"H": 0, "S": 1, "F": 2}


def _dp(a):
    return a.ctypes.data_as(C.c_void_p)


def factor_terms(prob, op: str):
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
    nt = lib.tt_transport_terms(*args, None)
    if nt < 0:
        raise _lib.TTError(1, lib.tt_last_error().decode())
    per = 3 * nv * nv + L * L + G * G
    out = np.zeros(nt * per, dtype=np.float64)
    lib.tt_transport_terms(*args, _dp(out))
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


def operator(prob, op: str, eps: float = 1e-13, device="cuda") -> TTMat:
    """Sum of the rank-1 terms (device tt_add), then device tt_round; plain TT
    cores (x, y, z, angle, group)."""
    terms = factor_terms(prob, op)
    rows = [f.shape[0] for f in terms[0]]
    d = len(rows)
    acc = None
    for t, fac in enumerate(terms):
        term = TTVec([n * n for n in rows], [1] * (d + 1), device)
        term.set_cores([f.reshape(1, -1, 1, order="F") for f in fac])
        if acc is None:
            acc = term
            continue
        nxt = TTVec(acc.n, [1] + [t + 1] * (d - 1) + [1], device)
        tt_add(acc, term, nxt)
        acc = nxt
    tt_round(acc, eps)
    R = acc.ranks()
    A = TTMat(rows, rows, R, device)
    # copy the rounded cores into the matrix container (same column-major layout)
    cores = acc.cores()
    A.set_cores([c.reshape(c.shape[0], m, m, c.shape[2], order="F") for c, m in zip(cores, rows)])
    return A


def operators(prob, eps: float = 1e-13, device="cuda"):
    return {k: operator(prob, k, eps, device) for k in ("H", "S", "F")}
