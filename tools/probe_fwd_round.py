"""Localise the accuracy loss of the device rounding on an exact index-forwarding
TT (device Alg. 1): build the TT on the host, run tt_orthogonalize(-1) and
tt_orthogonalize(+1) and tt_round(eps=0) on the device; print the per-core
orthogonality and the reconstruction error after each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_03347_b200 as tb  # noqa: E402
from oracle import transport as T  # noqa: E402
from oracle import tt as ott  # noqa: E402


def forward_tt(M):
    n = M.shape[0]
    l = int(round(np.log2(n)))
    h = l // 2
    rk = [4 ** min(t, l - t) for t in range(l + 1)]
    cores = []
    for t in range(l):
        c = np.zeros((rk[t], 4, rk[t + 1]))
        for a in range(rk[t]):
            for i in range(4):
                if t < h:
                    c[a, i, a + rk[t] * i] = 1.0
                elif t > h:
                    if a % 4 == i:
                        c[a, i, a // 4] = 1.0
        if t == h:
            for a in range(rk[t]):
                for i in range(4):
                    for b in range(rk[t + 1]):
                        row = col = 0
                        s = 0
                        for k in range(h):
                            dg = (a >> (2 * k)) & 3
                            row |= (dg & 1) << s; col |= (dg >> 1) << s; s += 1
                        row |= (i & 1) << s; col |= (i >> 1) << s; s += 1
                        for k in range(l - h - 1):
                            dg = (b >> (2 * k)) & 3
                            row |= (dg & 1) << s; col |= (dg >> 1) << s; s += 1
                        c[a, i, b] = M[row, col]
        cores.append(c)
    return cores


def orth_err(cores, side):
    out = []
    for c in cores:
        r0, n, r1 = c.shape
        if side < 0:
            Mx = c.reshape(r0, n * r1, order="F")
            out.append(np.max(np.abs(Mx @ Mx.T - np.eye(r0))))
        else:
            Mx = c.reshape(r0 * n, r1, order="F")
            out.append(np.max(np.abs(Mx.T @ Mx - np.eye(r1))))
    return out


for name, M in (("Ip-noBC256", T.Ip_minus_noBC(256)), ("rand64", np.random.default_rng(1).standard_normal((64, 64))),
                ("Ip-noBC64", T.Ip_minus_noBC(64))):
    X = forward_tt(M)
    full = ott.tt_full(X)
    print(name, "host forward TT exact:", np.max(np.abs(full - ott.tt_full(ott.tt_svd(full, [4] * len(X), 0.0)))))
    for op in ("orth-", "orth+", "round0"):
        G = tb.TTVec.from_cores(X)
        if op == "orth-":
            tb.tt_orthogonalize(G, -1)
        elif op == "orth+":
            tb.tt_orthogonalize(G, +1)
        else:
            tb.tt_round(G, 0.0)
        torch.cuda.synchronize()
        cs = G.cores()
        err = np.max(np.abs(ott.tt_full(cs) - full)) / np.abs(full).max()
        oe = orth_err(cs[1:], -1) if op == "orth-" else orth_err(cs[:-1], +1)
        print(f"  {op}: ranks {G.ranks()} recon err {err:.2e} orth err per core {[f'{v:.0e}' for v in oe]}",
              flush=True)
