"""ORACLE (test infrastructure only) — transport operators H, S, F.

Follows PAPER.md §3.2 and eq. Discretized_kNTE with
the readings of SURVEY.md §8(c).3 (listed in DESIGN.md):
  Z1  F = fission, S = scattering (labels at P:990-991 swapped)
  Z3  Intg^b = C_b 1_L w^T (full-L reading of P:1254)
  Z4  S energy factor = full transfer matrix sigma_s[g <- g']
  Z5  F energy factor = chi nu_sigma_f^T
  Z6  boundary rows follow the displayed matrices
  Z7  row -> cell association is octant dependent
  Z12 nv vertices per axis, nv-1 cells, Delta = extent / (nv-1)
  Z28 core order (x, y, z, angle, group), first index fastest
  Z34 heterogeneous cross sections by painted boxes, octant-shifted cells

Two independent constructions are provided and pinned against each other:
  * `dense_operators`: Kronecker sums of the per-octant factor matrices;
  * `eq4_apply`: the row equations of eq. Discretized_kNTE evaluated with
    explicit index loops (interior rows), generalised per octant (Z7).
"""
from __future__ import annotations

import math
import numpy as np

from . import tt as ott

# ----------------------------------------------------------- factors ---


def D_plus(n, h):
    """D^+_x: (1/h) lower bidiagonal, diag 1, sub-diagonal -1."""
    M = np.eye(n) - np.eye(n, k=-1)
    return M / h


def D_minus(n, h):
    """D^-_x: (1/h) upper bidiagonal, diag -1, super-diagonal 1."""
    M = -np.eye(n) + np.eye(n, k=1)
    return M / h


def Ip_minus(n):
    """Ip^-_x: 1/2 upper bidiagonal (1, 1), last row (0 .. 0 1)."""
    return 0.5 * (np.eye(n) + np.eye(n, k=1))


def Ip_plus(n):
    """Ip^+_x: 1/2 lower bidiagonal (1, 1), first row (1 0 .. 0)."""
    return 0.5 * (np.eye(n) + np.eye(n, k=-1))


def Ip_minus_noBC(n):
    """Ip^-_{x,noBC}: Ip^- with the last row zeroed."""
    M = Ip_minus(n)
    M[-1, :] = 0.0
    return M


def Ip_plus_noBC(n):
    """Ip^+_{x,noBC}: Ip^+ with the first row zeroed."""
    M = Ip_plus(n)
    M[0, :] = 0.0
    return M


def D_s(s, n, h):
    return D_plus(n, h) if s > 0 else D_minus(n, h)


def Ip_s(s, n):
    return Ip_plus(n) if s > 0 else Ip_minus(n)


def IpN_s(s, n):
    return Ip_plus_noBC(n) if s > 0 else Ip_minus_noBC(n)


def octant_of(quad):
    """Octant index b (0-based) of every ordinate, from the signs of (mu, eta, xi)."""
    mu, eta, xi = quad["mu"], quad["eta"], quad["xi"]
    return ((mu > 0).astype(int) + 2 * (eta > 0).astype(int) + 4 * (xi > 0).astype(int))


def C_b(quad, b):
    """C_b: L x L selector of octant block b."""
    return np.diag((octant_of(quad) == b).astype(float))


def cell_of_row(s, n):
    """Z7: in an octant with sign s on this axis, row (vertex) i stores the cell
    equation of cell i - [s > 0]; inflow-face rows are clamped into range."""
    c = np.arange(n) - (1 if s > 0 else 0)
    return np.clip(c, 0, n - 2)


def material_map(prob):
    """Material index of every cell (ncell^3 array indexed [cz, cy, cx])."""
    nc = prob["nv"] - 1
    mat = np.zeros((nc, nc, nc), dtype=int)
    for (lo, hi, m) in prob["boxes"]:
        mat[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = m
    return mat


def box_terms(prob):
    """Decompose the painted material field into a background plus separable
    box indicators: field = m0 + sum_t 1_box_t (m_t - parent_t) (Z34).
    Requires each box's footprint to be uniform before it is painted
    (nested or disjoint boxes)."""
    nc = prob["nv"] - 1
    mat = np.zeros((nc, nc, nc), dtype=int)
    terms = []
    for (lo, hi, m) in prob["boxes"]:
        foot = mat[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        parent = int(foot.flat[0])
        if not np.all(foot == parent):
            raise ValueError("boxes must be nested or disjoint")
        terms.append((lo, hi, m, parent))
        mat[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = m
    return terms


# ---------------------------------------------------- rank-1 term lists ---
# A term is (coefficient-free) list of 5 factor matrices in core order
# [F_x, F_y, F_z, F_angle, F_group]; the operator is the sum of their Kronecker
# products  F_group (x) F_angle (x) F_z (x) F_y (x) F_x  (paper order).


def _axis_indicator(s, n, lo, hi):
    c = cell_of_row(s, n)
    return np.diag(((c >= lo) & (c < hi)).astype(float))


def operator_terms(prob):
    """Rank-1 terms of H = H_x + H_y + H_z + H_sigma,
    S and F, each summed over the 8 octants (bci)."""
    if prob.get("dim", 3) == 1:
        return operator_terms_1d(prob)
    n = prob["nv"]
    h = prob["extent"] / (n - 1)
    quad = prob["quad"]
    G = prob["G"]
    mats = prob["materials"]
    chi = prob["chi"]
    L = len(quad["w"])
    w = quad["w"]
    I_G = np.eye(G)
    terms = box_terms(prob)
    H, S, F, V = [], [], [], []
    inv_v = prob.get("inv_v")
    for b in range(8):
        sx, sy, sz = (1 if b & 1 else -1, 1 if b & 2 else -1, 1 if b & 4 else -1)
        Cb = C_b(quad, b)
        Qmu = Cb @ np.diag(quad["mu"])
        Qeta = Cb @ np.diag(quad["eta"])
        Qxi = Cb @ np.diag(quad["xi"])
        Intg = Cb @ np.outer(np.ones(L), w)                       # Z3 full-L
        Dx, Dy, Dz = D_s(sx, n, h), D_s(sy, n, h), D_s(sz, n, h)
        Ix, Iy, Iz = Ip_s(sx, n), Ip_s(sy, n), Ip_s(sz, n)
        Nx, Ny, Nz = IpN_s(sx, n), IpN_s(sy, n), IpN_s(sz, n)
        H.append([Dx, Iy, Iz, Qmu, I_G])                            # H_x^{TT,b}
        H.append([Ix, Dy, Iz, Qeta, I_G])                           # H_y^{TT,b}
        H.append([Ix, Iy, Dz, Qxi, I_G])                            # H_z^{TT,b}
        # H_sigma^{TT,b} = diag(sigma) o C_b o Ip o Ip o Ip, with box terms (Z34)
        m0 = mats[0]
        H.append([Ix, Iy, Iz, Cb, np.diag(m0["sigma_t"])])
        S.append([Nx, Ny, Nz, Intg, m0["sigma_s"]])
        F.append([Nx, Ny, Nz, Intg, np.outer(chi, m0["nu_sigma_f"])])
        if inv_v is not None:
            # (V^{-1})^{TT,b} = diag(1/v) o (C_b (x) I) o Ip_z o Ip_y o Ip_x
            V.append([Ix, Iy, Iz, Cb, np.diag(inv_v)])
        for (lo, hi, m, parent) in terms:
            Ex = _axis_indicator(sx, n, lo[0], hi[0])
            Ey = _axis_indicator(sy, n, lo[1], hi[1])
            Ez = _axis_indicator(sz, n, lo[2], hi[2])
            dst = mats[m]["sigma_t"] - mats[parent]["sigma_t"]
            dss = mats[m]["sigma_s"] - mats[parent]["sigma_s"]
            dnf = mats[m]["nu_sigma_f"] - mats[parent]["nu_sigma_f"]
            H.append([Ex @ Ix, Ey @ Iy, Ez @ Iz, Cb, np.diag(dst)])
            if np.any(dss != 0):
                S.append([Ex @ Nx, Ey @ Ny, Ez @ Nz, Intg, dss])
            if np.any(dnf != 0):
                F.append([Ex @ Nx, Ey @ Ny, Ez @ Nz, Intg, np.outer(chi, dnf)])
    out = {"H": H, "S": S, "F": F}
    if inv_v is not None:
        out["V"] = V
    return out


def operator_terms_1d(prob):
    """1-D slab: the construction of P:1219-1293 restricted to the x
    factor; the two half-range blocks b = 0 (mu < 0), 1 (mu > 0) play the octants.
    Terms in core order [F_x, F_angle, F_group]."""
    n = prob["nv"]
    h = prob["extent"] / (n - 1)
    quad = prob["quad"]
    mu, w = quad["mu"], quad["w"]
    L = len(w)
    G = prob["G"]
    m0 = prob["materials"][0]
    chi = prob["chi"]
    H, S, F, V = [], [], [], []
    inv_v = prob.get("inv_v")
    for b, sx in ((0, -1), (1, 1)):
        Cb = np.diag(((mu > 0) == (sx > 0)).astype(float))
        H.append([D_s(sx, n, h), Cb @ np.diag(mu), np.eye(G)])
        H.append([Ip_s(sx, n), Cb, np.diag(m0["sigma_t"])])
        Intg = Cb @ np.outer(np.ones(L), w)
        S.append([IpN_s(sx, n), Intg, m0["sigma_s"]])
        F.append([IpN_s(sx, n), Intg, np.outer(chi, m0["nu_sigma_f"])])
        if inv_v is not None:
            V.append([Ip_s(sx, n), Cb, np.diag(inv_v)])          # P:1233-1237 in 1-D
    out = {"H": H, "S": S, "F": F}
    if inv_v is not None:
        out["V"] = V
    return out


def kron_term(term):
    if len(term) == 3:
        Fx, Fa, Fg = term
        return np.kron(Fg, np.kron(Fa, Fx))
    Fx, Fy, Fz, Fa, Fg = term
    return np.kron(Fg, np.kron(Fa, np.kron(Fz, np.kron(Fy, Fx))))


def slab_eq_apply(prob, psi):
    """Row equations of the 1-D diamond-difference slab (the 1-D form of eq.
    Discretized_kNTE) by explicit loops: for ordinate l with mu > 0
    the row of vertex i >= 1 is the balance of cell (i-1, i); for mu < 0 the row
    of vertex i <= n-2 is the balance of cell (i, i+1).  Returns (H psi, S psi,
    F psi, interior mask); inflow rows are NaN."""
    n = prob["nv"]
    h = prob["extent"] / (n - 1)
    mu, w = prob["quad"]["mu"], prob["quad"]["w"]
    L = len(w)
    m0 = prob["materials"][0]
    st, ss, nf = m0["sigma_t"][0], m0["sigma_s"][0, 0], m0["nu_sigma_f"][0]
    P = psi.reshape(L, n)
    phi = w @ P
    Hv = np.full(L * n, np.nan); Sv = np.full(L * n, np.nan); Fv = np.full(L * n, np.nan)
    mask = np.zeros(L * n, dtype=bool)
    for l in range(L):
        for i in range(n):
            lo, hi = (i - 1, i) if mu[l] > 0 else (i, i + 1)
            if lo < 0 or hi > n - 1:
                continue
            row = i + n * l
            Hv[row] = mu[l] / h * (P[l, hi] - P[l, lo]) + st / 2 * (P[l, lo] + P[l, hi])
            Sv[row] = ss / 2 * (phi[lo] + phi[hi])
            Fv[row] = nf / 2 * (phi[lo] + phi[hi])
            mask[row] = True
    return Hv, Sv, Fv, mask


def slab_keff_sweep(prob, tol=1e-12, max_it=100000, alpha=0.0):
    """Matrix-free Eq. 8 for the 1-D slab: H^{-1} is a transport sweep
    (per ordinate, forward substitution from the inflow face); S and F act
    through the scalar flux phi = sum_l w_l psi_l.  alpha != 0 solves the k problem
    of [alpha V^{-1} + H]: in the slab V^{-1} = Ip o C_b o diag(1/v)
    has the collision term's structure, so it enters as
    sigma_t + alpha / v.  Returns (k, psi, iterations)."""
    n = prob["nv"]
    h = prob["extent"] / (n - 1)
    mu, w = prob["quad"]["mu"], prob["quad"]["w"]
    L = len(w)
    m0 = prob["materials"][0]
    st, ss, nf = m0["sigma_t"][0], m0["sigma_s"][0, 0], m0["nu_sigma_f"][0]
    st = st + alpha * prob.get("inv_v", np.ones(1))[0]

    def rhs(psi, k):
        phi = w @ psi
        q = np.zeros((L, n))
        cell = (ss + nf / k) / 2 * (phi[:-1] + phi[1:])       # per cell (i, i+1)
        for l in range(L):
            if mu[l] > 0:
                q[l, 1:] = cell
            else:
                q[l, :-1] = cell
        return q

    def sweep(q):
        psi = np.zeros((L, n))
        for l in range(L):
            a = abs(mu[l]) / h
            if mu[l] > 0:                       # inflow at i = 0: psi_0 = 0
                for i in range(1, n):
                    psi[l, i] = (q[l, i] - (-a + st / 2) * psi[l, i - 1]) / (a + st / 2)
            else:                               # inflow at i = n-1
                for i in range(n - 2, -1, -1):
                    psi[l, i] = (q[l, i] - (-a + st / 2) * psi[l, i + 1]) / (a + st / 2)
        return psi

    def fsum(psi):
        phi = w @ psi
        return nf / 2 * np.sum(phi[:-1] + phi[1:])   # sum of F psi up to the factor L (cancels in k)

    psi = np.ones((L, n))
    k = 1.0
    for it in range(1, max_it + 1):
        new = sweep(rhs(psi, k))
        knew = k * fsum(new) / fsum(psi)
        psi = new / np.linalg.norm(new)
        if abs(knew - k) < tol:
            return knew, psi.reshape(-1), it
        k = knew
    return k, psi.reshape(-1), max_it


def keff_sweep_3d(prob, tol=1e-10, max_it=10000, alpha=0.0, verbose=False):
    """Matrix-free Eq. 8 for the 3-D vertex-DD problem with vacuum
    boundaries: H^{-1} is, per (group, ordinate), a
    transport sweep in the octant's direction solving the cell
    equations of eq. Discretized_kNTE (row vertex = the cell's
    downstream corner, Z7) for the downstream corner, with psi = 0 on inflow
    faces (Z33); S and F act through the scalar flux phi_g = sum_l w_l psi_{g,l}
    averaged over the 8 corners of each cell with that cell's cross sections
    (Z4, Z5, Z34).  alpha adds alpha/v_g to sigma_t (the alpha term of eq.
    Discretized_alphaNTE).  Sweeps run over wavefront planes
    i + j + k = const, vectorised over (group, ordinate).  Returns (k, psi, it)
    with psi shaped (G, L, n, n, n) [g, l, z, y, x]."""
    if prob.get("boundary", "vacuum") != "vacuum" or prob.get("dim", 3) != 3:
        raise ValueError("keff_sweep_3d: 3-D vacuum problems only")
    n = prob["nv"]
    nc = n - 1
    h = prob["extent"] / nc
    quad = prob["quad"]
    G = prob["G"]
    L = len(quad["w"])
    w = quad["w"]
    mats = prob["materials"]
    chi = prob["chi"]
    inv_v = prob.get("inv_v", np.ones(G))
    mat = material_map(prob)                                   # [cz, cy, cx]
    st = np.zeros((G, nc, nc, nc))
    for m, M in enumerate(mats):
        st[:, mat == m] = (M["sigma_t"] + alpha * inv_v)[:, None]
    octs = octant_of(quad)
    # wavefront planes of the +++ sweep (vertices 1..n-1 on every axis)
    ii, jj, kk = np.meshgrid(np.arange(1, n), np.arange(1, n), np.arange(1, n), indexing="ij")
    pl = (ii + jj + kk).ravel()
    vflat = (ii + n * (jj + n * kk)).ravel()
    cflat = ((ii - 1) + nc * ((jj - 1) + nc * (kk - 1))).ravel()
    planes = [(vflat[pl == p], cflat[pl == p]) for p in range(3, 3 * (n - 1) + 1)]
    corners = [(dx, dy, dz) for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)]

    def cell_avg(phi):                                         # phi [g, z, y, x] -> [g, cz, cy, cx]
        acc = np.zeros((phi.shape[0], nc, nc, nc))
        for (dx, dy, dz) in corners:
            acc += phi[:, dz:dz + nc, dy:dy + nc, dx:dx + nc]
        return acc / 8.0

    def source(psi, k):
        phi8 = cell_avg(np.einsum("l,glzyx->gzyx", w, psi))
        q = np.zeros((G, nc, nc, nc))
        for m, M in enumerate(mats):
            Mk = M["sigma_s"] + np.outer(chi, M["nu_sigma_f"]) / k
            sel = mat == m
            q[:, sel] = Mk @ phi8[:, sel]
        return q

    def fsum(psi):
        phi8 = cell_avg(np.einsum("l,glzyx->gzyx", w, psi))
        tot = 0.0
        for m, M in enumerate(mats):
            tot += np.sum(M["nu_sigma_f"][:, None] * phi8[:, mat == m])
        return tot

    def sweep(q):
        psi = np.zeros((G, L, n, n, n))
        for b in range(8):
            lb = np.nonzero(octs == b)[0]
            if lb.size == 0:
                continue
            flips = [ax for ax, bit in ((3, 1), (2, 2), (1, 4)) if not (b & bit)]   # axes of [g, z, y, x]
            qb = np.flip(q, axis=flips) if flips else q
            sb = np.flip(st, axis=flips) if flips else st
            qb = np.ascontiguousarray(qb).reshape(G, -1)
            sb = np.ascontiguousarray(sb).reshape(G, -1) / 8.0
            Lb = lb.size
            a = np.tile(np.abs(quad["mu"][lb]) / (4 * h), G)[:, None]
            bb = np.tile(np.abs(quad["eta"][lb]) / (4 * h), G)[:, None]
            c = np.tile(np.abs(quad["xi"][lb]) / (4 * h), G)[:, None]
            X = np.zeros((G * Lb, n ** 3))
            for (vi, ci) in planes:
                s8 = np.repeat(sb[:, ci], Lb, axis=0)
                rhs = np.repeat(qb[:, ci], Lb, axis=0)
                for (dx, dy, dz) in corners[:-1]:
                    coef = a * (2 * dx - 1) + bb * (2 * dy - 1) + c * (2 * dz - 1) + s8
                    rhs = rhs - coef * X[:, vi - (1 - dx) - n * (1 - dy) - n * n * (1 - dz)]
                X[:, vi] = rhs / (a + bb + c + s8)
            Xb = X.reshape(G, Lb, n, n, n)
            if flips:
                Xb = np.flip(Xb, axis=[ax + 1 for ax in flips])
            psi[:, lb] = Xb
        return psi

    psi = np.ones((G, L, n, n, n))
    k = 1.0
    f_old = fsum(psi)
    for it in range(1, max_it + 1):
        new = sweep(source(psi, k))
        f_new = fsum(new)
        knew = k * f_new / f_old
        nn = np.linalg.norm(new)
        psi = new / nn
        f_old = f_new / nn
        if verbose:
            print(it, knew, flush=True)
        if abs(knew - k) < tol:
            return knew, psi, it
        k = knew
    return k, psi, max_it


def dense_operators(prob):
    """Dense H, S, F as sums of Kronecker products."""
    T = operator_terms(prob)
    out = {}
    for key in T:
        out[key] = sum(kron_term(t) for t in T[key])
    if prob.get("boundary", "vacuum") == "reflective":
        out = _reflective(prob, out)
    return out


# ----------------------------------------------------- Eq.-4 index loop ---


def eq4_apply(prob, psi, k_eff=1.0, with_v=False):
    """Evaluate the row equations of eq. Discretized_kNTE with explicit
    index loops, generalised per octant (Z7): the cell of row (i,j,k) in an octant
    with signs s is (i - [s_x>0], j - [s_y>0], k - [s_z>0]).  Returns
    (Hpsi, Spsi, Fpsi, interior_mask) for the interior (cell-equation) rows (with_v:
    also V^{-1} psi from the alpha term of eq. Discretized_alphaNTE); the
    values at inflow-face rows are left as NaN.  psi is the dense vector
    (linearised x fastest, then y, z, angle, group)."""
    n = prob["nv"]
    h = prob["extent"] / (n - 1)
    quad = prob["quad"]
    G = prob["G"]
    L = len(quad["w"])
    mats = prob["materials"]
    chi = prob["chi"]
    mat = material_map(prob)
    P = psi.reshape(G, L, n, n, n)                 # [g, l, z, y, x]
    N = G * L * n ** 3
    Hv = np.full(N, np.nan); Sv = np.full(N, np.nan); Fv = np.full(N, np.nan)
    Vv = np.full(N, np.nan)
    inv_v = prob.get("inv_v", np.ones(G))
    mask = np.zeros(N, dtype=bool)
    # angular integral sum_l' w_l' psi_{g', l'} per vertex (used by both S and F)
    phi = np.einsum("l,glzyx->gzyx", quad["w"], P)
    for g in range(G):
        for l in range(L):
            mu, eta, xi = quad["mu"][l], quad["eta"][l], quad["xi"][l]
            for k in range(n):
                for j in range(n):
                    for i in range(n):
                        # vertex pair (lo, hi) along each axis for this octant
                        i0, i1 = (i - 1, i) if mu > 0 else (i, i + 1)
                        j0, j1 = (j - 1, j) if eta > 0 else (j, j + 1)
                        k0, k1 = (k - 1, k) if xi > 0 else (k, k + 1)
                        if min(i0, j0, k0) < 0 or max(i1, j1, k1) > n - 1:
                            continue                      # inflow-face (BC) row
                        row = i + n * (j + n * (k + n * (l + L * g)))
                        c = mat[k0, j0, i0]
                        st = mats[c]["sigma_t"][g]
                        sx = sum(P[g, l, kk, jj, i1] - P[g, l, kk, jj, i0]
                                 for kk in (k0, k1) for jj in (j0, j1))
                        sy = sum(P[g, l, kk, j1, ii] - P[g, l, kk, j0, ii]
                                 for kk in (k0, k1) for ii in (i0, i1))
                        sz = sum(P[g, l, k1, jj, ii] - P[g, l, k0, jj, ii]
                                 for jj in (j0, j1) for ii in (i0, i1))
                        s8 = sum(P[g, l, kk, jj, ii] for kk in (k0, k1)
                                 for jj in (j0, j1) for ii in (i0, i1))
                        Hv[row] = mu / (4 * h) * sx + eta / (4 * h) * sy + xi / (4 * h) * sz + st / 8 * s8
                        Vv[row] = inv_v[g] / 8 * s8        # alpha term of eq. Discretized_alphaNTE
                        scat = 0.0
                        fis = 0.0
                        for gp in range(G):
                            p8 = sum(phi[gp, kk, jj, ii] for kk in (k0, k1)
                                     for jj in (j0, j1) for ii in (i0, i1))
                            scat += mats[c]["sigma_s"][g, gp] * p8 / 8
                            fis += chi[g] * mats[c]["nu_sigma_f"][gp] * p8 / 8
                        Sv[row] = scat
                        Fv[row] = fis
                        mask[row] = True
    if with_v:
        return Hv, Sv, Fv, Vv, mask
    return Hv, Sv, Fv, mask


# --------------------------------------------------------- reflective ---


def _reflective(prob, ops):
    """Reading Z15 (not in the paper): each inflow-face row of ordinate l is
    replaced by psi_l(face) - psi_refl(l)(face) = 0; S and F rows there are zero.
    refl flips the cosine normal to the first inflow axis (x, y, z order)."""
    n = prob["nv"]
    quad = prob["quad"]
    G = prob["G"]
    L = len(quad["w"])
    H = ops["H"].copy(); S = ops["S"].copy(); F = ops["F"].copy()
    V = ops["V"].copy() if "V" in ops else None
    cos = np.stack([quad["mu"], quad["eta"], quad["xi"]], axis=1)
    for g in range(G):
        for l in range(L):
            for k in range(n):
                for j in range(n):
                    for i in range(n):
                        idx = (i, j, k)
                        axis = None
                        for a in range(3):
                            inflow = 0 if cos[l, a] > 0 else n - 1
                            if idx[a] == inflow:
                                axis = a
                                break
                        if axis is None:
                            continue
                        target = cos[l].copy(); target[axis] = -target[axis]
                        lr = int(np.argmin(np.sum((cos - target) ** 2, axis=1)))
                        row = i + n * (j + n * (k + n * (l + L * g)))
                        col = i + n * (j + n * (k + n * (lr + L * g)))
                        H[row, :] = 0.0; S[row, :] = 0.0; F[row, :] = 0.0
                        if V is not None:
                            V[row, :] = 0.0
                        H[row, row] = 1.0
                        H[row, col] -= 1.0
    out = {"H": H, "S": S, "F": F}
    if V is not None:
        out["V"] = V
    return out


# ------------------------------------------------------ TT / QTT forms ---


def term_tt(term):
    """Rank-1 TT-matrix of one term (eqn:TT_matrices P:726-729), plain TT cores."""
    return ott.rank1_ttm(term)


def qtt_matrix(Fm, eps=1e-14):
    """Algorithm 1 for one factor: reshape the 2^l x 2^l matrix to
    2x..x2, permute (i_1..i_l, j_1..j_l) -> (i_1, j_1, .., i_l, j_l) (bits LSB first,
    Z28), TT-SVD with modes 4 (row bit fastest), cores [r, 2, 2, r']."""
    n = Fm.shape[0]
    l = int(round(math.log2(n)))
    if 2 ** l != n or l == 0:
        raise ValueError("Alg. 1 needs a power-of-two mode >= 2")
    T = Fm.reshape([2] * l + [2] * l, order="F")          # (i_0..i_{l-1}, j_0..j_{l-1})
    perm = []
    for t in range(l):
        perm += [t, l + t]
    T = np.transpose(T, perm)                             # (i_0, j_0, i_1, j_1, ...)
    cores = ott.tt_svd(T.reshape(-1, order="F"), [4] * l, eps)
    return [c.reshape(c.shape[0], 2, 2, c.shape[2], order="F") for c in cores]


def term_qtt(term):
    """QTT form of one term: spatial factors via Alg. 1, angle and group kept as
    plain TT cores (mixed TT/QTT)."""
    cores = []
    for F in term[:-2]:
        cores += qtt_matrix(F)
    Fa, Fg = term[-2], term[-1]
    cores.append(Fa.reshape(1, Fa.shape[0], Fa.shape[1], 1))
    cores.append(Fg.reshape(1, Fg.shape[0], Fg.shape[1], 1))
    return cores


def ttm_sum_round(term_list, eps=1e-13, rmax=10**9):
    """Sum rank-1 TT-matrices (ranks add) then round them as TT-vectors
    with mode m_k n_k ('a rank reduction step could be necessary')."""
    rows = [c.shape[1] for c in term_list[0]]
    cols = [c.shape[2] for c in term_list[0]]
    acc = None
    for T in term_list:
        V = ott.ttm_as_tt(T)
        acc = V if acc is None else ott.tt_add(acc, V)
    rounded, _ = ott.tt_round(acc, eps, rmax)
    return ott.tt_as_ttm(rounded, rows, cols)


def tt_operators(prob, eps=1e-13, qtt=None):
    """H, S, F as TT-matrices (QTT spatial cores when prob['qtt'])."""
    if qtt is None:
        qtt = prob.get("qtt", False)
    T = operator_terms(prob)
    make = term_qtt if qtt else term_tt
    return {key: ttm_sum_round([make(t) for t in T[key]], eps) for key in T}


def ones_tt(mode_sizes):
    return [np.ones((1, n, 1)) for n in mode_sizes]


def qtt_modes(prob):
    n = prob["nv"]
    l = int(round(math.log2(n)))
    L = len(prob["quad"]["w"])
    return [2] * (prob.get("dim", 3) * l) + [L, prob["G"]]


def tt_modes(prob):
    n = prob["nv"]
    return [n] * prob.get("dim", 3) + [len(prob["quad"]["w"]), prob["G"]]
