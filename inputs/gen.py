"""Seeded input generators (problem data and random TT cores).

Everything here is *data*: random draws with NumPy PCG64 and problem
descriptions written out as plain arrays.  There is deliberately no operator
assembly, TT algebra or solver arithmetic in this module: the oracle
(`oracle/`) and the CUDA path (`paper_2309_03347_b200/`) each build their own
operators from these arrays.

Array conventions:
  * TT-vector core  : ndarray shape (r_{k-1}, n_k, r_k)        -- logical [a, i, b]
  * TT-matrix core  : ndarray shape (R_{k-1}, m_k, n_k, R_k)   -- logical [a, i, j, b]
    (i = row/output index, j = column/input index, Z27)
  * Values are drawn as one flat vector per core in column-major order (first
    index fastest), which is the device layout of include/tt.h.
  * Core order is (x-bits, y-bits, z-bits, angle, group), first core fastest
    in the linear index (Z28).
"""
from __future__ import annotations

import math
import numpy as np

__all__ = [
    "rng", "draw_core", "random_tt", "random_ttm", "c2_instance", "c2_slice",
    "c5_instance", "octant_signs", "quadrature_s2", "quadrature_ls_style",
    "problem_c1", "problem_c3", "problem_c4", "problem_small_hetero", "quadrature_gl_1d", "problem_slab",
]


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def draw_core(g: np.random.Generator, shape, scale: float = 1.0) -> np.ndarray:
    """One Gaussian core, drawn flat in column-major order then shaped."""
    size = int(np.prod(shape))
    flat = g.standard_normal(size) * scale
    return flat.reshape(shape, order="F")


def random_tt(g, modes, ranks):
    """TT-vector with given modes (len d) and ranks (len d+1, r0=rd=1).

    Entries N(0,1)/sqrt(r_{k-1}) (BASELINE.json configs[1]; reading Z25)."""
    d = len(modes)
    return [draw_core(g, (ranks[k], modes[k], ranks[k + 1]), 1.0 / math.sqrt(ranks[k]))
            for k in range(d)]


def random_ttm(g, rows, cols, ranks):
    d = len(rows)
    return [draw_core(g, (ranks[k], rows[k], cols[k], ranks[k + 1]), 1.0 / math.sqrt(ranks[k]))
            for k in range(d)]


def c2_instance(seed: int, d: int = 30, rlo: int = 20, rhi: int = 64, Rlo: int = 3, Rhi: int = 5):
    """BASELINE.json configs[1]: d QTT cores (2x2 modes), operator ranks U{3..5},
    vector ranks U{20..64}; draw order ranks, matrix cores, vector cores (Z26)."""
    g = rng(seed)
    R = [1] + [int(v) for v in g.integers(Rlo, Rhi + 1, size=d - 1)] + [1]
    r = [1] + [int(v) for v in g.integers(rlo, rhi + 1, size=d - 1)] + [1]
    A = random_ttm(g, [2] * d, [2] * d, R)
    X = random_tt(g, [2] * d, r)
    return {"A": A, "X": X, "R": R, "r": r, "d": d, "seed": seed}


def c2_slice(seed: int, d: int = 10):
    """d=10 slice of configs[1] used for the dense (1024-vector) parity check."""
    return c2_instance(seed, d=d)


def c5_instance(r: int, seed: int, d: int = 40, Rlo: int = 5, Rhi: int = 8):
    """BASELINE.json configs[4]: d cores, modes from {2,4,8,16}, interface rank r
    on every interior bond, operator ranks U{5..8}; X = Y (Galerkin)."""
    g = rng(seed)
    n = [int(v) for v in g.choice(np.array([2, 4, 8, 16]), size=d)]
    R = [1] + [int(v) for v in g.integers(Rlo, Rhi + 1, size=d - 1)] + [1]
    rr = [1] + [r] * (d - 1) + [1]
    A = random_ttm(g, n, n, R)
    X = random_tt(g, n, rr)
    return {"A": A, "X": X, "n": n, "R": R, "r": rr, "d": d, "seed": seed}


# --------------------------------------------------------------------------
# Quadrature (problem data).  Octant order of eq. hat-mu, PAPER.md P:1824-1839:
# b = 1..8 has signs (mu, eta, xi) = (-,-,-), (+,-,-), (-,+,-), (+,+,-),
#                                    (-,-,+), (+,-,+), (-,+,+), (+,+,+).
# --------------------------------------------------------------------------
def octant_signs():
    out = []
    for b in range(8):
        out.append((1 if b & 1 else -1, 1 if b & 2 else -1, 1 if b & 4 else -1))
    return out


def quadrature_s2():
    """S2 of BASELINE.json configs[0]: (+-1/sqrt3)^3 with equal weights 1/8."""
    a = 1.0 / math.sqrt(3.0)
    mu, eta, xi, w = [], [], [], []
    for (sx, sy, sz) in octant_signs():
        mu.append(sx * a); eta.append(sy * a); xi.append(sz * a); w.append(1.0 / 8.0)
    return {"mu": np.array(mu), "eta": np.array(eta), "xi": np.array(xi),
            "w": np.array(w), "per_octant": 1, "name": "S2"}


def quadrature_ls_style(N: int):
    """Level-symmetric-style S_N set: N(N+2)/8 directions per
    octant, levels mu_i^2 = mu_1^2 + (i-1) 2(1-3 mu_1^2)/(N-2), mu_1^2 = 1/(3(N-1)),
    triplets (i,j,k) 1-based with i+j+k = N/2+2 in lexicographic order, equal
    weights 1/L.  No published table is copied."""
    if N == 2:
        return quadrature_s2()
    m1 = 1.0 / (3.0 * (N - 1))
    lev = [math.sqrt(m1 + (i - 1) * 2.0 * (1.0 - 3.0 * m1) / (N - 2)) for i in range(1, N // 2 + 1)]
    trip = [(i, j, k) for i in range(1, N // 2 + 1) for j in range(1, N // 2 + 1)
            for k in range(1, N // 2 + 1) if i + j + k == N // 2 + 2]
    L = 8 * len(trip)
    mu, eta, xi, w = [], [], [], []
    for (sx, sy, sz) in octant_signs():
        for (i, j, k) in trip:
            mu.append(sx * lev[i - 1]); eta.append(sy * lev[j - 1]); xi.append(sz * lev[k - 1])
            w.append(1.0 / L)
    return {"mu": np.array(mu), "eta": np.array(eta), "xi": np.array(xi),
            "w": np.array(w), "per_octant": len(trip), "name": f"S{N}-LS-style"}


# --------------------------------------------------------------------------
# Problems.  A problem is: vertices per axis (power of two for QTT), extent,
# G, quadrature, boundary ("vacuum" | "reflective"), materials and boxes.
# Material m has sigma_t[g], sigma_s[g, g'] (transfer g' -> g, Z4),
# nu_sigma_f[g]; chi[g] is global (Z5).  Boxes are painted in order over a
# background material: cell (cx, cy, cz) takes the material of the LAST box
# [lo, hi)^3 (cell indices) that contains it, else material 0 (Z13, Z34).
# --------------------------------------------------------------------------
def inv_velocity(G: int):
    """1/v per group for the alpha problem (eq. Discretized_alphaNTE, P:341-349;
    reading Z39: the paper's velocities come with its unavailable library).
    One group: v = 1 (alpha in units of v cm^-1).  Multigroup: 1/v rising
    geometrically from 1 (fastest group) to 100 (slowest); no random draws."""
    return np.ones(1) if G == 1 else np.geomspace(1.0, 100.0, G)


def problem_c1(boundary: str = "vacuum"):
    """BASELINE.json configs[0]: unit cube, 8 vertices/axis (7 cells, Z12),
    G=1, S2, Sigma_t=1, Sigma_s=0.5, nu Sigma_f=0.6, chi=1."""
    return {
        "name": f"C1-{boundary}", "nv": 8, "extent": 1.0, "G": 1,
        "quad": quadrature_s2(), "boundary": boundary, "qtt": False,
        "materials": [{"sigma_t": np.array([1.0]), "sigma_s": np.array([[0.5]]),
                       "nu_sigma_f": np.array([0.6])}],
        "chi": np.array([1.0]), "boxes": [], "inv_v": inv_velocity(1),
    }


def _draw_material(g, G, fissile, upscatter_from=None):
    """SURVEY.md Z14 draws (problem data)."""
    st = g.uniform(0.5, 1.5, size=G)
    ss = np.zeros((G, G))
    for gp in range(G):
        ss[gp, gp] = 0.6 * st[gp]
        below = list(range(gp + 1, G))
        frac_down = 0.2
        if upscatter_from is not None and gp >= upscatter_from:
            up = list(range(upscatter_from - 1, gp))
            for gg in up:
                ss[gg, gp] += 0.05 * st[gp] / len(up)
            frac_down = 0.15
        for gg in below:
            ss[gg, gp] += frac_down * st[gp] / len(below)
    nsf = g.uniform(0.05, 0.3, size=G) if fissile else np.zeros(G)
    return {"sigma_t": st, "sigma_s": ss, "nu_sigma_f": nsf}


def problem_c3(seed: int = 3, nv: int = 64):
    """BASELINE.json configs[2]: [0,10]^3 cm, 64 vertices/axis, G=7 downscatter,
    S8 LS-style (80 ordinates), vacuum, fuel cells [16,48)^3 in a reflector.
    nv < 64 gives the same problem on a coarser grid (fuel cells
    [nv/4, 3nv/4)^3), used for parity at sizes the oracle finishes quickly."""
    g = rng(seed)
    G = 7
    refl = _draw_material(g, G, fissile=False)
    fuel = _draw_material(g, G, fissile=True)
    chi = np.zeros(G); chi[0] = 0.7; chi[1] = 0.3
    return {
        "name": "C3" if nv == 64 else f"C3-nv{nv}", "nv": nv, "extent": 10.0, "G": G,
        "quad": quadrature_ls_style(8), "boundary": "vacuum", "qtt": True, "materials": [refl, fuel], "chi": chi,
        "boxes": [((nv // 4,) * 3, (3 * nv // 4,) * 3, 1)], "seed": seed, "inv_v": inv_velocity(G),
    }


def problem_c4(seed: int = 4, nv: int = 256):
    """BASELINE.json configs[3]: 256 vertices/axis, G=30 with upscatter in groups
    26-30 (1-based), S16 LS-style (288), core/blanket/reflector (Z13).
    nv < 256 gives the same materials on a coarser grid (blanket cells
    [nv/8, 7nv/8)^3, core [nv/4, 3nv/4)^3), used for parity at sizes the
    oracle's matrix-free sweep finishes quickly."""
    g = rng(seed)
    G = 30
    refl = _draw_material(g, G, fissile=False, upscatter_from=26)
    blanket = _draw_material(g, G, fissile=True, upscatter_from=26)
    core = _draw_material(g, G, fissile=True, upscatter_from=26)
    chi = np.zeros(G); chi[0] = 0.7; chi[1] = 0.3
    b0, b1, c0, c1 = nv // 8, 7 * nv // 8, nv // 4, 3 * nv // 4
    return {
        "name": "C4" if nv == 256 else f"C4-nv{nv}", "nv": nv, "extent": 10.0, "G": G,
        "quad": quadrature_ls_style(16),
        "boundary": "vacuum", "qtt": True, "materials": [refl, blanket, core], "chi": chi,
        "boxes": [((b0,) * 3, (b1,) * 3, 1), ((c0,) * 3, (c1,) * 3, 2)],
        "seed": seed, "inv_v": inv_velocity(G),
    }


def quadrature_gl_1d(L: int):
    """1-D slab S_L set: Gauss-Legendre nodes on [-1, 1] with weights normalised to
    sum 1; ordered as the two half-range blocks [mu_-; mu_+]
    (P:1819-1822), each ascending.  (Reading: the paper does not name its 1-D set.)"""
    x, w = np.polynomial.legendre.leggauss(L)
    order = np.argsort(x)
    x, w = x[order], w[order] / np.sum(w)
    return {"mu": x, "w": w, "per_octant": L // 2, "name": f"GL-S{L}"}


def problem_slab(L: int = 8, nv: int = 1024, qtt: bool = True):
    """PAPER.md §3.5.1, Table 1: one-group Pu-239
    slab of width 3.707444 cm, nu = 3.24, sigma_f = 0.0816, sigma_s = 0.225216,
    sigma_t = 0.3264 cm^-1, vacuum boundaries, exactly critical (k = 1);
    1024 spatial points (vertices, reading Z12), L ordinates."""
    return {
        "name": f"slab-L{L}", "dim": 1, "nv": nv, "extent": 3.707444, "G": 1,
        "quad": quadrature_gl_1d(L), "boundary": "vacuum", "qtt": qtt,
        "materials": [{"sigma_t": np.array([0.3264]), "sigma_s": np.array([[0.225216]]),
                       "nu_sigma_f": np.array([3.24 * 0.0816])}],
        "chi": np.array([1.0]), "boxes": [], "inv_v": inv_velocity(1),
    }


def problem_small_hetero(seed: int = 7, nv: int = 8, G: int = 2, N: int = 2, qtt: bool = False):
    """Small two-region problem for dense cross-checks of heterogeneous assembly
    (8^3, G=2, two regions)."""
    g = rng(seed)
    m0 = _draw_material(g, G, fissile=False)
    m1 = _draw_material(g, G, fissile=True)
    chi = np.zeros(G); chi[0] = 1.0
    lo = nv // 4; hi = nv - nv // 4
    return {
        "name": f"hetero-{nv}", "nv": nv, "extent": 1.0, "G": G, "quad": quadrature_ls_style(N),
        "boundary": "vacuum", "qtt": qtt, "materials": [m0, m1], "chi": chi,
        "boxes": [((lo, lo, lo), (hi - 1, hi, hi), 1)], "seed": seed, "inv_v": inv_velocity(G),
    }
