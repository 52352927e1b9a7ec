"""Pins of the oracle transport assembly and eigen drivers (CPU only)."""
import copy
import os

import numpy as np
import pytest

import inputs
from oracle import transport as T
from oracle import tt as ott
from oracle import solvers as so

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def read_golden_matrices(name):
    out, cur = {}, None
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("["):
            cur = line[1:-1]
            out[cur] = []
        else:
            out[cur].append([float(v) for v in line.split()])
    return {k: np.array(v) for k, v in out.items()}


def test_factor_matrices_match_displayed():
    g = read_golden_matrices("factor_matrices_n4.txt")
    assert np.array_equal(T.D_plus(4, 1.0), g["D+"])
    assert np.array_equal(T.D_minus(4, 1.0), g["D-"])
    assert np.array_equal(T.Ip_minus(4), g["Ip-"])
    assert np.array_equal(T.Ip_plus(4), g["Ip+"])
    assert np.array_equal(T.Ip_minus_noBC(4), g["Ip-noBC"])
    assert np.array_equal(T.Ip_plus_noBC(4), g["Ip+noBC"])
    assert np.allclose(T.D_plus(4, 0.5), 2 * g["D+"])


def test_quadrature_sets():
    q = inputs.quadrature_s2()
    assert np.allclose(q["mu"] ** 2 + q["eta"] ** 2 + q["xi"] ** 2, 1.0)
    assert abs(q["w"].sum() - 1.0) < 1e-15
    for N, L in ((4, 24), (8, 80), (16, 288)):
        q = inputs.quadrature_ls_style(N)
        assert len(q["w"]) == L
        assert np.allclose(q["mu"] ** 2 + q["eta"] ** 2 + q["xi"] ** 2, 1.0, atol=1e-14)
        oc = T.octant_of(q)
        assert list(oc) == sorted(oc)                             # octant blocks, eq. hat-mu order
        assert abs(q["w"].sum() - 1.0) < 1e-14


@pytest.mark.parametrize("prob", [inputs.problem_c1(), inputs.problem_small_hetero(nv=4, G=2, N=4)],
                         ids=["C1", "hetero4"])
def test_eq4_rows_match_kronecker_assembly(prob):
    """eq. Discretized_kNTE index loop vs Kronecker sums."""
    ops = T.dense_operators(prob)
    g = inputs.rng(20)
    for _ in range(3):
        psi = g.standard_normal(ops["H"].shape[0])
        Hv, Sv, Fv, mask = T.eq4_apply(prob, psi)
        scale = np.abs(ops["H"]).max() * np.abs(psi).max()
        assert np.max(np.abs(Hv[mask] - (ops["H"] @ psi)[mask])) < 1e-13 * scale
        assert np.max(np.abs(Sv[mask] - (ops["S"] @ psi)[mask])) < 1e-14 * scale
        assert np.max(np.abs(Fv[mask] - (ops["F"] @ psi)[mask])) < 1e-14 * scale
    # number of BC rows: GL[nv^3 - (nv-1)^3] (P:1914 counts the faces)
    n = prob["nv"]
    L = len(prob["quad"]["w"])
    assert (~mask).sum() == prob["G"] * L * (n ** 3 - (n - 1) ** 3)
    # S and F vanish on the inflow-face rows (noBC interpolation)
    assert np.abs(ops["S"][~mask]).max() == 0.0
    assert np.abs(ops["F"][~mask]).max() == 0.0


def test_bc_rows_homogeneous_triangular():
    """Z33: the inflow-face rows of H couple only inflow-face unknowns of the same
    (g, l) and form a triangular system with a positive diagonal."""
    prob = inputs.problem_c1()
    H = T.dense_operators(prob)["H"]
    psi = np.ones(H.shape[0])
    _, _, _, mask = T.eq4_apply(prob, psi)
    bc = np.where(~mask)[0]
    assert np.abs(H[np.ix_(bc, np.where(mask)[0])]).max() == 0.0
    Hb = H[np.ix_(bc, bc)]
    assert np.all(np.diag(Hb) != 0.0)
    # H is (block) triangular in a sweep ordering: its eigenvalues are its diagonal
    ev = np.linalg.eigvals(Hb)
    assert np.allclose(np.sort(np.abs(ev)), np.sort(np.abs(np.diag(Hb))), rtol=1e-8)


def test_tt_operators_c1_exact_ranks_and_dense():
    prob = inputs.problem_c1()
    ops = T.dense_operators(prob)
    tops = T.tt_operators(prob)
    assert ott.ranks(tops["H"]) == [1, 3, 7, 8, 1, 1]             # Z29 exact ranks
    assert ott.ranks(tops["S"]) == [1, 2, 4, 8, 1, 1]
    assert ott.ranks(tops["F"]) == [1, 2, 4, 8, 1, 1]
    for k in "HSF":
        assert np.max(np.abs(ott.ttm_full(tops[k]) - ops[k])) < 1e-12 * np.abs(ops[k]).max()


def test_qtt_alg1_factor_and_operator():
    """Alg. 1 on displayed factor matrices; QTT operator of a small
    heterogeneous problem equals the dense assembly."""
    for M in (T.D_plus(8, 0.25), T.Ip_minus_noBC(8), np.eye(8)):
        cores = T.qtt_matrix(M)
        assert np.allclose(ott.ttm_full(cores), M, atol=1e-13)
        assert max(ott.ranks(cores)) <= 3                     # low-rank Toeplitz QTT
    prob = inputs.problem_small_hetero(nv=4, G=2, N=2, qtt=True)
    ops = T.dense_operators(prob)
    tops = T.tt_operators(prob)
    for k in "HSF":
        assert np.max(np.abs(ott.ttm_full(tops[k]) - ops[k])) < 1e-12 * np.abs(ops[k]).max()


def _small_c1(nv=4, boundary="vacuum"):
    p = inputs.problem_c1(boundary)
    p = copy.deepcopy(p)
    p["nv"] = nv
    return p


def test_keff_power_vs_ges_and_one_group_relation():
    """Eq. 8 power iteration vs the dense generalised eigenproblem, and
    the one-group relation k = nuSf lam / (1 - Ss lam), lam = rho(H^-1 M) with
    S = Ss M, F = nuSf M."""
    prob = _small_c1(4)
    ops = T.dense_operators(prob)
    k, psi, hist = so.keff_dense_power(ops["H"], ops["S"], ops["F"])
    kg, _ = so.keff_dense_ges(ops["H"], ops["S"], ops["F"])
    assert abs(k - kg) / kg < 1e-10
    Mop = ops["S"] / 0.5
    assert np.allclose(ops["F"], 0.6 * Mop, atol=1e-15)
    lam = np.max(np.linalg.eigvals(np.linalg.solve(ops["H"], Mop)).real)
    k1 = 0.6 * lam / (1 - 0.5 * lam)
    assert abs(k - k1) / k1 < 1e-10
    assert np.all(psi * np.sign(psi.sum()) > -1e-12)             # Psi >= 0
    # scale invariance in Psi0
    k2, _, _ = so.keff_dense_power(ops["H"], ops["S"], ops["F"], psi0=7.0 * np.ones(len(psi)))
    assert abs(k2 - k) < 1e-12


def test_keff_c1_vacuum_dense_matches_stored():
    """C1 vacuum (configs[0]) dense k; the stored value is written by
    tests/golden/make_c1_keff.py (oracle only)."""
    val = float(open(os.path.join(GOLD, "c1_keff_vacuum.txt")).read().split()[-1])
    prob = inputs.problem_c1()
    ops = T.dense_operators(prob)
    k, _, hist = so.keff_dense_power(ops["H"], ops["S"], ops["F"])
    assert abs(k - val) < 1e-12
    assert len(hist) < 60


def test_reflective_kinf_and_closed_form_sequence():
    """Reflective variant (Z15): k_inf = nuSf/(St - Ss) = 1.2 (configs[0]) and from
    psi0 = 1, k0 = 1 the sequence k_tau = 1.2 - 0.2 * 0.5^tau (closed form)."""
    prob = _small_c1(4, "reflective")
    ops = T.dense_operators(prob)
    k, psi, hist = so.keff_dense_power(ops["H"], ops["S"], ops["F"], minnorm=True, max_it=80)
    assert abs(k - 0.6 / (1.0 - 0.5)) < 1e-10
    for tau, kt in enumerate(hist[:10], start=1):
        assert abs(kt - (1.2 - 0.2 * 0.5 ** tau)) < 1e-10


def test_criticality_trichotomy():
    """scaling nuSf moves k through 1 monotonically."""
    prob = _small_c1(4)
    ks = []
    for s in (0.5, 1.0, 4.0):
        p = copy.deepcopy(prob)
        p["materials"][0]["nu_sigma_f"] = p["materials"][0]["nu_sigma_f"] * s
        ops = T.dense_operators(p)
        ks.append(so.keff_dense_power(ops["H"], ops["S"], ops["F"])[0])
    assert ks[0] < ks[1] < ks[2]
    assert abs(ks[1] / ks[0] - 2.0) < 1e-9 and abs(ks[2] / ks[1] - 4.0) < 1e-9
