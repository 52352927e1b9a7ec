"""Pins of the oracle's alpha-eigenvalue pieces (NEXT-2, CPU only): the velocity
operator V^{-1} against the row equations of eq.
Discretized_alphaNTE, closed forms, and the secant loop
(reading Z32) against a generalised eigensolve."""
import copy

import numpy as np
import scipy.linalg as sla

import inputs
from oracle import solvers as so
from oracle import transport as T
from oracle import tt as ott


def _cube(nv=4, nsf=0.6, boundary="vacuum"):
    p = copy.deepcopy(inputs.problem_c1(boundary))
    p["nv"] = nv
    p["materials"][0]["nu_sigma_f"] = np.array([nsf])
    return p


def test_velocity_operator_vs_row_equations():
    """Dense V^{-1} (Kronecker terms) = the alpha term of the Eq.-5 loop on interior rows."""
    g = inputs.rng(90)
    for prob in (_cube(4), inputs.problem_small_hetero(nv=4, G=2, N=4)):
        ops = T.dense_operators(prob)
        assert "V" in ops
        for _ in range(3):
            psi = g.standard_normal(ops["V"].shape[0])
            _, _, _, Vv, mask = T.eq4_apply(prob, psi, with_v=True)
            got = ops["V"] @ psi
            assert np.max(np.abs(got[mask] - Vv[mask])) <= 1e-13 * np.abs(Vv[mask]).max()


def test_alpha_shift_is_a_total_cross_section_shift():
    """For one group, V^{-1} has the structure of the collision term (P:1225 vs
    P:1233-1237), so H(sigma_t) + alpha V^{-1} = H(sigma_t + alpha / v) exactly."""
    for prob in (_cube(4), _cube(4, boundary="reflective"), inputs.problem_slab(4, nv=16)):
        a = 0.37
        ops = T.dense_operators(prob)
        shifted = copy.deepcopy(prob)
        shifted["materials"][0]["sigma_t"] = prob["materials"][0]["sigma_t"] + a * prob["inv_v"]
        Hs = T.dense_operators(shifted)["H"]
        assert np.max(np.abs(ops["H"] + a * ops["V"] - Hs)) <= 1e-13 * np.abs(Hs).max()


def test_alpha_reflective_closed_form():
    """Reflective homogeneous cube (Z15): k(alpha) = nuSf / (St + alpha/v - Ss), so
    alpha* = v (nuSf + Ss - St) = 0.1 for configs[0]'s data."""
    prob = _cube(4, boundary="reflective")
    ops = T.dense_operators(prob)
    a, k, hist = so.alpha_dense(ops["H"], ops["V"], ops["S"], ops["F"], tol=1e-11, minnorm=True)
    assert abs(a - 0.1) <= 1e-9
    assert abs(hist[0][1] - 1.2) <= 1e-10                    # alpha = 0: k_inf
    assert abs(hist[1][1] - 0.6 / 0.51) <= 1e-10             # alpha = 0.01
    assert len(hist) <= 8


def test_alpha_vs_generalised_eigensolve():
    """At the secant root, alpha is an eigenvalue of (S + F - H) psi = alpha V^{-1} psi
    (eq. OpFormAlphaNTE with k = 1), the rightmost one, with a one-signed
    eigenvector; the sign of alpha follows the criticality of k(0)."""
    for nsf, sign in ((2.8, 1.0), (2.0, -1.0)):
        prob = _cube(4, nsf=nsf)
        ops = T.dense_operators(prob)
        a, k, hist = so.alpha_dense(ops["H"], ops["V"], ops["S"], ops["F"], tol=1e-11)
        assert np.sign(a) == sign and np.sign(hist[0][1] - 1.0) == sign
        ev, vec = sla.eig(ops["S"] + ops["F"] - ops["H"], ops["V"])
        fin = np.isfinite(ev)
        ev, vec = ev[fin], vec[:, fin]
        i = int(np.argmin(np.abs(ev - a)))
        assert abs(ev[i] - a) <= 1e-8 * max(1.0, abs(a))
        assert abs(ev[i].imag) <= 1e-10
        real = ev[np.abs(ev.imag) <= 1e-10].real
        assert a >= real.max() - 1e-8
        v = vec[:, i].real
        v = v * np.sign(v[np.argmax(np.abs(v))])
        assert v.min() >= -1e-10 * np.abs(v).max()


def test_alpha_slab_critical_and_widened():
    """1-D Pu-239 slab: exactly critical, so alpha ~ 0; doubling the
    width makes it supercritical (k(0) > 1, alpha > 0).  The matrix-free secant
    equals the dense one."""
    p = inputs.problem_slab(8, nv=64)

    def keff(prob):
        return lambda a: T.slab_keff_sweep(prob, tol=1e-13, alpha=a)[0]

    a, k, hist = so.alpha_secant(keff(p), tol=1e-11)
    assert abs(a) <= 5e-3
    ops = T.dense_operators(p)
    ad, _, _ = so.alpha_dense(ops["H"], ops["V"], ops["S"], ops["F"], tol=1e-11)
    assert abs(a - ad) <= 1e-9
    w = copy.deepcopy(p)
    w["extent"] = 2 * p["extent"]
    a2, _, hist2 = so.alpha_secant(keff(w), tol=1e-11)
    assert hist2[0][1] > 1.0 and a2 > 0.0


def test_alpha_tt_matches_dense():
    """TT alpha loop (round(H + alpha V^{-1}), keff_tt per alpha) =
    dense alpha on the supercritical 4^3 cube."""
    prob = _cube(4, nsf=2.8)
    ops = T.dense_operators(prob)
    ad, _, _ = so.alpha_dense(ops["H"], ops["V"], ops["S"], ops["F"], tol=1e-11)
    tops = T.tt_operators(prob)
    modes = [4, 4, 4, 8, 1]
    g = inputs.rng(91)
    psi0 = [np.ones((1, n, 1)) for n in modes]
    z0 = inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1])
    at, kt, hist = so.alpha_tt(tops["H"], tops["V"], tops["S"], tops["F"], psi0, z0, tol=1e-10,
                               tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12)
    assert abs(at - ad) <= 1e-8 * abs(ad)
    assert ott.ranks(tops["V"]) == [1, 2, 4, 8, 1, 1]
