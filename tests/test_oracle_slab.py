"""1-D Pu-239 slab (§3.5.1; Table 1) in the
oracle: exactly critical benchmark, so k -> 1 as the number of ordinates grows
(P:1564).  CPU only."""
import numpy as np

import inputs
from oracle import solvers as so
from oracle import transport as T
from oracle import tt as ott


def test_slab_rows_and_dense_vs_sweep():
    for L in (2, 4):
        p = inputs.problem_slab(L)
        ops = T.dense_operators(p)
        psi = np.random.default_rng(L).standard_normal(ops["H"].shape[0])
        Hv, Sv, Fv, mask = T.slab_eq_apply(p, psi)
        assert np.max(np.abs(Hv[mask] - (ops["H"] @ psi)[mask])) < 1e-12
        assert np.max(np.abs(Sv[mask] - (ops["S"] @ psi)[mask])) < 1e-15
        assert np.max(np.abs(Fv[mask] - (ops["F"] @ psi)[mask])) < 1e-15
        assert (~mask).sum() == L                      # one inflow row per ordinate
        kd, _, _ = so.keff_dense_power(ops["H"], ops["S"], ops["F"], tol=1e-13)
        ks, _, _ = T.slab_keff_sweep(p, tol=1e-13)
        assert abs(kd - ks) < 1e-12


def test_slab_converges_to_critical():
    """Exactly critical (k = 1): k(L) increases toward 1 with L."""
    ks = [T.slab_keff_sweep(inputs.problem_slab(L), tol=1e-12)[0] for L in (2, 8, 32)]
    assert ks[0] < ks[1] < ks[2] < 1.0
    assert 1.0 - ks[2] < 5e-4
    assert 1.0 - ks[1] < 1e-2


def test_slab_qtt_keff_tt_vs_sweep():
    """TT/QTT fixed point (ISTT) vs the matrix-free full-grid iteration (ISFM)
    at L = 4 (agreement ~1e-7 at the 1e-6 tolerance; here tighter)."""
    p = inputs.problem_slab(4)
    tops = T.tt_operators(p, eps=1e-12)
    modes = T.qtt_modes(p)
    assert modes == [2] * 10 + [4, 1]
    g = inputs.rng(70)
    d = len(modes)
    psi0 = [np.ones((1, n, 1)) for n in modes]
    z0 = inputs.random_tt(g, modes, [1] + [3] * (d - 1) + [1])
    k, psi, hist = so.keff_tt(tops["H"], tops["S"], tops["F"], psi0, z0, tol_k=1e-11, eps_round=1e-11,
                              eps_solve=1e-11, rmax=40, dense_max=3000)
    ks, _, _ = T.slab_keff_sweep(p, tol=1e-13)
    assert abs(k - ks) < 1e-8
