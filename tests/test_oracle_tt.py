"""Pins of the oracle TT algebra (oracle/tt.py) against definitions that do not
go through the oracle itself: explicit slice products, np.kron, dense linear
algebra, closed forms.  CPU only."""
import math

import numpy as np
import pytest

import inputs
from oracle import tt as ott


def slice_product(cores, idx):
    """X(i_1..i_d) = G_1(i_1) ... G_d(i_d) (eqn:TT-vector) for one index."""
    M = np.eye(1)
    for G, i in zip(cores, idx):
        M = M @ G[:, i, :]
    return M[0, 0]


def lin(idx, dims):
    v, s = 0, 1
    for i, n in zip(idx, dims):
        v += i * s
        s *= n
    return v


def test_tt_full_matches_slice_products():
    g = inputs.rng(1)
    dims = [3, 4, 2, 5]
    X = inputs.random_tt(g, dims, [1, 2, 3, 4, 1])
    full = ott.tt_full(X)
    for _ in range(40):
        idx = [int(g.integers(0, n)) for n in dims]
        assert abs(full[lin(idx, dims)] - slice_product(X, idx)) < 1e-13


def test_ttm_full_matches_slice_products():
    g = inputs.rng(2)
    rows, cols = [2, 3, 2], [3, 2, 4]
    A = inputs.random_ttm(g, rows, cols, [1, 2, 3, 1])
    full = ott.ttm_full(A)
    for _ in range(40):
        i = [int(g.integers(0, n)) for n in rows]
        j = [int(g.integers(0, n)) for n in cols]
        M = np.eye(1)
        for Ak, a, b in zip(A, i, j):
            M = M @ Ak[:, a, b, :]
        assert abs(full[lin(i, rows), lin(j, cols)] - M[0, 0]) < 1e-13


def test_rank1_ttm_is_kron():
    """eqn:TT_matrices: rank-1 TT-matrix = tensor product of matrices; dense = kron
    with the first factor fastest (Z28)."""
    g = inputs.rng(3)
    Fs = [g.standard_normal((2, 3)), g.standard_normal((3, 3)), g.standard_normal((4, 2))]
    dense = np.kron(Fs[2], np.kron(Fs[1], Fs[0]))
    assert np.allclose(ott.ttm_full(ott.rank1_ttm(Fs)), dense, atol=1e-14, rtol=0)


def test_laplace_kronecker_sum():
    """L3 = L1 o I o I + I o L1 o I + I o I o L1."""
    n = 4
    L1 = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    I = np.eye(n)
    terms = [ott.ttm_as_tt(ott.rank1_ttm(f)) for f in ([L1, I, I], [I, L1, I], [I, I, L1])]
    S = ott.tt_add(ott.tt_add(terms[0], terms[1]), terms[2])
    S = ott.tt_as_ttm(S, [n] * 3, [n] * 3)
    dense = np.kron(L1, np.kron(I, I)) + np.kron(I, np.kron(L1, I)) + np.kron(I, np.kron(I, L1))
    assert np.allclose(ott.ttm_full(S), dense, atol=1e-14, rtol=0)
    assert ott.ranks(S) == [1, 3, 3, 1]


def test_matvec_dense_d10_slice():
    """Exact matvec vs dense 1024x1024 product (BASELINE.json configs[1] d=10 slice)."""
    inst = inputs.c2_slice(100)
    A, X = inst["A"], inst["X"]
    Y = ott.tt_matvec_fast(A, X)
    ref = ott.ttm_full(A) @ ott.tt_full(X)
    err = np.linalg.norm(ott.tt_full(Y) - ref) / np.linalg.norm(ref)
    assert err < 1e-13
    assert ott.ranks(Y) == [a * b for a, b in zip(inst["R"], inst["r"])]   # ranks multiply


def test_matvec_loop_equals_einsum_elementwise():
    g = inputs.rng(5)
    A = inputs.random_ttm(g, [2, 3, 2], [3, 2, 2], [1, 3, 2, 1])
    X = inputs.random_tt(g, [3, 2, 2], [1, 4, 3, 1])
    for a, b in zip(ott.tt_matvec(A, X), ott.tt_matvec_fast(A, X)):
        assert np.array_equal(a.shape, b.shape)
        assert np.max(np.abs(a - b)) < 1e-15


def test_matvec_identity_and_rank1():
    g = inputs.rng(6)
    X = inputs.random_tt(g, [2, 3, 4], [1, 3, 2, 1])
    I = ott.rank1_ttm([np.eye(2), np.eye(3), np.eye(4)])
    for a, b in zip(ott.tt_matvec(I, X), X):
        assert np.array_equal(a, b)
    Fs = [g.standard_normal((3, 2)), g.standard_normal((2, 3)), g.standard_normal((5, 4))]
    vs = [g.standard_normal(2), g.standard_normal(3), g.standard_normal(4)]
    x1 = [v.reshape(1, -1, 1) for v in vs]
    Y = ott.tt_matvec(ott.rank1_ttm(Fs), x1)
    for Yk, F, v in zip(Y, Fs, vs):
        assert np.allclose(Yk[0, :, 0], F @ v, atol=1e-14)


def test_add_dot_sum_norm():
    g = inputs.rng(7)
    dims = [2, 3, 4, 2]
    X = inputs.random_tt(g, dims, [1, 2, 3, 2, 1])
    Y = inputs.random_tt(g, dims, [1, 3, 1, 4, 1])
    Z = ott.tt_add(X, Y)
    assert ott.ranks(Z) == [1, 5, 4, 6, 1]
    assert np.allclose(ott.tt_full(Z), ott.tt_full(X) + ott.tt_full(Y), atol=1e-14)
    assert abs(ott.tt_dot(X, Y) - ott.tt_full(X) @ ott.tt_full(Y)) < 1e-12
    ones = [np.ones((1, n, 1)) for n in (2, 3, 4)]
    assert ott.tt_sum(ones) == 24.0
    a, b, c, e = (g.standard_normal(3) for _ in range(4))
    x = [a.reshape(1, 3, 1), b.reshape(1, 3, 1)]
    y = [c.reshape(1, 3, 1), e.reshape(1, 3, 1)]
    assert abs(ott.tt_dot(x, y) - (a @ c) * (b @ e)) < 1e-13
    assert abs(ott.tt_norm(X) - np.linalg.norm(ott.tt_full(X))) < 1e-12
    s = ott.tt_scale(X, -2.5)
    assert np.allclose(ott.tt_full(s), -2.5 * ott.tt_full(X), atol=1e-14)


def test_orthogonalize_rl():
    inst = inputs.c2_slice(101)
    Y = ott.tt_matvec_fast(inst["A"], inst["X"])
    full = ott.tt_full(Y)
    O, nrm = ott.tt_orthogonalize_rl(Y)
    assert np.linalg.norm(ott.tt_full(O) - full) / np.linalg.norm(full) < 1e-13
    assert abs(nrm - np.linalg.norm(full)) / nrm < 1e-13
    for k in range(1, len(O)):
        r0, n, r1 = O[k].shape
        M = O[k].reshape(r0, n * r1, order="F")
        assert np.max(np.abs(M @ M.T - np.eye(r0))) < 1e-13          # Z23 max-abs
        assert r0 <= n * r1
    Lo, nrm2 = ott.tt_orthogonalize_lr(Y)
    assert np.linalg.norm(ott.tt_full(Lo) - full) / np.linalg.norm(full) < 1e-13
    for k in range(len(Lo) - 1):
        r0, n, r1 = Lo[k].shape
        M = Lo[k].reshape(r0 * n, r1, order="F")
        assert np.max(np.abs(M.T @ M - np.eye(r1))) < 1e-13


def test_round_error_identity_and_bound():
    """||X - X'||^2 = sum of discarded sigma^2 (orthogonal
    truncation errors) and ||X - X'|| <= eps ||X|| when rmax does not bind."""
    inst = inputs.c2_slice(102)
    Y = ott.tt_matvec_fast(inst["A"], inst["X"])
    full = ott.tt_full(Y)
    for eps in (1e-1, 1e-2, 1e-3):
        R, info = ott.tt_round(Y, eps)
        err = np.linalg.norm(ott.tt_full(R) - full)
        assert abs(err ** 2 - sum(info["discarded_sq"])) <= 1e-10 * np.linalg.norm(full) ** 2
        assert err <= eps * np.linalg.norm(full) * (1 + 1e-12)
    # without truncation the bond singular values are those of the dense unfoldings
    R, info = ott.tt_round(Y, 0.0)
    dims = [2] * 10
    T = full.reshape(dims, order="F")
    for k in (2, 5, 7):
        M = T.reshape(2 ** (k + 1), -1, order="F")
        s = np.linalg.svd(M, compute_uv=False)
        p = len(info["sv"][k])
        assert np.allclose(info["sv"][k], s[:p], atol=1e-12 * s[0])


def test_round_special_cases():
    g = inputs.rng(8)
    dims = [3, 4, 3, 2]
    X = inputs.random_tt(g, dims, [1, 3, 4, 2, 1])
    R0, _ = ott.tt_round(X, 0.0)
    assert ott.ranks(R0) == ott.ranks(X)
    XX, _ = ott.tt_round(ott.tt_add(X, X), 1e-12)
    assert ott.ranks(XX) == ott.ranks(X)
    assert np.allclose(ott.tt_full(XX), 2 * ott.tt_full(X), atol=1e-12)
    # a known rank-2 tensor a o b o c + d o e o f: rounding recovers ranks [1,2,2,1]
    v = [g.standard_normal((5,)) for _ in range(6)]
    T1 = [v[0].reshape(1, 5, 1), v[1].reshape(1, 5, 1), v[2].reshape(1, 5, 1)]
    T2 = [v[3].reshape(1, 5, 1), v[4].reshape(1, 5, 1), v[5].reshape(1, 5, 1)]
    S = ott.tt_add(ott.tt_add(T1, T2), T1)
    R, _ = ott.tt_round(S, 1e-12)
    assert ott.ranks(R) == [1, 2, 2, 1]
    # rmax binds
    Rm, _ = ott.tt_round(ott.tt_matvec_fast(*[inputs.c2_slice(103)[k] for k in ("A", "X")]), 1e-14, rmax=5)
    assert max(ott.ranks(Rm)) <= 5


def test_trunc_rank_rule():
    s = np.array([4.0, 2.0, 1.0, 0.5])
    assert ott.trunc_rank(s, 0.5, 10) == 3            # tail {0.5}: 0.25 <= 0.25 inclusive
    assert ott.trunc_rank(s, math.sqrt(1.25), 10) == 2
    assert ott.trunc_rank(s, 0.0, 10) == 4
    assert ott.trunc_rank(s, 100.0, 10) == 1          # r >= 1
    assert ott.trunc_rank(s, 0.0, 2) == 2
    assert ott.trunc_rank(np.array([1.0, 0.0, 0.0]), 0.0, 10) == 1   # zeros dropped


def test_interfaces_and_local_apply_dense():
    """Phi after all cores = y^T A x; local apply = frames^T A frames x_k (dense)."""
    g = inputs.rng(9)
    dims = [2, 3, 2, 3]
    A = inputs.random_ttm(g, dims, dims, [1, 2, 3, 2, 1])
    X = inputs.random_tt(g, dims, [1, 2, 3, 2, 1])
    Y = inputs.random_tt(g, dims, [1, 2, 2, 3, 1])
    Ad = ott.ttm_full(A)
    Phi = np.ones((1, 1, 1))
    for k in range(4):
        Phi = ott.left_update(Phi, Y[k], A[k], X[k])
    ref = ott.tt_full(Y) @ Ad @ ott.tt_full(X)
    assert abs(Phi[0, 0, 0] - ref) < 1e-12 * (1 + abs(ref))
    Psi = np.ones((1, 1, 1))
    for k in range(3, -1, -1):
        Psi = ott.right_update(Psi, Y[k], A[k], X[k])
    assert abs(Psi[0, 0, 0] - ref) < 1e-12 * (1 + abs(ref))
    # local apply at core k=1 (0-based) against dense frames
    k = 1
    PhiL = ott.left_update(np.ones((1, 1, 1)), Y[0], A[0], X[0])
    PsiR = np.ones((1, 1, 1))
    for kk in range(3, k, -1):
        PsiR = ott.right_update(PsiR, Y[kk], A[kk], X[kk])
    y = ott.local_apply(PhiL, A[k], PsiR, X[k])
    FY = ott.frames_dense(Y, k)
    FX = ott.frames_dense(X, k)
    yd = FY.T @ Ad @ FX @ X[k].reshape(-1, order="F")
    assert np.allclose(y.reshape(-1, order="F"), yd, atol=1e-12)
    B = ott.local_matrix(PhiL, A[k], PsiR)
    assert np.allclose(B, FY.T @ Ad @ FX, atol=1e-12)
    # vector interfaces
    bvec = inputs.random_tt(g, dims, [1, 2, 2, 2, 1])
    phi = np.ones((1, 1))
    for kk in range(4):
        phi = ott.left_update_vec(phi, Y[kk], bvec[kk])
    assert abs(phi[0, 0] - ott.tt_full(Y) @ ott.tt_full(bvec)) < 1e-12
    phil = ott.left_update_vec(np.ones((1, 1)), Y[0], bvec[0])
    psir = np.ones((1, 1))
    for kk in range(3, k, -1):
        psir = ott.right_update_vec(psir, Y[kk], bvec[kk])
    rhs = ott.local_rhs(phil, bvec[k], psir)
    assert np.allclose(rhs.reshape(-1, order="F"), FY.T @ ott.tt_full(bvec), atol=1e-12)


def test_tt_svd_roundtrip():
    g = inputs.rng(10)
    T = g.standard_normal(4 * 5 * 6 * 7)
    cores = ott.tt_svd(T, [4, 5, 6, 7], 1e-10)
    assert np.linalg.norm(ott.tt_full(cores) - T) <= 1e-10 * np.linalg.norm(T)
    a, b, c = g.standard_normal(3), g.standard_normal(4), g.standard_normal(5)
    T = np.einsum("i,j,k->ijk", a, b, c).reshape(-1, order="F")
    cores = ott.tt_svd(T, [3, 4, 5], 1e-12)
    assert ott.ranks(cores) == [1, 1, 1, 1]
