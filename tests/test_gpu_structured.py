"""GPU parity of the structured (diagonal) operator-core forms of the ALS
local apply (a6) and interface updates (a5) against the oracle's plain
einsum contractions (oracle/tt.py), SURVEY.md §8(a) a6 / §8(c).5
"relative Frobenius <= 1e-12 per output array".  The cores are diagonal in
(i, j) like the angle / group factors of H."""
import numpy as np
import pytest
import torch

import inputs
from oracle import tt as ott

pytestmark = pytest.mark.gpu

tb = pytest.importorskip("paper_2309_03347_b200")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.reshape(-1, order="F"))).cuda()


def diag_core(g, R, m, Rp):
    """[R, m, m, Rp] core with A[g, i, j, g'] = 0 for i != j."""
    A = np.zeros((R, m, m, Rp))
    D = g.standard_normal((R, m, Rp))
    for i in range(m):
        A[:, i, i, :] = D[:, i, :]
    return A


SHAPES = [  # (rA, R, rB, m, rAp, Rp, rBp)
    (5, 3, 5, 4, 4, 2, 4),
    (33, 36, 33, 24, 7, 4, 7),      # C4 angle-core pattern (R >> Rp), scaled
    (20, 4, 20, 30, 1, 1, 1),       # group core: right boundary
    (17, 2, 9, 6, 11, 5, 13),       # Rp > R, rectangular ranks
    (64, 12, 64, 16, 30, 3, 30),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("absorb", [0, 1])
def test_local_apply_diag(shape, absorb):
    rA, R, rB, m, rAp, Rp, rBp = shape
    g = inputs.rng(71)
    Phi = g.standard_normal((rA, R, rB))
    Ak = diag_core(g, R, m, Rp)
    Psi = g.standard_normal((rAp, Rp, rBp))
    x = g.standard_normal((rB, m, rBp))
    ref = ott.local_apply(Phi, Ak, Psi, x).reshape(-1, order="F")
    y = torch.zeros(rA * m * rAp, dtype=torch.float64, device="cuda")
    dims = (rA, R, rB, m, m, rAp, Rp, rBp)
    tb.als_local_apply_structured(tb.CORE_DIAG, absorb, dims, _dev(Phi), _dev(Ak), _dev(Psi), _dev(x), y)
    assert rel(y.cpu().numpy(), ref) <= 1e-13


@pytest.mark.parametrize("shape", SHAPES)
def test_interfaces_diag(shape):
    rY, R, rX, m, rYp, Rp, rXp = shape
    g = inputs.rng(72)
    Phi = g.standard_normal((rY, R, rX))
    Ak = diag_core(g, R, m, Rp)
    Y = g.standard_normal((rY, m, rYp))
    X = g.standard_normal((rX, m, rXp))
    dims = (rY, R, rX, m, m, rYp, Rp, rXp)
    for absorb in (0, 1):
        out = torch.zeros(rYp * Rp * rXp, dtype=torch.float64, device="cuda")
        tb.als_update_interfaces_structured(tb.CORE_DIAG, absorb, +1, dims, _dev(Phi), _dev(Y), _dev(Ak), _dev(X), out)
        ref = ott.left_update(Phi, Y, Ak, X).reshape(-1, order="F")
        assert rel(out.cpu().numpy(), ref) <= 1e-13, f"left, absorb={absorb}"
    Psi = g.standard_normal((rYp, Rp, rXp))
    out = torch.zeros(rY * R * rX, dtype=torch.float64, device="cuda")
    tb.als_update_interfaces_structured(tb.CORE_DIAG, 0, -1, dims, _dev(Psi), _dev(Y), _dev(Ak), _dev(X), out)
    ref = ott.right_update(Psi, Y, Ak, X).reshape(-1, order="F")
    assert rel(out.cpu().numpy(), ref) <= 1e-13


def test_dense_kind_is_the_plain_call():
    g = inputs.rng(73)
    dims = (9, 3, 9, 4, 5, 6, 2, 6)
    rA, R, rB, m, n, rAp, Rp, rBp = dims
    Phi, Ak, Psi, x = (g.standard_normal(s) for s in ((rA, R, rB), (R, m, n, Rp), (rAp, Rp, rBp), (rB, n, rBp)))
    y = torch.zeros(rA * m * rAp, dtype=torch.float64, device="cuda")
    tb.als_local_apply_structured(tb.CORE_DENSE, 0, dims, _dev(Phi), _dev(Ak), _dev(Psi), _dev(x), y)
    assert rel(y.cpu().numpy(), ott.local_apply(Phi, Ak, Psi, x).reshape(-1, order="F")) <= 1e-13
    with pytest.raises(tb.TTError):   # a diagonal core must be square
        tb.als_local_apply_structured(tb.CORE_DIAG, 0, dims, _dev(Phi), _dev(Ak), _dev(Psi), _dev(x), y)


def test_core_kinds_of_transport_operators():
    """H's angle and group cores are diagonal; the
    QTT spatial cores (2 x 2) and S, F's angle cores (rank-1 Intg) are not."""
    from paper_2309_03347_b200 import transport as gtr
    prob = inputs.problem_c3(nv=8)
    ops = gtr.operators(prob, eps=1e-12)
    kinds, ratio = tb.core_kinds(ops["H"])
    d = len(kinds)
    assert kinds[d - 2] == tb.CORE_DIAG and kinds[d - 1] == tb.CORE_DIAG, (kinds, ratio)
    assert all(k == tb.CORE_DENSE for k in kinds[:d - 2])
    ks, _ = tb.core_kinds(ops["S"])
    assert ks[d - 2] == tb.CORE_DENSE
