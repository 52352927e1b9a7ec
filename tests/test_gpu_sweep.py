"""C5 (BASELINE.json configs[4]) at full size: a GPU double sweep of ALS local
applies + interface updates vs the oracle's contractions on the same cores
(relative Frobenius <= 1e-12 per array)."""
import numpy as np
import pytest

import inputs
from oracle import tt as ott

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2309_03347_b200.sweep import SweepProblem  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def host(t, shape):
    return t.cpu().numpy().reshape(shape, order="F")


@pytest.mark.parametrize("r", [64, 128])
def test_c5_double_sweep_interfaces(r):
    inst = inputs.c5_instance(r, seed=0)
    A, X = inst["A"], inst["X"]
    sp = SweepProblem(A, X)
    sp.build_right(normalize=False)
    sp.double_sweep()
    torch.cuda.synchronize()
    d = len(X)
    # oracle: all left interfaces, then right interfaces
    Phi = [np.ones((1, 1, 1))]
    for k in range(d - 1):
        Phi.append(ott.left_update(Phi[-1], X[k], A[k], X[k]))
    for k in (1, 7, 20, d - 1):
        shp = (sp.r[k], sp.R[k], sp.r[k])
        assert rel(host(sp.Phi[k], shp), Phi[k]) <= 1e-12, k
    Psi = {d: np.ones((1, 1, 1))}
    for k in range(d - 1, 0, -1):
        Psi[k] = ott.right_update(Psi[k + 1], X[k], A[k], X[k])
    for k in (1, 13, 33, d - 1):
        shp = (sp.r[k], sp.R[k], sp.r[k])
        assert rel(host(sp.Psi[k], shp), Psi[k]) <= 1e-12, k
    # the last local apply of the right-to-left sweep (core 1, 0-based)
    y = ott.local_apply(Phi[1], A[1], Psi[2], X[1])
    got = host(sp.y[:y.size], y.shape)
    assert rel(got, y) <= 1e-12


def test_c5_r256_single_visit():
    inst = inputs.c5_instance(256, seed=1, d=6)
    A, X = inst["A"], inst["X"]
    sp = SweepProblem(A, X)
    sp.build_right(normalize=False)
    sp.double_sweep()
    torch.cuda.synchronize()
    Phi = np.ones((1, 1, 1))
    for k in range(3):
        Phi = ott.left_update(Phi, X[k], A[k], X[k])
    shp = (sp.r[3], sp.R[3], sp.r[3])
    assert rel(host(sp.Phi[3], shp), Phi) <= 1e-12
