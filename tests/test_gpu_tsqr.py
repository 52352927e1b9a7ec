"""GPU parity of the tall-unfolding path (multi-level TSQR inside tt_orthogonalize
/ tt_round) against the oracle: orthogonality <= 1e-13 (max-abs, Z23),
reconstruction <= 1e-13, ranks = oracle, rounded tensor and bond singular
values vs oracle.  Shapes: unfoldings of 1800 x 64,
12000 x 4 and 57600 x 2 rows x columns (one to three TSQR levels), plus a
rank-deficient tall core."""
import numpy as np
import pytest

import inputs
from oracle import tt as ott

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2309_03347_b200 as tb  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


CASES = [([64, 900, 2], [1, 64, 2, 1]),      # R->L at core 1: 1800 x 64 (2 levels)
         ([4, 1000, 3], [1, 4, 12, 1]),      # R->L at core 1: 12000 x 4
         ([3, 30, 640, 3], [1, 3, 90, 3, 1]),  # L->R at core 2: 57600 x 3; R->L at core 2: 1920 x 90
         ([8, 288, 30], [1, 8, 30, 1])]      # the C4 angle pattern: 288*30 x 8 and 8*288 x 30


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("direction", [-1, 1])
def test_orthogonalize_tall(case, direction):
    modes, ranks = case
    g = inputs.rng(91)
    X = inputs.random_tt(g, modes, ranks)
    G = tb.TTVec.from_cores(X)
    nrm = tb.tt_orthogonalize(G, direction)
    torch.cuda.synchronize()
    O = G.cores()
    full = ott.tt_full(X)
    assert rel(ott.tt_full(O), full) <= 1e-13
    assert abs(nrm.item() - np.linalg.norm(full)) <= 1e-13 * np.linalg.norm(full)
    ref, _ = ott.tt_orthogonalize_rl(X) if direction < 0 else ott.tt_orthogonalize_lr(X)
    assert G.ranks() == ott.ranks(ref)
    for k in (range(1, len(O)) if direction < 0 else range(len(O) - 1)):
        r0, n, r1 = O[k].shape
        M = O[k].reshape(r0, n * r1, order="F").T if direction < 0 else O[k].reshape(r0 * n, r1, order="F")
        assert np.max(np.abs(M.T @ M - np.eye(M.shape[1]))) <= 1e-13


def test_orthogonalize_many_leaves_ragged_tail():
    """270001 x 150 unfolding: 451 leaves of 599 rows, the ragged last leaf has
    fewer rows (452 - ...) and the tree has three levels; plus a sum of rank-1
    terms (a rank-deficient tall unfolding, as in the operator assembly)."""
    g = inputs.rng(94)
    X = inputs.random_tt(g, [150, 270001], [1, 150, 1])
    G = tb.TTVec.from_cores(X)
    nrm = tb.tt_orthogonalize(G, -1)
    O = G.cores()
    M = O[1].reshape(O[1].shape[0], -1, order="F")
    assert np.max(np.abs(M @ M.T - np.eye(M.shape[0]))) <= 1e-13
    full = X[0].reshape(-1, 150) @ X[1].reshape(150, -1)
    assert rel(O[0].reshape(-1, O[0].shape[2]) @ M, full) <= 1e-13
    assert abs(nrm.item() - np.linalg.norm(full)) <= 1e-13 * np.linalg.norm(full)
    # rank-deficient: 24 rank-1 terms added as a rank-24 TT with 96-wide capacity
    terms = [inputs.random_tt(g, [8, 4000, 3], [1, 1, 1, 1]) for _ in range(24)]
    S = terms[0]
    for t in terms[1:]:
        S = ott.tt_add(S, t)
    S = [np.concatenate([S[0], S[0]], axis=2) * np.array([1.0] * 24 + [0.0] * 24), 
         np.concatenate([S[1], S[1]], axis=0), S[2]]
    S[1] = np.concatenate([S[1], S[1]], axis=2)
    S[2] = np.concatenate([S[2], 0.5 * S[2]], axis=0)
    G = tb.TTVec.from_cores(S)
    tb.tt_orthogonalize(G, -1)
    assert rel(ott.tt_full(G.cores()), ott.tt_full(S)) <= 1e-13
    tb.tt_round(G, 1e-12)
    assert G.ranks()[1] <= 24 and G.ranks()[2] <= 3
    assert rel(ott.tt_full(G.cores()), ott.tt_full(S)) <= 1e-11


def test_orthogonalize_tall_rank_deficient():
    """Tall core whose columns span only 3 of 16 directions: Householder keeps an
    orthonormal Q of full width (zero R rows), like the single-CTA path."""
    g = inputs.rng(92)
    X = inputs.random_tt(g, [16, 2000, 2], [1, 16, 2, 1])
    C = X[1].reshape(16, -1, order="F")
    C[3:, :] = g.standard_normal((13, 3)) @ C[:3, :]      # rank 3 in the row space
    X[1] = C.reshape(16, 2000, 2, order="F")
    G = tb.TTVec.from_cores(X)
    tb.tt_orthogonalize(G, -1)
    O = G.cores()
    assert rel(ott.tt_full(O), ott.tt_full(X)) <= 1e-13
    r0, n, r1 = O[1].shape
    M = O[1].reshape(r0, n * r1, order="F")
    assert np.max(np.abs(M @ M.T - np.eye(r0))) <= 1e-13


@pytest.mark.parametrize("case", CASES[:2] + CASES[3:])
def test_round_tall_vs_oracle(case):
    modes, ranks = case
    g = inputs.rng(93)
    X = inputs.random_tt(g, modes, ranks)
    for eps in (1e-2, 1e-10):
        G = tb.TTVec.from_cores(X)
        tb.tt_round(G, eps)
        ref, _ = ott.tt_round(X, eps)
        assert G.ranks() == ott.ranks(ref)
        full = ott.tt_full(ref)
        assert rel(ott.tt_full(G.cores()), full) <= 1e-12
