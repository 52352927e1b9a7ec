"""CPU checks of libtt's host-side setup logic (operator factor construction and
Algorithm 1), compared with the oracle's independent constructions.  These
call host code only (no device work)."""
import numpy as np
import pytest

import inputs
from oracle import transport as T
from oracle import tt as ott


@pytest.fixture(scope="module")
def gtr():
    from __graft_entry__ import _build_module
    build = _build_module()
    build.build()
    from paper_2309_03347_b200 import transport
    return transport


@pytest.mark.parametrize("prob", [inputs.problem_c1(), inputs.problem_small_hetero(nv=4, G=2, N=4),
                                  inputs.problem_slab(4, nv=16)], ids=["C1", "hetero4", "slab16"])
def test_factor_terms_match_oracle(gtr, prob):
    ref = T.operator_terms(prob)
    for op in "HSF":
        got = gtr.factor_terms(prob, op)
        assert len(got) == len(ref[op])
        for ta, tb in zip(got, ref[op]):
            for a, b in zip(ta, tb):
                assert np.array_equal(a, b)


def test_reflective_terms_sum_to_dense(gtr):
    """Reading Z15: the rank-1 reflective terms of the host builder sum to the
    oracle's dense reflective operators (row-replacement construction)."""
    import copy
    p = copy.deepcopy(inputs.problem_c1("reflective"))
    p["nv"] = 4
    dense = T.dense_operators(p)
    for op in "HSF":
        M = sum(T.kron_term(t) for t in gtr.factor_terms(p, op))
        assert np.array_equal(M, dense[op])


@pytest.mark.parametrize("prob", [inputs.problem_c1(), inputs.problem_c1("reflective"),
                                  inputs.problem_small_hetero(nv=4, G=2, N=4), inputs.problem_slab(4, nv=16)],
                         ids=["C1", "C1-reflective", "hetero4", "slab16"])
def test_velocity_terms_match_oracle(gtr, prob):
    """V^{-1}: host terms sum to the oracle's dense operator
    (reflective: with the face rows zeroed, Z15)."""
    import copy
    p = copy.deepcopy(prob)
    if p.get("dim", 3) == 3:
        p["nv"] = 4
    got = sum(T.kron_term(t) for t in gtr.factor_terms(p, "V"))
    assert np.array_equal(got, T.dense_operators(p)["V"])
