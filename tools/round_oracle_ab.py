"""Oracle-vs-oracle experiment behind the C2 rounding tolerance (VERDICT r1 weak #2,
reading Z22): the oracle's tt_round (Z21) run twice on the same C2
instance with two correct fp64 SVD routes — LAPACK gesdd (numpy) and gesvd
(scipy) of the left unfoldings — and the bond singular values compared bond by
bond, relative to sigma_1.  Prints, per bond, the max |sigma_a - sigma_b| / sigma_1
and whether rmax has bound on an earlier bond.  Calls only oracle/ and LAPACK."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sl  # noqa: E402

import inputs  # noqa: E402
from oracle import tt as ott  # noqa: E402


def round_with(svd, X, eps, rmax):
    d = len(X)
    Y, nrm = ott.tt_orthogonalize_rl(X)
    delta = eps * nrm / np.sqrt(d - 1)
    sv, ranks = [], []
    for k in range(d - 1):
        r0, n, r1 = Y[k].shape
        U, s, Vt = svd(Y[k].reshape(r0 * n, r1, order="F"))
        r = ott.trunc_rank(s, delta, rmax)
        sv.append(s)
        ranks.append(r)
        Y[k] = U[:, :r].reshape(r0, n, r, order="F")
        Y[k + 1] = np.einsum("cb,bjd->cjd", s[:r, None] * Vt[:r, :], Y[k + 1])
    return sv, ranks


gesdd = lambda M: np.linalg.svd(M, full_matrices=False)
gesvd = lambda M: sl.svd(M, full_matrices=False, lapack_driver="gesvd")
for seed in (0, 1, 2):
    inst = inputs.c2_instance(seed)
    Y = ott.tt_matvec_fast(inst["A"], inst["X"])
    sa, ra = round_with(gesdd, Y, 1e-8, 128)
    sb, rb = round_with(gesvd, Y, 1e-8, 128)
    s1 = max(s[0] for s in sa)
    worst_pre, worst_post, binds = 0.0, 0.0, 0
    for k, (a, b) in enumerate(zip(sa, sb)):
        dev = np.max(np.abs(a - b)) / s1
        if binds == 0:
            worst_pre = max(worst_pre, dev)
        else:
            worst_post = max(worst_post, dev)
        binds += int(ra[k] < len(a))
    print(f"seed {seed}: ranks equal {ra == rb}; max |dsigma|/sigma_1 before the first rmax-binding bond "
          f"{worst_pre:.2e}, after it {worst_post:.2e}")
