"""Device Alg. 1 diagnostics: reconstruction error of tt_qtt_matrix_dev vs the
matrix, for several eps and sizes; and of tt_round(eps=0) of the exact
index-forwarding TT (built here through the same ABI with eps=0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402
from oracle import transport as T  # noqa: E402
from oracle import tt as ott  # noqa: E402

box = np.diag(((np.arange(256) >= 64) & (np.arange(256) < 192)).astype(float)) @ T.Ip_plus(256)
for n in (64, 128, 256, 512, 1024):
    for name, M in (("Ip-noBC", T.Ip_minus_noBC(n)), ("Ip-", T.Ip_minus(n)), ("D+", T.D_plus(n, 10.0 / (n - 1))),
                    ("box", box if n == 256 else np.eye(n))):
        for eps in (0.0, 1e-15, 1e-14, 1e-13):
            gtr._QTT.done.clear()
            cores = gtr.qtt_matrix(M, eps=eps)
            err = np.max(np.abs(ott.ttm_full(cores) - M)) / np.abs(M).max()
            print(f"n {n:4d} {name:8s} eps {eps:.0e}: ranks {ott.ranks(cores)} err {err:.2e} "
                  f"(oracle ranks {ott.ranks(T.qtt_matrix(M)) if eps else '-'})", flush=True)
