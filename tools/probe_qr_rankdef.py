"""QR of rank-deficient square matrices on the device (tt_orthogonalize(+1) of a
d=2 TT whose first core is the m x p matrix): orthogonality of Q and
reconstruction, for exact-rank-r matrices of several sizes and structures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_03347_b200 as tb  # noqa: E402

g = np.random.default_rng(5)
cases = []
for m in (64, 96, 128, 160, 256):
    for r in (1, 3, 40):
        U = g.standard_normal((m, r)); V = g.standard_normal((r, m))
        cases.append((f"m={m} rank {r} dense", U @ V))
    A = np.zeros((m, m)); A[:, :3] = g.standard_normal((m, 3))
    cases.append((f"m={m} 3 cols then zeros", A))
    A = np.zeros((m, m)); A[:3, :] = g.standard_normal((3, m))
    cases.append((f"m={m} 3 rows then zeros", A))
    A = np.zeros((m, m)); idx = g.permutation(m)[:3]; A[idx, :] = g.standard_normal((3, m))
    cases.append((f"m={m} 3 scattered rows", A))
for name, A in cases:
    m, p = A.shape
    X = [A.reshape(1, m, p), np.eye(p).reshape(p, p, 1)]
    G = tb.TTVec.from_cores(X)
    tb.tt_orthogonalize(G, +1)
    torch.cuda.synchronize()
    c0, c1 = G.cores()
    Q = c0.reshape(m, -1, order="F")
    rec = Q @ c1.reshape(c1.shape[0], -1, order="F")
    print(f"{name:28s}: orth {np.max(np.abs(Q.T @ Q - np.eye(Q.shape[1]))):.1e} "
          f"recon {np.max(np.abs(rec - A)) / np.abs(A).max():.1e}", flush=True)
