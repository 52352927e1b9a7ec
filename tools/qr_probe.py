"""QR kernel microbenchmark: tt_orthogonalize(+1) of a d=2 TT whose first core is
an m x n left unfolding = one qr_kernel launch (+ the R-apply GEMM).  Prints the
mean time per call for AMEn/rounding shapes; with a QR_PHASE_TIMING build the
kernel also prints per-phase clock64 cycles (QRPH lines: m n hasQ copy panel
T trailing Q).  Usage: qr_probe.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_03347_b200 as tb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = np.random.default_rng(0)
for m, n in [(264, 132), (264, 136), (136, 132), (528, 132), (64, 32), (256, 64), (1000, 100)]:
    c0 = g.standard_normal((1, m, n))
    c1 = g.standard_normal((n, 2, 1))
    X = tb.TTVec.from_cores([c0, c1])
    Y = tb.TTVec.from_cores([c0, c1])
    for _ in range(3):
        tb.tt_copy(X, Y)
        tb.tt_orthogonalize(Y, +1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tb.tt_copy(X, Y)
        tb.tt_orthogonalize(Y, +1)
    e1.record()
    torch.cuda.synchronize()
    Q = Y.cores()[0].reshape(m, -1, order="F")
    orth = np.max(np.abs(Q.T @ Q - np.eye(Q.shape[1])))
    print(f"m {m:5d} n {n:4d}: {e0.elapsed_time(e1) / reps * 1e3:8.1f} us per orthogonalize (QR + R-apply), "
          f"orthogonality {orth:.1e}", flush=True)
