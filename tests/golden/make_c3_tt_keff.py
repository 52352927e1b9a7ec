"""Writes tests/golden/c3_tt_keff.txt from the oracle only: the CPU-TT k-eff
iteration (oracle.solvers.keff_tt: Eq. 8 in TT, B by amen_mv
P:1501-1506, AMEn with GMRES local solves, readings Z16-Z21) on the full
BASELINE.json configs[2] problem (C3: 64^3 QTT, G=7, S8 LS-style 80
ordinates, two regions), eps_round = eps_solve = 1e-6, rmax 64, <= 4 AMEn /
amen_mv sweeps per iteration, GMRES everywhere (dense_max 0, the device
path's local solver), z0 = inputs.random_tt(rng(61)) with kickrank 4, for a
bounded number of outer iterations from psi_0 = 1, k_0 = 1.  The GPU-TT
trajectory must follow it to |dk|/k <= 10 eps_solve.
Usage: make_c3_tt_keff.py [iterations]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import inputs  # noqa: E402
from oracle import solvers as so  # noqa: E402
from oracle import transport as T  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_tt_keff.txt")
t = time.time()
p = inputs.problem_c3()
tops = T.tt_operators(p)
modes = [c.shape[1] for c in tops["H"]]
d = len(modes)
z0 = inputs.random_tt(inputs.rng(61), modes, [1] + [4] * (d - 1) + [1])
psi0 = [np.ones((1, n, 1)) for n in modes]
k, psi, hist = so.keff_tt(tops["H"], tops["S"], tops["F"], psi0, z0, tol_k=0.0, eps_round=1e-6, eps_solve=1e-6,
                          max_outer=iters, dense_max=0, rmax=64, max_sweeps=4, mv_max_sweeps=4, matvec="amen_mv")
with open(out, "w") as f:
    f.write("# C3 (64^3) CPU-TT k-eff iterates by oracle.solvers.keff_tt (make_c3_tt_keff.py): eps 1e-6, rmax 64,\n")
    f.write("# 4 sweeps, amen_mv B, GMRES(60) local solves, z0 = random_tt(rng(61), kick 4); "
            f"{time.time() - t:.0f} s\n")
    f.write("# iteration k max_psi_rank\n")
    for i, h in enumerate(hist, start=1):
        f.write(f"{i} {h['k']:.17g} {max(h['ranks'])}\n")
print(open(out).read())
