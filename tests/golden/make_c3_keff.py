"""Writes tests/golden/c3_keff.txt from the oracle only: the matrix-free full-grid
k_eff (Eq. 8 with transport sweeps)
of BASELINE.json configs[2] (C3, 64^3) and of the same problem on coarser grids
(nv = 8, 16, 32), converged to |dk| < 1e-11.  Usage: make_c3_keff.py [nv ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import inputs  # noqa: E402
from oracle import transport as T  # noqa: E402

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_keff.txt")
nvs = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64]
rows = {}
if os.path.exists(out):
    for line in open(out):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            rows[int(f[0])] = line.rstrip("\n")
for nv in nvs:
    t = time.time()
    k, _, it = T.keff_sweep_3d(inputs.problem_c3(nv=nv), tol=1e-11)
    rows[nv] = f"{nv} {k:.17g} {it} {time.time() - t:.1f}"
    print(rows[nv], flush=True)
    with open(out, "w") as f:
        f.write("# C3 k_eff by the oracle's matrix-free sweep iteration to |dk| < 1e-11 (make_c3_keff.py)\n")
        f.write("# nv k iterations seconds\n")
        for key in sorted(rows):
            f.write(rows[key] + "\n")
