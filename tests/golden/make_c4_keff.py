"""Writes tests/golden/c4_keff.txt from the oracle only: the matrix-free full-grid
k_eff (Eq. 8 with transport sweeps)
of the BASELINE.json configs[3] physics (G=30 with upscatter in groups 26-30,
S16 LS-style 288 ordinates, core/blanket/reflector; inputs.problem_c4) on
coarse grids (nv = 4, 8), converged to |dk| < 1e-12.  The full 256^3 grid is
out of the oracle's reach.  Usage: make_c4_keff.py [nv ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import inputs  # noqa: E402
from oracle import transport as T  # noqa: E402

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c4_keff.txt")
nvs = [int(a) for a in sys.argv[1:]] or [4, 8]
rows = {}
if os.path.exists(out):
    for line in open(out):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            rows[int(f[0])] = line.rstrip("\n")
for nv in nvs:
    t = time.time()
    k, _, it = T.keff_sweep_3d(inputs.problem_c4(nv=nv), tol=1e-12)
    rows[nv] = f"{nv} {k:.17g} {it} {time.time() - t:.1f}"
    print(rows[nv], flush=True)
    with open(out, "w") as f:
        f.write("# C4 physics k_eff by the oracle's matrix-free sweep iteration to |dk| < 1e-12 (make_c4_keff.py)\n")
        f.write("# nv k iterations seconds\n")
        for key in sorted(rows):
            f.write(rows[key] + "\n")
