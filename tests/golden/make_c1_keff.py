"""Writes tests/golden/c1_keff_vacuum.txt from the oracle only (dense Eq.-8
power iteration, on BASELINE.json configs[0] vacuum)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import inputs  # noqa: E402
from oracle import transport as T, solvers as so  # noqa: E402

ops = T.dense_operators(inputs.problem_c1())
k, _, hist = so.keff_dense_power(ops["H"], ops["S"], ops["F"], tol=1e-13)
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c1_keff_vacuum.txt"), "w") as f:
    f.write("# C1 vacuum k_eff, dense power iteration to |dk|<1e-13 (oracle only; make_c1_keff.py)\n")
    f.write(f"{k:.17g}\n")
print(k, len(hist))
