"""GPU-TT C3 iterates (the settings of tests/golden/make_c3_tt_keff.py): k, AMEn
sweeps and psi ranks after 1, 2, 3 outer iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402

p = inputs.problem_c3()
ops = gtr.operators(p)
modes = gtr.modes(p)
d = len(modes)
for restart in (60, 40):
    for n in (1, 2, 3):
        z = tb.TTVec.from_cores(inputs.random_tt(inputs.rng(61), modes, [1] + [4] * (d - 1) + [1]))
        psi = tb.TTVec.from_cores([np.ones((1, m, 1)) for m in modes], rcap=[1] + [68] * (d - 1) + [1])
        r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, tol_k=0.0, eps_round=1e-6, eps_solve=1e-6,
                                rmax=64, matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4, restart=restart,
                                max_restarts=200, max_outer=n)
        torch.cuda.synchronize()
        print(restart, n, repr(r.k.item()), r.sweeps_hist[:n].tolist(), r.inner_hist[:n].tolist(), psi.ranks(),
              flush=True)
