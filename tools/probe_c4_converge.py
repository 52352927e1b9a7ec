"""C4 (configs[3]) to convergence: k-eff fixed point from psi_0 = 1 with
tol_k = 1e-6 and the fixed-point residual evaluated every iteration (reported,
S:468 / Z19), at rmax 128 and rmax 160 (refinement).  Usage:
probe_c4_converge.py [rmax ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402

rmaxs = [int(a) for a in sys.argv[1:]] or [128, 160]
prob = inputs.problem_c4()
ops = gtr.operators(prob, eps=1e-12)
modes = gtr.modes(prob)
d = len(modes)
for rmax in rmaxs:
    g = inputs.rng(61)
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1] + [4] * (d - 1) + [1]))
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [rmax + 4] * (d - 1) + [1])
    t = time.time()
    r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, tol_k=1e-6, tol_res=0.0, eps_round=1e-6,
                            eps_solve=1e-6, rmax=rmax, matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4,
                            restart=40, max_restarts=20, max_outer=200, hist_cap=256)
    torch.cuda.synchronize()
    it = r.iters.item()
    kh = r.k_hist[:it].cpu().numpy()
    print(f"rmax {rmax}: status {r.status.item()} iterations {it} time {time.time() - t:.1f} s k {r.k.item():.10f} "
          f"residual {r.res.item():.3e}", flush=True)
    print("  k history", " ".join(f"{v:.7f}" for v in kh), flush=True)
    print("  ranks", psi.ranks(), flush=True)
