"""One C1 k-eff solve limited to `--iters` outer iterations (for ncu launch lists)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs
import paper_2309_03347_b200 as tb
from paper_2309_03347_b200 import transport as gtr
ap = argparse.ArgumentParser(); ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--matvec", default="amen_mv"); a = ap.parse_args()
prob = inputs.problem_c1(); ops = gtr.operators(prob)
modes = [8, 8, 8, 8, 1]; g = inputs.rng(61)
psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 68, 68, 68, 68, 1])
z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1]))
torch.cuda.synchronize()
res = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12,
                          rmax=64, max_outer=a.iters, matvec=a.matvec)
torch.cuda.synchronize()
print("k", res.k.item(), "iters", res.iters.item())
