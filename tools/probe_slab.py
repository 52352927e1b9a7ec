"""Slab k-eff on the GPU: time, outer iterations and AMEn sweeps per iteration."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs
import paper_2309_03347_b200 as tb
from paper_2309_03347_b200 import transport as gtr
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-11
p = inputs.problem_slab(L)
t = time.time(); ops = gtr.operators(p, eps=1e-12); torch.cuda.synchronize(); print("assembly", time.time() - t, {k: v.ranks() for k, v in ops.items()})
modes = gtr.modes(p); d = len(modes)
for rep in range(2):
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [43] * (d - 1) + [1])
    z = tb.TTVec.from_cores(inputs.random_tt(inputs.rng(61), modes, [1] + [3] * (d - 1) + [1]))
    torch.cuda.synchronize(); t = time.time()
    res = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, rmax=40, tol_k=tol, eps_round=tol, eps_solve=tol)
    torch.cuda.synchronize(); dt = time.time() - t
    it = res.iters.item()
    print(f"L={L} tol={tol}: k={res.k.item():.12f} iters={it} time={dt:.2f}s  {it/dt:.2f} it/s  sweeps={res.sweeps_hist[:it].tolist()} ranks={psi.ranks()}")
