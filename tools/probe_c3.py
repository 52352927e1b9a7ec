"""C3 (configs[2]) / C4 (configs[3], NV=c4) on the device: QTT operator assembly
and the k-eff fixed point with B by amen_mv (NEXT-1).
Usage: probe_c3.py NV|c4 [eps] [rmax] [max_outer] [max_sweeps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "16"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
rmax = int(sys.argv[3]) if len(sys.argv) > 3 else 64
mo = int(sys.argv[4]) if len(sys.argv) > 4 else 200
ms = int(sys.argv[5]) if len(sys.argv) > 5 else 10
p = inputs.problem_c4() if cfg == "c4" else inputs.problem_c3(nv=int(cfg))
nv = p["nv"]
t = time.time()
ops = gtr.operators(p, eps=1e-12)
torch.cuda.synchronize()
print("assembly", round(time.time() - t, 2), {k: v.ranks() for k, v in ops.items()}, flush=True)
modes = gtr.modes(p)
d = len(modes)
kick = 4
g = inputs.rng(61)
psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [rmax + kick] * (d - 1) + [1])
z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1] + [kick] * (d - 1) + [1]))
t = time.time()
res = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, tol_k=eps, eps_round=eps, eps_solve=eps, rmax=rmax,
                          max_outer=mo, matvec="amen_mv", restart=40, max_restarts=20, max_sweeps=ms,
                          mv_max_sweeps=ms)
torch.cuda.synchronize()
dt = time.time() - t
it = res.iters.item()
print(f"nv={nv} eps={eps} k={res.k.item():.12f} iters={it} status={res.status.item()} time={dt:.2f}s "
      f"{it / dt:.3f} it/s sweeps={res.sweeps_hist[:it].tolist()} ranks={psi.ranks()}", flush=True)
print("k_hist", res.k_hist[:it].tolist())
