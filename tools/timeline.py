"""Real (non-serialised) kernel timeline summary of one k-eff solve from CUPTI
activity records: GPU busy fraction and per-kernel time.  Usage:
timeline.py c1|c3 [outer]"""
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 30
if cfg == "c1":
    p, rmax, kw = inputs.problem_c1(), 64, dict(tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12)
elif cfg == "c4":
    p, rmax, kw = inputs.problem_c4(), 128, dict(tol_k=1e-14, eps_round=1e-6, eps_solve=1e-6, max_sweeps=4,
                                                 mv_max_sweeps=4, max_restarts=20)
else:
    p, rmax, kw = inputs.problem_c3(), 64, dict(tol_k=1e-14, eps_round=1e-6, eps_solve=1e-6, max_sweeps=4,
                                                mv_max_sweeps=4, max_restarts=20)
ops = gtr.operators(p, eps=1e-12)
modes = gtr.modes(p)
d = len(modes)
g = inputs.rng(61)
z0 = inputs.random_tt(g, modes, [1] + [4] * (d - 1) + [1])


def solve():
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [rmax + 4] * (d - 1) + [1])
    z = tb.TTVec.from_cores(z0)
    r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, rmax=rmax, max_outer=outer, matvec="amen_mv", **kw)
    torch.cuda.synchronize()
    return r


solve()
if cfg != "c4":
    solve()
lc = C.CDLL(os.path.join(os.path.dirname(tb.__file__), "liblaunchcount.so"))
lc.lc_start()
r = solve()
a, o = C.c_ulonglong(0), C.c_ulonglong(0)
lc.lc_stop(C.byref(a), C.byref(o))
out = os.path.join("gpurun_out", f"timeline_{cfg}.txt")
os.makedirs("gpurun_out", exist_ok=True)
lc.lc_dump(out.encode())
lines = open(out).read().splitlines()
span, busy = map(int, lines[0].split())
rows = []
for l in lines[1:]:
    c, ns, name = l.split(" ", 2)
    name = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()[:70]
    rows.append((int(ns), int(c), name))
rows.sort(reverse=True)
it = r.iters.item()
print(f"{cfg}: {it} iterations, kernels {o.value} (all {a.value}), span {span / 1e6:.1f} ms, busy {busy / 1e6:.1f} ms "
      f"({100 * busy / span:.1f}%), {span / 1e6 / it:.2f} ms per iteration")
for ns, c, name in rows[:25]:
    print(f"{ns / 1e6:9.2f} ms {100 * ns / busy:5.1f}% {c:7d} x {ns / c / 1e3:7.1f} us  {name}")

gp = out + ".gaps"
if os.path.exists(gp):
    gl = []
    for l in open(gp).read().splitlines():
        c, ns, name = l.split(" ", 2)
        name = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()[:70]
        gl.append((int(ns), int(c), name))
    gl.sort(reverse=True)
    print(f"idle gaps > 5 us: {sum(c for _, c, _ in gl)} totalling {sum(n for n, _, _ in gl) / 1e6:.1f} ms, by the kernel that ends them:")
    for ns, c, name in gl[:12]:
        print(f"{ns / 1e6:9.2f} ms {c:7d} x {ns / c / 1e3:7.1f} us  {name}")
