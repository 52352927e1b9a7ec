"""C4 (configs[3]) steady-state probe: W warm-up fixed-point iterations in one
call, then K iterations timed with the fused-GMRES per-core profile and the
CUPTI kernel timeline.  Usage: probe_c4.py [W] [K] [c3|c4]"""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import _lib  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 6
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = sys.argv[3] if len(sys.argv) > 3 else "c4"
t0 = time.time()
prob = inputs.problem_c4() if cfg == "c4" else inputs.problem_c3()
rmax = 128 if cfg == "c4" else 64
ops = gtr.operators(prob, eps=1e-12)
torch.cuda.synchronize()
print(f"assembly {time.time() - t0:.1f} s; H ranks {ops['H'].ranks()}")
print("H kinds", tb.core_kinds(ops["H"]))
modes = gtr.modes(prob)
d = len(modes)
g = inputs.rng(61)
z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1] + [4] * (d - 1) + [1]))
psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [rmax + 4] * (d - 1) + [1])
kw = dict(tol_k=1e-14, eps_round=1e-6, eps_solve=1e-6, rmax=rmax, matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4,
          restart=int(os.environ.get("TT_RESTART", "40")), max_restarts=20)
t0 = time.time()
r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, max_outer=W, **kw)
torch.cuda.synchronize()
k = r.k.item()
print(f"warm-up {W} iterations {time.time() - t0:.1f} s, k {k:.10f}, sweeps {r.sweeps_hist[:W].tolist()}")
print("psi ranks", psi.ranks())
lib = _lib.lib()
lib.tt_fused_profile(1)
fl, fms, ffl = C.c_int64(0), C.c_double(0.0), (C.c_double * 3)()
lib.tt_fused_profile_read(C.byref(fl), C.byref(fms), ffl)
lib.tt_fused_profile(1)
cnt = (C.c_uint64 * 5)()
lib.tt_counters(cnt, 1)
lc = C.CDLL(os.path.join(os.path.dirname(tb.__file__), "liblaunchcount.so"))
lc.lc_start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, k0=k, max_outer=K, **kw)
e1.record()
torch.cuda.synchronize()
a, o = C.c_ulonglong(0), C.c_ulonglong(0)
lc.lc_stop(C.byref(a), C.byref(o))
ms = e0.elapsed_time(e1)
lib.tt_counters(cnt, 1)
cms, cst, cl = (C.c_double * 64)(), (C.c_double * 64)(), (C.c_int64 * 64)()
lib.tt_fused_profile_cores(cms, cst, cl)
lib.tt_fused_profile_read(C.byref(fl), C.byref(fms), ffl)
lib.tt_fused_profile(0)
print(f"timed {K} iterations: {ms:.1f} ms = {ms / K:.1f} ms/iter ({1e3 * K / ms:.3f} iter/s); k {r.k.item():.10f}; "
      f"sweeps {r.sweeps_hist[:K].tolist()}; gemm flops/iter {cnt[0] / K / 1e9:.1f} GF, qr {cnt[2] / K / 1e9:.1f}, "
      f"jacobi {cnt[3] / K / 1e9:.1f}")
print(f"fused GMRES: {fl.value} launches {fms.value:.1f} ms ({100 * fms.value / ms:.1f}%), steps {ffl[2]:.0f}, "
      f"apply GF {ffl[0] / 1e9:.1f}, vec GF {ffl[1] / 1e9:.1f}")
print("core  ms/iter  steps/iter  launches/iter  ms/step  n  r0 r1")
rk = psi.ranks()
for t in range(d):
    if cl[t]:
        print(f"{t:4d} {cms[t] / K:8.2f} {cst[t] / K:10.1f} {cl[t] / K:8.1f} {cms[t] / max(cst[t], 1):8.3f}  {modes[t]} "
              f"{rk[t]} {rk[t + 1]}")
out = os.path.join("gpurun_out", f"probe_{cfg}_timeline.txt")
os.makedirs("gpurun_out", exist_ok=True)
lc.lc_dump(out.encode())
lines = open(out).read().splitlines()
span, busy = map(int, lines[0].split())
rows = []
for line in lines[1:]:
    c, ns, name = line.split(" ", 2)
    name = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()[:70]
    rows.append((int(ns), int(c), name))
rows.sort(reverse=True)
print(f"kernels {o.value}, span {span / 1e6:.1f} ms, busy {busy / 1e6:.1f} ms ({100 * busy / span:.1f}%)")
for ns, c, name in rows[:16]:
    print(f"{ns / 1e6:9.2f} ms {100 * ns / busy:5.1f}% {c:7d} x {ns / c / 1e3:8.1f} us  {name}")
