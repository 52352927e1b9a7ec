"""Real kernel timeline (CUPTI) of one C5 double sweep replayed as a CUDA graph."""
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200.sweep import SweepProblem  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
inst = inputs.c5_instance(r, seed=0)
sp = SweepProblem(inst["A"], inst["X"], "cuda")
sp.build_right()
g = sp.capture()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
lc = C.CDLL(os.path.join(os.path.dirname(tb.__file__), "liblaunchcount.so"))
lc.lc_start()
g.replay()
torch.cuda.synchronize()
a, o = C.c_ulonglong(0), C.c_ulonglong(0)
lc.lc_stop(C.byref(a), C.byref(o))
out = "gpurun_out/timeline_c5.txt"
lc.lc_dump(out.encode())
lines = open(out).read().splitlines()
span, busy = map(int, lines[0].split())
print(f"r={r}: kernels {o.value}, span {span / 1e3:.1f} us, busy {busy / 1e3:.1f} us, flops {sp.flops() / 1e9:.1f} GF "
      f"-> {sp.flops() / span:.1f} GF/s over the span")
rows = []
for l in lines[1:]:
    c, ns, name = l.split(" ", 2)
    rows.append((int(ns), int(c), subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()[:90]))
for ns, c, name in sorted(rows, reverse=True)[:8]:
    print(f"{ns / 1e3:9.1f} us {100 * ns / busy:5.1f}% {c:5d} x {ns / c / 1e3:7.2f} us  {name}")
