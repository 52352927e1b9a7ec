"""Step-by-step timing probe of the libtt ops (debug aid; prints as it goes)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs
from oracle import tt as ott
import paper_2309_03347_b200 as tb

def step(name, f):
    torch.cuda.synchronize(); t = time.perf_counter()
    out = f(); torch.cuda.synchronize()
    print(f"{name}: {1e3*(time.perf_counter()-t):.2f} ms", flush=True)
    return out

inst = inputs.c2_slice(101)
Yc = ott.tt_matvec_fast(inst["A"], inst["X"])
print("ranks", ott.ranks(Yc), flush=True)
G = tb.TTVec.from_cores(Yc)
step("orth rl d10", lambda: tb.tt_orthogonalize(G, -1))
print("ranks after", G.ranks(), flush=True)
G = tb.TTVec.from_cores(Yc)
step("orth lr d10", lambda: tb.tt_orthogonalize(G, 1))
G = tb.TTVec.from_cores(Yc)
step("round d10 eps1e-1", lambda: tb.tt_round(G, 1e-1))
print("ranks", G.ranks(), flush=True)
G = tb.TTVec.from_cores(Yc)
step("round d10 eps1e-8", lambda: tb.tt_round(G, 1e-8))
print("ranks", G.ranks(), flush=True)
inst = inputs.c2_instance(0)
A = tb.TTMat.from_cores(inst["A"]); X = tb.TTVec.from_cores(inst["X"])
Y = step("matvec d30", lambda: tb.matvec_out(A, X))
step("round d30", lambda: tb.tt_round(Y, 1e-8, 128))
print("ranks", Y.ranks(), flush=True)
