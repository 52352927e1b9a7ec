import ctypes as C, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
import paper_2309_03347_b200 as tb
lc = C.CDLL(os.path.join(os.path.dirname(tb.__file__), "liblaunchcount.so"))
g = inputs.rng(5)
for r in (32, 64, 68, 96):
    for decay in (0, 1):
        d = 12
        ranks = [1] + [min(r, 2**k, 2**(d-k)) for k in range(1, d)] + [1]
        cores = inputs.random_tt(g, [2]*d, ranks)
        if decay:
            for k in range(d):
                c = cores[k]
                cores[k] = c * np.logspace(0, -10, c.shape[2]).reshape(1, 1, -1)
        X = tb.TTVec.from_cores(cores)
        for _ in range(2):
            Y = tb.TTVec.from_cores(cores); tb.tt_round(Y, 1e-14, 200)
        torch.cuda.synchronize()
        lc.lc_start()
        Y = tb.TTVec.from_cores(cores); tb.tt_round(Y, 1e-14, 200); torch.cuda.synchronize()
        a, o = C.c_ulonglong(0), C.c_ulonglong(0); lc.lc_stop(C.byref(a), C.byref(o))
        lc.lc_dump(b"/tmp/jt.txt")
        tot = {}
        for l in open("/tmp/jt.txt").read().splitlines()[1:]:
            c, ns, name = l.split(" ", 2)
            if "jacobi" in name or "qr_kernel" in name:
                tot[("jacobi" if "jacobi" in name else "qr")] = (int(c), int(ns) / 1e3)
        print(r, "decay" if decay else "flat", tot)
