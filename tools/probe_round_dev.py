"""GPU tt_round vs the oracle on C2 d=30 (rmax 128): per-bond max |dsigma| / sigma_1
before and after the first rmax-binding bond (the round-1 test tolerance question)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402
from oracle import tt as ott  # noqa: E402

for seed in (0, 1, 2):
    inst = inputs.c2_instance(seed)
    Y = tb.matvec_out(tb.TTMat.from_cores(inst["A"]), tb.TTVec.from_cores(inst["X"]))
    _, disc, sv = tb.tt_round(Y, 1e-8, 128, want_info=True)
    torch.cuda.synchronize()
    ref, info = ott.tt_round(ott.tt_matvec_fast(inst["A"], inst["X"]), 1e-8, 128)
    s1 = max(s[0] for s in info["sv"])
    binds, rows = 0, []
    for k, s in enumerate(info["sv"]):
        dev = np.max(np.abs(sv[k, :len(s)].cpu().numpy() - s)) / s1
        rows.append(f"{k}:{dev:.1e}{'*' if binds else ''}")
        binds += int(ott.ranks(ref)[k + 1] < len(s))
    print(f"seed {seed} ranks equal {Y.ranks() == ott.ranks(ref)}:", " ".join(rows), flush=True)
