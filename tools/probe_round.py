"""One C2 (configs[1]) instance: exact matvec then tt_round(1e-8, 128), for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402

dev = torch.device("cuda", 0)
inst = inputs.c2_instance(0)
A = tb.TTMat.from_cores(inst["A"], device=dev)
X = tb.TTVec.from_cores(inst["X"], device=dev)
Y = tb.matvec_out(A, X)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(reps):
    tb.tt_matvec(A, X, Y)
    tb.tt_round(Y, 1e-8, 128)
torch.cuda.synchronize()
print("ranks", Y.ranks())
