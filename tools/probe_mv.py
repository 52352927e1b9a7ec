"""64-instance batched exact matvec of C2 (configs[1]) for ncu captures:
prints the CUDA-event time and the algorithmic bytes per launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import inputs  # noqa: E402
import paper_2309_03347_b200 as tb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
insts = [inputs.c2_instance(b) for b in range(B)]
As = [tb.TTMat.from_cores(i["A"], device=dev) for i in insts]
Xs = [tb.TTVec.from_cores(i["X"], device=dev) for i in insts]
Ys = [tb.TTVec(a.m, [p * q for p, q in zip(a.Rcap, x.rcap)], dev) for a, x in zip(As, Xs)]
nbytes = sum(8 * sum(R0 * 4 * R1 + r0 * 2 * r1 + R0 * R1 * 2 * r0 * r1 for R0, R1, r0, r1 in
                     zip(i["R"][:-1], i["R"][1:], i["r"][:-1], i["r"][1:])) for i in insts)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
from paper_2309_03347_b200.tt import MatvecBatch  # noqa: E402
run = MatvecBatch(As, Xs, Ys)
for _ in range(3):
    run()
ts = []
for _ in range(reps):
    flush.fill_(1.0)
    torch.cuda._sleep(2_000_000)      # hide the host-side enqueue behind a GPU sleep
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
t = ts[len(ts) // 2]
print(f"B={B} bytes={nbytes} median_ms={t:.4f} GB/s={nbytes / t / 1e6:.1f}")
