#!/bin/bash
# Fused GMRES phase split on the C4 steady state: instrumented build (-DGM_PHASE_TIMING), one timed iteration.
TT_NVCC_EXTRA=-DGM_PHASE_TIMING python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
timeout 600 python tools/probe_c4.py 8 1 c4 > gpurun_out/gmph.log 2>&1
python - <<'PY'
names = ["top", "st3", "cgs1", "norm-barrier", "givens", "st1", "st2", "sum1", "upd1", "pass2", "upd2+norm"]
rows = []
for l in open("gpurun_out/gmph.log"):
    if l.startswith("GMPH"):
        f = l.split()
        rows.append((int(f[1]), int(f[2]), [int(x) for x in f[3:14]], int(f[14]) if len(f) > 14 else 0))
for cl in (0, 1):
    sel = [r for r in rows if r[0] == cl]
    n = sum(r[1] for r in sel)
    if not n: continue
    tot = [sum(r[2][i] for r in sel) for i in range(11)]
    print("cluster" if cl else "grid", "steps", n, "reorth", sum(r[3] for r in sel),
          " us/step:", " ".join(f"{names[i]} {tot[i] / n / 1965:.1f}" for i in range(11)), f"| total {sum(tot) / n / 1965:.1f}")
# the last 52 grid launches = the timed iteration's last sweeps
for r in [r for r in rows if r[0] == 0][-27:]:
    print(r[1], r[3], " ".join(f"{x / r[1] / 1965:.1f}" for x in r[2]))
PY
