#!/bin/bash
# C4 steady-state probe of the current build (tools/probe_c4.py 8 2) and the GMRES phase split
timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused|us  " | head -8
TT_NVCC_EXTRA=-DGM_PHASE_TIMING python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
timeout 600 python tools/probe_c4.py 8 1 c4 > gpurun_out/gmph.log 2>&1
python - <<'PY'
import collections
tot = collections.defaultdict(lambda: [0] * 9)
for l in open("gpurun_out/gmph.log"):
    if l.startswith("GMPH"):
        f = l.split(); t = tot[int(f[1])]; t[0] += 1; t[1] += int(f[2])
        for i in range(min(7, len(f) - 3)): t[2 + i] += int(f[3 + i])
for k, t in tot.items():
    print("cluster" if k else "grid", "steps", t[1], "cycles/step [top, stage3, cgs1, cgs2+norm, givens, stage1, stage2]", [round(x / t[1]) for x in t[2:]],
          "us/step %.1f" % (sum(t[2:]) / t[1] / 1965))
PY
