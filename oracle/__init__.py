"""ORACLE — test infrastructure only.

A plain, slow, fp64 CPU implementation (NumPy / SciPy LAPACK) of what the
hot path of arXiv 2309.03347 computes.  It shares no code with the CUDA path
(`paper_2309_03347_b200/`) and neither imports the other; only the seeded
generators in `inputs/` serve both.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.
The product path never routes through it.

Modules
  tt.py         TT / TT-matrix algebra: full, matvec, add, scale, dot,
                orthogonalize, round, interfaces, local apply (§2.2).
  transport.py  factor matrices, dense and Eq.-4 assembly, TT and QTT operators
                (§2.1.3-2.1.5, §3.2-3.3, App. A).
  solvers.py    dense power iteration / GES, AMEn linear solve, TT k-eff
                fixed point (PAPER.md eqs. k_eff_fixed_points,
                TT_k_eff_fixed_points, §3.4).

Parity status of every function is listed in DESIGN.md "Oracle pins".
"""
