"""CPU ORACLE — test infrastructure only, NOT part of the product path.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`.  The CUDA path
(`paper_2104_01439_b200/`) never imports it, and this package never imports
the CUDA path; the two share only the seeded generators in `workloads/`.

A plain, slow, obviously-correct fp64 (complex128) implementation of the hot
path of arXiv 2104.01439 ("PAPER"), written from the paper:

  fem.py      Q1 element matrices and element-loop CSR assembly of
              A(k, eps) = K - M(k, eps) - i B(k)
              canonical prolongation I and restriction I^T
  twogrid.py  damped Jacobi, two-grid V(nu,nu) cycle with a direct coarse
              solve (Alg. 1; coarse LU PAPER.md:511-512)
  fgmres.py   right-preconditioned flexible GMRES (Saad 1993)
              and the average convergence rate rho
  lfa.py      the paper's LFA symbols, used only as an
              independent pin of the V-cycle
  solve.py    end-to-end driver: spec -> iterations, solution, report

Every function is pinned by `tests/test_oracle_*.py` (-m "not gpu") against
closed forms, printed stencils, brute-force dense algebra or the paper's LFA.
Parity status per function is listed in DESIGN.md ("Oracle pins").
"""
