"""CPU oracle for the MGR-GMRES hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and only
as the checker or the timed CPU baseline; the product path
(``paper_1801_08464_b200``) never imports it and fails loudly when its CUDA
library is missing.

What it restates (each module cites the reference file:line it follows):

* ``oracle.sparse``  — ncpflow/sparse.py (CSR semantics, scipy products that
  drop exact zeros, extract keeping stored zeros).
* ``oracle.mgr``     — ncpflow/mgr.py (build_rp, setup_from_matrix,
  mgr_apply, F-solvers, block-diagonal relaxation).
* ``oracle.krylov``  — ncpflow/krylov.py (restarted right-preconditioned
  GMRES, CGS2, Givens, true-residual restarts).
* ``oracle.amg``     — the AMG the north star names (PMIS, extended+i,
  L1-Jacobi, dense-LU coarsest).  The reference has none of these
  (SURVEY.md §0 item 2); the contract is SURVEY.md §8(c), the heavy loops are
  C in ``oracle/csrc/amg_oracle.c``.  Strength, row-sign normalisation,
  Galerkin product and V-cycle structure follow ncpflow/amg.py.
* ``oracle.blockscale`` — per-cell block inverse / block scaling (the pinned
  readings D1-D3 of SURVEY.md §7).

Pinning: tests/test_oracle_vs_reference.py checks every restated piece
against the reference package itself (imported from /root/reference when it
is present, i.e. in the build container) and tests/golden/ holds fixtures
generated from it (tests/golden/make_golden.py).  PMIS / extended+i /
L1-Jacobi have no reference implementation, so they are pinned by the
reference's own AMG property tests (tests/test_amg.py analogues) and by
algorithm invariants; DESIGN.md records this as "parity pinned by
properties" for those three pieces.
"""
