"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference (``ldurepart``) algorithms on the
hot path: cavity generator, repartitioner, coefficient update and the Krylov
solvers.  Each function cites the reference ``file:line`` it follows
(paths relative to ``/root/reference/pkg/src/ldurepart/``).

Who may import this package: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` — and there only
as the checker or the timed CPU baseline.  The product package
``paper_2510_08536_b200`` never imports it; the product path fails loudly when
its CUDA library is missing instead of falling back here.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
``tests/golden/golden.npz``, produced by running the reference itself
(``tests/golden/make_golden.py``).  Jacobi-PCG is pinned indirectly (uniform
cavity diagonal ⇒ same iterates as the reference CG within rounding, SURVEY.md
App. B); BiCGStab has no reference implementation — parity unpinned.
"""
