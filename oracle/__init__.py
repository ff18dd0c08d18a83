"""CPU fp64 ORACLE for the dual-gradient hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2603_04621_b200``, ``include/``, the CUDA library) never imports,
links or executes it, and this package imports nothing from the product: the
two share no code; only the seeded input generator ``synth`` serves both.

Every function is a plain, slow, obviously-correct restatement of PAPER.md
(the arxiv 2603.04621 text) in float64, citing the passage it follows:

* ``projection`` -- Euclidean projections onto the simple-constraint polytopes
  (Eq. 4-5): simplex {x>=0, sum x<=r}, box-cut
  {0<=x<=u, sum x<=r}, box {0<=x<=u}.  Sort / breakpoint definitions.
* ``dual`` -- scores, x*_gamma(lambda), the dual objective g(lambda) (Eq. 2,
  PAPER.md:83-91), Danskin gradient A x* - b, Jacobi row norms
  and primal scaling.
* ``agd`` -- projected Nesterov accelerated gradient ascent with the adaptive
  Lipschitz step and gamma continuation, plain
  projected gradient ascent (Appendix A.2).
* ``layout`` -- the log2 length bucketing of PAPER.md:369 and this framework's
  tile/shard plan, for the bit-exact layout check.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie each function to something
other than itself: brute-force active-set enumeration, KKT conditions, finite
differences, exact LP optima (scipy HiGHS) for weak duality, closed forms, the
Appendix A.2 inequality, Lemma 1, and the paper's printed gamma schedule.
"""
