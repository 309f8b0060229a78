"""CPU oracle for the PHIF factorize / apply-inverse / PCG path.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package,
and only as the checker / the timed CPU baseline. The product package
`paper_1808_01364_b200` never imports it and has no CPU fallback.

What it restates:

* dense.py       - kernels.py:23-119 (dpotrf Cholesky with 0-based NotSpd pivot,
                   triangular solves, CPQR interpolative decomposition via dgeqp3),
                   plus `cpqr_dlaqp2`, a pure-numpy restatement of LAPACK's
                   dgeqp3/dlaqp2 pivot rule that pins the GPU CPQR kernel.
* hierarchy.py   - hierarchy.py:102-168 (classify_active group order and members).
* phif.py        - the absent `factorization` module, restated from SPEC.md:229-347
                   and PAPER.md:118-395 (eliminate -> precondition -> sequential
                   skeletonize per level, root Cholesky, record replay for
                   F, F^-1, G^-1, G^-T).
* krylov.py      - the absent `krylov.pcg`.
* diagnostics.py - the absent `diagnostics`: power_norm, e_s, e_a,
                   dense oracle.

Pinning: the primitives (dense.py, hierarchy.py) are checked against the
reference's own importable modules and against golden vectors generated from
them (tests/golden/make_golden.py). The factorization, krylov and diagnostics
modules do not exist in the reference, so their pin is SPEC.md's worked
examples plus exact-mode invariants.
"""
