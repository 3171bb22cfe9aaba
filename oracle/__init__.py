"""CPU oracle for the two-level Kuhn-P1 heat solve — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this package, and only as the checker or the
timed CPU baseline.  The product path (``paper_2110_12932_b200``) never
imports it and has no CPU fallback.

Contents (each function cites the reference file:line it restates):

- ``kuhn``      — matrix-free restatement of the reference discretization
                  (P1 on Kuhn-subdivided hexes, lumped mass, symmetric Dirichlet
                  elimination, 4-point Gaussian quadrature, swept-track deposit,
                  Kuhn-P1 point location / interpolation, interface node set).
- ``pcg``       — Jacobi-PCG mirroring ``scipy.sparse.linalg.cg`` (scipy 1.18.1)
                  operation for operation, as called by ``lpbfsim/fem.py:271-298``.
- ``assembly``  — literal element-by-element P1 assembly + CSR + scipy ``cg``,
                  the reference's own CPU algorithm (``lpbfsim/fem.py:129-194``);
                  used as the CPU baseline ("port") and as a second pin.
- ``twolevel``  — the multirate / uniform two-level drivers
                  (``lpbfsim/multirate.py:105-217``) over either backend.

Parity pin: ``tests/golden/make_golden.py`` runs the unmodified reference
(``lpbfsim`` 0.1.0 with numpy 2.3.5 / scipy 1.18.1) in the build container and
commits its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this oracle against those vectors.
"""
