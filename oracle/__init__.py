"""CPU oracle for the kronblur hot path — TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2410_00233_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` (as the checker) and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import it.  The product path runs on the GPU
through ``libkronblur_b200.so`` and fails loudly when that library is missing.

Contents (each function cites the reference file:line it restates; paths are
relative to the reference package root ``pkg/src/kronblur/``):

* :mod:`oracle.structured` — matrix-free R(A) products for a zero-BC PSF blur
  (closed form of ``rearrange.py:67-75`` ∘ ``blurmodel.py:87-121``) and the
  exact structured TSVD of R(A).
* :mod:`oracle.lowrank` — eGKB / RSVD / orthonormalize restated to take
  matvec callables (``lowrank.py:114-372``, ``linalg.py:134-199``).
* :mod:`oracle.sb` — Kronecker-sum apply, augmented operator, CGLS and split
  Bregman restated (``kronop.py:58-123``, ``regularizers.py:37-130``,
  ``cgls.py:50-116``, ``splitbregman.py:32-192``, ``metrics.py:28-57``).

Pinning: ``tests/golden/make_golden.py`` imports the reference itself (only in
the build container, where ``/root/reference`` exists) and writes the golden
fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
restatement against them bit-for-bit (eGKB/RSVD/CGLS/SB on dense inputs) and
to 1e-12 (structured R(A) vs the dense ``rearrange(build_blur_matrix(...))``).
"""
