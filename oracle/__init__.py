"""CPU oracle for the DPV-SLAM hot path — TEST INFRASTRUCTURE ONLY.

This package is the *checker*, never the product.  It restates, in plain
numpy float64, the reference algorithms of ``patchslam`` (pkg/src/patchslam,
numpy/scipy, float64) on the structure-of-arrays graph layout used by the
B200 package, plus a float64 restatement of the correlation lookup (PAPER.md
Eq. 4) that the reference does not implement.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The product
package ``paper_2408_01654_b200`` never imports it and has no CPU fallback.

Pinning: ``ba_oracle`` / ``geometry_oracle`` / ``cholesky_oracle`` /
``loop_oracle`` are checked
against golden fixtures produced by the real reference
(``tests/golden/make_golden.py``; ``tests/test_oracle_golden.py``).
``corr_oracle`` has no reference implementation (SPEC.md:14 puts Eq. 4 out of
scope): **parity unpinned** by the reference; it is pinned only by its own
known-answer tests (``tests/test_corr_oracle.py``).
"""
