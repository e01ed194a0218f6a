"""CPU oracle for the ImprovedGS+ densification hot path -- TEST INFRASTRUCTURE ONLY.

This package is a from-scratch CPU restatement (numpy) of the reference
``splitkit`` algorithms on the densification path (edge-importance map,
budgeted candidate selection, Long-Axis-Split).  It exists to CHECK the CUDA
product path, never to BE it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2603_08661_b200`` never imports it and fails
  loudly when its CUDA library is missing.

Pinning.  The reference itself is pure Python over numpy/scipy
(``/root/reference/pkg/src/splitkit``).  The third-party arithmetic it relies
on -- ``scipy.ndimage.convolve/correlate`` (scipy 1.18.1 here; the reference
pins only ``scipy>=1.10``, ``pkg/pyproject.toml:10-13``), ``np.hypot`` /
``np.arctan2`` (glibc 2.39 libm), ``np.median``, ``np.argsort(kind="stable")``
(numpy 2.3.5) -- is restated here in its published operation order (see
``oracle/edge.py`` for the NI_Correlate order).  The restatement is pinned
against golden vectors produced by running the real reference in the build
container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and
against the reference's own known-answer tests (``tests/test_oracle_golden.py``).
"""
