"""CPU oracle for the STFAS hot path — TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_1608_01102_b200``) runs exclusively on the CUDA library and fails
loudly when it is missing.

Contents
--------
``grid``    -- MAC grid metadata (restates ``pkg/src/smokectrl/fields.py:37-89``).
``ops``     -- fp64 numpy restatement of the reference raw kernels:
               div/grad/Laplacian/Poisson/projection (``fields.py:145-358``),
               Taylor advection and its adjoints, self-advection S(a,w), its
               Jacobian and transpose (``advection.py:43-441``).
``sim``     -- forward step and AO sweep (``simulator.py:56-122``,
               ``ao.py:27-254``).
``stfas``   -- the STFAS / NSO solver that the reference only specifies
               (``SPEC.md:285-374``, PAPER Eq. 8/9, Alg. 2, Appendix A):
               KKT residual, coloured time-line SCGS smoother, cell/face R/P,
               FAS V-cycle, ``solve_nso``.
``dense``   -- dense Newton solve of the Eq. 8 KKT system on tiny grids
               (``SPEC.md:315``, ``:526``) used as a known-answer oracle.

Parity pinning
--------------
* Sub-operators (``ops``, ``sim``) are pinned against golden vectors produced
  by the *reference itself* (``tests/golden/make_golden.py`` imports
  ``/root/reference/pkg/src/smokectrl`` in the build container and commits the
  ``.npz`` fixtures).
* The STFAS layer has no reference implementation: it is
  pinned to the SPEC known-answer tests instead — the residual vanishes at the
  dense-Newton KKT solution, its Jacobian matches finite differences, the
  smoother reproduces a dense single-cell solve and ``solve_nso`` converges to
  the dense-Newton solution (``tests/test_oracle_stfas.py``).  There are no
  reference golden vectors for STFAS: "parity unpinned" w.r.t. reference code
  at that level, pinned w.r.t. the SPEC KATs.
"""
