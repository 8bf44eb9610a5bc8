"""CPU ORACLE for the B200 WMG tomography hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_1310_0956_b200`` never
imports, links or executes anything in here.

Contents
--------
``cproj``      ctypes wrapper of ``wmg_oracle.c``: the reference line kernel
               (geometry.py:88-128) as an exact CSR, plus W x / W^T y / row and
               column sums with the reference's summation orders.
``geometry``   host-side restatement of ``Geometry`` / ``build_geometry`` /
               ``_snapped_trig`` (geometry.py:34-85).
``solvers``    numpy restatements of ``sirt_solve`` / ``normal_operator`` /
               ``bicgstab_solve`` (solvers.py:79-243) plus the new CGLS,
               flexible PCG-NE (WMG-CGLS) and GMRES definitions, all using the
               deterministic DET_SUM reduction shared bit for bit with the GPU.
``multilevel`` restatement of the Haar operators, hierarchy and WTG V-cycle
               (multilevel.py:36-208) on scipy sparse matrices.

Parity pinning: ``tests/golden/make_golden.py`` imports the reference (only in
the build container, where ``/root/reference`` exists) and freezes hashes and
vectors under ``tests/golden/``; ``tests/test_oracle.py`` checks the oracle
against them.
"""
