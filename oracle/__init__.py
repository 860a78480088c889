"""CPU oracle for the elastic-distance hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2102_05221_b200`` never
imports, links or executes anything under ``oracle/``.

Contents
--------
``ek_oracle.c`` / ``eko.py``
    Our plain-C restatement of the reference engines (``base``/``ea``/
    ``eapruned``, the variant facade, the diagonal upper bound, the serial
    1-NN scan, the all-pairs loop, the z-normalised subsequence scan), with
    a ctypes front end.  Cell counts follow the reference exactly.
``refdrive.py``
    Drives the reference's OWN compiled kernel (``oracle/_ref/_speedups*.so``,
    built by ``oracle/Makefile`` from ``/root/reference/pkg/src/elastik/
    _speedups.pyx``) through a restatement of the reference's Python glue
    (``make_recurrence`` payloads, ``nn_search``).  Used to pin ``eko`` and as
    the ``--impl reference`` CPU arm of ``bench.py``.

Parity pins: ``tests/test_oracle_pins.py`` checks ``eko`` against the golden
fixtures produced from the live reference by ``tests/golden/make_golden.py``
and against the reference's known-answer tests (Fig. 1 cost 9 / 36 cells,
Fig. 4 counts, infeasible window, WDTW/ERP/MSM/TWE scalar KATs).
"""
