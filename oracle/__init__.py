"""TEST INFRASTRUCTURE — the parity oracle for the particle hot path.

Nothing under ``oracle/`` is part of the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it, and only as the checker / the timed
CPU reference, never as the code path being measured or shipped.

* ``oracle.port``  — ctypes wrapper of ``nau_oracle.c``, a plain-C restatement of
  the reference algorithm (each function cites /root/reference/proj file:line).
* ``oracle.ref``   — ctypes wrapper of ``_ref/libnauticle_ref.so``: the reference
  C++ sources compiled unmodified against ``shim/`` (Eigen / doctest subsets).
  It pins ``port`` (tests/test_oracle.py) and produced ``tests/golden/``.
"""
