"""B200-native particle hot path of Nauticle (arXiv 1710.08259).

* ``csrc/``      hand-written sm_100a CUDA + the C-ABI (include/nauticle_gpu.h)
                 -> ``libnau_b200.so`` (built by __graft_entry__.build())
* ``nau``        ctypes binding of that C-ABI (Context, operators, errors)
* ``scenes``     seeded synthetic inputs of the BASELINE.json configurations
"""
from . import nau  # noqa: F401

__all__ = ["nau"]
