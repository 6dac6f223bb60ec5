"""B200-native first-order finite-volume hot path (arXiv:1701.05431).

The product is ``libfv2d.so`` (C ABI, ``include/fv2d.h``) built from
``csrc/``; :mod:`paper_1701_05431_b200.fv2d` is its thin ctypes binding.
:mod:`paper_1701_05431_b200.inputs` holds the seeded initial-condition
generators shared with the test oracle.
"""
__all__ = ["fv2d", "inputs"]
