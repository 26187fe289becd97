"""paper_1412_1127_b200 — B200-native execution of the OpenACC `reduction(op:var)` clause (IPMACC, arxiv 1412.1127).

The product is ``libipm.so`` (C ABI in ``include/ipm.h``, CUDA sm_100a kernels in ``csrc/``); ``ipm`` is its thin
Python binding. See DESIGN.md.
"""
from . import ipm  # noqa: F401  (raises if libipm.so is missing: there is no CPU fallback)

__all__ = ["ipm"]
