"""B200-native (sm_100a) decision-evaluation path of BiScale (arXiv 2602.18755).

The product is ``libbiscale_gpu.so`` (C ABI in ``include/biscale_gpu.h``);
``pdsim`` mirrors the reference's ``pdsim`` C++ interface on top of it.
"""
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["LIB_PATH", "lib"]
