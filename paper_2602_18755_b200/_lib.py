"""Loader for the in-tree sm_100a library ``libbiscale_gpu.so``.

There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every entry point of the package raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import _abi

PKG = Path(__file__).resolve().parent
# BS_LIB_PATH: an alternative in-tree build (A/B experiments of compile-time variants)
LIB_PATH = Path(os.environ.get("BS_LIB_PATH", str(PKG / "libbiscale_gpu.so")))

_lock = threading.Lock()
_lib = None


class NativeLibraryMissing(ImportError):
    pass


def lib() -> C.CDLL:
    """The loaded C-ABI library with prototypes set (loads once)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the sm_100a path has no CPU fallback)")
            handle = C.CDLL(str(LIB_PATH))
            for name, restype, argtypes in _abi.PROTOTYPES:
                fn = getattr(handle, name)
                fn.restype = restype
                fn.argtypes = argtypes
            if handle.bs_abi_version() != 1:
                raise NativeLibraryMissing("libbiscale_gpu.so ABI version mismatch")
            _lib = handle
        return _lib


def exported_symbols() -> list[str]:
    return [name for name, _, _ in _abi.PROTOTYPES]
