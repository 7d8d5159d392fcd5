"""Loader for the in-tree CUDA library. There is no fallback: if the library is
missing or cannot be loaded, every entry point raises."""
import ctypes as C
import os
import pathlib

from . import _abi

# UT_LIBRARY selects another build of the same library (A/B performance runs of
# in-tree variants under _lib/); unset, the in-tree product library is used.
LIB_PATH = pathlib.Path(os.environ.get("UT_LIBRARY") or
                        pathlib.Path(__file__).resolve().parent / "_lib" / "libutrack_b200.so")
_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_08222_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        handle = C.CDLL(str(LIB_PATH))
        _abi.declare_product(handle)
        if handle.ut_abi_version() != _abi.UT_ABI_VERSION:
            raise NativeLibraryMissing("libutrack_b200.so ABI version mismatch")
        _lib = handle
    return _lib
