import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2505_08222_b200 import _native, _abi
lib = _native.lib(); _abi.declare_debug(lib)
for kind in (2, 3, 4):
    bad = C.c_uint64()
    assert lib.ut_debug_ieee_check(kind, 7, 1 << 28, 0, C.byref(bad)) == 0
    print(_native.LIB_PATH.name, "kind", kind, "mismatches", bad.value, "of", 1 << 28, flush=True)
