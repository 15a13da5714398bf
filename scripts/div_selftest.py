import ctypes, sys
sys.path.insert(0, "/root/repo")
from paper_2202_05628_b200 import _lib
L = _lib.lib()
bad = ctypes.c_ulonglong(0)
buf = (ctypes.c_double * 48)()
for seed in (12345, 777):
    assert L.artemis_debug_division_selftest(1 << 28, seed, ctypes.byref(bad), buf) == 0
    print("seed", seed, "mismatches", bad.value)
    for k in range(min(16, bad.value)):
        print(int(buf[3*k]), repr(buf[3*k+1]), repr(buf[3*k+2]), (buf[3*k+1]).hex(), (buf[3*k+2]).hex())
