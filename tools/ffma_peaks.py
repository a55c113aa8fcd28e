import sys, ctypes; sys.path.insert(0,'/root/repo')
from paper_2006_06762_b200 import runtime as rt
lib=rt.load()
for fn in ("lt_ffma_peak","lt_ffma_peak_reg"):
    t,m=ctypes.c_double(),ctypes.c_double()
    rt.check(getattr(lib,fn)(0,ctypes.byref(t),ctypes.byref(m)),fn)
    print(fn, round(t.value,2), "TFLOP/s", round(m.value,3), "ms")
