"""Per-panel timeline of one LU (direct launches, event timestamps).
usage: timeline.py K N [panels to print]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix
k = int(sys.argv[1]); n = int(sys.argv[2])
A0 = DeviceMatrix(k, n, n); A0.generate(0, n, 5)
W = DeviceMatrix(k, n, n)
W.copy_from(A0); W.lu_factor()       # warm-up
W.copy_from(A0); nat.sync()
nat.prof_enable(True); nat.prof_reset()
W.lu_factor(); nat.sync()
cnt = ctypes.c_int64()
L = nat.lib()
nat.check(L.mpcore_debug_timeline(None, 0, ctypes.byref(cnt)), "tl")
buf = np.zeros(3 * cnt.value)
nat.check(L.mpcore_debug_timeline(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), buf.size, ctypes.byref(cnt)), "tl")
nat.prof_enable(False)
t = buf.reshape(-1, 3)
names = nat.PROF_SLOTS
t0 = t[:, 1].min()
print("LU wall (first start -> last end): %.1f us, launches %d" % (t[:, 2].max() - t0, len(t)))
for row in t[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print("%-8s %9.1f %9.1f  (%6.1f)" % (names[int(row[0])], row[1] - t0, row[2] - t0, row[2] - row[1]))
