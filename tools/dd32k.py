"""Single-GPU one-call solve of the config-4 system (DD n=32768, seeded
recipe as bench --config 4 builds it) vs. the time of the distributed
protocol at one rank."""
import ctypes, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix, DeviceVector
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
k = 2
L = nat.lib()
W = DeviceMatrix(k, n, n + 1)
A0 = DeviceMatrix(k, n, n); A0.generate(0, n, 210712554)
xt = DeviceVector(k, n); xt.generate(2, n, 210712554)
b = DeviceVector(k, n)
nat.check(L.mpcore_mat_vec(A0.handle, xt.handle, b.handle), "mv")
x = DeviceVector(k, n)
sw = np.zeros(n, dtype=np.int32); ss = ctypes.c_int32()
a0p, bp, wp, xp = A0.device_ptr(), b.device_ptr(), W.device_ptr(), x.device_ptr()
def step():
    nat.check(L.mpcore_dev_copy2d(k, n, n, wp, n + 1, n * (n + 1), a0p, n, n * n), "A")
    nat.check(L.mpcore_dev_copy2d(k, n, 1, wp + n * 8, n + 1, n * (n + 1), bp, 1, n), "b")
    nat.check(L.mpcore_dev_solve_system(k, n, wp, n + 1, n * (n + 1), 0, xp,
              sw.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(ss)), "solve")
step()
t = nat.StreamTimer()
t.start(); step(); ms = t.stop()
print("DD n=%d one-call solve: %.1f ms, %.1f GFLOP/s" % (n, ms, (2/3) * n**3 / ms / 1e6))
