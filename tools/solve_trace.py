"""Owner timeline of the triangular sweeps (MPCORE_TRACE_SOLVE=1).
usage: solve_trace.py K N"""
import ctypes, os, sys
import numpy as np
os.environ["MPCORE_TRACE_SOLVE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix, DeviceVector, device_solve
k = int(sys.argv[1]); n = int(sys.argv[2])
A = DeviceMatrix(k, n, n); A.generate(0, n, 5)
b = DeviceVector(k, n); b.generate(2, n, 5)
x = DeviceVector(k, n)
piv = A.lu_factor()
for _ in range(3):
    device_solve(A, piv, b, x)
nat.sync()
nb = (n + 31) // 32
buf = np.zeros(2 * nb * 8, dtype=np.uint64)
nat.check(nat.lib().mpcore_debug_solve_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), buf.size), "trace")
t = buf.reshape(2, nb, 8).astype(np.int64)
for sw, name in ((0, "forward"), (1, "backward")):
    T = t[sw]; t0 = T[:, 0].min(); T6 = T[:, 6].copy()
    print("== %s: total %.1f us" % (name, (T[:, 3].max() - t0) / 1e3))
    order = range(nb) if sw == 0 else range(nb - 1, -1, -1)
    prev_end = None
    for i, blk in enumerate(order):
        s, a, c, d, cs, lastv, _, fp = (T[blk] - t0) / 1e3
        iters = T6[blk]
        if i < 6 or i % 8 == 0 or i > nb - 4:
            print("blk %3d start %7.1f full-done %7.1f crit-done %7.1f diag-done %7.1f | crit %5.1f diag %5.1f gap-from-prev-diag %5.1f | crit-start %7.1f first-poll %7.1f all-valid %7.1f iters %d"
                  % (blk, s, a, c, d, c - max(a, prev_end or 0), d - c, c - (prev_end or 0), cs, fp, lastv, iters))
        prev_end = d
