"""Device time of one LU solve (both sweeps) at size n.
usage: solve_time.py K N"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix, DeviceVector, device_solve
k = int(sys.argv[1]); n = int(sys.argv[2])
A = DeviceMatrix(k, n, n); A.generate(0, n, 5)
b = DeviceVector(k, n); b.generate(2, n, 5)
x = DeviceVector(k, n)
piv = A.lu_factor()
device_solve(A, piv, b, x); nat.sync()
nat.prof_enable(True); nat.prof_reset()
for _ in range(3):
    device_solve(A, piv, b, x)
nat.sync()
ms, c = nat.prof_read()["solve"]
print("k=%d n=%d solve %.2f ms" % (k, n, ms / c))
