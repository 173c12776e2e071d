"""One LU of a seeded K x N x N matrix (for profiler captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix
k = int(sys.argv[1]); n = int(sys.argv[2])
A = DeviceMatrix(k, n, n); A.generate(0, n, 5)
A.lu_factor(); nat.sync()
print("lu done", k, n)
