"""One LU + solve (default TD, n=2048; the bench's one-call path) for
profiling under ncu.
Direct launches (no graph) so each kernel is a separate ncu target."""
import os, sys
os.environ.setdefault("MPCORE_NO_GRAPH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix, DeviceVector, device_solve_system
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
A0 = DeviceMatrix(k, n, n); A0.generate(0, n, 5)
b = DeviceVector(k, n); b.generate(2, n, 5)
W = DeviceMatrix(k, n, n); x = DeviceVector(k, n)
for rep in range(int(os.environ.get("REPS", "1"))):
    W.copy_from(A0)
    device_solve_system(W, b, x)      # the bench's one-call path
nat.sync()
print("ok")
