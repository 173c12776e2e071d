"""Host-side timing of each API call of one bench step (diagnostics)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix, DeviceVector, device_solve
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
A0 = DeviceMatrix(k, n, n); A0.generate(0, n, 5)
b = DeviceVector(k, n); b.generate(2, n, 5)
W = DeviceMatrix(k, n, n); x = DeviceVector(k, n)
for rep in range(4):
    t = [time.perf_counter()]
    W.copy_from(A0); t.append(time.perf_counter())
    piv = W.lu_factor(); t.append(time.perf_counter())
    device_solve(W, piv, b, x); t.append(time.perf_counter())
    del piv; t.append(time.perf_counter())
    print("copy %.2f  lu %.2f  solve %.2f  release %.2f ms" % tuple(
        (t[i + 1] - t[i]) * 1e3 for i in range(4)))
