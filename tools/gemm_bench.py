"""Config-1 GEMM (C = A*B, n x n, DD/TD/QD) through the C ABI: device time
per product and FP64 issue rate (dead-code-free instruction counts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix
MADD = {2: 29, 3: 214, 4: 326}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = nat.lib()
for k in (2, 3, 4):
    A = DeviceMatrix(k, n, n); A.generate(0, n, 210712551)
    B = DeviceMatrix(k, n, n); B.generate(1, n, 210712551)
    C = DeviceMatrix(k, n, n)
    nat.check(L.mpcore_mat_mul(A.handle, B.handle, C.handle), "mm")
    t0 = time.perf_counter()
    for _ in range(reps):
        nat.check(L.mpcore_mat_mul(A.handle, B.handle, C.handle), "mm")
    dt = (time.perf_counter() - t0) / reps
    print("k=%d n=%d  %.2f ms  %.1f GFLOP/s (2n^3/t)  %.2f T FP64 instr/s" % (
        k, n, dt * 1e3, 2 * n ** 3 / dt / 1e9, n ** 3 * MADD[k] / dt / 1e12))
