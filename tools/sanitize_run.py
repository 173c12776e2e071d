"""compute-sanitizer workload (SURVEY §5 sanitizers): small LU + solve
paths whose kernels use the cross-CTA word protocols (panel, sweeps), the
one-call [A | b] path, the GEMM and the long residual.  Each result is
checked bitwise against the oracle (test infrastructure), so a clean
sanitizer log comes with a correct answer.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from oracle import gen  # noqa: E402
from paper_2107_12550_b200 import _native as nat  # noqa: E402
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,  # noqa: E402
                                          device_solve, device_solve_system)

cases = [(3, 257), (2, 513)]
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]]
for k, n in cases:
    seed = 4242 + n
    A = gen.planes(k, (n, n), 0, n, seed)
    xt = gen.planes(k, (n,), 2, n, seed)
    b = oracle.matvec(A, xt)
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, b)
    M = DeviceMatrix.from_planes(A)
    piv = M.lu_factor()
    bv = DeviceVector.from_planes(b)
    x = DeviceVector(k, n)
    device_solve(M, piv, bv, x)
    assert np.asarray(piv.swaps()).tobytes() == sw_ref.tobytes()
    assert M.download().tobytes() == lu_ref.tobytes()
    assert x.download().tobytes() == x_ref.tobytes()
    M1 = DeviceMatrix.from_planes(A)
    x1 = DeviceVector(k, n)
    device_solve_system(M1, bv, x1)
    assert x1.download().tobytes() == x_ref.tobytes()
    B = gen.planes(k, (n, n), 1, n, seed)
    Bd = DeviceMatrix.from_planes(B)
    C = DeviceMatrix(k, n, n)
    Ad = DeviceMatrix.from_planes(A)
    nat.check(nat.lib().mpcore_mat_mul(Ad.handle, Bd.handle, C.handle), "mm")
    assert C.download().tobytes() == oracle.gemm(A, B).tobytes()
    nat.sync()
    print("k=%d n=%d: LU, solve, one-call solve, GEMM bitwise vs oracle" % (k, n))
print("sanitize_run ok")
