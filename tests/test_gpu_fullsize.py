"""Parity at the benchmark sizes: the exact bench workloads (BASELINE
config 2, TD n = 2048 with the bench seed; DD n = 4096, whose panels span
128 CTAs) factored and solved on the GPU must equal the oracle bit for bit
-- pivots, factors and solution.  The oracle (C++ restatement, OpenMP over
rows) needs ~10-20 s per case on the GPU box's host cores."""

import numpy as np
import pytest

import oracle
from oracle import gen
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          device_solve, device_solve_system)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,n,seed", [(3, 2048, 210712552), (2, 4096, 77)])
def test_bench_workload_bitwise(k, n, seed):
    # the bench's own inputs: device generator + device mat_vec
    A0 = DeviceMatrix(k, n, n)
    A0.generate(0, n, seed)
    xt = DeviceVector(k, n)
    xt.generate(2, n, seed)
    b = DeviceVector(k, n)
    nat.check(nat.lib().mpcore_mat_vec(A0.handle, xt.handle, b.handle), "mv")
    A = A0.download()
    bh = b.download()
    assert A.tobytes() == gen.planes(k, (n, n), 0, n, seed).tobytes()
    assert bh.tobytes() == oracle.matvec(A, xt.download()).tobytes()
    piv = A0.lu_factor()
    x = DeviceVector(k, n)
    device_solve(A0, piv, b, x)
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, bh)
    assert np.asarray(piv.swaps()).tobytes() == sw_ref.tobytes()
    assert A0.download().tobytes() == lu_ref.tobytes()
    assert x.download().tobytes() == x_ref.tobytes()
    # the bench's one-call path (b as an extra column of the LU)
    A1 = DeviceMatrix.from_planes(A)
    x1 = DeviceVector(k, n)
    piv1 = device_solve_system(A1, b, x1)
    assert np.asarray(piv1.swaps()).tobytes() == sw_ref.tobytes()
    assert A1.download().tobytes() == lu_ref.tobytes()
    assert x1.download().tobytes() == x_ref.tobytes()


def test_bench_qd_workload_bitwise():
    # BASELINE config 2 for QD (n = 2048, the bench seed): one-call path
    k, n, seed = 4, 2048, 210712552
    A0 = DeviceMatrix(k, n, n)
    A0.generate(0, n, seed)
    xt = DeviceVector(k, n)
    xt.generate(2, n, seed)
    b = DeviceVector(k, n)
    nat.check(nat.lib().mpcore_mat_vec(A0.handle, xt.handle, b.handle), "mv")
    A, bh = A0.download(), b.download()
    x = DeviceVector(k, n)
    piv = device_solve_system(A0, b, x)
    lu_ref, sw_ref = oracle.lu(A)
    assert np.asarray(piv.swaps()).tobytes() == sw_ref.tobytes()
    assert A0.download().tobytes() == lu_ref.tobytes()
    assert x.download().tobytes() == oracle.solve(lu_ref, sw_ref, bh).tobytes()


@pytest.mark.parametrize("k,n", [(2, 2048), (3, 1024), (4, 768)])
def test_config1_gemm_bitwise(k, n):
    # BASELINE config 1 recipe (slots A: 0, B: 1) at or near full size
    seed = 210712551
    A = DeviceMatrix(k, n, n)
    A.generate(0, n, seed)
    B = DeviceMatrix(k, n, n)
    B.generate(1, n, seed)
    C = DeviceMatrix(k, n, n)
    nat.check(nat.lib().mpcore_mat_mul(A.handle, B.handle, C.handle), "mm")
    assert C.download().tobytes() == \
        oracle.gemm(A.download(), B.download()).tobytes()
