"""Edge shapes on the GPU, bitwise vs the oracle: tiny and block-boundary
sizes (n = 1..3, 31..33, 63..65, 95..97) for every precision through both
the two-call (lu_factor + lu_solve) and the one-call solve, singular
matrices at the first and the last step, and a zero right-hand side."""

import numpy as np
import pytest

import oracle
from oracle import gen
from paper_2107_12550_b200.errors import SingularMatrixError
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          device_solve, device_solve_system)

pytestmark = pytest.mark.gpu

SIZES = [1, 2, 3, 31, 32, 33, 63, 64, 65, 95, 96, 97]


@pytest.mark.parametrize("k", [2, 3, 4])
def test_block_boundaries(k):
    for n in SIZES:
        A = gen.planes(k, (n, n), 0, n, 600 + n)
        b = gen.planes(k, (n,), 2, n, 600 + n)
        lu_ref, sw_ref = oracle.lu(A)
        x_ref = oracle.solve(lu_ref, sw_ref, b)
        dm = DeviceMatrix.from_planes(A)
        piv = dm.lu_factor()
        bv, xv = DeviceVector.from_planes(b), DeviceVector(k, n)
        device_solve(dm, piv, bv, xv)
        assert np.asarray(piv.swaps()).tobytes() == sw_ref.tobytes(), n
        assert dm.download().tobytes() == lu_ref.tobytes(), n
        assert xv.download().tobytes() == x_ref.tobytes(), n
        dm2, xv2 = DeviceMatrix.from_planes(A), DeviceVector(k, n)
        piv2 = device_solve_system(dm2, bv, xv2)
        assert np.asarray(piv2.swaps()).tobytes() == sw_ref.tobytes(), n
        assert dm2.download().tobytes() == lu_ref.tobytes(), n
        assert xv2.download().tobytes() == x_ref.tobytes(), n


@pytest.mark.parametrize("k,n,col", [(2, 50, 0), (3, 50, 49), (4, 33, 32),
                                     (2, 70, 31)])
def test_singular_steps(k, n, col):
    A = gen.planes(k, (n, n), 0, n, 31 + col)
    A[:, :, col] = 0.0
    with pytest.raises(oracle.Singular) as e:
        oracle.lu(A)
    with pytest.raises(SingularMatrixError) as e2:
        DeviceMatrix.from_planes(A).lu_factor()
    assert e2.value.step == e.value.step
    b = gen.planes(k, (n,), 2, n, 1)
    with pytest.raises(SingularMatrixError) as e3:
        device_solve_system(DeviceMatrix.from_planes(A),
                            DeviceVector.from_planes(b), DeviceVector(k, n))
    assert e3.value.step == e.value.step


def test_zero_rhs():
    k, n = 3, 45
    A = gen.planes(k, (n, n), 0, n, 8)
    b = np.zeros((k, n))
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, b)
    xv = DeviceVector(k, n)
    device_solve_system(DeviceMatrix.from_planes(A), DeviceVector.from_planes(b),
                        xv)
    assert xv.download().tobytes() == x_ref.tobytes()
