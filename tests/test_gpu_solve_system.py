"""One-call solve (mpcore_solve_system / mpcore_dev_solve_system): the
right-hand side rides along the factorisation as an extra column, so its
exchanges and updates are the forward substitution.  Factors, pivots and
solution must equal the two-call path (lu_factor + lu_solve) and the
oracle bit for bit, for every precision, ragged n and panel widths, and a
singular matrix must report the same step."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
from oracle import gen
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.errors import SingularMatrixError
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          device_solve_system)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,n,nb", [(2, 300, 0), (3, 257, 16), (4, 100, 7),
                                    (2, 64, 0), (3, 33, 0), (2, 1, 0),
                                    (4, 130, 32)])
def test_solve_system_matches_oracle(k, n, nb):
    seed = 4040 + n
    A = gen.planes(k, (n, n), 0, n, seed)
    b = gen.planes(k, (n,), 2, n, seed)
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, b)
    dm, bv, xv = DeviceMatrix.from_planes(A), DeviceVector.from_planes(b), \
        DeviceVector(k, n)
    piv = device_solve_system(dm, bv, xv, nb)
    assert np.asarray(piv.swaps()).tobytes() == sw_ref.tobytes()
    assert dm.download().tobytes() == lu_ref.tobytes()
    assert xv.download().tobytes() == x_ref.tobytes()


def test_dev_solve_system_augmented_buffer():
    k, n = 3, 200
    A = gen.planes(k, (n, n), 0, n, 99)
    b = gen.planes(k, (n,), 2, n, 99)
    aug = np.zeros((k, n, n + 3))          # ld = n + 3 > n + 1
    aug[:, :, :n] = A
    aug[:, :, n] = b
    d = torch.from_numpy(aug).cuda()
    x = torch.zeros((k, n), dtype=torch.float64, device="cuda")
    sw = np.zeros(n, dtype=np.int32)
    step = ctypes.c_int32()
    torch.cuda.synchronize()
    st = nat.lib().mpcore_dev_solve_system(
        k, n, d.data_ptr(), n + 3, n * (n + 3), 0, x.data_ptr(),
        sw.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(step))
    assert st == 0 and step.value == -1
    lu_ref, sw_ref = oracle.lu(A)
    assert sw.tobytes() == sw_ref.tobytes()
    out = d.cpu().numpy()
    assert np.ascontiguousarray(out[:, :, :n]).tobytes() == lu_ref.tobytes()
    assert x.cpu().numpy().tobytes() == \
        oracle.solve(lu_ref, sw_ref, b).tobytes()


def test_solve_system_singular():
    k, n = 2, 40
    A = gen.planes(k, (n, n), 0, n, 5)
    A[:, :, 7] = 0.0                      # column 7 dependent -> step 7
    b = gen.planes(k, (n,), 2, n, 5)
    with pytest.raises(oracle.Singular) as ei:
        oracle.lu(A)
    dm, bv, xv = DeviceMatrix.from_planes(A), DeviceVector.from_planes(b), \
        DeviceVector(k, n)
    with pytest.raises(SingularMatrixError) as ej:
        device_solve_system(dm, bv, xv)
    assert ej.value.step == ei.value.step
