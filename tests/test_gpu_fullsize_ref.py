"""Parity at the benchmark sizes pinned to the REFERENCE itself (not only
to the oracle restatement): tests/golden/make_golden_fullsize.py ran the
reference's lane path on the exact bench inputs -- lu_factor_pp + lu_solve
(linalg.py:422-538) for TD n = 512 / 1024 / 2048, DD n = 1024 and QD
n = 2048 (the BASELINE config-2 workloads), and mat_mul_blocked
(linalg.py:577-617) for the BASELINE config-1 GEMMs at n = 2048 (a 96-row
band of C: each row of the lane path depends only on its row of A).  The
fixtures hold SHA-256 digests of the exact float64 planes (inputs too,
which pins the device generator), the swaps and the solution as hex.
Checked here: the product path (device generator, mat_vec, LU, solve; the
two-call API and the bench's one-call [A | b] path; the GEMM) bit for
bit."""

import glob
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          device_solve, device_solve_system)

pytestmark = pytest.mark.gpu
GOLD = [json.load(open(p)) for p in sorted(glob.glob(os.path.join(
    os.path.dirname(__file__), "golden", "fullsize_*.json")))]
LU = [g for g in GOLD if g["kind"] == "lu"]
GEMM = [g for g in GOLD if g["kind"] == "gemm"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()
                          ).hexdigest()


def x_hex(x):
    return [[float(v).hex() for v in row] for row in x]


@pytest.mark.parametrize("g", LU, ids=lambda g: "k%d_n%d" % (g["k"], g["n"]))
def test_lu_solve_matches_reference(g):
    k, n, seed = g["k"], g["n"], g["seed"]
    A = DeviceMatrix(k, n, n)
    A.generate(0, n, seed)
    xt = DeviceVector(k, n)
    xt.generate(2, n, seed)
    b = DeviceVector(k, n)
    nat.check(nat.lib().mpcore_mat_vec(A.handle, xt.handle, b.handle), "mv")
    A_h = A.download()
    assert sha(A_h) == g["sha_A"]
    assert sha(b.download()) == g["sha_b"]
    # two-call API: lu_factor + lu_solve
    piv = A.lu_factor()
    x = DeviceVector(k, n)
    device_solve(A, piv, b, x)
    assert [int(s) for s in piv.swaps()] == g["swaps"]
    assert sha(A.download()) == g["sha_lu"]
    assert x_hex(x.download()) == g["x_hex"]
    # the bench's one-call path ([A | b] factored together)
    A1 = DeviceMatrix.from_planes(A_h)
    x1 = DeviceVector(k, n)
    piv1 = device_solve_system(A1, b, x1)
    assert [int(s) for s in piv1.swaps()] == g["swaps"]
    assert sha(A1.download()) == g["sha_lu"]
    assert x_hex(x1.download()) == g["x_hex"]


@pytest.mark.parametrize("g", GEMM, ids=lambda g: "k%d_n%d" % (g["k"], g["n"]))
def test_gemm_matches_reference(g):
    k, n, seed = g["k"], g["n"], g["seed"]
    A = DeviceMatrix(k, n, n)
    A.generate(0, n, seed)
    B = DeviceMatrix(k, n, n)
    B.generate(1, n, seed)
    assert sha(A.download()) == g["sha_A"]
    assert sha(B.download()) == g["sha_B"]
    C = DeviceMatrix(k, n, n)
    nat.check(nat.lib().mpcore_mat_mul(A.handle, B.handle, C.handle), "mm")
    band = np.ascontiguousarray(C.download()[:, g["rows"], :])
    assert [[float(v).hex() for v in band[c, 0, :16]] for c in range(k)] == \
        g["C_row0_hex"]
    assert sha(band) == g["sha_C_rows"]
