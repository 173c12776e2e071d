"""The reference acceptance suite's dual-path criterion (test_acceptance.py:
444-481) with the GPU as the third path: the same 50 random instances
(np.random.default_rng(88); n in 2..128; DD/TD/QD in turn) through this
package's drop-in API -- lu_factor_pp, lu_solve, mat_vec,
elementwise_mul_batch / _add_batch, axpy_batch -- must equal the
reference's lane path bit for bit (digests made by running the reference,
tests/golden/make_golden_criterion8.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2107_12550_b200.linalg import (DenseMatrix, McDomain, Vector,
                                          axpy_batch, elementwise_add_batch,
                                          elementwise_mul_batch, lu_factor_pp,
                                          lu_solve, mat_vec)

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "criterion8.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()
                          ).hexdigest()


def test_fifty_instances_bitwise_vs_reference():
    rng = np.random.default_rng(88)
    sizes = [int(x) for x in rng.integers(2, 33, size=40)]
    sizes += [int(x) for x in rng.integers(33, 128, size=9)] + [128]
    assert sizes == [g["n"] for g in GOLD]
    for idx, (n, g) in enumerate(zip(sizes, GOLD)):
        dom = McDomain(g["tag"])
        rows = rng.uniform(-1.0, 1.0, size=(n, n))
        rhs = rng.uniform(-1.0, 1.0, size=n)
        assert sha(rows) == g["sha_rows"] and sha(rhs) == g["sha_rhs"]
        A = DenseMatrix.from_rows(dom, rows.tolist())
        b = Vector.from_values(dom, rhs.tolist())
        lu = A.copy()
        piv = lu_factor_pp(lu)
        assert piv.swaps == g["swaps"], idx
        assert sha(lu.data) == g["lu"], idx
        x = lu_solve(lu, piv, b)
        assert sha(x.data) == g["x"], idx
        y = mat_vec(A, x)
        assert sha(y.data) == g["y"], idx
        w = elementwise_mul_batch(x, y)
        assert sha(w.data) == g["w"], idx
        assert sha(elementwise_add_batch(w, y).data) == g["s"], idx
        ax = axpy_batch(x.get(0), w, y.copy())
        assert sha(ax.data) == g["axpy"], idx
