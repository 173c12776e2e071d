"""The oracle (test infrastructure) on the reference acceptance suite's 50
dual-path instances (test_acceptance.py:444-481), against digests made by
running the reference (tests/golden/make_golden_criterion8.py): LU, solve,
mat_vec and the batch kernels bit for bit."""

import hashlib
import json
import os

import numpy as np

import oracle
from paper_2107_12550_b200.linalg import DenseMatrix, McDomain, Vector

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "criterion8.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()
                          ).hexdigest()


def test_oracle_matches_reference_on_criterion8():
    rng = np.random.default_rng(88)
    sizes = [int(x) for x in rng.integers(2, 33, size=40)]
    sizes += [int(x) for x in rng.integers(33, 128, size=9)] + [128]
    for idx, (n, g) in enumerate(zip(sizes, GOLD)):
        dom = McDomain(g["tag"])
        rows = rng.uniform(-1.0, 1.0, size=(n, n))
        rhs = rng.uniform(-1.0, 1.0, size=n)
        A = DenseMatrix.from_rows(dom, rows.tolist()).data
        b = Vector.from_values(dom, rhs.tolist()).data
        lu, sw = oracle.lu(A)
        assert [int(s) for s in sw] == g["swaps"], idx
        assert sha(lu) == g["lu"], idx
        x = oracle.solve(lu, sw, b)
        assert sha(x) == g["x"], idx
        y = oracle.matvec(A, x)
        assert sha(y) == g["y"], idx
        w = oracle.elementwise("mul", x, y)
        assert sha(w) == g["w"], idx
        assert sha(oracle.elementwise("add", w, y)) == g["s"], idx
        assert sha(oracle.axpy(x[:, 0], w, y)) == g["axpy"], idx
