"""The reference acceptance suite's dual-path criterion (test_acceptance.py:
444-481: 50 random instances, n in 2..128, DD/TD/QD cycling) run through
the REFERENCE lane path, recorded as SHA-256 digests of every result so the
GPU path joins as a third path (tests/test_gpu_criterion8.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_criterion8.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import mpcore  # noqa: E402
from mpcore.linalg import (DenseMatrix, McDomain, Vector, axpy_batch,  # noqa: E402
                           elementwise_add_batch, elementwise_mul_batch,
                           lu_factor_pp, lu_solve, mat_vec)

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/")
TAGS = ["dd", "td", "qd"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()
                          ).hexdigest()


def main():
    rng = np.random.default_rng(88)
    sizes = [int(x) for x in rng.integers(2, 33, size=40)]
    sizes += [int(x) for x in rng.integers(33, 128, size=9)] + [128]
    out = []
    for idx, n in enumerate(sizes):
        dom = McDomain(TAGS[idx % 3])
        rows = rng.uniform(-1.0, 1.0, size=(n, n))
        rhs = rng.uniform(-1.0, 1.0, size=n)
        A = DenseMatrix.from_rows(dom, rows.tolist())
        b = Vector.from_values(dom, rhs.tolist())
        lu = A.copy()
        piv = lu_factor_pp(lu, simd=True)
        x = lu_solve(lu, piv, b, simd=True)
        y = mat_vec(A, x, simd=True)
        w = elementwise_mul_batch(x, y, simd=True)
        s = elementwise_add_batch(w, y, simd=True)
        alpha = x.get(0)
        ax = axpy_batch(alpha, w, y.copy(), simd=True)
        out.append(dict(n=n, tag=TAGS[idx % 3], sha_rows=sha(rows),
                        sha_rhs=sha(rhs), swaps=list(piv.swaps),
                        lu=sha(lu.data), x=sha(x.data), y=sha(y.data),
                        w=sha(w.data), s=sha(s.data), axpy=sha(ax.data)))
    with open(os.path.join(HERE, "criterion8.json"), "w") as fh:
        json.dump(out, fh)
    print("criterion 8: %d instances" % len(out))


if __name__ == "__main__":
    main()
