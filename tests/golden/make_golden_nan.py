"""Golden LU runs with NaN / Inf entries, made by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_nan.py

The reference's pivot is np.argmax over |head| (linalg.py:429): the first
NaN wins if any, else the first maximum; NaNs then propagate through its
EFT kernels.  Recorded: the inputs (seeded recipe + placed specials), the
swap list and the factors (NaN payloads are platform-specific, so the tests
compare NaN positions and every other bit).
"""

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(1, "/root/reference/pkg/src")

import mpcore  # noqa: E402
from mpcore.errors import SingularMatrixError  # noqa: E402
from mpcore.linalg import DenseMatrix, McDomain, lu_factor_pp  # noqa: E402

from oracle import gen  # noqa: E402

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/")

CASES = [
    # (k, n, [(row, col, head value)])
    (2, 8, [(3, 0, np.nan), (6, 2, np.inf)]),
    (3, 12, [(5, 4, np.nan), (9, 4, np.nan), (7, 4, np.inf)]),
    (4, 10, [(2, 2, np.nan)]),
    (2, 40, [(30, 10, -np.inf), (35, 20, np.nan)]),
    (3, 33, [(32, 31, np.nan), (0, 5, np.inf)]),
]


def main():
    warnings.simplefilter("ignore")
    out = {}
    for idx, (k, n, specials) in enumerate(CASES):
        A = gen.planes(k, (n, n), 0, n, 900 + idx)
        for r, c, v in specials:
            A[0, r, c] = v
            A[1:, r, c] = 0.0
        M = DenseMatrix(McDomain({2: "dd", 3: "td", 4: "qd"}[k]), n, n,
                        A.copy())
        try:
            sw = np.array(lu_factor_pp(M, simd=True).swaps, dtype=np.int32)
            step = -1
        except SingularMatrixError as e:
            sw = np.zeros(0, dtype=np.int32)
            step = e.step
        out["A%d" % idx] = A
        out["lu%d" % idx] = M.data
        out["sw%d" % idx] = sw
        out["step%d" % idx] = np.array([step])
        print("case", idx, "k=%d n=%d" % (k, n), "swaps", sw[:6], "step", step)
    np.savez(os.path.join(HERE, "lu_nan.npz"), **out)


if __name__ == "__main__":
    main()
