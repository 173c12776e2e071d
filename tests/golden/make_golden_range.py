"""Golden vectors at the ends of the binary64 range, from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_range.py

The reference's two_prod is Dekker's splitting form (mcfloat.py:79-102).  It
equals the FMA form (p = a*b, e = fma(a, b, -p)) only while the split
cannot overflow (|a|, |b| < 2**996) and no partial product underflows;
outside that band the reference produces its own bits (NaN error terms for
huge operands, inexact tails near underflow), and a drop-in must produce the
same ones.  These fixtures hold operands and systems whose products land
there: heads near 2**+-1000, subnormals, zeros beside huge partners, and
LU / GEMM inputs scaled so their products underflow or their split
overflows.

Reference entry points (file:line in /root/reference/pkg/src/mpcore):
  kernel_add / kernel_mul        mcfloat.py:268-275
  _div_t                         mcfloat.py:304-318
  lu_factor_pp / lu_solve        linalg.py:452-469, 524-538 (lane paths)
  mat_mul_blocked                linalg.py:577-617
"""

import os
import random
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import mpcore  # noqa: E402  (the reference)
from mpcore import mcfloat  # noqa: E402
from mpcore.errors import SingularMatrixError  # noqa: E402
from mpcore.linalg import (DenseMatrix, McDomain, Vector,  # noqa: E402
                           lu_factor_pp, lu_solve, mat_mul_blocked)

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/"), \
    mpcore.__file__
warnings.simplefilter("ignore")
np.seterr(all="ignore")


def operand(rng, k, e):
    """A k-component value with head ~2**e (lower parts 2**-53 apart),
    renormalised by the reference; subnormal tails flush as it does."""
    terms = [rng.uniform(-1, 1) * 2.0 ** (e - 53 * i - rng.randint(0, 3))
             if e - 53 * i > -1080 else 0.0 for i in range(k + 1)]
    return list(mcfloat.renormalize(terms, k))


def exps(rng):
    r = rng.random()
    if r < 0.3:
        return rng.randint(-1074, -900)     # products underflow
    if r < 0.6:
        return rng.randint(960, 1023)       # split overflows from 2**996
    if r < 0.8:
        return rng.randint(-480, -440)      # pairs land near 2**-960
    return rng.randint(-40, 40)


def pairs(k, seed, count):
    rng = random.Random(seed)
    a, b = [], []
    for _ in range(count):
        ea, eb = exps(rng), exps(rng)
        r = rng.random()
        if r < 0.05:
            x, y = [0.0] * k, operand(rng, k, rng.randint(990, 1023))
        elif r < 0.10:
            x, y = operand(rng, k, rng.randint(990, 1023)), [0.0] * k
        elif r < 0.15:      # a huge operand with a product in range
            x, y = operand(rng, k, rng.randint(997, 1010)), \
                operand(rng, k, rng.randint(-200, -100))
        else:
            x, y = operand(rng, k, ea), operand(rng, k, eb)
        a.append(x)
        b.append(y)
    return (np.array(a, dtype=np.float64).T.copy(),
            np.array(b, dtype=np.float64).T.copy())


def kernels(k, seed):
    a, b = pairs(k, seed, 2000)
    add = np.stack([np.asarray(x, dtype=np.float64)
                    for x in mcfloat.kernel_add(k)(*a, *b)])
    mul = np.stack([np.asarray(x, dtype=np.float64)
                    for x in mcfloat.kernel_mul(k)(*a, *b)])
    nd = 400
    da, db = a[:, :nd].copy(), b[:, :nd].copy()
    for i in range(nd):
        if db[0, i] == 0.0:
            db[:, i] = 0.0
            db[0, i] = 3.0
    div = np.zeros((k, nd))
    for i in range(nd):
        div[:, i] = mcfloat._div_t(tuple(da[:, i]), tuple(db[:, i]), k)
    return dict(a=a, b=b, add=add, mul=mul, div_a=da, div_b=db, div=div)


def scaled_planes(k, shape, scale_exp, seed):
    rng = random.Random(seed)
    vals = [operand(rng, k, scale_exp + rng.randint(-3, 0))
            for _ in range(int(np.prod(shape)))]
    return np.array(vals, dtype=np.float64).T.reshape((k,) + shape).copy()


def system(k, n, scale_exp, seed):
    dom = McDomain({2: "dd", 3: "td", 4: "qd"}[k])
    A = scaled_planes(k, (n, n), scale_exp, seed)
    b = scaled_planes(k, (n,), scale_exp, seed + 1)
    lu = DenseMatrix(dom, n, n, A.copy())
    try:
        piv = lu_factor_pp(lu, simd=True)
    except SingularMatrixError as e:
        return dict(A=A, b=b, lu=lu.data.copy(), step=np.int32(e.step))
    x = lu_solve(lu, piv, Vector(dom, n, b.copy()), simd=True)
    return dict(A=A, b=b, lu=lu.data.copy(), step=np.int32(-1),
                swaps=np.array(piv.swaps, dtype=np.int32), x=x.data.copy())


def gemm(k, m, kk, nn, ea, eb, seed):
    dom = McDomain({2: "dd", 3: "td", 4: "qd"}[k])
    A = scaled_planes(k, (m, kk), ea, seed)
    B = scaled_planes(k, (kk, nn), eb, seed + 1)
    C = mat_mul_blocked(DenseMatrix(dom, m, kk, A.copy()),
                        DenseMatrix(dom, kk, nn, B.copy()), simd=True)
    return dict(A=A, B=B, C=C.data.copy())


def main():
    for k in (2, 3, 4):
        out = {}
        for key, v in kernels(k, 9100 + k).items():
            out["kern_" + key] = v
        # LU + solve: products near underflow (entries ~2**-485: l*u
        # ~2**-970) and split overflow (entries up to 2**998)
        for tag, se in (("tiny", -485), ("huge", 998)):
            for key, v in system(k, 40, se, 9200 + k).items():
                out["lu_%s_%s" % (tag, key)] = v
        for key, v in gemm(k, 20, 24, 18, -500, -470, 9300 + k).items():
            out["gemm_" + key] = v
        np.savez_compressed(os.path.join(HERE, "range_k%d.npz" % k), **out)
        print("range_k%d.npz" % k, {a: b.shape for a, b in out.items()})


if __name__ == "__main__":
    main()
