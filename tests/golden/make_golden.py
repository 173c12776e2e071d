"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only,
never copied) and records inputs + outputs of the hot-path functions as
small .npz fixtures next to this script.  The GPU box never needs the
reference: the tests compare the oracle and the CUDA path against these
files.

Reference entry points exercised (file:line in /root/reference/pkg/src/mpcore):
  kernel_add / kernel_mul        mcfloat.py:268-275   (_add2.._mul4, 189-257)
  _div_t                          mcfloat.py:304-318
  lu_factor_pp (lane path)        linalg.py:452-469   (_lu_lanes 422-449)
  lu_solve (lane path)            linalg.py:524-538   (_solve_lanes 496-521)
  mat_vec                         linalg.py:545-574
  mat_mul_blocked                 linalg.py:577-617
  axpy_batch                      linalg.py:624-645
"""

import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import mpcore  # noqa: E402  (the reference)
from mpcore import mcfloat  # noqa: E402
from mpcore.linalg import (  # noqa: E402
    DenseMatrix, McDomain, Vector, axpy_batch, lu_factor_pp, lu_solve,
    mat_mul_blocked, mat_vec)
from mpcore.errors import SingularMatrixError  # noqa: E402

from oracle import gen  # noqa: E402  (input recipe only; no oracle arithmetic)

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/"), \
    mpcore.__file__


def ref_renorm(raw):
    """add_k(raw, 0) with the reference kernel (mcfloat.py:268-270)."""
    k = raw.shape[0]
    flat = raw.reshape(k, -1)
    z = np.zeros_like(flat[0])
    out = mcfloat.kernel_add(k)(*[flat[c] for c in range(k)], *([z] * k))
    return np.stack([np.asarray(o, dtype=np.float64) for o in out]).reshape(
        raw.shape)


def ref_planes(k, shape, slot, n, seed):
    count = int(np.prod(shape))
    raw = gen.raw_planes(k, count, slot, n, seed)
    return ref_renorm(raw).reshape((k,) + tuple(shape))


def rand_operands(rng, k, count):
    """Canonical k-component operands with varied magnitudes, signs,
    exact zeros and cancellation-prone pairs."""
    heads = []
    for _ in range(count):
        r = rng.random()
        if r < 0.04:
            heads.append([0.0] * k)
            continue
        e = rng.randint(-30, 30)
        terms = [rng.uniform(-1, 1) * 2.0 ** (e - 53 * i - rng.randint(0, 3))
                 for i in range(k + 1)]
        heads.append(list(mcfloat.renormalize(terms, k)))
    return np.array(heads, dtype=np.float64).T.copy()


def kernels(k, seed):
    rng = random.Random(seed)
    n = 3000
    a = rand_operands(rng, k, n)
    b = rand_operands(rng, k, n)
    # cancellation pairs: b = -a perturbed in the tail
    for i in range(0, n, 17):
        b[:, i] = -a[:, i]
        b[k - 1, i] = b[k - 1, i] * 0.5
    add = mcfloat.kernel_add(k)(*a, *b)
    mul = mcfloat.kernel_mul(k)(*a, *b)
    add = np.stack([np.asarray(x, dtype=np.float64) for x in add])
    mul = np.stack([np.asarray(x, dtype=np.float64) for x in mul])
    # division: scalar reference on nonzero divisors
    nd = 600
    div = np.zeros((k, nd))
    bd = b[:, :nd].copy()
    for i in range(nd):
        if bd[0, i] == 0.0:
            bd[:, i] = 0.0
            bd[0, i] = 3.0
        div[:, i] = mcfloat._div_t(tuple(a[:, i]), tuple(bd[:, i]), k)
    return dict(a=a, b=b, add=add, mul=mul, div_a=a[:, :nd].copy(),
                div_b=bd, div=div)


def system(k, n, seed, config_slot_x=2):
    dom = McDomain({2: "dd", 3: "td", 4: "qd"}[k])
    A = ref_planes(k, (n, n), 0, n, seed)
    x = ref_planes(k, (n,), config_slot_x, n, seed)
    Am = DenseMatrix(dom, n, n, A.copy())
    xv = Vector(dom, n, x.copy())
    b = mat_vec(Am, xv, simd=True).data.copy()
    lu = Am.copy()
    piv = lu_factor_pp(lu, simd=True)
    sol = lu_solve(lu, piv, Vector(dom, n, b.copy()), simd=True)
    return dict(A=A, x_true=x, b=b, lu=lu.data.copy(),
                swaps=np.array(piv.swaps, dtype=np.int32),
                x=sol.data.copy())


def products(k, m, kk, nn, seed):
    dom = McDomain({2: "dd", 3: "td", 4: "qd"}[k])
    A = ref_planes(k, (m, kk), 0, 4096, seed)
    B = ref_planes(k, (kk, nn), 1, 4096, seed)
    C = mat_mul_blocked(DenseMatrix(dom, m, kk, A.copy()),
                        DenseMatrix(dom, kk, nn, B.copy()), simd=True)
    v = ref_planes(k, (kk,), 2, 4096, seed)
    y = mat_vec(DenseMatrix(dom, m, kk, A.copy()), Vector(dom, kk, v.copy()),
                simd=True)
    alpha = tuple(ref_planes(k, (1,), 3, 4096, seed)[:, 0])
    yy = Vector(dom, kk, ref_planes(k, (kk,), 1, 4096, seed + 1)[:, :].copy())
    y0 = yy.data.copy()
    axpy_batch(mcfloat.MultiComp(alpha, validate=False), Vector(dom, kk, v),
               yy, simd=True)
    return dict(A=A, B=B, C=C.data.copy(), v=v, y=y.data.copy(),
                alpha=np.array(alpha), axpy_x=v, axpy_y0=y0,
                axpy_y=yy.data.copy())


def pinned():
    """Small known-answer systems from the reference's own tests."""
    out = {}
    cases = {
        # test_linalg.py:123-142 / test_ffi.py:108-125
        "spd2": ([[2, 1], [1, 3]], [3, 4]),
        "perm2": ([[0, 1], [1, 0]], [5, 7]),
        "ffi2": ([[4, 3], [6, 3]], [10, 12]),
        # test_linalg.py:262-275 (head tie -> first row)
        "tie3": ([[0.5, 2.0, 1.0], [1.0, 0.25, -3.0], [-1.0, 1.0, 0.125]],
                 [1, 2, 3]),
    }
    for k in (2, 3, 4):
        dom = McDomain({2: "dd", 3: "td", 4: "qd"}[k])
        for name, (rows, rhs) in cases.items():
            A = DenseMatrix.from_rows(dom, rows)
            a0 = A.data.copy()
            piv = lu_factor_pp(A)
            x = lu_solve(A, piv, Vector.from_values(dom, rhs))
            out["%s_k%d_A" % (name, k)] = a0
            out["%s_k%d_b" % (name, k)] = Vector.from_values(dom, rhs).data
            out["%s_k%d_lu" % (name, k)] = A.data.copy()
            out["%s_k%d_swaps" % (name, k)] = np.array(piv.swaps, np.int32)
            out["%s_k%d_x" % (name, k)] = x.data.copy()
        # singular steps (test_linalg.py:145-155)
        for name, rows in (("sing1", [[1, 2], [2, 4]]),
                           ("sing0", [[0, 1], [0, 2]])):
            A = DenseMatrix.from_rows(dom, rows)
            out["%s_k%d_A" % (name, k)] = A.data.copy()
            try:
                lu_factor_pp(A)
                step = -1
            except SingularMatrixError as e:
                step = e.step
            out["%s_k%d_step" % (name, k)] = np.array([step], np.int32)
    return out


def main():
    for k in (2, 3, 4):
        np.savez_compressed(os.path.join(HERE, "kernels_k%d.npz" % k),
                            **kernels(k, 7000 + k))
        print("kernels k", k)
        sysd = {}
        for n, seed in ((23, 11), (64, 12)):
            for key, val in system(k, n, seed).items():
                sysd["n%d_%s" % (n, key)] = val
        np.savez_compressed(os.path.join(HERE, "lu_k%d.npz" % k), **sysd)
        print("lu k", k)
        np.savez_compressed(os.path.join(HERE, "prod_k%d.npz" % k),
                            **products(k, 24, 20, 28, 9000 + k))
        print("prod k", k)
    np.savez_compressed(os.path.join(HERE, "pinned.npz"), **pinned())
    # config 0: DD LU + solve, n = 128, seed 210712550 (x_true = ones)
    n, k = 128, 2
    dom = McDomain("dd")
    seed = gen.config_seed(0)
    A = ref_planes(k, (n, n), 0, n, seed)
    ones = np.zeros((k, n))
    ones[0] = 1.0
    b = mat_vec(DenseMatrix(dom, n, n, A.copy()), Vector(dom, n, ones.copy()),
                simd=True).data.copy()
    lu = DenseMatrix(dom, n, n, A.copy())
    piv = lu_factor_pp(lu, simd=True)
    x = lu_solve(lu, piv, Vector(dom, n, b.copy()), simd=True)
    np.savez_compressed(os.path.join(HERE, "config0.npz"), A=A, b=b,
                        lu=lu.data, swaps=np.array(piv.swaps, np.int32),
                        x=x.data)
    print("config0")


if __name__ == "__main__":
    main()
