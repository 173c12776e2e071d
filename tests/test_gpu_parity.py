"""Parity of the sm_100a path (through the C ABI) with the reference:
bitwise against the reference's own golden vectors, and bitwise against the
CPU oracle (pinned to the reference) at sizes the golden files don't cover.
"""

import numpy as np
import pytest

import oracle
from oracle import gen
from conftest import golden
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          PivotHandle, device_solve)

pytestmark = pytest.mark.gpu
KS = (2, 3, 4)


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def dev_elementwise(op, x, y):
    k, n = x.shape
    hx, hy = DeviceVector.from_planes(x), DeviceVector.from_planes(y)
    ho = DeviceVector(k, n)
    nat.check(nat.lib().mpcore_elementwise(op, hx.handle, hy.handle,
                                           ho.handle), "elementwise")
    return ho.download()


def dev_lu(A, nb=0):
    dm = DeviceMatrix.from_planes(A)
    piv = dm.lu_factor(nb)
    return dm, piv


def dev_solve(dm, piv, b):
    bv = DeviceVector.from_planes(b)
    xv = DeviceVector(b.shape[0], b.shape[1])
    device_solve(dm, piv, bv, xv)
    return xv.download()


def dev_matvec(A, x):
    dm, xv = DeviceMatrix.from_planes(A), DeviceVector.from_planes(x)
    yv = DeviceVector(A.shape[0], A.shape[1])
    nat.check(nat.lib().mpcore_mat_vec(dm.handle, xv.handle, yv.handle),
              "mat_vec")
    return yv.download()


def dev_gemm(A, B):
    da, db = DeviceMatrix.from_planes(A), DeviceMatrix.from_planes(B)
    dc = DeviceMatrix(A.shape[0], A.shape[1], B.shape[2])
    nat.check(nat.lib().mpcore_mat_mul(da.handle, db.handle, dc.handle),
              "mat_mul")
    return dc.download()


@pytest.mark.parametrize("k", KS)
def test_kernels_vs_reference_golden(k):
    g = golden("kernels_k%d.npz" % k)
    assert same(dev_elementwise(0, g["a"], g["b"]), g["add"])
    assert same(dev_elementwise(1, g["a"], g["b"]), g["mul"])
    assert same(dev_elementwise(2, g["div_a"], g["div_b"]), g["div"])


@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("n", (23, 64))
def test_lu_solve_vs_reference_golden(k, n):
    g = golden("lu_k%d.npz" % k)
    for nb in (0, 8, 16):
        dm, piv = dev_lu(g["n%d_A" % n], nb)
        assert same(piv.swaps(), g["n%d_swaps" % n])
        assert same(dm.download(), g["n%d_lu" % n])
        assert same(dev_solve(dm, piv, g["n%d_b" % n]), g["n%d_x" % n])
    assert same(dev_matvec(g["n%d_A" % n], g["n%d_x_true" % n]),
                g["n%d_b" % n])


@pytest.mark.parametrize("k", KS)
def test_products_vs_reference_golden(k):
    g = golden("prod_k%d.npz" % k)
    assert same(dev_gemm(g["A"], g["B"]), g["C"])
    assert same(dev_matvec(g["A"], g["v"]), g["y"])
    x, y = DeviceVector.from_planes(g["axpy_x"]), \
        DeviceVector.from_planes(g["axpy_y0"])
    al = np.ascontiguousarray(g["alpha"])
    nat.check(nat.lib().mpcore_axpy(nat.dptr(al), k, x.handle, y.handle),
              "axpy")
    assert same(y.download(), g["axpy_y"])


@pytest.mark.parametrize("k", KS)
def test_pinned_systems(k):
    g = golden("pinned.npz")
    for name in ("spd2", "perm2", "ffi2", "tie3"):
        dm, piv = dev_lu(g["%s_k%d_A" % (name, k)])
        assert same(piv.swaps(), g["%s_k%d_swaps" % (name, k)])
        assert same(dm.download(), g["%s_k%d_lu" % (name, k)])
        assert same(dev_solve(dm, piv, g["%s_k%d_b" % (name, k)]),
                    g["%s_k%d_x" % (name, k)])
    from paper_2107_12550_b200.errors import SingularMatrixError
    for name in ("sing1", "sing0"):
        with pytest.raises(SingularMatrixError) as e:
            dev_lu(g["%s_k%d_A" % (name, k)])
        assert e.value.step == int(g["%s_k%d_step" % (name, k)][0])


def test_config0_vs_reference_golden():
    g = golden("config0.npz")
    n = 128
    dA = DeviceMatrix(2, n, n)
    dA.generate(0, n, gen.config_seed(0))
    assert same(dA.download(), g["A"])          # device generator == recipe
    ones = np.zeros((2, n))
    ones[0] = 1.0
    assert same(dev_matvec(g["A"], ones), g["b"])
    dm, piv = dev_lu(g["A"])
    assert same(piv.swaps(), g["swaps"])
    assert same(dm.download(), g["lu"])
    assert same(dev_solve(dm, piv, g["b"]), g["x"])


@pytest.mark.parametrize("k", KS)
def test_generator_matches_oracle_recipe(k):
    n = 97
    dA = DeviceMatrix(k, n, n)
    dA.generate(0, n, 12345)
    assert same(dA.download(), gen.planes(k, (n, n), 0, n, 12345))
    dx = DeviceVector(k, n)
    dx.generate(2, n, 12345)
    assert same(dx.download(), gen.planes(k, (n,), 2, n, 12345))


@pytest.mark.parametrize("k,n", [(2, 300), (3, 257), (4, 200), (2, 513),
                                 (3, 100), (4, 33)])
def test_lu_solve_vs_oracle(k, n):
    seed = 777 + n
    A = gen.planes(k, (n, n), 0, n, seed)
    x_true = gen.planes(k, (n,), 2, n, seed)
    b = oracle.matvec(A, x_true)
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, b)
    for nb in (0, 16, 7):
        dm, piv = dev_lu(A, nb)
        assert same(piv.swaps(), sw_ref)
        assert same(dm.download(), lu_ref)
        assert same(dev_solve(dm, piv, b), x_ref)


@pytest.mark.parametrize("k,m,kk,nn", [(2, 130, 70, 90), (3, 65, 129, 33),
                                       (4, 40, 50, 61), (2, 256, 256, 256)])
def test_gemm_vs_oracle(k, m, kk, nn):
    A = gen.planes(k, (m, kk), 0, 512, 99)
    B = gen.planes(k, (kk, nn), 1, 512, 99)
    assert same(dev_gemm(A, B), oracle.gemm(A, B))


def test_abi_2x2_known_answer():
    # test_ffi.py:108-125 / 233-261: [[4,3],[6,3]] x = [10,12] -> (1, 2)
    from paper_2107_12550_b200 import ffi
    st, h = ffi.matrix_new(2, 2, 2)
    assert st == 0
    for (i, j), t in {(0, 0): "4", (0, 1): "3", (1, 0): "6",
                      (1, 1): "3"}.items():
        assert ffi.set_element_from_decimal(h, i, j, t) == 0
    st, b = ffi.vector_new(2, 2)
    ffi.set_element_from_decimal(b, 0, 0, "10")
    ffi.set_element_from_decimal(b, 1, 0, "12")
    st, x = ffi.vector_new(2, 2)
    st, piv = ffi.lu_factor(h)
    assert st == 0
    assert ffi.lu_solve_handles(h, piv, b, x) == 0
    assert ffi.get_element_components(x, 0, 0) == (0, (1.0, 0.0))
    assert ffi.get_element_components(x, 1, 0) == (0, (2.0, 0.0))
    for hh in (h, b, piv, x):
        assert ffi.release(hh) == 0
    assert ffi.release(x) == 1
