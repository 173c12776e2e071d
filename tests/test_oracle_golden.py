"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference implementation itself (tests/golden/make_golden.py), plus the
reference's own known-answer pins (test_mcfloat.py:66-81, test_linalg.py:
123-155, 262-275).  Everything compares bytes, not tolerances."""

import numpy as np
import pytest

import oracle
from oracle import gen
from conftest import golden

KS = (2, 3, 4)


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def test_eft_pins():
    s, e = oracle.two_sum(np.array([1.0, 2.0 ** 53, 0.0]),
                          np.array([2.0 ** -53, 1.0, 0.0]))
    assert list(s) == [1.0, 2.0 ** 53, 0.0]
    assert list(e) == [2.0 ** -53, 1.0, 0.0]
    v = 1.0 + 2.0 ** -27
    p, e = oracle.two_prod(np.array([v, 0.0]), np.array([v, 12.5]))
    assert list(p) == [1.0 + 2.0 ** -26, 0.0]
    assert list(e) == [2.0 ** -54, 0.0]


@pytest.mark.parametrize("k", KS)
def test_kernels_bitwise(k):
    g = golden("kernels_k%d.npz" % k)
    assert same(oracle.elementwise("add", g["a"], g["b"]), g["add"])
    assert same(oracle.elementwise("mul", g["a"], g["b"]), g["mul"])
    assert same(oracle.elementwise("div", g["div_a"], g["div_b"]), g["div"])


@pytest.mark.parametrize("k", KS)
def test_identities(k):
    g = golden("kernels_k%d.npz" % k)
    a = g["a"]
    z = np.zeros_like(a)
    one = np.zeros_like(a)
    one[0] = 1.0
    assert same(oracle.elementwise("add", a, z), a)   # test_mcfloat.py:207
    assert same(oracle.elementwise("mul", a, one), a)


@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("n", (23, 64))
def test_lu_solve_bitwise(k, n):
    g = golden("lu_k%d.npz" % k)
    A = g["n%d_A" % n]
    lu, swaps = oracle.lu(A)
    assert same(swaps, g["n%d_swaps" % n])
    assert same(lu, g["n%d_lu" % n])
    x = oracle.solve(lu, swaps, g["n%d_b" % n])
    assert same(x, g["n%d_x" % n])
    assert same(oracle.matvec(A, g["n%d_x_true" % n]), g["n%d_b" % n])


@pytest.mark.parametrize("k", KS)
def test_products_bitwise(k):
    g = golden("prod_k%d.npz" % k)
    assert same(oracle.gemm(g["A"], g["B"]), g["C"])
    assert same(oracle.matvec(g["A"], g["v"]), g["y"])
    assert same(oracle.axpy(g["alpha"], g["axpy_x"], g["axpy_y0"]),
                g["axpy_y"])


@pytest.mark.parametrize("k", KS)
def test_pinned_systems(k):
    g = golden("pinned.npz")
    for name in ("spd2", "perm2", "ffi2", "tie3"):
        lu, swaps = oracle.lu(g["%s_k%d_A" % (name, k)])
        assert same(swaps, g["%s_k%d_swaps" % (name, k)])
        assert same(lu, g["%s_k%d_lu" % (name, k)])
        x = oracle.solve(lu, swaps, g["%s_k%d_b" % (name, k)])
        assert same(x, g["%s_k%d_x" % (name, k)])
    assert list(g["tie3_k%d_swaps" % k])[0] == 1
    for name in ("sing1", "sing0"):
        with pytest.raises(oracle.Singular) as e:
            oracle.lu(g["%s_k%d_A" % (name, k)])
        assert e.value.step == int(g["%s_k%d_step" % (name, k)][0])


def test_config0_bitwise():
    g = golden("config0.npz")
    A = gen.planes(2, (128, 128), 0, 128, gen.config_seed(0))
    assert same(A, g["A"])
    ones = np.zeros((2, 128))
    ones[0] = 1.0
    assert same(oracle.matvec(A, ones), g["b"])
    lu, swaps = oracle.lu(A)
    assert same(swaps, g["swaps"])
    assert same(lu, g["lu"])
    assert same(oracle.solve(lu, swaps, g["b"]), g["x"])


def test_threading_does_not_change_bits():
    g = golden("lu_k3.npz")
    A = g["n64_A"]
    oracle.set_threads(1)
    lu1, s1 = oracle.lu(A)
    oracle.set_threads(max(2, oracle.num_threads()))
    lu2, s2 = oracle.lu(A)
    assert same(lu1, lu2) and same(s1, s2)
