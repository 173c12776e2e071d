"""Operands at the ends of the binary64 range.

The reference's two_prod is Dekker's splitting form (mcfloat.py:79-102); the
CUDA path forms the same pair as p = a*b, e = fma(a, b, -p).  The two are
bit-identical inside the band DESIGN §2 states -- the split cannot overflow
(|a|, |b| < 2**996), both operands normal and |p| >= 2**-959, or an operand
is +-0 beside a partner below 2**996 -- and differ outside it (Dekker's NaN
error terms for huge operands; its tails near underflow).  Goldens from the
reference itself (tests/golden/make_golden_range.py): add / mul / div on
2000 / 400 pairs per k with heads near 2**+-1000, subnormals and zeros beside
huge partners; LU + solve of matrices with entries near 2**-485 and up to
2**998; a GEMM whose heads multiply near 2**-970 (and its TD / QD tails
far below).

  * the oracle (Dekker, like the reference) reproduces every golden;
  * the oracle built with the FMA form differs from the reference only on
    elements with a pair outside the band;
  * the GPU reproduces the FMA-form oracle everywhere, and therefore the
    reference on every in-band element.
NaN payloads are platform-specific: NaN positions and every other bit are
compared."""

import numpy as np
import pytest

import oracle
from conftest import golden

KS = (2, 3, 4)


def same_nan_aware(a, b):
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    if a.shape != b.shape or not np.array_equal(na, nb):
        return False
    return a[~na].tobytes() == b[~nb].tobytes()


def differs(a, b):
    """Per element (column of planar (k, n)): any component differs."""
    a, b = np.asarray(a), np.asarray(b)
    eq = (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))
    return ~eq.all(axis=0)


def _field(x):
    return (np.asarray(x, dtype=np.float64).view(np.uint64) >> 52) & 0x7ff


def pair_in_band(a, b):
    """Dekker's e == the FMA form's e for every pair (elementwise)."""
    with np.errstate(all="ignore"):
        p = a * b
    ea, eb, ep = _field(a), _field(b), _field(p)
    za, zb = (a == 0.0), (b == 0.0)
    normal = (ea >= 1) & (ea <= 2018) & (eb >= 1) & (eb <= 2018) & \
        (ep >= 64) & (ep <= 2046)
    return normal | (za & (eb <= 2018)) | (zb & (ea <= 2018))


def mul_in_band(a, b):
    """Every two_prod of kernel_mul(k) (mcfloat.py:198-257) in the band."""
    k = a.shape[0]
    pairs = [(0, 0)] if k == 2 else \
        [(0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0)]
    ok = np.ones(a.shape[1], dtype=bool)
    for i, j in pairs:
        ok &= pair_in_band(a[i], b[j])
    return ok


@pytest.mark.parametrize("k", KS)
def test_oracle_range_edges_match_reference(k):
    g = golden("range_k%d.npz" % k)
    assert same_nan_aware(oracle.elementwise("add", g["kern_a"], g["kern_b"]),
                          g["kern_add"])
    assert same_nan_aware(oracle.elementwise("mul", g["kern_a"], g["kern_b"]),
                          g["kern_mul"])
    assert same_nan_aware(oracle.elementwise("div", g["kern_div_a"],
                                             g["kern_div_b"]), g["kern_div"])
    for tag in ("tiny", "huge"):
        assert int(g["lu_%s_step" % tag]) < 0
        lu, sw = oracle.lu(g["lu_%s_A" % tag])
        assert sw.tobytes() == g["lu_%s_swaps" % tag].tobytes()
        assert same_nan_aware(lu, g["lu_%s_lu" % tag])
        x = oracle.solve(lu, sw, g["lu_%s_b" % tag])
        assert same_nan_aware(x, g["lu_%s_x" % tag])
    assert same_nan_aware(oracle.gemm(g["gemm_A"], g["gemm_B"]), g["gemm_C"])


@pytest.mark.parametrize("k", KS)
def test_fma_form_differs_only_outside_band(k):
    g = golden("range_k%d.npz" % k)
    a, b = g["kern_a"], g["kern_b"]
    with oracle.fma_two_prod():
        add = oracle.elementwise("add", a, b)
        mul = oracle.elementwise("mul", a, b)
        lu_t, sw_t = oracle.lu(g["lu_tiny_A"])
    assert same_nan_aware(add, g["kern_add"])      # no two_prod in add
    d = differs(mul, g["kern_mul"])
    inb = mul_in_band(a, b)
    assert not (d & inb).any()                      # in band: identical
    assert d.sum() > 100                            # the goldens do leave it
    # products near 2**-970 with normal operands stay exact both ways
    assert sw_t.tobytes() == g["lu_tiny_swaps"].tobytes()
    assert same_nan_aware(lu_t, g["lu_tiny_lu"])


@pytest.mark.gpu
@pytest.mark.parametrize("k", KS)
def test_gpu_range_edges(k):
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                              device_solve)
    g = golden("range_k%d.npz" % k)
    if nat.LIB_PATH.endswith("libmpcore_exact.so"):
        _exact_checks()    # this process runs the exact-range build
        return

    def ew(op, x, y):
        hx, hy = DeviceVector.from_planes(x), DeviceVector.from_planes(y)
        ho = DeviceVector(x.shape[0], x.shape[1])
        nat.check(nat.lib().mpcore_elementwise(op, hx.handle, hy.handle,
                                               ho.handle), "elementwise")
        return ho.download()

    a, b = g["kern_a"], g["kern_b"]
    add, mul = ew(0, a, b), ew(1, a, b)
    div = ew(2, g["kern_div_a"], g["kern_div_b"])
    with oracle.fma_two_prod():
        assert same_nan_aware(mul, oracle.elementwise("mul", a, b))
        assert same_nan_aware(div, oracle.elementwise(
            "div", g["kern_div_a"], g["kern_div_b"]))
    # the reference's own bits: every add, every in-band product
    assert same_nan_aware(add, g["kern_add"])
    inb = mul_in_band(a, b)
    assert same_nan_aware(mul[:, inb], g["kern_mul"][:, inb])
    for tag in ("tiny", "huge"):
        A, rhs = g["lu_%s_A" % tag], g["lu_%s_b" % tag]
        with oracle.fma_two_prod():
            lu_f, sw_f = oracle.lu(A)
            x_f = oracle.solve(lu_f, sw_f, rhs)
        for nb in (0, 8):
            dm = DeviceMatrix.from_planes(A)
            piv = dm.lu_factor(nb)
            sw = np.asarray(piv.swaps(), dtype=np.int32)
            assert sw.tobytes() == sw_f.tobytes()
            assert same_nan_aware(dm.download(), lu_f)
            bv = DeviceVector.from_planes(rhs)
            xv = DeviceVector(k, rhs.shape[1])
            device_solve(dm, piv, bv, xv)
            assert same_nan_aware(xv.download(), x_f)
            if tag == "tiny":   # in band: the reference's bits
                assert sw.tobytes() == g["lu_tiny_swaps"].tobytes()
                assert same_nan_aware(xv.download(), g["lu_tiny_x"])
    da = DeviceMatrix.from_planes(g["gemm_A"])
    db = DeviceMatrix.from_planes(g["gemm_B"])
    dc = DeviceMatrix(k, g["gemm_A"].shape[1], g["gemm_B"].shape[2])
    nat.check(nat.lib().mpcore_mat_mul(da.handle, db.handle, dc.handle),
              "mat_mul")
    # (its TD / QD tails multiply below 2**-1000: outside the band)
    with oracle.fma_two_prod():
        assert same_nan_aware(dc.download(),
                              oracle.gemm(g["gemm_A"], g["gemm_B"]))


def _exact_checks():
    """Run in a process with MPCORE_EXACT_RANGE=1: the exact-range build
    against the reference's goldens, every element."""
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                              device_solve)
    assert nat.LIB_PATH.endswith("libmpcore_exact.so"), nat.LIB_PATH
    for k in KS:
        g = golden("range_k%d.npz" % k)

        def ew(op, x, y):
            hx, hy = DeviceVector.from_planes(x), DeviceVector.from_planes(y)
            ho = DeviceVector(x.shape[0], x.shape[1])
            nat.check(nat.lib().mpcore_elementwise(op, hx.handle, hy.handle,
                                                   ho.handle), "elementwise")
            return ho.download()

        assert same_nan_aware(ew(0, g["kern_a"], g["kern_b"]), g["kern_add"])
        assert same_nan_aware(ew(1, g["kern_a"], g["kern_b"]), g["kern_mul"])
        assert same_nan_aware(ew(2, g["kern_div_a"], g["kern_div_b"]),
                              g["kern_div"])
        for tag in ("tiny", "huge"):
            for nb in (0, 8):
                dm = DeviceMatrix.from_planes(g["lu_%s_A" % tag])
                piv = dm.lu_factor(nb)
                assert np.asarray(piv.swaps(), dtype=np.int32).tobytes() == \
                    g["lu_%s_swaps" % tag].tobytes()
                assert same_nan_aware(dm.download(), g["lu_%s_lu" % tag])
                rhs = g["lu_%s_b" % tag]
                bv = DeviceVector.from_planes(rhs)
                xv = DeviceVector(k, rhs.shape[1])
                device_solve(dm, piv, bv, xv)
                assert same_nan_aware(xv.download(), g["lu_%s_x" % tag])
        da = DeviceMatrix.from_planes(g["gemm_A"])
        db = DeviceMatrix.from_planes(g["gemm_B"])
        dc = DeviceMatrix(k, g["gemm_A"].shape[1], g["gemm_B"].shape[2])
        nat.check(nat.lib().mpcore_mat_mul(da.handle, db.handle, dc.handle),
                  "mat_mul")
        assert same_nan_aware(dc.download(), g["gemm_C"])
    print("exact-range build: all range goldens bit-identical")


@pytest.mark.gpu
def test_gpu_exact_range_build_matches_reference_everywhere():
    """MPCORE_EXACT_RANGE=1 loads libmpcore_exact.so, whose two_prod takes
    the reference's Dekker sequence outside the band: then every golden --
    huge operands' NaNs included -- is reproduced bit for bit."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, MPCORE_EXACT_RANGE="1")
    code = ("import sys; sys.path[:0] = [%r, %r]; import test_range_edges "
            "as t; t._exact_checks()" % (here, os.path.dirname(here)))
    r = subprocess.run([sys.executable, "-c", code], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bit-identical" in r.stdout
