"""The reference's handle-surface tests (test_ffi.py) re-run against the
native library: same statuses, same values, handles never reused."""

import json
import os

import pytest

from conftest import GOLDEN
from paper_2107_12550_b200 import ffi

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "longside.json")) as fh:
    G = json.load(fh)


def new_matrix(k, rows, cols):
    st, h = ffi.matrix_new(k, rows, cols)
    assert st == ffi.OK
    return h


def new_vector(k, n):
    st, h = ffi.vector_new(k, n)
    assert st == ffi.OK
    return h


def fill(h, entries):
    for key, text in entries.items():
        i, j = key if isinstance(key, tuple) else (key, 0)
        assert ffi.set_element_from_decimal(h, i, j, text) == ffi.OK


def test_release_lifecycle():
    h = new_matrix(2, 1, 1)
    assert ffi.release(h) == ffi.OK
    assert ffi.release(h) == ffi.BAD_HANDLE
    assert ffi.set_element_from_decimal(h, 0, 0, "1") == ffi.BAD_HANDLE
    assert ffi.get_element_components(h, 0, 0)[0] == ffi.BAD_HANDLE


def test_handles_never_reused():
    a = new_vector(2, 1)
    ffi.release(a)
    b = new_vector(2, 1)
    assert b != a
    ffi.release(b)


def test_new_rejects_bad_shape_or_k():
    assert ffi.matrix_new(5, 2, 2)[0] == ffi.BAD_DIMENSION
    assert ffi.matrix_new(2, 0, 2)[0] == ffi.BAD_DIMENSION
    assert ffi.vector_new(1, 3)[0] == ffi.BAD_DIMENSION
    assert ffi.vector_new(3, 0)[0] == ffi.BAD_DIMENSION


def test_element_text_matches_reference():
    # decimal at 53k+64 bits then k heads; hex exact (ffi.py:167-186)
    for case in G["parse"]:
        k = case["k"]
        h = new_vector(k, 1)
        assert ffi.set_element_from_decimal(h, 0, 0, case["text"]) == ffi.OK
        st, comps = ffi.get_element_components(h, 0, 0)
        assert st == ffi.OK
        assert [c.hex() for c in comps] == case["comps"], case
        ffi.release(h)


def test_element_errors():
    h = new_matrix(2, 2, 2)
    assert ffi.set_element_from_decimal(h, 2, 0, "1") == ffi.BAD_DIMENSION
    assert ffi.set_element_from_decimal(h, 0, 0, "zz") == ffi.BAD_PARSE
    assert ffi.set_element_from_decimal(h, 0, 0, "1e400") == ffi.OVERFLOW
    assert ffi.get_element_components(h, 0, 5)[0] == ffi.BAD_DIMENSION
    v = new_vector(2, 2)
    assert ffi.set_element_from_decimal(v, 0, 1, "1") == ffi.BAD_DIMENSION
    ffi.release(h)
    ffi.release(v)


def test_wrong_kind_is_invalid_handle():
    h = new_matrix(2, 2, 2)
    fill(h, {(0, 0): "4", (0, 1): "3", (1, 0): "6", (1, 1): "3"})
    st, piv = ffi.lu_factor(h)
    assert st == ffi.OK
    assert ffi.set_element_from_decimal(piv, 0, 0, "1") == ffi.BAD_HANDLE
    assert ffi.lu_factor(piv)[0] == ffi.BAD_HANDLE
    assert ffi.report_iterations(h)[0] == ffi.BAD_HANDLE
    ffi.release(h)
    ffi.release(piv)


def test_singular_factor_status():
    h = new_matrix(4, 2, 2)
    fill(h, {(0, 0): "1", (0, 1): "2", (1, 0): "2", (1, 1): "4"})
    st, piv = ffi.lu_factor(h)
    assert st == ffi.SINGULAR and piv == 0
    ffi.release(h)


def test_solve_shape_and_k_mismatches():
    h = new_matrix(2, 2, 2)
    fill(h, {(0, 0): "2", (0, 1): "0", (1, 0): "0", (1, 1): "2"})
    st, piv = ffi.lu_factor(h)
    b3 = new_vector(2, 3)
    x2 = new_vector(2, 2)
    assert ffi.lu_solve_handles(h, piv, b3, x2) == ffi.BAD_DIMENSION
    btd = new_vector(3, 2)
    assert ffi.lu_solve_handles(h, piv, btd, x2) == ffi.BAD_DIMENSION
    assert ffi.lu_solve_handles(h, piv, 999999, x2) == ffi.BAD_HANDLE
    for hh in (h, piv, b3, x2, btd):
        ffi.release(hh)


def test_rectangular_factor_is_dimension_error():
    h = new_matrix(3, 2, 3)
    assert ffi.lu_factor(h)[0] == ffi.BAD_DIMENSION
    ffi.release(h)
