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


# --------------------------------------------------------------- refine ----
from paper_2107_12550_b200.longfloat import (format_decimal, format_hex,
                                             parse_hex)


def write_bf(path, rows_hex, bits):
    with open(path, "w") as fh:
        fh.write("mpmat %d %d bf %d\n" % (len(rows_hex), len(rows_hex[0]), bits))
        for row in rows_hex:
            fh.write(" ".join(row) + "\n")


@pytest.mark.parametrize("exact_fro", [False, True])
@pytest.mark.parametrize("idx", range(5))
def test_native_refine_matches_reference(tmp_path, idx, exact_fro,
                                         monkeypatch):
    """mpcore_refine (ffi.py:243-258): native long arithmetic + GPU short
    solves (and the GPU long residual) reproduce the reference's IR run bit
    for bit -- with check_stop decided from the rigorous ||A||_F bounds
    where they suffice (default) and with the exact ||A||_F always formed
    (MPCORE_REFINE_EXACT_FRO)."""
    if exact_fro:
        monkeypatch.setenv("MPCORE_REFINE_EXACT_FRO", "1")
    case = G["refine"][idx]
    p = case["long_bits"]
    a_path, b_path = str(tmp_path / "A.mpmat"), str(tmp_path / "b.mpmat")
    write_bf(a_path, case["A"], p)
    write_bf(b_path, [[h] for h in case["b"]], p)
    st, rep = ffi.refine(a_path, b_path, case["short_k"], p, case["rtol"], "0",
                         40)
    assert st == ffi.OK, st
    assert ffi.report_iterations(rep) == (ffi.OK, case["iterations"])
    assert ffi.report_stop_reason(rep) == (ffi.OK, case["stop_reason"])
    st, count = ffi.report_residual_count(rep)
    assert count == len(case["history"])
    for i, h in enumerate(case["history"]):
        want = format_decimal(parse_hex(h).round(p), 60)
        assert ffi.report_residual_entry(rep, i, 60) == (ffi.OK, want)
    for i, h in enumerate(case["solution"]):
        v = parse_hex(h).round(p)
        assert ffi.report_solution_entry(rep, i, 40) == (ffi.OK,
                                                         format_decimal(v, 40))
        # default digits: ceil(prec*log10 2)+2 (bigfloat.py:489-490)
        assert ffi.report_solution_entry(rep, i, 0) == (ffi.OK,
                                                        format_decimal(v))
    assert ffi.report_residual_entry(rep, count, 20)[0] == ffi.BAD_DIMENSION
    ffi.release(rep)
    assert ffi.report_iterations(rep)[0] == ffi.BAD_HANDLE


def test_native_refine_errors(tmp_path):
    # test_ffi.py:204-215
    st, rep = ffi.refine(str(tmp_path / "nope.mpmat"),
                         str(tmp_path / "nope2.mpmat"), 2, 424, "1e-30", "0", 5)
    assert (st, rep) == (ffi.BAD_PARSE, 0)
    case = G["refine"][4]
    a_path, b_path = str(tmp_path / "A.mpmat"), str(tmp_path / "b.mpmat")
    write_bf(a_path, case["A"], case["long_bits"])
    write_bf(b_path, [[h] for h in case["b"]], case["long_bits"])
    assert ffi.refine(a_path, b_path, 7, 424, "1e-30", "0", 5) == (ffi.INTERNAL, 0)
    assert ffi.refine(a_path, b_path, 2, 424, "abc", "0", 5)[0] == ffi.BAD_PARSE
    assert ffi.refine(a_path, b_path, 2, 424, "0", "0", 5)[0] == ffi.INTERNAL
