"""BASELINE config 3 on the GPU: the native refinement driver on the
generated kappa = 1e30 systems reproduces the reference's own IR runs
(tests/golden/config3_ir.json, made by running the reference's
iterative_refinement on the same files) -- iterations, stop reason,
residual history (40 digits) and solution (60 digits) -- both in memory
(mpcore_refine_config3) and through the .mpmat files (mpcore_refine)."""

import ctypes
import json
import os

import pytest

from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200 import ffi
from paper_2107_12550_b200.refine import refine_config3

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "config3_ir.json")))


def report_text(h):
    hist = [ffi.report_residual_entry(h, i, 40)[1]
            for i in range(ffi.report_residual_count(h)[1])]
    sol = [ffi.report_solution_entry(h, i, 60)[1]
           for i in range(ffi.report_solution_count(h)[1])]
    return (ffi.report_iterations(h)[1], ffi.report_stop_reason(h)[1], hist,
            sol)


def check(g, rep):
    it, stop, hist, sol = rep
    assert it == g["iterations"]
    assert stop == g["stop_reason"]
    assert hist == g["history"]
    assert sol == g["solution"]


@pytest.mark.parametrize("g", GOLD, ids=lambda g: "n%d" % g["n"])
def test_config3_in_memory_matches_reference(g):
    L = nat.lib()
    h = ctypes.c_uint64()
    assert L.mpcore_refine_config3(g["n"], g["seed"], g["kappa_exp10"], 3,
                                   512, b"1e-100", b"0", 20, 0,
                                   ctypes.byref(h)) == 0
    try:
        check(g, report_text(h.value))
    finally:
        L.mpcore_release(h.value)


@pytest.mark.parametrize("g", GOLD[:1], ids=lambda g: "n%d" % g["n"])
def test_config3_files_match_reference(tmp_path, g):
    L = nat.lib()
    pa, pb = str(tmp_path / "A.mpmat"), str(tmp_path / "b.mpmat")
    assert L.mpcore_write_config3(g["n"], g["seed"], g["kappa_exp10"], 512, 0,
                                  pa.encode(), pb.encode()) == 0
    st, h = ffi.refine(pa, pb, 3, 512, "1e-100", "0", 20)
    assert st == 0
    try:
        check(g, report_text(h))
    finally:
        ffi.release(h)


def test_config3_full_size_converges():
    r = refine_config3(n=1024)
    assert r["stop_reason"] == "converged"
    assert 1 <= r["iterations"] <= 20
    # |x - 1| is bounded by kappa * (relative residual); well below 1e-60
    assert float(r["max_abs_err_vs_ones"]) < 1e-60
