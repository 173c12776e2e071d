"""BASELINE config 3 at its full size, pinned to the REFERENCE itself:
the reference's iterative_refinement (refine.py:121-197) was run on the
n = 1024, kappa = 1e30, 512-bit system written by mpcore_write_config3
(tests/golden/make_golden_fullsize.py config3_1024; ~4 min of reference
CPU time).  The native driver must reproduce the iteration count, the stop
reason, the residual history (40 digits) and the solution (60 digits,
SHA-256 of the text) exactly -- with the ||A||_F-bounds shortcut and with
the exact norm, with the one-call factor_solve (asynchronous, overlapping
the host conversion, or not) and with factor() then solve() -- both in
memory and through the .mpmat files.  (MPCORE_RESIDUAL_VARIANT is read once
per process, so the warp-per-row residual variant is pinned by
tests/test_gpu_long_residual.py instead.)"""

import ctypes
import hashlib
import json
import os

import pytest

from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200 import ffi

pytestmark = pytest.mark.gpu
G = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                "fullsize_config3_1024.json")))


def report(h):
    hist = [ffi.report_residual_entry(h, i, 40)[1]
            for i in range(ffi.report_residual_count(h)[1])]
    sol = [ffi.report_solution_entry(h, i, 60)[1]
           for i in range(ffi.report_solution_count(h)[1])]
    return (ffi.report_iterations(h)[1], ffi.report_stop_reason(h)[1], hist,
            sol)


def check(rep):
    it, stop, hist, sol = rep
    assert it == G["iterations"]
    assert stop == G["stop_reason"]
    assert hist == G["history"]
    assert sol[:8] == G["solution_head"]
    assert hashlib.sha256("\n".join(sol).encode()).hexdigest() == \
        G["solution_sha"]


@pytest.mark.parametrize("mode", ["bounds", "exact_fro", "split_factor",
                                  "no_overlap", "host_convert"])
def test_config3_n1024_matches_reference(mode, monkeypatch):
    # bounds: the production path (asynchronous factorisation overlapping
    # the fixed-width conversion, products-off-the-chain residual)
    if mode == "exact_fro":
        monkeypatch.setenv("MPCORE_REFINE_EXACT_FRO", "1")
    if mode == "split_factor":
        monkeypatch.setenv("MPCORE_REFINE_SPLIT_FACTOR", "1")
    if mode == "no_overlap":
        monkeypatch.setenv("MPCORE_REFINE_NO_OVERLAP", "1")
    if mode == "host_convert":   # (default: the conversion on the GPU)
        monkeypatch.setenv("MPCORE_REFINE_HOST_CONVERT", "1")
    h = ctypes.c_uint64()
    assert nat.lib().mpcore_refine_config3(
        G["n"], G["seed"], G["kappa_exp10"], 3, 512, b"1e-100", b"0", 20, 0,
        ctypes.byref(h)) == 0
    try:
        check(report(h.value))
    finally:
        nat.lib().mpcore_release(h.value)


def test_config3_n1024_files_match_reference(tmp_path):
    pa, pb = str(tmp_path / "A.mpmat"), str(tmp_path / "b.mpmat")
    assert nat.lib().mpcore_write_config3(G["n"], G["seed"], G["kappa_exp10"],
                                          512, 0, pa.encode(), pb.encode()) == 0
    # the generator writes exactly the files the reference was run on
    assert hashlib.sha256(open(pa, "rb").read()).hexdigest() == G["sha_A"]
    assert hashlib.sha256(open(pb, "rb").read()).hexdigest() == G["sha_b"]
    st, h = ffi.refine(pa, pb, 3, 512, "1e-100", "0", 20)
    assert st == 0
    try:
        check(report(h))
    finally:
        ffi.release(h)
