"""Host long-precision side against golden vectors made by the reference
(tests/golden/make_golden_ir.py): decimal/hex parsing into k components,
decimal formatting, check_stop pins (test_refine.py:38-58) and full
iterative-refinement runs.  The IR runs here use a checker-backed short
solver (the CPU oracle) in place of the GPU so the host loop is exercised
without a device; tests/test_gpu_refine.py runs the same cases on the GPU.
"""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN
from paper_2107_12550_b200 import refine as R
from paper_2107_12550_b200.linalg import DenseMatrix, Vector
from paper_2107_12550_b200.longfloat import (BfDomain, LF, format_decimal,
                                             format_hex, parse_decimal,
                                             parse_hex)
from paper_2107_12550_b200.errors import DomainError

with open(os.path.join(GOLDEN, "longside.json")) as fh:
    G = json.load(fh)


def test_parse_matches_reference():
    for case in G["parse"]:
        k, t = case["k"], case["text"]
        s = t.strip()
        if s.lstrip("+-").lower().startswith("0x"):
            v = parse_hex(s)
        else:
            v = parse_decimal(s, 53 * k + 64)
        comps = v.to_components(k)
        assert [c.hex() for c in comps] == case["comps"], (k, t)


def test_format_matches_reference():
    for case in G["format"]:
        v = parse_decimal(case["text"], case["prec"])
        assert format_hex(v) == case["hex"]
        assert format_decimal(v, case["digits"]) == case["out"], case


def bf(text, bits=212):
    return parse_decimal(text, bits)


def test_check_stop_pins():
    # test_refine.py:38-58
    args = dict(x_norm=bf("1"), a_fro=bf("10"), n=4, rtol=bf("1e-2"),
                atol=bf("0"))
    assert R.check_stop(bf("0.19"), **args) is True
    assert R.check_stop(bf("0.21"), **args) is False
    assert R.check_stop(bf("0"), **args) is True
    one, zero = bf("1"), bf("0")
    assert R.check_stop(bf("0.5"), one, one, 9, zero, one) is True
    assert R.check_stop(zero, zero, one, 4, bf("1e-2"), zero) is False
    with pytest.raises(DomainError):
        R.check_stop(zero, one, one, 0, one, zero)


def test_config_validation():
    with pytest.raises(DomainError):
        R.RefineConfig(short_k=5)
    with pytest.raises(DomainError):
        R.RefineConfig(short_k=2, long_bits=106)
    with pytest.raises(DomainError):
        R.RefineConfig(max_iter=0)


class OracleShort:
    """Checker-backed stand-in for DeviceShortSolver (CPU tests only)."""

    def __init__(self, k, a_planes, nb=0):
        self.lu, self.swaps = oracle.lu(a_planes)

    def solve(self, b_planes):
        return oracle.solve(self.lu, self.swaps, b_planes)


def load_system(case):
    dom = BfDomain(case["long_bits"])
    n = case["n"]
    A = DenseMatrix.zeros(dom, n, n)
    A.data = [[parse_hex(e).round(dom.p) for e in row] for row in case["A"]]
    b = Vector.zeros(dom, n)
    b.data = [parse_hex(e).round(dom.p) for e in case["b"]]
    return A, b


@pytest.mark.parametrize("idx", range(5))
def test_refinement_matches_reference(monkeypatch, idx):
    case = G["refine"][idx]
    monkeypatch.setattr(R, "make_short_solver", OracleShort)
    A, b = load_system(case)
    cfg = R.RefineConfig(short_k=case["short_k"], long_bits=case["long_bits"],
                         rtol=case["rtol"], atol=0, max_iter=40)
    rep = R.iterative_refinement(A, b, cfg)
    assert rep.iterations == case["iterations"]
    assert rep.stop_reason == case["stop_reason"]
    assert [format_hex(h) for h in rep.residual_history] == case["history"]
    assert [format_hex(x) for x in rep.solution.data] == case["solution"]


@pytest.mark.parametrize("prec", [53, 64, 65, 106, 300, 424, 512, 576, 640])
def test_fixed_width_long_arithmetic_matches_generic(prec):
    # the refinement loop's fixed-width add/sub/mul (fastfloat.h) against
    # the generic big-integer path (bigfloat.py single-rounding semantics)
    import ctypes
    from paper_2107_12550_b200 import _native as nat
    m = ctypes.c_int64()
    assert nat.lib().mpcore_debug_longfloat_selftest(
        40000, 1234 + prec, prec, ctypes.byref(m)) == 0
    assert m.value == 0
