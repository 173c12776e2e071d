"""The reference's bigfloat surface (bigfloat.py:73-158, 404-466) as
exported by this package -- BigFloat, PrecisionContext, bf_parse_decimal,
bf_to_multicomp, bf_from_multicomp (__init__.py:62-78) -- against fixtures
made by the reference itself (tests/golden/make_golden_sqrt.py), and the
oracle's mc_sqrt restatement against the reference's mc_sqrt goldens."""

import json
import os

import numpy as np
import pytest

import oracle
import paper_2107_12550_b200 as mp
from paper_2107_12550_b200 import bigfloat as bfm

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "bigfloat_api.json")))


@pytest.mark.parametrize("row", CASES, ids=lambda r: "%s@%d" % (r["text"][:12], r["p"]))
def test_parse_peel_and_sum_match_reference(row):
    v = mp.bf_parse_decimal(row["text"], mp.PrecisionContext(row["p"]))
    assert isinstance(v, mp.BigFloat)
    assert bfm.bf_format_hex(v) == row["hex"]
    assert v.prec == row["prec"]
    for k in (2, 3, 4):
        m = mp.bf_to_multicomp(v, k)
        assert isinstance(m, mp.MultiComp)
        assert [float(c).hex() for c in m.components] == row["mc%d" % k]
        assert bfm.bf_format_hex(mp.bf_from_multicomp(m)) == row["back%d" % k]
        assert bfm.bf_format_hex(mp.bf_from_multicomp(
            m, mp.PrecisionContext(200))) == row["back%d_200" % k]


def test_bigfloat_constructor_and_operators():
    a = mp.BigFloat(1, 3, -1, 53)          # 1.5
    b = mp.BigFloat(-1, 1, -2, 106)        # -0.25
    assert (a.sign, a.man, a.exp, a.prec) == (1, 3, -1, 53)
    assert float(a) == 1.5 and float(b) == -0.25
    s = a + b
    assert float(s) == 1.25 and s.prec == 106     # max operand precision
    assert float(a * b) == -0.375 and float(a - b) == 1.75
    assert float(a / b) == -6.0
    assert a > b and b < a and a == mp.BigFloat(1, 6, -2, 20)
    assert hash(a) == hash(mp.BigFloat(1, 6, -2, 20))
    assert mp.BigFloat(0, 0, 0, 53).is_zero()
    assert repr(a).startswith("BigFloat(0x1.8p+0")


def test_errors_follow_reference():
    with pytest.raises(mp.ParseError):
        mp.bf_parse_decimal("1.2.3", mp.PrecisionContext(53))
    with pytest.raises(mp.DomainError):
        mp.PrecisionContext(1)
    with pytest.raises(mp.DivideByZeroError):
        bfm.bf_div(mp.BigFloat(1, 1, 0, 53), mp.BigFloat(0, 0, 0, 53),
                   mp.PrecisionContext(53))


@pytest.mark.parametrize("k", [2, 3, 4])
def test_oracle_sqrt_matches_reference(k):
    d = np.load(os.path.join(HERE, "golden", "sqrt.npz"))
    a, s = d["a_k%d" % k], d["sqrt_k%d" % k]
    assert oracle.elementwise("sqrt", a, a).tobytes() == s.tobytes()
