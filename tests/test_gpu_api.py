"""The drop-in Python API on the GPU: reference test cases
(test_linalg.py:123-155, 262-299; test_refine.py) through
paper_2107_12550_b200's lu_factor_pp / lu_solve / mat_mul_blocked /
mat_vec / iterative_refinement, compared with the reference's golden
outputs."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
import paper_2107_12550_b200 as mp
from paper_2107_12550_b200 import refine as R
from paper_2107_12550_b200.longfloat import format_hex, parse_hex

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "longside.json")) as fh:
    G = json.load(fh)


@pytest.mark.parametrize("name", ["dd", "td", "qd"])
def test_pinned_api(name):
    dom = mp.McDomain(name)
    A = mp.DenseMatrix.from_rows(dom, [[2, 1], [1, 3]])
    b = mp.Vector.from_values(dom, [3, 4])
    piv = mp.lu_factor_pp(A)
    assert piv.swaps == [0, 1]
    x = mp.lu_solve(A, piv, b)
    assert [x.get(i).components[0] for i in range(2)] == [1.0, 1.0]
    A = mp.DenseMatrix.from_rows(dom, [[0, 1], [1, 0]])
    piv = mp.lu_factor_pp(A)
    assert piv.swaps == [1, 1]
    with pytest.raises(mp.SingularMatrixError) as e:
        mp.lu_factor_pp(mp.DenseMatrix.from_rows(dom, [[1, 2], [2, 4]]))
    assert e.value.step == 1
    with pytest.raises(mp.DimensionError):
        mp.lu_factor_pp(mp.DenseMatrix.zeros(dom, 2, 3))


@pytest.mark.parametrize("k", (2, 3, 4))
def test_api_matches_golden(k):
    g = golden("lu_k%d.npz" % k)
    dom = mp.McDomain({2: "dd", 3: "td", 4: "qd"}[k])
    n = 64
    A = mp.DenseMatrix(dom, n, n, g["n64_A"].copy())
    piv = mp.lu_factor_pp(A)
    assert piv.swaps == g["n64_swaps"].tolist()
    assert A.data.tobytes() == g["n64_lu"].tobytes()
    x = mp.lu_solve(A, piv, mp.Vector(dom, n, g["n64_b"].copy()))
    assert x.data.tobytes() == g["n64_x"].tobytes()
    gp = golden("prod_k%d.npz" % k)
    C = mp.mat_mul_blocked(mp.DenseMatrix(dom, 24, 20, gp["A"]),
                           mp.DenseMatrix(dom, 20, 28, gp["B"]), block=3)
    assert C.data.tobytes() == gp["C"].tobytes()


def test_paper_names():
    g = golden("lu_k3.npz")
    dom = mp.McDomain("td")
    af = mp.DenseMatrix(dom, 23, 23, g["n23_A"].copy())
    af_ch = []
    mp.TDLUdecompPM(af, af_ch)
    assert af_ch == g["n23_swaps"].tolist()
    xf = mp.Vector.zeros(dom, 23)
    mp.SolveTDLSPM(xf, af, mp.Vector(dom, 23, g["n23_b"].copy()), af_ch)
    assert xf.data.tobytes() == g["n23_x"].tobytes()


@pytest.mark.parametrize("idx", range(5))
def test_refinement_on_gpu_matches_reference(idx):
    case = G["refine"][idx]
    dom = mp.BfDomain(case["long_bits"])
    n = case["n"]
    A = mp.DenseMatrix.zeros(dom, n, n)
    A.data = [[parse_hex(e).round(dom.p) for e in row] for row in case["A"]]
    b = mp.Vector.zeros(dom, n)
    b.data = [parse_hex(e).round(dom.p) for e in case["b"]]
    cfg = R.RefineConfig(short_k=case["short_k"], long_bits=case["long_bits"],
                         rtol=case["rtol"], atol=0, max_iter=40)
    rep = R.iterative_refinement(A, b, cfg)
    assert rep.iterations == case["iterations"]
    assert rep.stop_reason == case["stop_reason"]
    assert [format_hex(h) for h in rep.residual_history] == case["history"]
    assert [format_hex(x) for x in rep.solution.data] == case["solution"]
