"""BASELINE config 3 system (csrc/testsys.cpp), host only: the generator is
deterministic, independent of the thread count and pinned by the files the
reference's own driver ran on (tests/golden/make_golden_config3.py); A has
the prescribed singular values; b = A*ones in the reference's mat_vec
order at 512 bits."""

import hashlib
import json
import os

import mpmath
import pytest

from paper_2107_12550_b200 import _native as nat

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "config3_ir.json")))


def write(tmp_path, n, kappa=30.0, threads=0, seed=210712553, tag=""):
    pa, pb = tmp_path / ("A%s.mpmat" % tag), tmp_path / ("b%s.mpmat" % tag)
    st = nat.lib().mpcore_write_config3(n, seed, kappa, 512, threads,
                                        str(pa).encode(), str(pb).encode())
    assert st == 0
    return pa, pb


def sha(p):
    return hashlib.sha256(p.read_bytes()).hexdigest()


def parse_hex(tok):
    neg = tok.startswith("-")
    t = tok.lstrip("-")
    assert t.startswith("0x")
    mant, e = t[2:].split("p")
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    man = int(ip + fp, 16) if (ip + fp) else 0
    exp = int(e) - 4 * len(fp)
    v = mpmath.mpf((man, exp)) if man else mpmath.mpf(0)
    return -v if neg else v


def load(p):
    lines = p.read_text().split("\n")
    hdr = lines[0].split()
    rows, cols = int(hdr[1]), int(hdr[2])
    return [[parse_hex(t) for t in lines[1 + i].split()] for i in range(rows)]


@pytest.mark.parametrize("g", GOLD, ids=lambda g: "n%d" % g["n"])
def test_generator_pinned_to_reference_run(tmp_path, g):
    pa, pb = write(tmp_path, g["n"], g["kappa_exp10"], seed=g["seed"])
    assert sha(pa) == g["sha_A"] and sha(pb) == g["sha_b"]


def test_thread_count_invariant(tmp_path):
    a1, b1 = write(tmp_path, 37, threads=1, tag="1")
    a4, b4 = write(tmp_path, 37, threads=4, tag="4")
    assert sha(a1) == sha(a4) and sha(b1) == sha(b4)


def test_singular_values_and_rhs(tmp_path):
    n = 16
    pa, pb = write(tmp_path, n)
    with mpmath.workprec(700):
        A = mpmath.matrix(load(pa))
        b = [r[0] for r in load(pb)]
        # b = A * ones, rounded to 512 bits after every addition, row-major
        with mpmath.workprec(512):
            for i in range(n):
                acc = mpmath.mpf(0)
                for j in range(n):
                    acc = acc + A[i, j]
                assert acc == b[i]
        s = sorted(mpmath.svd_r(A, compute_uv=False), reverse=True)
        for kk, sv in enumerate(s):
            want = mpmath.mpf(10) ** (-mpmath.mpf(30) * kk / (n - 1))
            assert abs(sv / want - 1) < mpmath.mpf(10) ** -100
