"""Division digits on the GPU take RN(a/b) from a reciprocal hint
(mc.cuh ddiv_y: RN(a y) and two remainder corrections) instead of the
division routine.  These cases are built so the head quotient a0/b0 lies a
few units of the last place of a - m b from a rounding midpoint m — the only
inputs where a correction could round the wrong way — plus divisors at both
ends of the binade and operands outside the hinted exponent range.  Every
result is compared bit for bit with the oracle's div (host IEEE division,
mcfloat.py:304-318)."""
import random

import numpy as np
import pytest

import oracle
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceVector

pytestmark = pytest.mark.gpu


def _mk(mant, e):
    """the double mant * 2^e for a 53-bit integer mantissa"""
    return float(np.ldexp(float(mant), e))


def near_midpoint_pairs(count, seed):
    """(a0, b0) with a0 - m b0 = t * 2^-s for a quotient midpoint m and a
    small integer t: M * B = A * 2^s + t, M odd (54 bits), A, B 53 bits."""
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        M = rng.getrandbits(54) | (1 << 53) | 1
        t = rng.choice((-5, -3, -2, -1, 1, 2, 3, 5))
        for s in (54, 53):
            mod = 1 << s
            B = (t * pow(M, -1, mod)) % mod
            if not (1 << 52) <= B < (1 << 53):
                continue
            P = M * B - t
            if P % mod:
                continue
            A = P >> s
            if (1 << 52) <= A < (1 << 53):
                ea, eb = rng.randint(-60, 60), rng.randint(-60, 60)
                sa = -1.0 if rng.random() < 0.5 else 1.0
                out.append((sa * _mk(A, ea), _mk(B, eb)))
                break
    return out


def special_pairs(seed):
    rng = random.Random(seed)
    out = []
    for _ in range(2000):
        # divisors at the ends of the binade, near sqrt(2)
        b = rng.choice((2.0 - rng.randint(1, 1 << 20) * 2.0 ** -52,
                        1.0 + rng.randint(0, 1 << 12) * 2.0 ** -52,
                        float.fromhex("0x1.6a09e667f3bcdp+0")
                        + rng.randint(-4096, 4096) * 2.0 ** -52))
        a = rng.uniform(-2, 2)
        out.append((a * 2.0 ** rng.randint(-40, 40), b * 2.0 ** rng.randint(-40, 40)))
    # around and outside the hinted exponent range (|e| <= 423) and zeros;
    # products stay normal (two_prod's FMA form equals Dekker's there only)
    for e in (-700, -424, -423, -422, 0, 422, 423, 424, 700):
        for f in (-1.5, 1.0, 1.25, 1.9999999999999998):
            out.append((f * 2.0 ** e, 3.0))
            out.append((1.7, f * 2.0 ** e))
            if abs(e) <= 424:
                out.append((f * 2.0 ** e, 1.3 * 2.0 ** -e))
    out += [(0.0, 3.0), (-0.0, 3.0), (0.0, -3.0)]
    return out


def run_pairs(k, pairs, seed):
    n = len(pairs)
    rng = np.random.default_rng(seed)
    raw_a = np.zeros((k, n))
    raw_b = np.zeros((k, n))
    raw_a[0] = [p[0] for p in pairs]
    raw_b[0] = [p[1] for p in pairs]
    for c in range(1, k):
        raw_a[c] = raw_a[c - 1] * 2.0 ** -53 * rng.uniform(-1, 1, n)
        raw_b[c] = raw_b[c - 1] * 2.0 ** -53 * rng.uniform(-1, 1, n)
    a = oracle.renormalize_planes(raw_a)
    b = oracle.renormalize_planes(raw_b)
    keep = b[0] != 0
    a, b = np.ascontiguousarray(a[:, keep]), np.ascontiguousarray(b[:, keep])
    want = oracle.elementwise("div", a, b)
    hx, hy = DeviceVector.from_planes(a), DeviceVector.from_planes(b)
    ho = DeviceVector(k, a.shape[1])
    nat.check(nat.lib().mpcore_elementwise(2, hx.handle, hy.handle, ho.handle),
              "elementwise")
    got = ho.download()
    # NaN payloads differ between host and device: NaN-aware, else bitwise
    nan_g, nan_w = np.isnan(got), np.isnan(want)
    diff = (got.view(np.int64) != want.view(np.int64)) & ~(nan_g & nan_w)
    bad = np.nonzero((diff | (nan_g != nan_w)).any(axis=0))[0]
    assert bad.size == 0, ("k=%d: %d mismatches, first a=%r b=%r"
                           % (k, bad.size, a[:, bad[0]], b[:, bad[0]]))


@pytest.mark.parametrize("k", (2, 3, 4))
def test_div_near_midpoints(k):
    run_pairs(k, near_midpoint_pairs(20000, 17 + k), k)


@pytest.mark.parametrize("k", (2, 3, 4))
def test_div_binade_ends_and_ranges(k):
    run_pairs(k, special_pairs(29 + k), 100 + k)
