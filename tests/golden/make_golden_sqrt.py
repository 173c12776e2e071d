"""Golden vectors for mc_sqrt (mcfloat.py:324-340 _sqrt_t, 596-601 mc_sqrt)
made by the REFERENCE:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_sqrt.py

Per k: 1500 canonical nonnegative operands (exact zeros, exponents over
2^-300 .. 2^300, values near perfect squares and near powers of two) and
the reference's results, plus the Python bigfloat surface fixtures used by
tests/test_bigfloat_api.py (bf_parse_decimal / bf_to_multicomp /
bf_from_multicomp round trips).
"""
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import mpcore  # noqa: E402
from mpcore import mcfloat  # noqa: E402
from mpcore.bigfloat import (PrecisionContext, bf_format_hex,  # noqa: E402
                             bf_from_multicomp, bf_parse_decimal,
                             bf_to_multicomp)

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/")


def operands(rng, k, count):
    out = []
    for i in range(count):
        r = rng.random()
        if r < 0.03:
            out.append([0.0] * k)
            continue
        if r < 0.1:   # near a perfect square / a power of two
            base = float(rng.randint(1, 1 << 20)) ** 2 if r < 0.07 else 1.0
            e = rng.randint(-40, 40)
            terms = [base * 2.0 ** (2 * e)] + [
                rng.uniform(-1, 1) * 2.0 ** (2 * e - 53 * (j + 1))
                for j in range(k)]
        else:
            e = rng.randint(-300, 300)
            terms = [rng.uniform(0, 1) * 2.0 ** e] + [
                rng.uniform(-1, 1) * 2.0 ** (e - 53 * j - rng.randint(0, 3))
                for j in range(1, k + 1)]
        v = list(mcfloat.renormalize(terms, k))
        if v[0] < 0:
            v = [-c for c in v]
        out.append(v)
    return np.array(out, dtype=np.float64).T.copy()


def main():
    res = {}
    for k in (2, 3, 4):
        rng = random.Random(8100 + k)
        a = operands(rng, k, 1500)
        s = np.zeros_like(a)
        for i in range(a.shape[1]):
            s[:, i] = mcfloat.mc_sqrt(mcfloat.MultiComp(
                tuple(a[:, i]), validate=False)).components
        res["a_k%d" % k] = a
        res["sqrt_k%d" % k] = s
    np.savez_compressed(os.path.join(HERE, "sqrt.npz"), **res)
    # bigfloat surface round trips
    texts = ["1", "-0.1", "3.14159265358979323846264338327950288419716939937510",
             "1e-300", "-2.5e+280", "0", "123456789012345678901234567890.5",
             "0.3333333333333333333333333333333333333333333333333333333333"]
    cases = []
    for t in texts:
        for p in (53, 106, 200, 512):
            v = bf_parse_decimal(t, PrecisionContext(p))
            row = dict(text=t, p=p, hex=bf_format_hex(v), prec=v.prec)
            for k in (2, 3, 4):
                m = bf_to_multicomp(v, k)
                row["mc%d" % k] = [float(c).hex() for c in m.components]
                back = bf_from_multicomp(m, None)
                row["back%d" % k] = bf_format_hex(back)
                row["back%d_200" % k] = bf_format_hex(
                    bf_from_multicomp(m, PrecisionContext(200)))
            cases.append(row)
    with open(os.path.join(HERE, "bigfloat_api.json"), "w") as fh:
        json.dump(cases, fh, indent=0)
    print("sqrt + bigfloat api goldens written")


if __name__ == "__main__":
    main()
