"""Golden vectors for the long-precision side, made by the REFERENCE itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ir.py

Records (as JSON, exact hex text via bf_format_hex):
  * iterative_refinement runs (refine.py:121-197) on small generated
    systems (testgen.build_system, the paper's R*D*R^-1 family) for
    short_k = 2, 3, 4: iterations, stop reason, residual history, solution;
  * decimal/hex element parsing (ffi.py:167-186 -> bf_to_multicomp);
  * bf_format_decimal outputs (bigfloat.py:483-509);
  * check_stop pins (refine.py:104-118).
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import mpcore  # noqa: E402
from mpcore.bigfloat import (PrecisionContext, bf_format_decimal,  # noqa
                             bf_format_hex, bf_parse_decimal, bf_parse_hex,
                             bf_to_multicomp)
from mpcore.linalg import BfDomain, convert_matrix, convert_vector  # noqa
from mpcore.refine import RefineConfig, iterative_refinement  # noqa
from mpcore.testgen import ProblemSpec, build_system  # noqa

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/")


def hexv(v):
    return bf_format_hex(v)


def main():
    out = {"refine": [], "parse": [], "format": []}
    for n, seed, k, long_bits, rtol in ((12, 1, 2, 424, "1e-100"),
                                        (12, 1, 3, 424, "1e-100"),
                                        (12, 1, 4, 424, "1e-100"),
                                        (20, 3, 3, 512, "1e-100"),
                                        (8, 5, 2, 300, "1e-60")):
        sysd = build_system(ProblemSpec(n=n, seed=seed))
        dom = BfDomain(long_bits)
        A = convert_matrix(sysd.A, dom)
        b = convert_vector(sysd.b, dom)
        cfg = RefineConfig(short_k=k, long_bits=long_bits, rtol=rtol,
                           atol=0, max_iter=40)
        rep = iterative_refinement(A, b, cfg)
        out["refine"].append(dict(
            n=n, seed=seed, short_k=k, long_bits=long_bits, rtol=rtol,
            A=[[hexv(e) for e in row] for row in A.data],
            b=[hexv(e) for e in b.data],
            iterations=rep.iterations, stop_reason=rep.stop_reason,
            history=[hexv(h) for h in rep.residual_history],
            solution=[hexv(e) for e in rep.solution.data]))
        print("refine", n, k, rep.iterations, rep.stop_reason)
    texts = ["0.1", "1", "-3.25", "1e-100", "123456789012345678901234567890",
             "2.718281828459045235360287471352662497757", ".5", "7.",
             "-0.000001234e-20", "1e300", "-1e-320", "0x1.8p+1", "-0x1p-1074",
             "0x1.123456789abcdef0123p-3", "3.14159265358979323846264338327950288419716939937510"]
    for k in (2, 3, 4):
        for t in texts:
            s = t.strip()
            if s.lstrip("+-").lower().startswith("0x"):
                v = bf_parse_hex(s)
            else:
                v = bf_parse_decimal(s, PrecisionContext(53 * k + 64))
            comps = list(bf_to_multicomp(v, k).components)
            out["parse"].append(dict(k=k, text=t, comps=[c.hex() for c in comps]))
    for t, p, d in (("0.1", 424, 20), ("1e-100", 424, 40), ("-3.25", 100, 5),
                    ("123456.789", 200, 3), ("0", 100, 10), ("9.9999", 60, 2),
                    ("2", 64, 1), ("1.5e-30", 300, None)):
        v = bf_parse_decimal(t, PrecisionContext(p))
        out["format"].append(dict(text=t, prec=p, digits=d, hex=hexv(v),
                                  out=bf_format_decimal(v, d)))
    with open(os.path.join(HERE, "longside.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
