"""Golden IR runs on the config-3 system family, made by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_config3.py

The config-3 generator (A = U diag(sigma) W, kappa = 1e30, b = A*ones at
512 bits; csrc/testsys.cpp) writes .mpmat files through
mpcore_write_config3 (host only, no GPU); the reference's own matfile
loader reads them and its iterative_refinement (refine.py:121-197, TD short
side, rtol 1e-100, atol 0) runs on them.  Recorded per size: the SHA-256
of both files (pins the generator), iterations, stop reason, residual
history and solution as bf_format_decimal text (the report API's format).
"""

import ctypes
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(1, "/root/reference/pkg/src")

import mpcore  # noqa: E402
from mpcore.bigfloat import bf_format_decimal  # noqa: E402
from mpcore.matfile import load_matrix, load_vector  # noqa: E402
from mpcore.refine import RefineConfig, iterative_refinement  # noqa: E402

from paper_2107_12550_b200 import _native as nat  # noqa: E402

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/")

SEED = 210712553


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def main():
    out = []
    tmp = tempfile.mkdtemp()
    for n, kappa in ((24, 30.0), (40, 30.0), (33, 20.0)):
        pa = os.path.join(tmp, "A%d.mpmat" % n)
        pb = os.path.join(tmp, "b%d.mpmat" % n)
        st = nat.lib().mpcore_write_config3(n, SEED, kappa, 512, 0,
                                            pa.encode(), pb.encode())
        assert st == 0, st
        A = load_matrix(pa)
        b = load_vector(pb)
        cfg = RefineConfig(short_k=3, long_bits=512, rtol="1e-100", atol=0,
                           max_iter=20)
        rep = iterative_refinement(A, b, cfg)
        out.append(dict(
            n=n, kappa_exp10=kappa, seed=SEED, sha_A=sha(pa), sha_b=sha(pb),
            iterations=rep.iterations, stop_reason=rep.stop_reason,
            history=[bf_format_decimal(h, 40) for h in rep.residual_history],
            solution=[bf_format_decimal(e, 60) for e in rep.solution.data]))
        print("config3 golden n=%d: %d iterations, %s" % (
            n, rep.iterations, rep.stop_reason))
    with open(os.path.join(HERE, "config3_ir.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    main()
