"""Full-size golden fixtures made by running the REFERENCE at the bench sizes.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_fullsize.py JOB

Run in the build container (the only place /root/reference exists); each JOB
is one single-threaded reference run (minutes to ~an hour of numpy lane
work), so the jobs are launched side by side and each writes its own
`fullsize_<JOB>.json`.  Factors are too large to commit, so the fixtures
hold SHA-256 digests of the exact little-endian float64 planes (inputs too,
which pins the seeded recipe), the pivot swaps in full and the solution
planes as exact hex.  The GPU tests (tests/test_gpu_fullsize_ref.py) rebuild
the same inputs on the device, run the product path and compare digests.

Jobs (reference entry points under /root/reference/pkg/src/mpcore):
  lu_td512, lu_dd1024, lu_td1024, lu_td2048, lu_qd2048
      lu_factor_pp + lu_solve, lane path (linalg.py:422-469, 496-538);
      A = slot 0, x_true = slot 2 of the seeded recipe (oracle/gen.py),
      b = mat_vec(A, x_true) (linalg.py:545-574).  td2048 / qd2048 are the
      exact BASELINE config-2 bench workloads (seed 210712552).
  gemm_dd2048, gemm_td2048, gemm_qd2048
      mat_mul_blocked (linalg.py:577-617) of the BASELINE config-1 inputs
      (n = 2048, A slot 0, B slot 1, seed 210712551).  The lane path is a
      rank-1 sweep over the inner index, so each row of C depends only on
      its row of A: the reference is run on a 96-row band of A (rows
      0..47 and 2000..2047) against the full B, and the digests cover those
      rows of C.
  config3_1024
      iterative_refinement (refine.py:121-197) on the BASELINE config-3
      system (n = 1024, kappa = 1e30, 512 bits, rtol 1e-100, atol 0,
      maxtimes 20; files from mpcore_write_config3, as
      make_golden_config3.py does at n = 24/33/40).
"""

import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import mpcore  # noqa: E402  (the reference)
from mpcore import mcfloat  # noqa: E402
from mpcore.linalg import (DenseMatrix, McDomain, Vector, lu_factor_pp,  # noqa: E402
                           lu_solve, mat_mul_blocked, mat_vec)

from oracle import gen  # noqa: E402  (input recipe only)

assert os.path.realpath(mpcore.__file__).startswith("/root/reference/"), \
    mpcore.__file__

DOM = {2: "dd", 3: "td", 4: "qd"}
GEMM_ROWS = list(range(0, 48)) + list(range(2000, 2048))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()
                          ).hexdigest()


def ref_renorm(raw):
    k = raw.shape[0]
    flat = raw.reshape(k, -1)
    z = np.zeros_like(flat[0])
    out = mcfloat.kernel_add(k)(*[flat[c] for c in range(k)], *([z] * k))
    return np.stack([np.asarray(o, dtype=np.float64) for o in out]).reshape(
        raw.shape)


def ref_planes(k, shape, slot, n, seed):
    count = int(np.prod(shape))
    return ref_renorm(gen.raw_planes(k, count, slot, n, seed)).reshape(
        (k,) + tuple(shape))


def lu_job(k, n, seed):
    dom = McDomain(DOM[k])
    A = ref_planes(k, (n, n), 0, n, seed)
    xt = ref_planes(k, (n,), 2, n, seed)
    b = mat_vec(DenseMatrix(dom, n, n, A.copy()), Vector(dom, n, xt.copy()),
                simd=True).data.copy()
    lu = DenseMatrix(dom, n, n, A.copy())
    t0 = time.time()
    piv = lu_factor_pp(lu, simd=True)
    x = lu_solve(lu, piv, Vector(dom, n, b.copy()), simd=True)
    return dict(kind="lu", k=k, n=n, seed=seed, sha_A=sha(A), sha_b=sha(b),
                sha_lu=sha(lu.data), swaps=[int(s) for s in piv.swaps],
                x_hex=[[float(v).hex() for v in row] for row in x.data],
                ref_seconds=time.time() - t0)


def gemm_job(k, n, seed):
    dom = McDomain(DOM[k])
    A = ref_planes(k, (n, n), 0, n, seed)
    B = ref_planes(k, (n, n), 1, n, seed)
    band = np.ascontiguousarray(A[:, GEMM_ROWS, :])
    t0 = time.time()
    C = mat_mul_blocked(DenseMatrix(dom, len(GEMM_ROWS), n, band),
                        DenseMatrix(dom, n, n, B.copy()), simd=True)
    return dict(kind="gemm", k=k, n=n, seed=seed, rows=GEMM_ROWS,
                sha_A=sha(A), sha_B=sha(B), sha_C_rows=sha(C.data),
                C_row0_hex=[[float(v).hex() for v in C.data[c, 0, :16]]
                            for c in range(k)],
                ref_seconds=time.time() - t0)


def config3_job(n=1024, kappa=30.0, seed=210712553):
    from mpcore.bigfloat import bf_format_decimal
    from mpcore.matfile import load_matrix, load_vector
    from mpcore.refine import RefineConfig, iterative_refinement
    from paper_2107_12550_b200 import _native as nat
    tmp = tempfile.mkdtemp()
    pa, pb = os.path.join(tmp, "A.mpmat"), os.path.join(tmp, "b.mpmat")
    assert nat.lib().mpcore_write_config3(n, seed, kappa, 512, 0,
                                          pa.encode(), pb.encode()) == 0
    fsha = [hashlib.sha256(open(p, "rb").read()).hexdigest()
            for p in (pa, pb)]
    A = load_matrix(pa)
    b = load_vector(pb)
    cfg = RefineConfig(short_k=3, long_bits=512, rtol="1e-100", atol=0,
                       max_iter=20)
    t0 = time.time()
    rep = iterative_refinement(A, b, cfg)
    sol = [bf_format_decimal(e, 60) for e in rep.solution.data]
    return dict(kind="config3", n=n, kappa_exp10=kappa, seed=seed,
                sha_A=fsha[0], sha_b=fsha[1], iterations=rep.iterations,
                stop_reason=rep.stop_reason,
                history=[bf_format_decimal(h, 40)
                         for h in rep.residual_history],
                solution_sha=hashlib.sha256(
                    "\n".join(sol).encode()).hexdigest(),
                solution_head=sol[:8], ref_seconds=time.time() - t0)


JOBS = {
    "lu_td512": lambda: lu_job(3, 512, 210712552),
    "lu_dd1024": lambda: lu_job(2, 1024, 77),
    "lu_td1024": lambda: lu_job(3, 1024, 210712552),
    "lu_td2048": lambda: lu_job(3, 2048, 210712552),
    "lu_qd2048": lambda: lu_job(4, 2048, 210712552),
    "gemm_dd2048": lambda: gemm_job(2, 2048, 210712551),
    "gemm_td2048": lambda: gemm_job(3, 2048, 210712551),
    "gemm_qd2048": lambda: gemm_job(4, 2048, 210712551),
    "config3_1024": config3_job,
}


def main():
    job = sys.argv[1]
    out = JOBS[job]()
    with open(os.path.join(HERE, "fullsize_%s.json" % job), "w") as fh:
        json.dump(out, fh, indent=0)
    print(job, "done in %.1f s" % out["ref_seconds"])


if __name__ == "__main__":
    main()
