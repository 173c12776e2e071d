"""A/B: one-call LU + solve (nb = 32, one level) vs the distributed driver
at one rank (outer nb, inner 32: two-level blocking, K = nb updates), both
on [A | b], bitwise-checked; CUDA-event time per solve (restore included).

    python tools/twolevel_ab.py K N [NB ...]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat  # noqa: E402
from paper_2107_12550_b200.dist import Layout, dist_lu_solve  # noqa: E402

k, n = int(sys.argv[1]), int(sys.argv[2])
nbs = [int(a) for a in sys.argv[3:]] or [64, 128, 256]
reps = int(os.environ.get("REPS", "10"))
seed = 210712552
L = nat.lib()
W0 = torch.zeros((k, n, n + 1), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
nat.check(L.mpcore_dev_generate_cyclic(k, W0.data_ptr(), n + 1, n * (n + 1), n,
                                       n, 32, 1, 0, 0, n, seed), "gen")
xt = torch.zeros((k, n), dtype=torch.float64, device="cuda")
nat.check(L.mpcore_dev_generate_cyclic(k, xt.data_ptr(), n, n, 1, n, 32, 1, 0,
                                       2, n, seed), "gen x") if False else None
xt[0] = 1.0
b = torch.zeros_like(xt)
nat.check(L.mpcore_dev_matvec(k, n, n, W0.data_ptr(), n + 1, n * (n + 1),
                              xt.data_ptr(), b.data_ptr()), "mv")
W0[:, :, n] = b
W = W0.clone()
x = torch.zeros_like(xt)
sw = np.zeros(n, dtype=np.int32)
st = nat._i32(-1)
torch.cuda.synchronize()


def onecall():
    W.copy_(W0)
    torch.cuda.synchronize()
    nat.check(L.mpcore_dev_solve_system(k, n, W.data_ptr(), n + 1,
                                        n * (n + 1), 0, x.data_ptr(),
                                        nat.iptr(sw), ctypes.byref(st)), "1c")


def timed(f):
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), \
            torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


t1 = timed(onecall)
ref_x = x.cpu().numpy().copy()
ref_lu = W.cpu().numpy().copy()
print("k=%d n=%d one-call: %.3f ms (%.1f GFLOP/s)" % (
    k, n, t1, (2 / 3) * n ** 3 / t1 / 1e6), flush=True)
for nb in nbs:
    M = W0.clone()
    xd = torch.zeros_like(xt)

    def dist():
        M.copy_(W0)
        dist_lu_solve(Layout(n, nb, 1), {0: M}, {0: xd}, k)
    t2 = timed(dist)
    same = (xd.cpu().numpy().tobytes() == ref_x.tobytes() and
            M.cpu().numpy().tobytes() == ref_lu.tobytes())
    _, ph, _ = dist_lu_solve(Layout(n, nb, 1), {0: M.copy_(W0)}, {0: xd}, k,
                             phases=True)
    print("  two-level nb=%d: %.3f ms (%.1f GFLOP/s) bitwise=%s phases %s" % (
        nb, t2, (2 / 3) * n ** 3 / t2 / 1e6, same,
        {a: round(v, 2) for a, v in ph.items()}), flush=True)
