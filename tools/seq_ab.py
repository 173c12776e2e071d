"""A/B: one-call LU after the distributed driver in the same process."""
import os
import subprocess
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes  # noqa
from paper_2107_12550_b200 import _native as nat  # noqa
from paper_2107_12550_b200.dist import Layout, dist_lu_solve, DeviceBackend  # noqa

k, nb, seed = 2, 256, 210712554
L = nat.lib()


def system(n):
    W0 = torch.zeros((k, n, n + 1), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    nat.check(L.mpcore_dev_generate_cyclic(k, W0.data_ptr(), n + 1, n * (n + 1), n, n,
                                           nb, 1, 0, 0, n, seed), "gen")
    xt = torch.zeros((k, n), dtype=torch.float64, device="cuda"); xt[0] = 1
    b = torch.zeros_like(xt)
    nat.check(L.mpcore_dev_matvec(k, n, n, W0.data_ptr(), n + 1, n * (n + 1),
                                  xt.data_ptr(), b.data_ptr()), "mv")
    W0[:, :, n] = b
    torch.cuda.synchronize()
    return W0


def onecall(W0, tag):
    n = W0.shape[1]
    W = W0.clone(); x = torch.zeros((k, n), dtype=torch.float64, device="cuda")
    sw = np.zeros(n, dtype=np.int32); st = nat._i32(-1)
    torch.cuda.synchronize()
    r = L.mpcore_dev_solve_system(k, n, W.data_ptr(), n + 1, n * (n + 1), 0,
                                  x.data_ptr(), nat.iptr(sw), ctypes.byref(st))
    print(tag, "onecall n=%d status %d step %d" % (n, r, st.value), flush=True)


def dist(W0, tag):
    n = W0.shape[1]
    M = W0.clone(); x = torch.zeros((k, n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    try:
        dist_lu_solve(Layout(n, nb, 1), {0: M}, {0: x}, k)
        print(tag, "dist n=%d ok" % n, flush=True)
    except Exception as e:
        print(tag, "dist n=%d FAILED %s" % (n, e), flush=True)


A = system(16384)
B = system(8192)
onecall(A, "1")
dist(B, "2")
onecall(A, "3")
onecall(A, "4")
dist(A, "5")
dist(A, "6")
onecall(A, "7")
