"""Native distributed driver vs the one-call LU + solve at one rank, on the
config-4 recipe: bitwise pivots and x (diagnostics).

    python tools/dist_check.py N [N ...]     (env: MPCORE_DIST_SERIAL, MPCORE_NO_GRAPH)
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat  # noqa: E402
from paper_2107_12550_b200.dist import (DeviceBackend, Layout,  # noqa: E402
                                        dist_lu_solve)

k, nb, seed = 2, 256, 210712554
L = nat.lib()
for n in [int(a) for a in sys.argv[1:]]:
    be = DeviceBackend(k)
    W = be.alloc(n, n + 1)
    base, ld, plane = be.view(W)
    torch.cuda.synchronize()
    nat.check(L.mpcore_dev_generate_cyclic(k, base, ld, plane, n, n, nb, 1, 0,
                                           0, n, seed), "gen")
    xt = torch.zeros((k, n), dtype=torch.float64, device="cuda")
    xt[0] = 1.0
    b = torch.zeros_like(xt)
    torch.cuda.synchronize()
    nat.check(L.mpcore_dev_matvec(k, n, n, base, ld, plane, xt.data_ptr(),
                                  b.data_ptr()), "mv")
    W[:, :, n] = b
    M = W.clone()
    torch.cuda.synchronize()
    x1 = torch.zeros_like(xt)
    sw1 = np.zeros(n, dtype=np.int32)
    st = nat._i32(-1)
    t0 = time.time()
    nat.check(L.mpcore_dev_solve_system(k, n, base, n + 1, n * (n + 1), 0,
                                        x1.data_ptr(), nat.iptr(sw1),
                                        ctypes.byref(st)), "one-call")
    t1 = time.time()
    x = torch.zeros_like(xt)
    try:
        sw, ph, nl = dist_lu_solve(Layout(n, nb, 1), {0: M}, {0: x}, k,
                                   phases=True)
        t2 = time.time()
        ok_sw = sw.tobytes() == sw1.tobytes()
        first = int(np.argmax(sw != sw1)) if not ok_sw else -1
        ok_x = x.cpu().numpy().tobytes() == x1.cpu().numpy().tobytes()
        ok_lu = M[:, :, :n].cpu().numpy().tobytes() == \
            W[:, :, :n].cpu().numpy().tobytes()
        print("n=%d one-call %.3f s dist %.3f s swaps %s (first diff %d) "
              "lu %s x %s phases %s launches %d" % (
                  n, t1 - t0, t2 - t1, ok_sw, first, ok_lu, ok_x,
                  {a: round(v, 1) for a, v in ph.items()}, nl), flush=True)
    except Exception as ex:
        print("n=%d dist failed: %s" % (n, ex), flush=True)
    del W, M
    torch.cuda.empty_cache()
