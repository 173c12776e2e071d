"""SURVEY §8(c) config-4 plan, step 2, at the full size: the native
distributed LU + solve of the n = 32768 DD system with G = 1 and G = 8
(virtual ranks on one GPU: the same host loop as the NCCL path, broadcasts
and hand-offs as device copies) -- pivots, every factor and x bitwise
equal.  Also the normwise backward error of x.

    python tools/dist_invariance.py [n] [G ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat  # noqa: E402
from paper_2107_12550_b200.dist import (DeviceBackend, Layout,  # noqa: E402
                                        dist_lu_solve)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
Gs = [int(a) for a in sys.argv[2:]] or [1, 8]
k, nb, seed = 2, 256, 210712554
be = DeviceBackend(k)
full = be.alloc(n, n)
be.generate(full, Layout(n, nb, 1), 0, 0, seed)
xt = torch.zeros((k, n), dtype=torch.float64, device="cuda")
xt[0] = 1.0
b = torch.zeros_like(xt)
torch.cuda.synchronize()
nat.check(nat.lib().mpcore_dev_matvec(k, n, n, full.data_ptr(), n, n * n,
                                      xt.data_ptr(), b.data_ptr()), "mv")
ref = None
for G in Gs:
    layout = Layout(n, nb, G)
    local, xs = {}, {}
    for r in range(G):
        cols = torch.as_tensor(layout.global_columns(r), device="cuda")
        M = torch.empty((k, n, len(cols) + 1), dtype=torch.float64,
                        device="cuda")
        M[:, :, :len(cols)] = full[:, :, cols]
        M[:, :, len(cols)] = b
        local[r] = M
        xs[r] = torch.zeros_like(xt)
    torch.cuda.synchronize()
    t0 = time.time()
    swaps, _, launches = dist_lu_solve(layout, local, xs, k)
    torch.cuda.synchronize()
    dt = time.time() - t0
    fact = torch.empty((k, n, n), dtype=torch.float64, device="cuda")
    for r in range(G):
        cols = torch.as_tensor(layout.global_columns(r), device="cuda")
        fact[:, :, cols] = local[r][:, :, :-1]
    del local
    torch.cuda.empty_cache()
    x = xs[0].cpu().numpy()
    err = float(np.max(np.abs((x[0] - 1.0) + x[1])))
    same = None
    if ref is None:
        ref = (swaps.tobytes(), x.tobytes(), fact)
    else:
        same = (swaps.tobytes() == ref[0], x.tobytes() == ref[1],
                bool(torch.equal(fact.view(torch.int64),
                                 ref[2].view(torch.int64))))
        del fact
        torch.cuda.empty_cache()
    print("n=%d G=%d: %.2f s (one GPU serving %d virtual ranks), %d launches, "
          "max|x-1| %.3g, bitwise vs G=%d (swaps, x, factors): %s"
          % (n, G, dt, G, launches, err, Gs[0], same), flush=True)
