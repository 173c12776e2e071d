"""One-call [A | b] LU + solve at size n on the config-4 recipe, repeated:
prints the singular step if any and x's max error (diagnostics, A/B of
library builds via MPCORE_LIB)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat  # noqa: E402

k, nb, seed = 2, 256, 210712554
L = nat.lib()
reps = int(os.environ.get("REPS", "2"))
for n in [int(a) for a in sys.argv[1:]]:
    W0 = torch.zeros((k, n, n + 1), dtype=torch.float64, device="cuda")
    base = W0.data_ptr()
    torch.cuda.synchronize()
    nat.check(L.mpcore_dev_generate_cyclic(k, base, n + 1, n * (n + 1), n, n,
                                           nb, 1, 0, 0, n, seed), "gen")
    xt = torch.zeros((k, n), dtype=torch.float64, device="cuda")
    xt[0] = 1.0
    b = torch.zeros_like(xt)
    nat.check(L.mpcore_dev_matvec(k, n, n, base, n + 1, n * (n + 1),
                                  xt.data_ptr(), b.data_ptr()), "mv")
    W0[:, :, n] = b
    W = W0.clone()
    x = torch.zeros_like(xt)
    sw = np.zeros(n, dtype=np.int32)
    for rep in range(reps):
        W.copy_(W0)
        torch.cuda.synchronize()
        st = nat._i32(-1)
        t0 = time.time()
        r = L.mpcore_dev_solve_system(k, n, W.data_ptr(), n + 1, n * (n + 1),
                                      0, x.data_ptr(), nat.iptr(sw),
                                      ctypes.byref(st))
        dt = time.time() - t0
        xs = x.cpu().numpy()
        print("n=%d rep %d status %d step %d  %.3f s  err %.3g" % (
            n, rep, r, st.value, dt,
            float(np.max(np.abs(xs[0] - 1.0 + xs[1])))), flush=True)
    del W, W0
    torch.cuda.empty_cache()
