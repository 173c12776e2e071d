"""Per-kernel-class time of the distributed LU protocol on one GPU
(LocalComm, G virtual ranks), plus host wall time.
usage: dist_prof.py N [G] [K]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.dist import DeviceBackend, Layout, LocalComm, dist_lu_factor
n = int(sys.argv[1]); G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
layout = Layout(n, 256, G)
be = DeviceBackend(k)
local = {}
for r in range(G):
    M = be.alloc(n, layout.local_cols(r)); be.generate(M, layout, r, 0, 210712554); local[r] = M
pristine = {r: M.clone() for r, M in local.items()}
dist_lu_factor(be, LocalComm(), layout, local); torch.cuda.synchronize()
for r in local: local[r].copy_(pristine[r])
torch.cuda.synchronize()
t0 = time.perf_counter()
dist_lu_factor(be, LocalComm(), layout, local); torch.cuda.synchronize()
wall = time.perf_counter() - t0
for r in local: local[r].copy_(pristine[r])
torch.cuda.synchronize()
nat.prof_enable(True); nat.prof_reset()
t0 = time.perf_counter()
dist_lu_factor(be, LocalComm(), layout, local); torch.cuda.synchronize()
wall_p = time.perf_counter() - t0
p = nat.prof_read(); nat.prof_enable(False)
print("n=%d G=%d k=%d wall %.1f ms (%.1f GF/s), profiled wall %.1f ms" % (n, G, k, wall * 1e3, (2/3) * n**3 / wall / 1e9, wall_p * 1e3))
print({s: (round(v[0], 1), v[1]) for s, v in p.items() if v[1]})
