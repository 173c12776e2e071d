"""Per-panel chain of one LU in graph mode (MPCORE_LU_STAMPS kernel stamps):
panel time, gap panel(P) exit -> exchange+U12(P) entry, its time, gap to
panel(P+1) entry (the next-panel update and launch latency).
usage: lu_stamps.py K N [one-call]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix
k = int(sys.argv[1]); n = int(sys.argv[2])
L = nat.lib()
A0 = DeviceMatrix(k, n, n); A0.generate(0, n, 5)
W = DeviceMatrix(k, n, n)
for _ in range(2):
    W.copy_from(A0); W.lu_factor()
W.copy_from(A0); nat.sync()
nat.check(L.mpcore_debug_lu_stamps(4 * n, None), "arm")
W.lu_factor(); nat.sync()
buf = np.zeros(4 * n, dtype=np.uint64)
nat.check(L.mpcore_debug_lu_stamps(4 * n, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))), "read")
s = buf.reshape(n, 4).astype(np.float64)
Js = [J for J in range(n) if buf[4 * J + 1] != 0]
t0 = s[Js[0], 0]
rows = []
for i, J in enumerate(Js):
    pe, px, te, tx = s[J]
    nxt = s[Js[i + 1], 0] if i + 1 < len(Js) else np.nan
    have_t = buf[4 * J + 3] != 0
    rows.append((J, (pe - t0) / 1e3, (px - pe) / 1e3,
                 (te - px) / 1e3 if have_t else np.nan,
                 (tx - te) / 1e3 if have_t else np.nan,
                 (nxt - tx) / 1e3 if have_t else np.nan))
r = np.array(rows)
print("J  start_us  panel_us  gap_to_trsm  trsm_us  trsm_exit_to_next_panel")
for row in r[:: max(1, len(r) // 16)]:
    print("%5d %9.1f %8.1f %8.1f %8.1f %8.1f" % tuple(row))
last = s[Js[-1]]
print("LU (first panel entry -> last exchange exit): %.1f us" % ((max(last[1], last[3]) - t0) / 1e3))
for a, b in ((0, len(r) // 2), (len(r) // 2, len(r))):
    seg = r[a:b]
    print("panels %d-%d: panel %.1f, gap->trsm %.1f, trsm %.1f, trsm->next panel %.1f (sums, us)" % (
        a, b - 1, np.nansum(seg[:, 2]), np.nansum(seg[:, 3]), np.nansum(seg[:, 4]), np.nansum(seg[:, 5])))
