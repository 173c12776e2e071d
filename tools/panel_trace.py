"""Per-phase latency of the panel kernel (MPCORE_TRACE_PANEL=J).
slots 0..6: clock64 at phase ends (cycles), slot 7: globaltimer at start."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix
k = int(sys.argv[1]); n = int(sys.argv[2])
A = DeviceMatrix(k, n, n); A.generate(0, n, 5)
A.lu_factor()
G = nat.sm_count()
buf = np.zeros(G * 33 * 8, dtype=np.uint64)
nat.check(nat.lib().mpcore_debug_panel_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), buf.size), "trace")
t = buf.reshape(G, 33, 8).astype(np.int64)
ks = t[:, 32, :4].copy()
mk = t[0, 32, 4:6].copy()   # stamp kernels just before / after the launch
g_used = int((t[:, 0, 7] > 0).sum())
t = t[:g_used]
names = ["poll", "pivot+div", "B_ROW", "mult", "B_REM", "la+pub"]
print("CTAs traced:", g_used, " (cycles, median over CTAs)")
d = np.diff(t[:, :31, :7], axis=2)          # phase durations
for jj in (0, 5, 10, 20, 30):
    med = np.median(d[:, jj, :], axis=0)
    print("col %2d " % jj + "  ".join("%s %6.0f" % (names[s], med[s]) for s in range(6)))
per = np.median(np.diff(t[:, :31, 0], axis=1), axis=0); per = per[np.isfinite(per)]
print("period (cycles):", per[:10].astype(int), " median", int(np.median(per)))
start_ns = t[:, :31, 7]
print("period (ns, globaltimer):", np.median(np.diff(start_ns, axis=1), axis=0)[:10].astype(int))
ks = ks[:g_used]
e0 = ks[:, 0].min()
print("kernel stamps (ns from first CTA entry; median/max over CTAs): entry %d/%d  prologue-done %d/%d  loop-done %d/%d  exit %d/%d" % tuple(
    v for c in range(4) for v in (np.median(ks[:, c] - e0), (ks[:, c] - e0).max())))
if mk[0] > 0:
    print("stream stamps (ns): before-launch -> first CTA entry %d, last CTA exit -> after-launch %d" % (
        e0 - mk[0], mk[1] - ks[:, 3].max()))
