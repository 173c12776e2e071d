import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MPCORE_SELFTEST_VERBOSE"] = "1"
from paper_2107_12550_b200 import _native as nat
for prec, k in [(53, 2), (512, 3), (106, 2)]:
    m = ctypes.c_int64(-1)
    t = time.time()
    st = nat.lib().mpcore_debug_convert_selftest(20000, 31 * prec + k, prec, k, ctypes.byref(m))
    print(prec, k, st, m.value, "%.3f s" % (time.time() - t), flush=True)
