"""ctypes binding of libmpcore.so (include/mpcore.h).

The library is the only execution path: if it is missing or no sm_100 device
is usable, calls raise NativeError loudly.  There is no CPU fallback.
"""

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPCORE_EXACT_RANGE=1: the build whose two_prod reproduces the reference's
# Dekker bits outside the binary64 band too (mc.cuh; 12-19 % slower)
LIB_PATH = os.environ.get("MPCORE_LIB") or os.path.join(
    _HERE, "libmpcore_exact.so" if os.environ.get("MPCORE_EXACT_RANGE", "0")
    not in ("", "0") else "libmpcore.so")  # (MPCORE_LIB: A/B builds)

OK, BAD_HANDLE, BAD_DIMENSION, SINGULAR, BAD_PARSE, OVERFLOW, INTERNAL = \
    range(7)

_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_cp = ctypes.c_char_p

_PROTOS = {
    # reference ABI (build_lib.py:31-57)
    "mpcore_version": (_i32, [ctypes.c_char_p, _i32]),
    "mpcore_simd_enabled": (_i32, []),
    "mpcore_matrix_new": (_i32, [_i32, _i32, _i32, ctypes.POINTER(_u64)]),
    "mpcore_vector_new": (_i32, [_i32, _i32, ctypes.POINTER(_u64)]),
    "mpcore_release": (_i32, [_u64]),
    "mpcore_set_element_from_decimal": (_i32, [_u64, _i32, _i32, _cp]),
    "mpcore_get_element_components": (_i32, [_u64, _i32, _i32, _dp, _i32]),
    "mpcore_lu_factor": (_i32, [_u64, ctypes.POINTER(_u64)]),
    "mpcore_lu_solve": (_i32, [_u64, _u64, _u64, _u64]),
    "mpcore_refine": (_i32, [_cp, _cp, _i32, _i32, _cp, _cp, _i32,
                             ctypes.POINTER(_u64)]),
    "mpcore_report_iterations": (_i32, [_u64, _ip]),
    "mpcore_report_stop_reason": (_i32, [_u64, ctypes.c_char_p, _i32]),
    "mpcore_report_residual_count": (_i32, [_u64, _ip]),
    "mpcore_report_residual_entry": (_i32, [_u64, _i32, _i32,
                                            ctypes.c_char_p, _i32]),
    "mpcore_report_solution_count": (_i32, [_u64, _ip]),
    "mpcore_report_solution_entry": (_i32, [_u64, _i32, _i32,
                                            ctypes.c_char_p, _i32]),
    # extensions
    "mpcore_object_info": (_i32, [_u64, _ip, _ip, _ip, _ip]),
    "mpcore_set_planes": (_i32, [_u64, _dp, _i64]),
    "mpcore_get_planes": (_i32, [_u64, _dp, _i64]),
    "mpcore_set_planes_async": (_i32, [_u64, _dp, _i64]),
    "mpcore_get_planes_async": (_i32, [_u64, _dp, _i64]),
    "mpcore_copy": (_i32, [_u64, _u64]),
    "mpcore_pivot_new": (_i32, [_i32, _ip, ctypes.POINTER(_u64)]),
    "mpcore_pivot_get": (_i32, [_u64, _ip, _i32]),
    "mpcore_host_alloc": (_i32, [_i64, ctypes.POINTER(ctypes.c_void_p)]),
    "mpcore_host_free": (_i32, [ctypes.c_void_p]),
    "mpcore_lu_factor_ex": (_i32, [_u64, _i32, ctypes.POINTER(_u64), _ip]),
    "mpcore_mat_mul": (_i32, [_u64, _u64, _u64]),
    "mpcore_mat_vec": (_i32, [_u64, _u64, _u64]),
    "mpcore_elementwise": (_i32, [_i32, _u64, _u64, _u64]),
    "mpcore_axpy": (_i32, [_dp, _i32, _u64, _u64]),
    "mpcore_generate": (_i32, [_u64, _i32, _i64, _u64]),
    "mpcore_lu_decomp_pm": (_i32, [_i32, _i32, _dp, _ip, _ip]),
    "mpcore_solve_ls_pm": (_i32, [_i32, _i32, _dp, _ip, _dp, _dp]),
    "mpcore_set_device": (_i32, [_i32]),
    "mpcore_device_name": (_i32, [ctypes.c_char_p, _i32]),
    "mpcore_sm_count": (_i32, [_ip]),
    "mpcore_last_error": (_i32, [ctypes.c_char_p, _i32]),
    "mpcore_sync": (_i32, []),
    "mpcore_prof_enable": (_i32, [_i32]),
    "mpcore_prof_reset": (_i32, []),
    "mpcore_prof_read": (_i32, [_dp, ctypes.POINTER(_i64), _i32]),
    "mpcore_fp64_peak": (_i32, [_dp, _dp]),
    "mpcore_debug_panel_trace": (_i32, [ctypes.POINTER(_u64), _i64]),
    "mpcore_debug_lu_stamps": (_i32, [_i64, ctypes.POINTER(_u64)]),
    "mpcore_stream_event_record": (_i32, [_i32]),
    "mpcore_debug_long_residual_selftest": (_i32, [_i32, _i32, _u64, _i32, ctypes.POINTER(_i64)]),
    "mpcore_stream_event_elapsed": (_i32, [_i32, _i32, ctypes.POINTER(ctypes.c_double)]),
    "mpcore_solve_system": (_i32, [_u64, _u64, _u64, _i32, ctypes.POINTER(_u64),
                                   ctypes.POINTER(_i32)]),
    "mpcore_dev_solve_system": (_i32, [_i32, _i32, _u64, _i64, _i64, _i32,
                                       _u64, ctypes.POINTER(_i32),
                                       ctypes.POINTER(_i32)]),
    "mpcore_refine_config3": (_i32, [_i32, _u64, ctypes.c_double, _i32, _i32,
                                     ctypes.c_char_p, ctypes.c_char_p, _i32,
                                     _i32, ctypes.POINTER(_u64)]),
    "mpcore_write_config3": (_i32, [_i32, _u64, ctypes.c_double, _i32, _i32,
                                    ctypes.c_char_p, ctypes.c_char_p]),
    "mpcore_report_timings": (_i32, [_u64, ctypes.POINTER(ctypes.c_double),
                                     _i32, ctypes.POINTER(_i32)]),
    "mpcore_debug_solve_trace": (_i32, [ctypes.POINTER(_u64), _i64]),
    "mpcore_debug_longfloat_selftest": (_i32, [_i64, _u64, _i32,
                                               ctypes.POINTER(_i64)]),
    "mpcore_debug_timeline": (_i32, [ctypes.POINTER(ctypes.c_double), _i64,
                                     ctypes.POINTER(_i64)]),
    # device-pointer building blocks (dist.py)
    "mpcore_object_device_ptr": (_i32, [_u64, ctypes.POINTER(_u64)]),
    "mpcore_dev_lu_block": (_i32, [_i32, _i32, _i32, _u64, _i64, _i64, _i32,
                                   _ip, _ip]),
    "mpcore_dev_laswp": (_i32, [_i32, _u64, _i64, _i64, _i32, _i32, _i32,
                                _ip, _i32]),
    "mpcore_dev_trsm": (_i32, [_i32, _i32, _i32, _u64, _i64, _i64, _u64,
                               _i64, _i64]),
    "mpcore_dev_gemm": (_i32, [_i32, _i32, _i32, _i32, _i32, _i32, _u64,
                               _i64, _i64, _u64, _i64, _i64, _u64, _i64,
                               _i64]),
    "mpcore_dev_copy2d": (_i32, [_i32, _i32, _i32, _u64, _i64, _i64, _u64,
                                 _i64, _i64]),
    "mpcore_dev_lu_solve": (_i32, [_i32, _i32, _u64, _i64, _i64, _ip, _u64,
                                   _u64]),
    "mpcore_dev_matvec": (_i32, [_i32, _i32, _i32, _u64, _i64, _i64, _u64,
                                 _u64]),
    "mpcore_dev_generate_cyclic": (_i32, [_i32, _u64, _i64, _i64, _i32, _i32,
                                          _i32, _i32, _i32, _i32, _i64,
                                          _u64]),
    "mpcore_debug_check_guards": (_i32, [ctypes.POINTER(_i64),
                                         ctypes.POINTER(_i64)]),
    "mpcore_debug_convert_selftest": (_i32, [_i64, _u64, _i32, _i32,
                                             ctypes.POINTER(_i64)]),
    # the native distributed LU + solve (dist.cu; BASELINE config 4)
    "mpcore_dist_unique_id": (_i32, [ctypes.c_char_p, _i32]),
    "mpcore_dist_comm_init": (_i32, [_i32, _i32, ctypes.c_char_p, _i32,
                                     ctypes.POINTER(_u64)]),
    "mpcore_dist_comm_destroy": (_i32, [_u64]),
    "mpcore_dist_lu_solve": (_i32, [_u64, _i32, _i32, _i32, _i32, _i32, _ip,
                                    ctypes.POINTER(_u64),
                                    ctypes.POINTER(_i64),
                                    ctypes.POINTER(_i64), _ip,
                                    ctypes.POINTER(_u64), _u64, _ip, _ip,
                                    _dp, ctypes.POINTER(_i64)]),
}

# The 16 symbols of the reference ABI (build_lib.py:31-57).
REFERENCE_SYMBOLS = [
    "mpcore_version", "mpcore_simd_enabled", "mpcore_matrix_new",
    "mpcore_vector_new", "mpcore_release", "mpcore_set_element_from_decimal",
    "mpcore_get_element_components", "mpcore_lu_factor", "mpcore_lu_solve",
    "mpcore_refine", "mpcore_report_iterations", "mpcore_report_stop_reason",
    "mpcore_report_residual_count", "mpcore_report_residual_entry",
    "mpcore_report_solution_count", "mpcore_report_solution_entry",
]
ALL_SYMBOLS = list(_PROTOS)

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """libmpcore failed (status code + library message)."""

    def __init__(self, status, where, message=""):
        super().__init__("%s failed with status %d%s" % (
            where, status, (": " + message) if message else ""))
        self.status = status
        self.message = message


def lib():
    """Load libmpcore.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        "libmpcore.so not built (%s); run "
                        "`python -c 'import __graft_entry__ as g; g.build()'`"
                        % LIB_PATH)
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _PROTOS.items():
                    f = getattr(L, name, None)
                    if f is None and os.environ.get("MPCORE_LIB"):
                        continue   # an older A/B build
                    if f is None:
                        raise ImportError("libmpcore lacks " + name)
                    f.restype = res
                    f.argtypes = args
                _lib = L
    return _lib


def last_error():
    buf = ctypes.create_string_buffer(512)
    lib().mpcore_last_error(buf, 512)
    return buf.value.decode("ascii", "replace")


def check(st, where):
    if st != OK:
        raise NativeError(st, where, last_error())
    return st


def dptr(a):
    return a.ctypes.data_as(_dp)


def iptr(a):
    return a.ctypes.data_as(_ip)


def new_matrix(k, rows, cols):
    h = _u64()
    check(lib().mpcore_matrix_new(k, rows, cols, ctypes.byref(h)),
          "matrix_new")
    return h.value


def new_vector(k, n):
    h = _u64()
    check(lib().mpcore_vector_new(k, n, ctypes.byref(h)), "vector_new")
    return h.value


def release(h):
    return lib().mpcore_release(h)


def set_planes(h, planes):
    a = np.ascontiguousarray(planes, dtype=np.float64)
    check(lib().mpcore_set_planes(h, dptr(a), a.size), "set_planes")


# host arrays an asynchronous copy still reads or writes: kept alive here
# until sync() returns (a dropped array would otherwise be freed under the
# DMA); keyed by id so a loop re-using the same staging buffers without
# sync() does not grow it
_inflight = {}


def set_planes_async(h, planes):
    """Asynchronous upload (mpcore_set_planes_async): `planes` must be a
    C-contiguous float64 array (page-locked for a truly asynchronous copy)
    that stays unchanged until the next library call that uses the object
    returns."""
    if not (isinstance(planes, np.ndarray) and planes.dtype == np.float64
            and planes.flags.c_contiguous):
        raise ValueError("set_planes_async needs a C-contiguous float64 array")
    check(lib().mpcore_set_planes_async(h, dptr(planes), planes.size),
          "set_planes_async")
    _inflight[id(planes)] = planes


def get_planes_async(h, out):
    """Asynchronous download into `out` (C-contiguous float64, page-locked
    for a truly asynchronous copy); valid after sync()."""
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64
            and out.flags.c_contiguous):
        raise ValueError("get_planes_async needs a C-contiguous float64 array")
    check(lib().mpcore_get_planes_async(h, dptr(out), out.size),
          "get_planes_async")
    _inflight[id(out)] = out


def get_planes(h, shape, out=None):
    if out is None:
        out = np.empty(shape, dtype=np.float64)
    check(lib().mpcore_get_planes(h, dptr(out), out.size), "get_planes")
    return out


def lu_factor(h, nb=0):
    """-> (status, pivot handle, singular step)."""
    piv = _u64()
    step = _i32(-1)
    st = lib().mpcore_lu_factor_ex(h, nb, ctypes.byref(piv),
                                   ctypes.byref(step))
    return st, piv.value, step.value


def pivot_get(h, n):
    out = np.empty(n, dtype=np.int32)
    check(lib().mpcore_pivot_get(h, iptr(out), n), "pivot_get")
    return out


def pivot_new(swaps):
    s = np.ascontiguousarray(swaps, dtype=np.int32)
    h = _u64()
    check(lib().mpcore_pivot_new(len(s), iptr(s), ctypes.byref(h)),
          "pivot_new")
    return h.value


class Handle:
    """Owning wrapper: releases the library object when collected."""

    __slots__ = ("h", "__weakref__")

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.mpcore_release(self.h)
        except Exception:
            pass
        self.h = 0


_DEVICE_OK = None


def device_available():
    """True when libmpcore is built and finds its sm_100 device (cached)."""
    global _DEVICE_OK
    if _DEVICE_OK is None:
        try:
            v = _i32()
            _DEVICE_OK = lib().mpcore_sm_count(ctypes.byref(v)) == OK
        except Exception:
            _DEVICE_OK = False
    return _DEVICE_OK


class _PinnedHolder:
    """numpy base object keeping a PinnedBuffer alive (array interface)."""

    def __init__(self, pb, shape):
        self._pb = pb
        self.__array_interface__ = {
            "shape": tuple(shape), "typestr": "<f8",
            "data": (pb.ptr.value, False), "version": 3}


def pinned_zeros(shape):
    """float64 zeros in page-locked host memory (mpcore_host_alloc): the
    containers' planes, so every host<->device copy of the drop-in API runs
    at DMA speed.  The memory lives as long as the returned array."""
    pb = PinnedBuffer(shape)
    a = np.asarray(_PinnedHolder(pb, pb.shape))
    a[...] = 0.0
    return a


class PinnedBuffer:
    """Page-locked host array (mpcore_host_alloc) viewed as numpy."""

    def __init__(self, shape, dtype=np.float64):
        self.shape = tuple(shape)
        nbytes = int(np.prod(self.shape)) * np.dtype(dtype).itemsize
        self.ptr = ctypes.c_void_p()
        check(lib().mpcore_host_alloc(max(nbytes, 8), ctypes.byref(self.ptr)),
              "host_alloc")
        buf = (ctypes.c_char * max(nbytes, 8)).from_address(self.ptr.value)
        self.array = np.frombuffer(buf, dtype=dtype,
                                   count=int(np.prod(self.shape))).reshape(
                                       self.shape)

    def free(self):
        if self.ptr is not None and self.ptr.value:
            lib().mpcore_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


PROF_SLOTS = ["panel", "laswp", "trsm", "update", "solve", "gemm", "matvec",
              "elementwise", "gen", "update_next"]


def prof_enable(on=True):
    check(lib().mpcore_prof_enable(1 if on else 0), "prof_enable")


def prof_reset():
    check(lib().mpcore_prof_reset(), "prof_reset")


def prof_read():
    n = len(PROF_SLOTS)
    ms = np.zeros(n)
    cnt = np.zeros(n, dtype=np.int64)
    check(lib().mpcore_prof_read(dptr(ms), cnt.ctypes.data_as(
        ctypes.POINTER(_i64)), n), "prof_read")
    return {s: (float(ms[i]), int(cnt[i])) for i, s in enumerate(PROF_SLOTS)}


def fp64_peak():
    a = ctypes.c_double()
    b = ctypes.c_double()
    check(lib().mpcore_fp64_peak(ctypes.byref(a), ctypes.byref(b)),
          "fp64_peak")
    return a.value, b.value


def device_name():
    buf = ctypes.create_string_buffer(256)
    check(lib().mpcore_device_name(buf, 256), "device_name")
    return buf.value.decode()


def sm_count():
    v = _i32()
    check(lib().mpcore_sm_count(ctypes.byref(v)), "sm_count")
    return v.value


def sync():
    check(lib().mpcore_sync(), "sync")
    _inflight.clear()


class StreamTimer:
    """Device time between start() and stop(): CUDA events recorded on the
    library's stream (every kernel and host<->device copy of libmpcore runs
    there), slots a and b of mpcore_stream_event_record."""

    def __init__(self, a=0, b=1):
        self.a, self.b = a, b

    def start(self):
        check(lib().mpcore_stream_event_record(self.a), "event record")

    def stop(self):
        """-> elapsed milliseconds (waits for the stop event)."""
        check(lib().mpcore_stream_event_record(self.b), "event record")
        ms = ctypes.c_double()
        check(lib().mpcore_stream_event_elapsed(self.a, self.b,
                                                ctypes.byref(ms)),
              "event elapsed")
        return ms.value
