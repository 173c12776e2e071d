"""Handle-level call surface with the reference's names and status codes
(/root/reference/pkg/src/mpcore/ffi.py:1-306), forwarding to the native
C ABI (include/mpcore.h).  Every function returns the status (and value)
exactly as the reference's does, so host code written against mpcore.ffi
runs unchanged."""

import ctypes

from . import _native as nat

OK, BAD_HANDLE, BAD_DIMENSION, SINGULAR, BAD_PARSE, OVERFLOW, INTERNAL = \
    range(7)

__all__ = [
    "OK", "BAD_HANDLE", "BAD_DIMENSION", "SINGULAR", "BAD_PARSE",
    "OVERFLOW", "INTERNAL", "version", "simd_enabled", "matrix_new",
    "vector_new", "release", "set_element_from_decimal",
    "get_element_components", "lu_factor", "lu_solve_handles", "refine",
    "report_iterations", "report_stop_reason", "report_residual_count",
    "report_residual_entry", "report_solution_count",
    "report_solution_entry",
]


def _L():
    return nat.lib()


def _text(fn, *args, cap=4096):
    buf = ctypes.create_string_buffer(cap)
    st = fn(*args, buf, cap)
    return st, buf.value.decode("ascii", "replace")


def version():
    return _text(_L().mpcore_version, cap=64)[1]


def simd_enabled():
    return _L().mpcore_simd_enabled()


def matrix_new(k, rows, cols):
    h = ctypes.c_uint64()
    st = _L().mpcore_matrix_new(k, rows, cols, ctypes.byref(h))
    return st, h.value


def vector_new(k, n):
    h = ctypes.c_uint64()
    st = _L().mpcore_vector_new(k, n, ctypes.byref(h))
    return st, h.value


def release(h):
    return _L().mpcore_release(h)


def set_element_from_decimal(h, i, j, text):
    return _L().mpcore_set_element_from_decimal(
        h, i, j, text.encode("ascii", "replace"))


def get_element_components(h, i, j):
    out = (ctypes.c_double * 4)()
    st = _L().mpcore_get_element_components(h, i, j, out, 4)
    if st != OK:
        return st, ()
    kind = ctypes.c_int32()
    k = ctypes.c_int32()
    _L().mpcore_object_info(h, ctypes.byref(kind), ctypes.byref(k), None,
                            None)
    return OK, tuple(out[:k.value])


def lu_factor(h):
    piv = ctypes.c_uint64()
    st = _L().mpcore_lu_factor(h, ctypes.byref(piv))
    return st, piv.value


def lu_solve_handles(lu_h, piv_h, b_h, x_h):
    return _L().mpcore_lu_solve(lu_h, piv_h, b_h, x_h)


def refine(a_path, b_path, short_k, long_bits, rtol, atol, max_iter):
    h = ctypes.c_uint64()
    st = _L().mpcore_refine(a_path.encode(), b_path.encode(), short_k,
                            long_bits, rtol.encode(), atol.encode(), max_iter,
                            ctypes.byref(h))
    return st, h.value


def _int(fn, h):
    v = ctypes.c_int32()
    st = fn(h, ctypes.byref(v))
    return st, v.value


def report_iterations(h):
    return _int(_L().mpcore_report_iterations, h)


def report_stop_reason(h):
    st, t = _text(_L().mpcore_report_stop_reason, h, cap=64)
    return (st, t) if st == OK else (st, "")


def report_residual_count(h):
    return _int(_L().mpcore_report_residual_count, h)


def report_residual_entry(h, idx, digits):
    st, t = _text(_L().mpcore_report_residual_entry, h, idx, digits)
    return (st, t) if st == OK else (st, "")


def report_solution_count(h):
    return _int(_L().mpcore_report_solution_count, h)


def report_solution_entry(h, idx, digits):
    st, t = _text(_L().mpcore_report_solution_entry, h, idx, digits)
    return (st, t) if st == OK else (st, "")
