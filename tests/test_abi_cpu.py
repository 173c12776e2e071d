"""C-ABI library checks that need no GPU: libmpcore.so loads, exports every
symbol include/mpcore.h declares (including the reference's 16,
build_lib.py:31-57), answers the device-free calls, and fails loudly (status
6 + message) instead of falling back to the CPU when no device exists."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2107_12550_b200 import _native as nat

HEADER = os.path.join(ROOT, "include", "mpcore.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mpcore_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_reference_abi():
    syms = header_symbols()
    for s in nat.REFERENCE_SYMBOLS:
        assert s in syms, s
    assert len(nat.REFERENCE_SYMBOLS) == 16


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (mpcore_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    lib = nat.lib()
    for s in header_symbols():
        assert hasattr(lib, s)


def test_bindings_cover_header():
    assert sorted(nat.ALL_SYMBOLS) == header_symbols()


def test_version_and_simd(monkeypatch):
    buf = ctypes.create_string_buffer(32)
    assert nat.lib().mpcore_version(buf, 32) == 0
    assert buf.value.decode() == "0.1.0"
    small = ctypes.create_string_buffer(3)
    assert nat.lib().mpcore_version(small, 3) == 2     # truncation
    assert small.value == b"0."
    monkeypatch.delenv("MPCORE_SIMD", raising=False)
    assert nat.lib().mpcore_simd_enabled() == 1
    for text, want in (("0", 0), ("off", 0), ("FALSE", 0), (" No ", 0),
                       ("1", 1), ("on", 1)):
        monkeypatch.setenv("MPCORE_SIMD", text)
        assert nat.lib().mpcore_simd_enabled() == want


def test_null_and_shape_errors_without_device():
    L = nat.lib()
    h = ctypes.c_uint64()
    assert L.mpcore_matrix_new(2, 2, 2, None) == 2
    assert L.mpcore_matrix_new(5, 2, 2, ctypes.byref(h)) == 2
    assert L.mpcore_matrix_new(2, 0, 2, ctypes.byref(h)) == 2
    assert L.mpcore_vector_new(1, 3, ctypes.byref(h)) == 2
    assert L.mpcore_release(123456789) == 1
    assert L.mpcore_lu_factor(99999, None) == 2
    piv = ctypes.c_uint64()
    assert L.mpcore_lu_factor(99999, ctypes.byref(piv)) == 1
    assert L.mpcore_lu_solve(1, 2, 3, 4) == 1
    assert L.mpcore_report_iterations(77, ctypes.byref(ctypes.c_int32())) == 1


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="has a GPU")
def test_no_device_fails_loudly():
    L = nat.lib()
    h = ctypes.c_uint64()
    st = L.mpcore_matrix_new(2, 4, 4, ctypes.byref(h))
    assert st == 6
    msg = nat.last_error()
    assert "device" in msg.lower() or "cuda" in msg.lower()
