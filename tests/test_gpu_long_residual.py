"""The IR residual b - A x at long precision on the GPU (SURVEY §8(f) row 1,
csrc/residual.cu) against the host's fixed-width arithmetic (itself checked
against the generic big-integer path, test_longside.py) on random systems
with cancellation rows, zeros and all-ones mantissas: bit for bit.  The
golden IR runs (test_gpu_config3.py, test_gpu_ffi.py) go through it too."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [0, 1, 2, 5])
@pytest.mark.parametrize("prec", [53, 64, 65, 106, 200, 300, 424, 511, 512])
@pytest.mark.parametrize("n", [1, 7, 33])
def test_device_residual_matches_host(prec, n, variant):
    # variant 5: products kernel + chain kernel (production), 2: products
    # on producer warps beside the chain, 0: warp per row,
    # 1: thread per row
    from paper_2107_12550_b200 import _native as nat
    m = ctypes.c_int64(-1)
    nat.check(nat.lib().mpcore_debug_long_residual_selftest(
        n, prec, 2107 + prec * 31 + n, variant, ctypes.byref(m)),
        "residual selftest")
    assert m.value == 0


@pytest.mark.parametrize("variant", [0, 2, 5])
def test_device_residual_larger(variant):
    from paper_2107_12550_b200 import _native as nat
    m = ctypes.c_int64(-1)
    nat.check(nat.lib().mpcore_debug_long_residual_selftest(
        256, 512, 99, variant, ctypes.byref(m)), "residual selftest")
    assert m.value == 0
