"""The refinement driver's long -> short conversion on the GPU
(csrc/convert.cu, linalg.py:761-770 with
bf_to_multicomp, bigfloat.py:419-432): rounding each exact value once to
the working precision and peeling its k binary64 heads must give the
host's fixed-width results bit for bit (which test_longside.py pins to the
generic big-integer path) -- values of 1 .. 640 bits, exponents at both
ends of the binary64 range (the out-of-range flag included), runs of ones
and exact halves.  The config-3 goldens (test_gpu_config3*.py) run through
it end to end."""

import ctypes

import pytest

from paper_2107_12550_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", [53, 64, 65, 106, 200, 424, 511, 512, 640])
@pytest.mark.parametrize("k", [2, 3, 4])
def test_device_conversion_matches_host(prec, k):
    m = ctypes.c_int64(-1)
    nat.check(nat.lib().mpcore_debug_convert_selftest(
        20000, 31 * prec + k, prec, k, ctypes.byref(m)), "convert selftest")
    assert m.value == 0
