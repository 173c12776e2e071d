"""mc_sqrt on the device (mc.cuh sqrt<K>, elementwise op 3) against the
reference's own results (tests/golden/sqrt.npz, mcfloat.py:324-340):
bitwise, as a 1500-lane batch and through the scalar mc_sqrt API."""

import os

import numpy as np
import pytest

import paper_2107_12550_b200 as mp
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceVector

pytestmark = pytest.mark.gpu
D = np.load(os.path.join(os.path.dirname(__file__), "golden", "sqrt.npz"))


@pytest.mark.parametrize("k", [2, 3, 4])
def test_batch_sqrt_bitwise(k):
    a, s = D["a_k%d" % k], D["sqrt_k%d" % k]
    X = DeviceVector.from_planes(a)
    O = DeviceVector(k, a.shape[1])
    nat.check(nat.lib().mpcore_elementwise(3, X.handle, X.handle, O.handle),
              "sqrt")
    assert O.download().tobytes() == s.tobytes()


@pytest.mark.parametrize("k", [2, 3, 4])
def test_scalar_mc_sqrt_bitwise(k):
    a, s = D["a_k%d" % k], D["sqrt_k%d" % k]
    for i in range(0, a.shape[1], 97):
        r = mp.mc_sqrt(mp.MultiComp(tuple(a[:, i]), validate=False))
        assert r.components == tuple(s[:, i])


def test_negative_raises():
    with pytest.raises(mp.DomainError):
        mp.mc_sqrt(mp.MultiComp((-2.0, 0.0)))
    neg = DeviceVector.from_planes(np.array([[1.0, -4.0], [0.0, 0.0]]))
    out = DeviceVector(2, 2)
    assert nat.lib().mpcore_elementwise(3, neg.handle, neg.handle,
                                        out.handle) == nat.INTERNAL
