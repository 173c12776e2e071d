"""NaN / Inf entries: the pivot is np.argmax over |head| (linalg.py:429) --
the first NaN if there is one, else the first maximum -- and the factors
follow the reference's kernels.  Goldens from the reference itself
(tests/golden/make_golden_nan.py); NaN payloads are platform-specific, so
factors compare NaN positions and every other bit."""

import numpy as np
import pytest

import oracle
from conftest import golden


def same_nan_aware(a, b):
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    if a.shape != b.shape or not np.array_equal(na, nb):
        return False
    return a[~na].tobytes() == b[~nb].tobytes()


G = golden("lu_nan.npz")
IDS = sorted(int(k[1:]) for k in G.files if k.startswith("A"))


@pytest.mark.parametrize("idx", IDS)
def test_oracle_nan_pivots_match_reference(idx):
    A = G["A%d" % idx]
    lu, sw = oracle.lu(A)
    assert sw.tobytes() == G["sw%d" % idx].tobytes()
    assert same_nan_aware(lu, G["lu%d" % idx])


@pytest.mark.gpu
@pytest.mark.parametrize("idx", IDS)
def test_gpu_nan_pivots_match_reference(idx):
    from paper_2107_12550_b200.linalg import DeviceMatrix
    A = G["A%d" % idx]
    dm = DeviceMatrix.from_planes(A)
    piv = dm.lu_factor()
    assert np.asarray(piv.swaps(), dtype=np.int32).tobytes() == \
        G["sw%d" % idx].tobytes()
    assert same_nan_aware(dm.download(), G["lu%d" % idx])
