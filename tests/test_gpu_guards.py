"""Write-overrun checks of every kernel family (the substitute for
compute-sanitizer memcheck, which this GPU pool does not run): objects are
allocated between 64 KiB guard zones (MPCORE_DEBUG_GUARD=1) and the zones
must be intact after LU, solves, the one-call solve, GEMM (non-square),
mat_vec, the elementwise kernels (add/mul/div/sqrt), axpy and the
generator at ragged sizes; the distributed driver's local matrices and x
get guard margins of their own.  A deliberate overrun (a copy one element
before an object's planes) must be detected.  Results are also checked
bitwise against the oracle, so a clean run comes with correct answers."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
from oracle import gen
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.dist import Layout, dist_lu_solve
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          device_solve, device_solve_system)

pytestmark = pytest.mark.gpu


def guards():
    c, b = ctypes.c_int64(), ctypes.c_int64()
    nat.check(nat.lib().mpcore_debug_check_guards(ctypes.byref(c),
                                                  ctypes.byref(b)), "guards")
    return c.value, b.value


@pytest.fixture
def guarded(monkeypatch):
    monkeypatch.setenv("MPCORE_DEBUG_GUARD", "1")
    yield


@pytest.mark.parametrize("k,n", [(2, 1), (3, 2), (4, 31), (2, 33), (3, 97),
                                 (4, 130), (2, 257), (3, 300)])
def test_kernels_stay_in_bounds(guarded, k, n):
    seed = 900 + n
    A = gen.planes(k, (n, n), 0, n, seed)
    xt = gen.planes(k, (n,), 2, n, seed)
    objs = []
    M = DeviceMatrix.from_planes(A)
    bh = oracle.matvec(A, xt)
    b = DeviceVector.from_planes(bh)
    x = DeviceVector(k, n)
    objs += [M, b, x]
    piv = M.lu_factor()
    device_solve(M, piv, b, x)
    lu_ref, sw_ref = oracle.lu(A)
    assert x.download().tobytes() == oracle.solve(lu_ref, sw_ref, bh).tobytes()
    M1 = DeviceMatrix.from_planes(A)
    x1 = DeviceVector(k, n)
    objs += [M1, x1]
    device_solve_system(M1, b, x1)
    assert x1.download().tobytes() == x.download().tobytes()
    # GEMM with a non-square inner dimension, mat_vec, elementwise, axpy
    m2, n2 = n + 3, max(1, n - 1)
    Ag = gen.planes(k, (m2, n), 0, 4096, seed)
    Bg = gen.planes(k, (n, n2), 1, 4096, seed)
    Ad, Bd, Cd = (DeviceMatrix.from_planes(Ag), DeviceMatrix.from_planes(Bg),
                  DeviceMatrix(k, m2, n2))
    objs += [Ad, Bd, Cd]
    nat.check(nat.lib().mpcore_mat_mul(Ad.handle, Bd.handle, Cd.handle), "mm")
    assert Cd.download().tobytes() == oracle.gemm(Ag, Bg).tobytes()
    y = DeviceVector(k, m2)
    objs.append(y)
    nat.check(nat.lib().mpcore_mat_vec(Ad.handle, x.handle, y.handle), "mv")
    pos = xt * np.where(xt[0] < 0, -1.0, 1.0)   # |x|, canonical form kept
    X, O = DeviceVector.from_planes(pos), DeviceVector(k, n)
    objs += [X, O]
    for op in (0, 1, 2, 3):
        nat.check(nat.lib().mpcore_elementwise(op, X.handle, X.handle,
                                               O.handle), "ew")
    alpha = np.ascontiguousarray(xt[:, 0])
    nat.check(nat.lib().mpcore_axpy(nat.dptr(alpha), k, X.handle, O.handle),
              "axpy")
    G = DeviceMatrix(k, n, n)
    objs.append(G)
    G.generate(0, n, seed)
    nat.sync()
    checked, bad = guards()
    assert checked >= len(objs)
    assert bad == 0


def test_overrun_is_detected(guarded):
    V = DeviceVector(2, 8)
    p = V.device_ptr()
    src = DeviceVector.from_planes(np.ones((2, 8)))
    # one element before plane 0: inside the lower guard zone
    nat.check(nat.lib().mpcore_dev_copy2d(1, 1, 1, p - 8, 1, 1,
                                          src.device_ptr(), 1, 1), "copy")
    checked, bad = guards()
    assert bad >= 1
    del V        # (release the corrupted object before the next test)


def _guarded_tensor(shape, margin=4096):
    """A contiguous view inside a larger buffer whose margins hold a
    sentinel bit pattern."""
    numel = int(np.prod(shape))
    buf = torch.empty(numel + 2 * margin, dtype=torch.float64, device="cuda")
    buf.view(torch.int64)[:] = 0x5A5A5A5A5A5A5A5A
    return buf, buf[margin:margin + numel].view(shape), margin


def _margins_intact(buf, margin):
    v = buf.view(torch.int64)
    return bool((v[:margin] == 0x5A5A5A5A5A5A5A5A).all()) and \
        bool((v[-margin:] == 0x5A5A5A5A5A5A5A5A).all())


@pytest.mark.parametrize("k,n,nb,G", [(2, 300, 64, 3), (3, 257, 100, 2),
                                      (4, 130, 32, 1)])
def test_distributed_driver_stays_in_bounds(k, n, nb, G):
    layout = Layout(n, nb, G)
    A = gen.planes(k, (n, n), 0, n, 77 + n)
    xt = gen.planes(k, (n,), 2, n, 77 + n)
    b = oracle.matvec(A, xt)
    bufs, local, xs = [], {}, {}
    for r in range(G):
        cols = layout.global_columns(r)
        Mh = np.zeros((k, n, len(cols) + 1))
        Mh[:, :, :len(cols)] = A[:, :, cols]
        Mh[:, :, -1] = b
        buf, M, mg = _guarded_tensor(Mh.shape)
        M.copy_(torch.from_numpy(Mh))
        xb, xv, xm = _guarded_tensor((k, n))
        bufs += [(buf, mg), (xb, xm)]
        local[r], xs[r] = M, xv
    torch.cuda.synchronize()
    dist_lu_solve(layout, local, xs, k)
    torch.cuda.synchronize()
    lu_ref, sw_ref = oracle.lu(A)
    assert xs[0].cpu().numpy().tobytes() == \
        oracle.solve(lu_ref, sw_ref, b).tobytes()
    for buf, mg in bufs:
        assert _margins_intact(buf, mg)
