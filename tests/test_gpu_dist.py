"""The distributed LU's device path on one B200: one process serves G
virtual ranks (LocalComm: the broadcast shares the owner's buffer), so the
GPU primitives (tall-block LU, LASWP, blocked TRSM, trailing GEMM, cyclic
generator) run exactly as each rank would run them.  Factors and pivots
must equal the reference's bit for bit (via the pinned oracle), and the
device generator must produce every rank's local columns of the recipe."""

import numpy as np
import pytest
import torch

import oracle
from oracle import gen
from paper_2107_12550_b200.dist import (DeviceBackend, Layout, LocalComm,
                                        dist_lu_factor)

pytestmark = pytest.mark.gpu


def assemble(local, layout, k):
    full = np.zeros((k, layout.n, layout.n))
    for r, M in local.items():
        full[:, :, layout.global_columns(r)] = M.cpu().numpy()
    return full


@pytest.mark.parametrize("k,n,nb,G", [(2, 256, 64, 2), (3, 200, 32, 3),
                                      (4, 160, 64, 2), (2, 300, 128, 4),
                                      (2, 513, 256, 2), (3, 96, 32, 1)])
def test_virtual_ranks_match_reference(k, n, nb, G):
    seed = 31337 + n
    layout = Layout(n, nb, G)
    be = DeviceBackend(k)
    local = {}
    for r in range(G):
        M = be.alloc(n, layout.local_cols(r))
        be.generate(M, layout, r, 0, seed)
        local[r] = M
    A = gen.planes(k, (n, n), 0, n, seed)
    assert assemble(local, layout, k).tobytes() == A.tobytes()
    swaps = dist_lu_factor(be, LocalComm(), layout, local)
    lu_ref, sw_ref = oracle.lu(A)
    assert swaps.tobytes() == sw_ref.tobytes()
    assert assemble(local, layout, k).tobytes() == lu_ref.tobytes()


def test_dev_trsm_blocked_matches_oracle():
    k, w, ncols = 3, 96, 40
    L = gen.planes(k, (w, w), 0, 512, 5)
    U = gen.planes(k, (w, ncols), 1, 512, 5)
    Uo = U.copy()
    lib = oracle.lib()
    import ctypes
    F = ctypes.POINTER(ctypes.c_double)
    lib.mcref_trsm(k, w, ncols, L.ctypes.data_as(F), w, w * w,
                   Uo.ctypes.data_as(F), ncols, w * ncols)
    be = DeviceBackend(k)
    buf = torch.from_numpy(L).cuda()
    M = torch.from_numpy(U).cuda()
    be.trsm(buf, w, M, 0, 0, ncols)
    assert M.cpu().numpy().tobytes() == Uo.tobytes()
