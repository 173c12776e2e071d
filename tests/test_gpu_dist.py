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
                                      (2, 513, 256, 2), (3, 96, 32, 1),
                                      (2, 2048, 256, 4), (2, 2100, 256, 3)])
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


@pytest.mark.parametrize("k,m,w", [(2, 4100, 32), (3, 2200, 32),
                                   (4, 4740, 64), (2, 9000, 48)])
def test_tall_block_lu_matches_oracle(k, m, w):
    # tall blocks spread the panel over > 64 CTAs (the 5-slot poll path, up
    # to one CTA per SM); w > 32 exercises the inner panel blocking
    import ctypes
    A = gen.planes(k, (m, w), 0, m, 4242 + m)
    ref = A.copy()
    sw_ref = np.zeros(w, dtype=np.int32)
    step = np.zeros(1, dtype=np.int32)
    I32 = ctypes.POINTER(ctypes.c_int32)
    F = ctypes.POINTER(ctypes.c_double)
    st = oracle.lib().mcref_lu_block(k, m, w, ref.ctypes.data_as(F), w, m * w,
                                     sw_ref.ctypes.data_as(I32),
                                     step.ctypes.data_as(I32))
    assert st == 0 and step[0] == -1
    be = DeviceBackend(k)
    M = torch.from_numpy(A).cuda()
    sw = be.lu_block(M, 0, 0, w)
    assert sw.tobytes() == sw_ref.tobytes()
    assert M.cpu().numpy().tobytes() == ref.tobytes()


def test_config4_rank_invariance_large():
    # SURVEY 8(c) config-4 plan: the column-block-cyclic factorisation is
    # byte-identical for every rank count (here G = 1, 4, 8 virtual ranks
    # on one GPU) at a size the oracle cannot reach; n = 16384 DD, nb = 256
    k, n, nb, seed = 2, 16384, 256, 210712554
    full = {}
    for G in (1, 4, 8):
        layout = Layout(n, nb, G)
        be = DeviceBackend(k)
        local = {}
        for r in range(G):
            M = be.alloc(n, layout.local_cols(r))
            be.generate(M, layout, r, 0, seed)
            local[r] = M
        swaps = dist_lu_factor(be, LocalComm(), layout, local)
        A = torch.empty((k, n, n), dtype=torch.float64, device="cuda")
        for r, M in local.items():
            A[:, :, torch.as_tensor(layout.global_columns(r),
                                    device="cuda")] = M
        del local
        full[G] = (swaps, A)
        if G != 1:
            assert swaps.tobytes() == full[1][0].tobytes()
            assert torch.equal(A.view(torch.int64), full[1][1].view(torch.int64))
            del full[G]
        torch.cuda.empty_cache()
