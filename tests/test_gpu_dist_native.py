"""The native, device-ordered distributed LU + solve (csrc/dist.cu, C ABI
mpcore_dist_lu_solve) against the reference's chain, bit for bit.

One GPU serves G virtual ranks through the library's local transport (the
same host loop as the NCCL path; broadcasts and the back-substitution
hand-offs become device copies), and the NCCL transport itself runs at
world size 1.  Checked: pivots, every rank's factored local columns, y =
L^-1 P b in the replicated right-hand-side column, and x, against the
pinned oracle (reference lane path, linalg.py:422-538); panels narrower
and wider than 32 (multi-chunk exchanges), ragged last blocks, more ranks
than blocks, the singular step."""

import numpy as np
import pytest
import torch

import oracle
from oracle import gen
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.dist import (DIST_PHASES, DeviceBackend, Layout,
                                        NcclComm, dist_lu_solve)
from paper_2107_12550_b200.errors import SingularMatrixError

pytestmark = pytest.mark.gpu


def build(k, n, nb, G, seed, A=None):
    """Local matrices (k, n, lc + 1) with b = A x_true in the last column;
    returns (layout, local, xs, A, b)."""
    layout = Layout(n, nb, G)
    be = DeviceBackend(k)
    if A is None:
        A = gen.planes(k, (n, n), 0, n, seed)
    xt = gen.planes(k, (n,), 2, n, seed)
    b = oracle.matvec(A, xt)
    local, xs = {}, {}
    for r in range(G):
        cols = layout.global_columns(r)
        M = np.zeros((k, n, len(cols) + 1))
        M[:, :, :len(cols)] = A[:, :, cols]
        M[:, :, len(cols)] = b
        local[r] = torch.from_numpy(M).to(be.device)
        xs[r] = torch.zeros((k, n), dtype=torch.float64, device=be.device)
    torch.cuda.synchronize()
    return layout, local, xs, A, b


@pytest.mark.parametrize("k,n,nb,G", [
    (2, 256, 64, 2), (3, 200, 32, 3), (4, 160, 64, 2), (2, 300, 128, 4),
    (2, 513, 256, 2), (3, 96, 32, 1), (2, 1100, 256, 1), (3, 700, 48, 3),
    (2, 130, 16, 5), (4, 257, 100, 2), (2, 64, 256, 3)])
def test_native_virtual_ranks_match_reference(k, n, nb, G):
    layout, local, xs, A, b = build(k, n, nb, G, 4711 + n)
    swaps, _, launches = dist_lu_solve(layout, local, xs, k)
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, b)
    assert swaps.tobytes() == sw_ref.tobytes()
    for r in range(G):
        cols = layout.global_columns(r)
        M = local[r].cpu().numpy()
        assert M[:, :, :len(cols)].tobytes() == \
            np.ascontiguousarray(lu_ref[:, :, cols]).tobytes()
        assert xs[r].cpu().numpy().tobytes() == x_ref.tobytes()
    # y (the replicated b column) equals the one-GPU [A | b] LU's column n
    aug = np.concatenate([A, b[:, :, None]], axis=2)
    W = torch.from_numpy(np.ascontiguousarray(aug)).cuda()
    x1 = torch.zeros((k, n), dtype=torch.float64, device="cuda")
    sw1 = np.zeros(n, dtype=np.int32)
    st = nat._i32(-1)
    torch.cuda.synchronize()
    nat.check(nat.lib().mpcore_dev_solve_system(
        k, n, W.data_ptr(), n + 1, n * (n + 1), 0, x1.data_ptr(),
        nat.iptr(sw1), nat.ctypes.byref(st)), "solve_system")
    y1 = W.cpu().numpy()[:, :, n]
    for r in range(G):
        assert local[r].cpu().numpy()[:, :, -1].tobytes() == \
            np.ascontiguousarray(y1).tobytes()
    assert launches > 0


def test_native_repeat_and_phases():
    # repeated calls reuse the cached workspace and the tall-block LU graphs
    k, n, nb = 2, 1024, 256
    layout, local, xs, A, b = build(k, n, nb, 1, 99)
    M0 = local[0].clone()
    lu_ref, sw_ref = oracle.lu(A)
    x_ref = oracle.solve(lu_ref, sw_ref, b)
    for it in range(3):
        local[0].copy_(M0)
        swaps, ph, _ = dist_lu_solve(layout, local, xs, k, phases=True)
        assert swaps.tobytes() == sw_ref.tobytes()
        assert xs[0].cpu().numpy().tobytes() == x_ref.tobytes()
        assert set(ph) == set(DIST_PHASES) and ph["total"] > 0
        assert ph["update"] > 0 and ph["factor"] > 0


def test_native_nccl_world1_matches_local():
    k, n, nb = 3, 600, 128
    layout, local, xs, A, b = build(k, n, nb, 1, 5150)
    comm = NcclComm(1, 0)
    try:
        swaps, _, _ = dist_lu_solve(layout, local, xs, k, comm=comm)
    finally:
        comm.close()
    lu_ref, sw_ref = oracle.lu(A)
    assert swaps.tobytes() == sw_ref.tobytes()
    assert local[0].cpu().numpy()[:, :, :n].tobytes() == lu_ref.tobytes()
    assert xs[0].cpu().numpy().tobytes() == \
        oracle.solve(lu_ref, sw_ref, b).tobytes()


@pytest.mark.parametrize("G", [1, 2])
def test_native_singular_step(G):
    # column 70 is a copy of column 3 after scaling rows: exact zero pivot
    k, n, nb = 2, 160, 32
    A = np.zeros((k, n, n))
    A[0] = np.eye(n)
    A[0, :, 70] = 0.0            # a zero column -> singular at step 70
    layout, local, xs, _, _ = build(k, n, nb, G, 1, A=A)
    with pytest.raises(SingularMatrixError) as ei:
        dist_lu_solve(layout, local, xs, k)
    assert ei.value.step == 70


@pytest.mark.parametrize("k,n,G", [(2, 2048, 2), (2, 4096, 4), (3, 2048, 3)])
def test_native_config4_path_vs_oracle(k, n, G):
    # SURVEY §8(c) config-4 plan, step 1: the nb = 256 column-cyclic path
    # byte-compared with the oracle at n = 2048 / 4096
    layout, local, xs, A, b = build(k, n, 256, G, 210712554 + n)
    swaps, _, _ = dist_lu_solve(layout, local, xs, k)
    lu_ref, sw_ref = oracle.lu(A)
    assert swaps.tobytes() == sw_ref.tobytes()
    for r in range(G):
        cols = layout.global_columns(r)
        assert local[r].cpu().numpy()[:, :, :len(cols)].tobytes() == \
            np.ascontiguousarray(lu_ref[:, :, cols]).tobytes()
    assert xs[0].cpu().numpy().tobytes() == \
        oracle.solve(lu_ref, sw_ref, b).tobytes()


def test_native_rank_invariance_n16384():
    # step 2 of the plan at n = 16384 (DD, 4.3 GB): G = 1, 4 and 8 virtual
    # ranks give the same pivots, factors and x bit for bit
    k, n, nb = 2, 16384, 256
    seed = 210712554
    ref = None
    for G in (1, 4, 8):
        layout = Layout(n, nb, G)
        be = DeviceBackend(k)
        full = be.alloc(n, n)
        be.generate(full, Layout(n, nb, 1), 0, 0, seed)
        xt = torch.zeros((k, n), dtype=torch.float64, device="cuda")
        xt[0] = 1.0
        bb = torch.zeros_like(xt)
        torch.cuda.synchronize()
        nat.check(nat.lib().mpcore_dev_matvec(k, n, n, full.data_ptr(), n,
                                              n * n, xt.data_ptr(),
                                              bb.data_ptr()), "mv")
        local, xs = {}, {}
        for r in range(G):
            cols = torch.as_tensor(layout.global_columns(r), device="cuda")
            M = torch.empty((k, n, len(cols) + 1), dtype=torch.float64,
                            device="cuda")
            M[:, :, :len(cols)] = full[:, :, cols]
            M[:, :, len(cols)] = bb
            local[r] = M
            xs[r] = torch.zeros_like(xt)
        del full
        torch.cuda.synchronize()
        swaps, _, _ = dist_lu_solve(layout, local, xs, k)
        # factors back in global column order, compared bitwise on the GPU
        fact = torch.empty((k, n, n), dtype=torch.float64, device="cuda")
        for r in range(G):
            cols = torch.as_tensor(layout.global_columns(r), device="cuda")
            fact[:, :, cols] = local[r][:, :, :-1]
        res = (swaps.tobytes(), xs[0].cpu().numpy().tobytes())
        if ref is None:
            ref, ref_fact = res, fact
        else:
            assert res == ref
            assert torch.equal(fact.view(torch.int64),
                               ref_fact.view(torch.int64))
            del fact
        del local, xs
        torch.cuda.empty_cache()
