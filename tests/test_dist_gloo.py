"""The distributed (column-block-cyclic) LU protocol of
paper_2107_12550_b200/dist.py, run on CPU with a checker backend (the
oracle's block primitives, each in the reference's chain order):

  * one process acting for G = 1, 2, 3 ranks (LocalComm);
  * world_size 2 over torch.distributed gloo (TorchComm), 127.0.0.1.

Both must reproduce the reference factorisation bit for bit (pivots and
factors), which also pins the layout math, the pivot/panel broadcast and
the order of row exchanges / TRSM / trailing updates."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from oracle import gen
from paper_2107_12550_b200.dist import (Layout, LocalComm, TorchComm,
                                        dist_lu_factor)
from paper_2107_12550_b200.errors import SingularMatrixError

_F64 = ctypes.POINTER(ctypes.c_double)


class OracleBackend:
    """CPU checker backend: torch CPU tensors (gloo-broadcastable) viewed as
    numpy, arithmetic by the oracle."""

    def __init__(self, k):
        self.k = k
        self.L = oracle.lib()

    def alloc(self, rows, cols):
        return torch.zeros((self.k, rows, cols), dtype=torch.float64)

    def _ptr(self, M, row0=0, col0=0):
        a = M.numpy()
        k, rows, cols = a.shape
        addr = a.ctypes.data + (row0 * cols + col0) * 8
        return ctypes.cast(addr, _F64), cols, rows * cols

    def int_buffer(self, n):
        return torch.zeros(n, dtype=torch.int32)

    def ints_to_host(self, t):
        return t.numpy().copy()

    def ints_from_host(self, t, arr):
        t.copy_(torch.from_numpy(np.ascontiguousarray(arr, np.int32)))

    def lu_block(self, M, row0, col0, width):
        p, ld, pl = self._ptr(M, row0, col0)
        m = M.shape[1] - row0
        sw = np.zeros(width, np.int32)
        step = np.zeros(1, np.int32)
        st = self.L.mcref_lu_block(self.k, m, width, p, ld, pl,
                                   sw.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   step.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        if st == 3:
            raise SingularMatrixError("singular", step=row0 + int(step[0]))
        return sw + row0

    def pack(self, M, row0, col0, width, buf):
        rows = M.shape[1] - row0
        buf[:, :rows, :width] = M[:, row0:, col0:col0 + width]

    def laswp(self, M, col0, ncols, row0, swaps):
        if ncols <= 0:
            return
        a = M.numpy()
        for i, r in enumerate(swaps):
            j = row0 + i
            if r != j:
                tmp = a[:, j, col0:col0 + ncols].copy()
                a[:, j, col0:col0 + ncols] = a[:, r, col0:col0 + ncols]
                a[:, r, col0:col0 + ncols] = tmp

    def trsm(self, buf, w, M, row0, col0, ncols):
        pl_, ldl, pll = self._ptr(buf)
        pu, ldu, plu = self._ptr(M, row0, col0)
        self.L.mcref_trsm(self.k, w, ncols, pl_, ldl, pll, pu, ldu, plu)

    def gemm_update(self, buf, w, M, row0, col0, ncols):
        mrows = M.shape[1] - row0 - w
        if mrows <= 0 or ncols <= 0:
            return
        pa, lda, pla = self._ptr(buf, w, 0)
        pb, ldb, plb = self._ptr(M, row0, col0)
        pc, ldc, plc = self._ptr(M, row0 + w, col0)
        self.L.mcref_gemm_update(self.k, mrows, ncols, w, pa, lda, pla, pb,
                                 ldb, plb, pc, ldc, plc)


def local_blocks(A, layout, ranks, backend):
    out = {}
    for r in ranks:
        cols = layout.global_columns(r)
        M = backend.alloc(layout.n, len(cols))
        M.copy_(torch.from_numpy(np.ascontiguousarray(A[:, :, cols])))
        out[r] = M
    return out


def assemble(local, layout):
    full = np.zeros((local[next(iter(local))].shape[0], layout.n, layout.n))
    for r, M in local.items():
        full[:, :, layout.global_columns(r)] = M.numpy()
    return full


@pytest.mark.parametrize("lookahead", [True, False])
@pytest.mark.parametrize("k,n,nb,G", [(2, 96, 16, 1), (2, 96, 16, 2),
                                      (3, 80, 32, 3), (4, 70, 16, 2),
                                      (2, 130, 32, 4), (3, 64, 64, 2)])
def test_local_world_matches_reference_lu(k, n, nb, G, lookahead):
    A = gen.planes(k, (n, n), 0, n, 4242 + n)
    lu_ref, sw_ref = oracle.lu(A)
    layout = Layout(n, nb, G)
    be = OracleBackend(k)
    local = local_blocks(A, layout, range(G), be)
    swaps = dist_lu_factor(be, LocalComm(), layout, local, lookahead)
    assert swaps.tobytes() == sw_ref.tobytes()
    assert assemble(local, layout).tobytes() == lu_ref.tobytes()


def test_layout_math():
    lay = Layout(1000, 64, 3)
    assert lay.nblocks == 16 and lay.width(15) == 1000 - 15 * 64
    cols = np.concatenate([lay.global_columns(r) for r in range(3)])
    assert sorted(cols.tolist()) == list(range(1000))
    for r in range(3):
        assert lay.local_cols(r) == len(lay.global_columns(r))
        g = lay.global_columns(r)
        for P in range(lay.nblocks):
            t0 = lay.trailing_start(r, P)
            assert (g[t0:] > (P + 1) * 64 - 1).all()
            assert (g[:t0] < (P + 1) * 64).all()
        for b in lay.blocks_of(r):
            off = lay.local_offset(r, b)
            assert g[off] == b * 64


def test_singular_reported_on_every_rank():
    k, n = 2, 48
    A = gen.planes(k, (n, n), 0, n, 7)
    A[:, :, 20] = 0.0                      # column 20 entirely zero
    with pytest.raises(oracle.Singular) as e:
        oracle.lu(A)
    layout = Layout(n, 16, 2)
    be = OracleBackend(k)
    local = local_blocks(A, layout, range(2), be)
    with pytest.raises(SingularMatrixError) as e2:
        dist_lu_factor(be, LocalComm(), layout, local)
    assert e2.value.step == e.value.step


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, k, n, nb, out_dir, lookahead=True):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = gen.planes(k, (n, n), 0, n, 99 + n)
        layout = Layout(n, nb, world)
        be = OracleBackend(k)
        local = local_blocks(A, layout, [rank], be)
        swaps = dist_lu_factor(be, TorchComm(), layout, local, lookahead)
        np.save(os.path.join(out_dir, "rank%d.npy" % rank), local[rank].numpy())
        np.save(os.path.join(out_dir, "swaps%d.npy" % rank), swaps)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,n,nb,world,lookahead",
                         [(2, 100, 16, 2, True), (3, 72, 32, 2, False),
                          (2, 90, 16, 3, True)])
def test_gloo_world_matches_reference_lu(tmp_path, k, n, nb, world, lookahead):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), k, n, nb, str(tmp_path),
                            lookahead),
             nprocs=world, join=True)
    A = gen.planes(k, (n, n), 0, n, 99 + n)
    lu_ref, sw_ref = oracle.lu(A)
    layout = Layout(n, nb, world)
    full = np.zeros_like(A)
    for r in range(world):
        full[:, :, layout.global_columns(r)] = np.load(tmp_path / ("rank%d.npy" % r))
        assert np.load(tmp_path / ("swaps%d.npy" % r)).tobytes() == sw_ref.tobytes()
    assert full.tobytes() == lu_ref.tobytes()


def _id_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.dist import NcclComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = NcclComm.exchange_id(world, rank)
        with open(os.path.join(out_dir, "id%d" % rank), "wb") as fh:
            fh.write(uid)
        # no GPU here: creating the communicator must fail loudly (status
        # 6 with the library's message), never fall back
        try:
            NcclComm(world, rank)
            ok = "created"
        except nat.NativeError as e:
            ok = "refused %d" % e.status
        with open(os.path.join(out_dir, "init%d" % rank), "w") as fh:
            fh.write(ok)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_nccl_bootstrap_id_over_gloo(tmp_path):
    # the native distributed driver's bootstrap at world size 2: one NCCL
    # unique id drawn on rank 0 (libnccl via dlopen), identical on every rank
    import torch.multiprocessing as mp
    from paper_2107_12550_b200 import _native as nat
    if torch.cuda.is_available():
        pytest.skip("CPU-only check (the GPU suite covers the communicator)")
    mp.spawn(_id_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2,
             join=True)
    ids = [open(tmp_path / ("id%d" % r), "rb").read() for r in range(2)]
    assert len(ids[0]) == 128 and ids[0] == ids[1] and any(ids[0])
    for r in range(2):
        assert open(tmp_path / ("init%d" % r)).read() == \
            "refused %d" % nat.INTERNAL
