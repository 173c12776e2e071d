"""Distributed DD/TD/QD LU with partial pivoting: 1-D column-block-cyclic
layout over G GPUs, panel + pivot broadcast (BASELINE config 4; SURVEY
§2.4, §8(e)).

Block column b (columns [b*nb, (b+1)*nb)) lives on rank b % G.  For each
panel P (owner o = P % G):
  1. o factors its tall block rows [J, n) x the panel's nb columns in place
     (pivot search over all rows; libmpcore's blocked LU on the block);
  2. o packs the factored block (L21 with L11/U11 on top) contiguously and
     broadcasts it with the nb pivot indices (NCCL over NVLink via
     torch.distributed, one process per GPU);
  3. every rank applies the row exchanges, in order, to its local columns,
     solves U12 = L11^-1 A12 on its trailing local columns and updates its
     trailing block A22 <- fold_j add(A22, mul(-L21_j, U12_j)).
Every matrix element sees the reference's chain of add(., mul(-m, u)) in
the reference's order (linalg.py:422-449), so the factors and pivots are
bitwise those of the single-GPU factorisation and of the reference.

The orchestration below is backend-agnostic: DeviceBackend drives the GPU
through libmpcore's device-pointer entry points; the CPU tests plug in a
checker backend (tests/test_dist_gloo.py) and run the same protocol on gloo
with world_size 2.  `local_ranks` lets one process act for several ranks
(one GPU emulating G ranks serially, broadcast = sharing the buffer).
"""

import ctypes

import numpy as np

from . import _native as nat
from .errors import SingularMatrixError

__all__ = ["Layout", "DeviceBackend", "TorchComm", "LocalComm",
           "dist_lu_factor", "NcclComm", "dist_lu_solve", "DIST_PHASES"]


class Layout:
    """1-D column-block-cyclic layout of an n x n matrix over `world` ranks."""

    def __init__(self, n, nb, world):
        self.n, self.nb, self.world = int(n), int(nb), int(world)
        self.nblocks = (self.n + self.nb - 1) // self.nb

    def owner(self, b):
        return b % self.world

    def width(self, b):
        return min(self.nb, self.n - b * self.nb)

    def blocks_of(self, rank):
        return list(range(rank, self.nblocks, self.world))

    def local_cols(self, rank):
        return sum(self.width(b) for b in self.blocks_of(rank))

    def local_offset(self, rank, b):
        """Local column of block b's first column on its owner."""
        assert self.owner(b) == rank
        # every block before the globally last one is full
        return (b // self.world) * self.nb

    def trailing_start(self, rank, P):
        """First local column of rank's blocks with global index > P."""
        cnt = 0 if P < rank else (P - rank) // self.world + 1
        return min(cnt * self.nb, self.local_cols(rank))

    def global_columns(self, rank):
        cols = []
        for b in self.blocks_of(rank):
            cols.extend(range(b * self.nb, b * self.nb + self.width(b)))
        return np.array(cols, dtype=np.int64)


class LocalComm:
    """World of ranks all served by this process: broadcast shares the
    owner's buffer (nothing moves)."""

    def broadcast(self, buf, root):
        return buf

    def ibroadcast(self, buf, root):
        return None

    def wait(self, handle):
        pass

    def barrier(self):
        pass


class TorchComm:
    """torch.distributed broadcast (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def broadcast(self, buf, root):
        self.dist.broadcast(buf, src=root, group=self.group)
        if buf.is_cuda:
            import torch
            torch.cuda.current_stream().synchronize()
        return buf

    def ibroadcast(self, buf, root):
        """Start a broadcast (NCCL: on its own stream, so the sender's next
        kernels overlap it); wait() before reading the buffer."""
        return (self.dist.broadcast(buf, src=root, group=self.group,
                                    async_op=True), buf)

    def wait(self, handle):
        if handle is None:
            return
        work, buf = handle
        work.wait()
        if buf.is_cuda:
            import torch
            torch.cuda.current_stream().synchronize()

    def barrier(self):
        self.dist.barrier(group=self.group)


class DeviceBackend:
    """Local blocks and panel buffers as torch CUDA tensors (planar
    (k, rows, cols) float64), compute through libmpcore."""

    def __init__(self, k, device=None):
        import torch
        self.torch = torch
        self.k = k
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.L = nat.lib()

    # -- storage -----------------------------------------------------------
    def alloc(self, rows, cols):
        return self.torch.zeros((self.k, rows, cols), dtype=self.torch.float64,
                                device=self.device)

    def view(self, M, row0=0, col0=0):
        """(base address, ld, plane) of element (row0, col0)."""
        k, rows, cols = M.shape
        return (M.data_ptr() + (row0 * cols + col0) * 8, cols, rows * cols)

    def to_host(self, M):
        return M.cpu().numpy()

    def int_buffer(self, n):
        return self.torch.zeros(n, dtype=self.torch.int32, device=self.device)

    def ints_to_host(self, t):
        return t.cpu().numpy()

    def ints_from_host(self, t, arr):
        t.copy_(self.torch.from_numpy(np.ascontiguousarray(arr, np.int32)))

    # -- compute -----------------------------------------------------------
    def sync(self):
        self.torch.cuda.current_stream().synchronize()

    def generate(self, M, layout, rank, slot, seed):
        if M.numel() == 0:          # a rank without blocks (world > nblocks)
            return
        base, ld, plane = self.view(M)
        self.sync()
        nat.check(self.L.mpcore_dev_generate_cyclic(
            self.k, base, ld, plane, M.shape[1], M.shape[2], layout.nb,
            layout.world, rank, slot, layout.n, seed), "generate_cyclic")

    def lu_block(self, M, row0, col0, width):
        """Factor rows [row0, n) x cols [col0, col0+width) in place; returns
        the swaps as absolute row indices."""
        base, ld, plane = self.view(M, row0, col0)
        m = M.shape[1] - row0
        sw = np.zeros(width, dtype=np.int32)
        step = nat._i32(-1)
        self.sync()
        st = self.L.mpcore_dev_lu_block(self.k, m, width, base, ld, plane, 0,
                                        nat.iptr(sw), nat.ctypes.byref(step))
        if st == nat.SINGULAR:
            raise SingularMatrixError(
                "no nonzero pivot at elimination step %d" % (row0 + step.value),
                step=row0 + step.value)
        nat.check(st, "lu_block")
        return sw + row0

    def pack(self, M, row0, col0, width, buf):
        rows = M.shape[1] - row0
        dst = buf[:, :rows, :width]
        base_d, ldd, pd = buf.data_ptr(), buf.shape[2], buf.shape[1] * buf.shape[2]
        base_s, lds, ps = self.view(M, row0, col0)
        self.sync()
        nat.check(self.L.mpcore_dev_copy2d(self.k, rows, width, base_d, ldd,
                                           pd, base_s, lds, ps), "copy2d")
        return dst

    def laswp(self, M, col0, ncols, row0, swaps):
        if ncols <= 0:
            return
        base, ld, plane = self.view(M)
        sw = np.ascontiguousarray(swaps, dtype=np.int32)
        self.sync()
        nat.check(self.L.mpcore_dev_laswp(self.k, base, ld, plane, col0, ncols,
                                          row0, nat.iptr(sw), len(sw)),
                  "laswp")

    def trsm(self, buf, w, M, row0, col0, ncols):
        bl, ldl, pl = buf.data_ptr(), buf.shape[2], buf.shape[1] * buf.shape[2]
        bu, ldu, pu = self.view(M, row0, col0)
        self.sync()
        nat.check(self.L.mpcore_dev_trsm(self.k, w, ncols, bl, ldl, pl, bu,
                                         ldu, pu), "trsm")

    def gemm_update(self, buf, w, M, row0, col0, ncols):
        mrows = M.shape[1] - row0 - w
        if mrows <= 0 or ncols <= 0:
            return
        ldb, pb = buf.shape[2], buf.shape[1] * buf.shape[2]
        a = buf.data_ptr() + (w * ldb) * 8            # L21: rows w.. of buf
        bu, ldu, pu = self.view(M, row0, col0)         # U12
        bc, ldc, pc = self.view(M, row0 + w, col0)     # A22
        self.sync()
        nat.check(self.L.mpcore_dev_gemm(self.k, 1, 0, mrows, ncols, w, a, ldb,
                                         pb, bu, ldu, pu, bc, ldc, pc),
                  "gemm_update")


def _local_ranges(layout, rank, P):
    """Local column ranges of `rank` outside panel P's block."""
    lc = layout.local_cols(rank)
    if layout.owner(P) != rank:
        return [(0, lc)]
    off = layout.local_offset(rank, P)
    w = layout.width(P)
    return [(0, off), (off + w, lc - off - w)]


def dist_lu_factor(backend, comm, layout, local, lookahead=True):
    """Factor the distributed matrix in place.

    local: {rank: local block (backend storage)} for the ranks this process
    serves (all of them under LocalComm).  Returns the global swap list
    (swaps[j] = r, the reference's PivotRecord.swaps, linalg.py:348-354).
    Raises SingularMatrixError(step) on every rank alike.

    Look-ahead: while applying panel P, the owner of panel
    P+1 first brings that block up to date (exchanges, U12, update of its
    columns only), factors it and starts its broadcast, and only then runs
    the bulk of its update for P -- so the next panel travels while every
    rank updates.  Only the order across column blocks changes; each
    element's chain is the same, so the result is identical either way.
    """
    n, G = layout.n, layout.world
    nbk = layout.nblocks
    swaps_all = np.zeros(n, dtype=np.int32)
    bufs = [backend.alloc(n, layout.nb), backend.alloc(n, layout.nb)]
    ibufs = [backend.int_buffer(layout.nb + 1),
             backend.int_buffer(layout.nb + 1)]

    def factor_pack(P, slot):
        """Owner of P: factor its block, pack it, stage pivots + status."""
        J, w, owner = P * layout.nb, layout.width(P), layout.owner(P)
        M = local[owner]
        off = layout.local_offset(owner, P)
        status = np.zeros(layout.nb + 1, dtype=np.int32)
        try:
            status[:w] = backend.lu_block(M, J, off, w)
            status[layout.nb] = -1
        except SingularMatrixError as e:
            status[layout.nb] = e.step
        backend.pack(M, J, off, w, bufs[slot])
        backend.ints_from_host(ibufs[slot], status)

    def send(P, slot):
        """Every rank, in panel order: start P's broadcasts."""
        owner = layout.owner(P)
        return (comm.ibroadcast(ibufs[slot], owner),
                comm.ibroadcast(bufs[slot], owner))

    def update(M, rank, P, sw, buf, c0, nc, exchange_ranges):
        """Panel P applied to local columns: exchanges on the given ranges,
        then U12 and the trailing update on [c0, c0 + nc)."""
        J, w = P * layout.nb, layout.width(P)
        for a, m in exchange_ranges:
            backend.laswp(M, a, m, J, sw)
        if nc > 0:
            backend.trsm(buf, w, M, J, c0, nc)
            backend.gemm_update(buf, w, M, J, c0, nc)

    if layout.owner(0) in local:
        factor_pack(0, 0)
    pending = send(0, 0)
    for P in range(nbk):
        J, w = P * layout.nb, layout.width(P)
        slot = P % 2
        comm.wait(pending[0])
        status = backend.ints_to_host(ibufs[slot])
        if status[layout.nb] >= 0:
            raise SingularMatrixError(
                "no nonzero pivot at elimination step %d" % status[layout.nb],
                step=int(status[layout.nb]))
        comm.wait(pending[1])
        buf = bufs[slot]
        sw = status[:w].copy()
        swaps_all[J:J + w] = sw
        nxt = P + 1 < nbk
        # (one rank has nobody to overlap with: keep the launches fewer)
        ahead = lookahead and nxt and G > 1
        if ahead:
            # the next panel's owner: that block first, then factor + send
            o1 = layout.owner(P + 1)
            if o1 in local:
                M = local[o1]
                off1, w1 = layout.local_offset(o1, P + 1), layout.width(P + 1)
                update(M, o1, P, sw, buf, off1, w1, [(off1, w1)])
                factor_pack(P + 1, 1 - slot)
            pending = send(P + 1, 1 - slot)
        for rank, M in local.items():
            t0 = layout.trailing_start(rank, P)
            nt = layout.local_cols(rank) - t0
            ranges = _local_ranges(layout, rank, P)
            if ahead and rank == layout.owner(P + 1):
                # block P+1 (the first trailing block) is already done
                w1 = layout.width(P + 1)
                ranges = _split_out(ranges, t0, w1)
                t0, nt = t0 + w1, nt - w1
            update(M, rank, P, sw, buf, t0, nt, ranges)
        if nxt and not ahead:
            if layout.owner(P + 1) in local:
                factor_pack(P + 1, 1 - slot)
            pending = send(P + 1, 1 - slot)
    return swaps_all


def _split_out(ranges, a0, m0):
    """Column ranges minus [a0, a0 + m0)."""
    out = []
    for a, m in ranges:
        b = a + m
        if b <= a0 or a >= a0 + m0:
            if m > 0:
                out.append((a, m))
            continue
        if a < a0:
            out.append((a, a0 - a))
        if b > a0 + m0:
            out.append((a0 + m0, b - a0 - m0))
    return out


# ------------------------------------------------------------------------
# The native driver (libmpcore dist.cu): the same protocol, device-ordered.
# The functions above are its executable specification on any backend
# (tests/test_dist_gloo.py runs them on CPU over gloo); the product path
# for BASELINE config 4 is dist_lu_solve below: one C-ABI call per solve,
# pivots on the device, the panel loop, broadcasts (live rows only),
# look-ahead and the column-cyclic back substitution all enqueued by the
# library on its own streams, ordered after / before the caller's stream.

DIST_PHASES = ("total", "factor", "bcast", "exch_trsm", "update", "back")


class NcclComm:
    """libmpcore's own NCCL communicator for this rank.  The unique id is
    drawn on rank 0 and shared through the caller's torch.distributed
    group (any backend; one small object broadcast at setup)."""

    def __init__(self, world, rank, group=None):
        uid = self.exchange_id(world, rank, group)
        h = nat._u64()
        nat.check(nat.lib().mpcore_dist_comm_init(world, rank, uid, 128,
                                                  ctypes.byref(h)),
                  "dist_comm_init")
        self.handle, self.world, self.rank = h.value, world, rank

    @staticmethod
    def exchange_id(world, rank, group=None):
        """Rank 0 draws the 128-byte NCCL unique id (mpcore_dist_unique_id)
        and every rank receives it over the torch.distributed group; ->
        bytes."""
        obj = [None]
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            nat.check(nat.lib().mpcore_dist_unique_id(buf, 128),
                      "dist_unique_id")
            obj[0] = buf.raw
        if world > 1:
            import torch.distributed as dist
            dist.broadcast_object_list(obj, src=0, group=group)
        assert isinstance(obj[0], bytes) and len(obj[0]) == 128
        return obj[0]

    def close(self):
        if self.handle:
            nat.lib().mpcore_dist_comm_destroy(self.handle)
            self.handle = 0


def dist_lu_solve(layout, local, xs, k, comm=None, stream=None, phases=False):
    """Factor the distributed matrix and solve (one library call).

    local: {rank: device tensor (k, n, local_cols + 1)}, the last column
    holding b (every rank) -- y = L^-1 P b on exit; xs: {rank: device tensor
    (k, n)} receiving x.  comm: an NcclComm (this process serves its one
    rank) or None (every rank of the layout served here on one device).
    stream: the CUDA stream (int handle) the work is ordered after and that
    waits for it; default: torch's current stream (the legacy default
    stream is passed as cudaStreamLegacy).  Returns (swaps, phase_ms or
    None, launches); raises SingularMatrixError(step) like lu_factor_pp."""
    ranks = sorted(local)
    R = len(ranks)
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    if stream == 0:
        stream = 1          # cudaStreamLegacy: torch's legacy default stream
    arr = lambda t, vals: (t * R)(*vals)  # noqa: E731
    for r in ranks:
        M = local[r]
        assert M.shape[0] == k and M.shape[1] == layout.n
        assert M.shape[2] == layout.local_cols(r) + 1 and M.is_contiguous()
    rk = arr(ctypes.c_int32, ranks)
    bases = arr(nat._u64, [local[r].data_ptr() for r in ranks])
    lds = arr(ctypes.c_int64, [local[r].shape[2] for r in ranks])
    planes = arr(ctypes.c_int64, [local[r].shape[1] * local[r].shape[2]
                                  for r in ranks])
    cols = arr(ctypes.c_int32, [local[r].shape[2] for r in ranks])
    xp = arr(nat._u64, [xs[r].data_ptr() for r in ranks])
    swaps = np.zeros(layout.n, dtype=np.int32)
    step = nat._i32(-1)
    ph = (ctypes.c_double * len(DIST_PHASES))() if phases else None
    nl = ctypes.c_int64(0)
    st = nat.lib().mpcore_dist_lu_solve(
        comm.handle if comm is not None else 0, k, layout.n, layout.nb,
        layout.world, R, rk, bases, lds, planes, cols, xp, int(stream),
        nat.iptr(swaps), ctypes.byref(step),
        ctypes.cast(ph, nat._dp) if ph is not None else None,
        ctypes.byref(nl))
    if st == nat.SINGULAR:
        raise SingularMatrixError(
            "no nonzero pivot at elimination step %d" % step.value,
            step=step.value)
    nat.check(st, "dist_lu_solve")
    return (swaps, dict(zip(DIST_PHASES, list(ph))) if ph is not None
            else None, nl.value)
