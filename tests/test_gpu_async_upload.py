"""mpcore_set_planes_async (the pipelined e2e path of bench.py): uploads on
their own stream, ordered before every later library call -- results are
those of the synchronous upload, bit for bit, including when the next
upload overlaps a running solve, and releasing an object with an upload in
flight is safe."""

import numpy as np
import pytest

import oracle
from oracle import gen
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                          device_solve_system)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,n", [(2, 200), (3, 257), (4, 96)])
def test_async_upload_pipelined_solves_match_oracle(k, n):
    seeds = [11, 12, 13]
    hosts = []
    for s in seeds:
        A = gen.planes(k, (n, n), 0, n, s)
        b = oracle.matvec(A, gen.planes(k, (n,), 2, n, s))
        hA = nat.PinnedBuffer((k, n, n))
        hA.array[...] = A
        hb = nat.PinnedBuffer((k, n))
        hb.array[...] = b
        lu, sw = oracle.lu(A)
        hosts.append((hA, hb, oracle.solve(lu, sw, b)))
    Es = [DeviceMatrix(k, n, n), DeviceMatrix(k, n, n)]
    bs = [DeviceVector(k, n), DeviceVector(k, n)]
    x = DeviceVector(k, n)
    nat.set_planes_async(Es[0].handle, hosts[0][0].array)
    nat.set_planes_async(bs[0].handle, hosts[0][1].array)
    for i in range(len(seeds)):
        if i + 1 < len(seeds):  # the next system uploads during this solve
            nat.set_planes_async(Es[(i + 1) % 2].handle, hosts[i + 1][0].array)
            nat.set_planes_async(bs[(i + 1) % 2].handle, hosts[i + 1][1].array)
        device_solve_system(Es[i % 2], bs[i % 2], x)
        assert x.download().tobytes() == hosts[i][2].tobytes()


def test_async_upload_then_release_and_reuse():
    k, n = 3, 128
    A = gen.planes(k, (n, n), 0, n, 5)
    hA = nat.PinnedBuffer((k, n, n))
    hA.array[...] = A
    M = DeviceMatrix(k, n, n)
    nat.set_planes_async(M.handle, hA.array)
    del M                             # released: the copy completes first
    M2 = DeviceMatrix(k, n, n)
    nat.set_planes_async(M2.handle, hA.array)
    assert M2.download().tobytes() == A.tobytes()
    with pytest.raises(ValueError):
        nat.set_planes_async(M2.handle, A[:, :, ::2])


@pytest.mark.parametrize("k,n", [(2, 130), (3, 64)])
def test_async_download_pipelined_products(k, n):
    # mat_mul with async uploads and downloads, two buffers per operand:
    # every product equals the oracle's, and rewriting a C whose download
    # is in flight waits for it
    L = nat.lib()
    systems = []
    for s in (3, 4, 5):
        A = gen.planes(k, (n, n), 0, n, s)
        B = gen.planes(k, (n, n), 1, n, s)
        hA, hB, hC = (nat.PinnedBuffer((k, n, n)) for _ in range(3))
        hA.array[...] = A
        hB.array[...] = B
        systems.append((hA, hB, hC, oracle.gemm(A, B)))
    EA = [DeviceMatrix(k, n, n) for _ in range(2)]
    EB = [DeviceMatrix(k, n, n) for _ in range(2)]
    EC = [DeviceMatrix(k, n, n) for _ in range(2)]
    for i, (hA, hB, hC, _) in enumerate(systems):
        nat.set_planes_async(EA[i % 2].handle, hA.array)
        nat.set_planes_async(EB[i % 2].handle, hB.array)
        nat.check(L.mpcore_mat_mul(EA[i % 2].handle, EB[i % 2].handle,
                                   EC[i % 2].handle), "mm")
        nat.get_planes_async(EC[i % 2].handle, hC.array)
    nat.sync()
    for hA, hB, hC, want in systems:
        assert hC.array.tobytes() == want.tobytes()
