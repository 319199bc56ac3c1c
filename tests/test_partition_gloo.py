"""N>1 host path on CPU: two gloo ranks drive the partition communicator exactly as
libpkgpu does (through the C callback pointers of pkgpu_partition): allocation, then an
in-place sum over ranks."""
import ctypes
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1705_02043_b200 as pk


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = pk.TorchDistComm(device="cpu")
        assert (comm.rank, comm.nranks) == (rank, world)
        comm.begin_call()
        part = pk._Partition(comm.rank, comm.nranks, comm.c_alloc, comm.c_allreduce, None)
        # what the library does: alloc, fill (each rank owns a disjoint slice), allreduce
        ptr = part.alloc(None, 10 * 8)
        buf = comm._bufs[ptr]
        buf.zero_()
        buf[rank * 5:(rank + 1) * 5] = torch.arange(5, dtype=torch.float64) + 100 * rank
        rc = part.allreduce(None, ptr, 10, None)
        q.put((rank, rc, buf.tolist(), comm.error is None))
        comm.end_call()
    finally:
        dist.destroy_process_group()


def test_partition_comm_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [0.0, 1.0, 2.0, 3.0, 4.0, 100.0, 101.0, 102.0, 103.0, 104.0]
    for rank, rc, buf, ok in res:
        assert rc == 0 and ok
        assert buf == expect


def test_partition_descriptor_layout():
    # pkgpu_partition: int rank, int nranks, alloc fn, allreduce fn, void* user, alltoallv fn, allgather fn
    assert ctypes.sizeof(pk._Partition) == 4 + 4 + 8 + 8 + 8 + 8 + 8


def _worker_v2(rank, world, port, q):
    """The halo (alltoallv) and modulus-split (allgather) callbacks through the C pointers."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = pk.TorchDistComm(device="cpu")
        comm.begin_call()
        part = pk._Partition(comm.rank, comm.nranks, comm.c_alloc, comm.c_allreduce, None, comm.c_alltoallv,
                             comm.c_allgather)
        # alltoallv: rank r sends (r + 1) * (q + 1) values 100 r + q to rank q
        sc = [(rank + 1) * (qq + 1) for qq in range(world)]
        rc = [(qq + 1) * (rank + 1) for qq in range(world)]
        sptr, rptr = part.alloc(None, 8 * sum(sc)), part.alloc(None, 8 * sum(rc))
        sb = comm._bufs[sptr]
        o = 0
        for qq in range(world):
            sb[o:o + sc[qq]] = 100 * rank + qq
            o += sc[qq]
        SC, RC = (ctypes.c_int64 * world)(*sc), (ctypes.c_int64 * world)(*rc)
        rc1 = part.alltoallv(None, sptr, SC, rptr, RC, None)
        got = comm._bufs[rptr][:sum(rc)].tolist()
        # allgather: 3 doubles per rank, block r = r + [0.25, 0.5, 0.75]
        gptr = part.alloc(None, 8 * 3 * world)
        gb = comm._bufs[gptr]
        gb.zero_()
        gb[3 * rank:3 * rank + 3] = torch.tensor([0.25, 0.5, 0.75], dtype=torch.float64) + rank
        rc2 = part.allgather(None, gptr, 24, None)
        q.put((rank, rc1, rc2, got, gb[:3 * world].tolist(), comm.error is None))
        comm.end_call()
    finally:
        dist.destroy_process_group()


def test_partition_halo_and_allgather_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_v2, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rc1, rc2, got, gath, ok in res:
        assert rc1 == 0 and rc2 == 0 and ok
        expect = []
        for src in range(2):
            expect += [100.0 * src + rank] * ((src + 1) * (rank + 1))
        assert got == expect
        assert gath == [0.25, 0.5, 0.75, 1.25, 1.5, 1.75]
