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
    # pkgpu_partition: int rank, int nranks, alloc fn, allreduce fn, void* user
    assert ctypes.sizeof(pk._Partition) == 4 + 4 + 8 + 8 + 8
