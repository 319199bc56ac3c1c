"""Partitioned evaluate (pkgpu_evaluate_partitioned) across two PROCESSES: one
rank per process, torch.distributed over gloo (CUDA tensors; both processes share cuda:0
here -- the GPU box has one GPU -- and the collectives are host-side, so no kernel waits on
another process's kernel). The result must match the single-process evaluate."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_path):
    import torch.distributed as dist

    import paper_1705_02043_b200 as pk
    from test_gpu_partition import golden_req

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        req, _ = golden_req(name)
        ctx = pk.Context(0)
        comm = pk.TorchDistComm(device=0)
        res = pk.evaluate(req, context=ctx, comm=comm)
        np.save(out_path.format(rank=rank), res.potentials)
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["lap_sp_p8_clu", "sto_tp_p6"])
def test_partitioned_two_processes(name, tmp_path):
    import torch.multiprocessing as mp

    import paper_1705_02043_b200 as pk
    from test_gpu_partition import golden_req

    req, spread = golden_req(name)
    single = pk.evaluate(req).potentials
    out = str(tmp_path / "pot_{rank}.npy")
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    pots = [np.load(out.format(rank=r)) for r in range(2)]
    assert np.array_equal(pots[0], pots[1])  # every rank returns the full, identical result
    err = float(np.linalg.norm(pots[0] - single) / np.linalg.norm(single))
    print(f"{name} 2 processes: rel-L2 vs single process {err:.3e}")
    assert err <= max(1e-12, 3 * spread)
