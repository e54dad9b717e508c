"""Two processes, one GPU: the CUDA-IPC plumbing of the multi-GPU slab path.

Each process builds its rank's context (``assemble(grid, rank=r, nranks=2)``),
the 64-byte arena handles are exchanged over a gloo group (``connect_ranks``)
and every rank maps the other's arena (``vs_ipc_attach``: cudaIpcOpenMemHandle,
arena layout, peer pointers, the shared barrier counter).  Nothing is SOLVED
here: the fused kernels of the two ranks would wait on one another, and
separate launches that wait on one another are not guaranteed to be
co-resident on one GPU (profiling guide) -- the data path itself is covered
by the emulated-rank tests (one cooperative launch over all ranks' data) and
by the gloo CPU test of the schedule.  What this test pins is that the
handles, the arena sizes and the mapping agree between processes.
"""
import os
import socket

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fluid, q):
    import torch.distributed as dist

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import paper_2307_05266_b200 as vx

        s = vx.assemble(vx.VoxelGrid(fluid), 0, device=0, rank=rank, nranks=world)
        vx.connect_ranks(s)
        dist.barrier()
        out = (rank, s.m_u, s.m_p, s.rank, s.nranks)
        del s
        dist.barrier()
        dist.destroy_process_group()
        q.put(("ok", out))
    except BaseException as e:  # noqa: BLE001
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}"))


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_handles_attach_between_processes(world):
    import torch.multiprocessing as mp

    g = load_golden("spheres3d")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, g["fluid"], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    bad = [r for r in res if r[0] != "ok"]
    assert not bad, bad
    outs = sorted(r[1] for r in res)
    assert [o[0] for o in outs] == list(range(world))
    assert len({(o[1], o[2]) for o in outs}) == 1  # every rank reports the global sizes
    assert all(o[4] == world for o in outs)
