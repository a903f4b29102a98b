"""GPU, two processes: the sharded solve's multi-process path (one shard per
process, push transport over CUDA IPC, coordination through a host all-gather
over torch.distributed gloo instead of NCCL) run as two ranks that share the
one GPU of this box. The iterates must be bit-identical to the single-device
engine. (NCCL cannot put two ranks on one GPU; the CUDA IPC stores, the
system-scope epoch flags and the cross-rank stop agreement are the same code
either way.)"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ITERS = 200


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _lp(kind):
    from paper_2510_24429_b200 import lpgen
    if kind == "staircase":
        return lpgen.staircase_lp(stages=16, cols_per_stage=200, rows_per_stage=100, seed=6)[0]
    return lpgen.random_equality_lp(1500, 6000, 8, seed=9)[0]


def _worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2510_24429_b200.pdhg import PdhgConfig, ShardedEngine
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allgather(blob: bytes):
        t = torch.frombuffer(bytearray(blob), dtype=torch.uint8) if blob else torch.zeros(0, dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [bytes(p.numpy().tobytes()) for p in parts]

    try:
        with ShardedEngine(_lp(kind), device=0, rank=rank, nranks=world,
                           host_allgather=allgather) as eng:
            res = eng.solve(PdhgConfig(max_iterations=ITERS))
            d = eng.describe()
        q.put((rank, res.iterate.x, res.iterate.y, res.iterations, d))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e), None, None, None))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["random", "staircase"])
def test_two_process_push_transport_bit_identical(kind):
    from paper_2510_24429_b200.pdhg import PdhgConfig, run_pdhg
    one = run_pdhg(_lp(kind), PdhgConfig(max_iterations=ITERS))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, x, y, its, d in outs:
        assert y is not None, x
        assert its == one.iterations
        assert np.array_equal(x, one.iterate.x), rank
        assert np.array_equal(y, one.iterate.y), rank
        assert d["shards"] == 2
        if kind == "staircase":
            assert d["halo_x"] and d["halo_y"]
