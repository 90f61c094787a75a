"""World-size-2 checks of bench.py's multi-GPU host logic on CPU (gloo): the
query shards of the ranks are disjoint seeded streams, the step time is the max
over ranks, and the job rate counts every rank's queries (weak scaling, no
data-path collective)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import workloads
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 1000, 40)
    Q = bench.rank_queries(cfg, 40, rank)
    local_ms = 10.0 + 5.0 * rank                      # rank 1 is the slow one
    ms = bench.max_over_ranks(local_ms, dist)
    rate = bench.whole_job_rate(40, world, ms)
    # gather the shards to rank 0 to check disjointness
    t = torch.from_numpy(Q.copy())
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    if rank == 0:
        out.put((ms, rate, [g.numpy() for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ms, rate, shards = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ms == 15.0                                  # max over ranks
    assert rate == pytest.approx(2 * 40 / 0.015)       # all ranks' queries / slowest time
    a, b = shards
    assert a.shape == b.shape == (40, 64)
    assert not np.any(np.all(a[:, None, :] == b[None, :, :], axis=-1))   # disjoint streams
    np.testing.assert_allclose(np.linalg.norm(a, axis=1), 1.0, rtol=1e-5)
