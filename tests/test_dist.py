"""Multi-process (world_size 2, gloo, CPU) check of bench.py's N>1 plumbing:
per-rank sketch-column sharding (distinct seeds / blocks), barrier, and the
max-over-ranks timing used for the whole-job value."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    from paper_2401_15758_b200 import api

    dist = bench.dist_init(world, backend="gloo")
    seed = bench.rank_seed(rank)
    block = api.gaussian_matrix(64, 3, seed)
    ms = 10.0 + 5.0 * rank  # rank-specific "timing"
    bench.dist_barrier(dist)
    ms_max = bench.dist_max(dist, ms)
    value = world * 3 * 2 / (ms_max / 1000.0)
    q.put((rank, seed, block.sum(), ms_max, value))
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert res[0][1] != res[1][1]  # distinct per-rank sketch blocks
    assert res[0][2] != res[1][2]
    assert res[0][3] == res[1][3] == 15.0  # max over ranks
    assert np.isclose(res[0][4], 2 * 3 * 2 / 0.015)
