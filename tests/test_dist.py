"""Multi-process (gloo, world_size 2) checks of the sharding / timing plumbing on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_01239_b200 import dist as fdist


def test_shard_range_partition():
    for total in (0, 1, 7, 65536, 16384, 8):
        for world in (1, 2, 3, 4, 8):
            spans = [fdist.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        fdist.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = fdist.shard_range(65536, rank, world)
    # each rank "generates" its shard from (seed, global index): check disjointness via a sum
    idx = torch.arange(b, e, dtype=torch.float64)
    total = fdist.sum_over_ranks(float(idx.sum()))
    mx = fdist.max_over_ranks(10.0 * (rank + 1))
    seeds = [fdist.instance_seed(0, r) for r in range(world)]
    dist.barrier()
    q.put((rank, b, e, total, mx, seeds))
    dist.destroy_process_group()


def test_gloo_world2_sharding_and_timing_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0][1:3] == (0, 32768) and res[1][1:3] == (32768, 65536)
    assert all(r[3] == 65536 * 65535 / 2 for r in res)
    assert all(r[4] == 20.0 for r in res)
    assert res[0][5] == [0, 1]
