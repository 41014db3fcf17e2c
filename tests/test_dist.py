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


def _bench_worker(rank, world, port, q):
    """The bench's rank loop on CPU: instances_for_rank -> per-rank 'steps' -> fdist.summarize (the
    exact reduction / all_gather code bench.py calls)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = fdist.instances_for_rank(8, rank, world)
    times = [10.0 * (rank + 1)] * 3            # ms per step; rank world-1 is the slowest
    s = fdist.summarize(times, len(inst), {"rank": rank, "instances": inst, "branch_b": rank}, device=None)
    q.put((rank, s))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_bench_summarize_and_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for rank, s in res:
        # max over ranks of the per-rank total, sum of units, whole-job value
        assert s["total_ms"] == 30.0 * world
        assert s["units_all"] == 8
        assert abs(s["value"] - 8 * 3 / (30.0 * world / 1e3)) < 1e-9
        assert abs(s["ms_per_step"] - 10.0 * world) < 1e-12
        # every rank holds every rank's record, in rank order
        assert [r["rank"] for r in s["per_rank"]] == list(range(world))
        got = sorted(i for r in s["per_rank"] for i in r["instances"])
        assert got == list(range(8))                       # 8/k instances per rank, disjoint, complete
        assert all(len(r["instances"]) == 8 // world for r in s["per_rank"])
        assert [r["branch_b"] for r in s["per_rank"]] == list(range(world))
        assert [r["elapsed_ms"] for r in s["per_rank"]] == [30.0 * (r + 1) for r in range(world)]
