"""Multi-rank host logic on CPU (gloo, world_size 2): chip ownership and the
max-over-ranks timing reduction bench.py uses for N > 1."""
import os

import pytest
import torch.multiprocessing as mp

from paper_2510_23221_b200.sharding import chips_for_rank, owner_of_chip


@pytest.mark.parametrize("n,world", [(5000, 8), (5000, 3), (7, 2), (3, 4), (1, 1)])
def test_chip_partition_is_exact_and_contiguous(n, world):
    seen = []
    for r in range(world):
        rg = chips_for_rank(n, r, world)
        seen.extend(rg)
        for c in rg:
            assert owner_of_chip(c, n, world) == r
    assert seen == list(range(n))


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2510_23221_b200.sharding import chips_for_rank, max_over_ranks, sum_over_ranks

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    chips = chips_for_rank(10, rank, world)
    t = max_over_ranks(1.0 + rank)          # per-rank device time
    tot = sum_over_ranks(len(chips))
    q.put((rank, list(chips), t, tot))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] == [0, 1, 2, 3, 4] and out[1][1] == [5, 6, 7, 8, 9]
    assert out[0][2] == out[1][2] == 2.0       # max over ranks
    assert out[0][3] == out[1][3] == 10.0      # every chip owned exactly once
