"""CPU tests of the slab-decomposition host logic (gloo, world size 2): row
partitioning, halo exchange of ghost rows and the Gram all-reduce, with the
same functions the GPU path uses (paper_2510_23221_b200/dd.py)."""
import os

import pytest
import torch
import torch.multiprocessing as mp

from paper_2510_23221_b200.dd import halo_exchange, partition_rows


@pytest.mark.parametrize("ny,world", [(512, 8), (512, 3), (40, 2), (7, 7)])
def test_partition_rows(ny, world):
    parts = partition_rows(ny, world)
    assert parts[0][0] == 0 and sum(n for _, n in parts) == ny
    for (y0, n), (y1, _) in zip(parts, parts[1:]):
        assert y0 + n == y1 and n >= 1
    assert max(n for _, n in parts) - min(n for _, n in parts) <= 1


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2510_23221_b200.dd import TorchComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nz, nx, S = 3, 5, 4
    parts = partition_rows(9, world)
    y0, nyl = parts[rank]
    # global field value = 1000*iz + 10*iy_global + ix + 0.01*col; ghost rows = -1
    v = torch.full((nz, nyl + 2, nx, S), -1.0, dtype=torch.float64)
    for iz in range(nz):
        for iyl in range(1, nyl + 1):
            for ix in range(nx):
                for c in range(S):
                    v[iz, iyl, ix, c] = 1000 * iz + 10 * (y0 + iyl - 1) + ix + 0.01 * c
    halo_exchange(v, nyl, rank, world, dist)

    class _S:
        pass

    sl = _S()
    sl.red = torch.arange(6, dtype=torch.float64) * (rank + 1)
    TorchComm().allreduce([sl], 4)
    # per-sample residual partials (num, den) of the slab-local outputs
    nd = torch.tensor([[1.0 + rank, 2.0 * (rank + 1)], [0.5, 0.25]], dtype=torch.float64)
    TorchComm().sum([nd])
    q.put((rank, y0, nyl, v.numpy().copy(), sl.red.numpy().copy(), nd.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_halo_and_allreduce_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, y0, nyl, v, red, nd in out:
        assert nd.tolist() == [[3.0, 6.0], [1.0, 0.5]]
        nz, _, nx, S = v.shape
        # ghost row 0 holds global row y0-1 (or stays -1 at the domain edge)
        for iz in range(nz):
            for ix in range(nx):
                lo = v[iz, 0, ix, 1]
                hi = v[iz, nyl + 1, ix, 1]
                assert lo == (-1.0 if y0 == 0 else 1000 * iz + 10 * (y0 - 1) + ix + 0.01)
                assert hi == (-1.0 if y0 + nyl == 9 else 1000 * iz + 10 * (y0 + nyl) + ix + 0.01)
        # first 4 entries summed over ranks (1 + 2) * i, the rest untouched
        assert list(red[:4]) == [3.0 * i for i in range(4)]
        assert red[4] == 4.0 * (rank + 1) and red[5] == 5.0 * (rank + 1)
