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


# ------------------------------------------------ lookahead loop (host logic)
class _FakeDevice:
    """In-order model of one rank's stream for dd_block_cg's host loops: the
    control word (cmd, sa) as the control kernels set it, BK_DD_GATED steps
    skipped while a verification is pending, and a log of the steps that
    actually ran. Verifications are scripted: ctl_update at iteration m asks
    for one when m is in `verify_at`; the verification then restarts
    (m in `restart_at`), finishes (m in `done_at`) or continues."""

    def __init__(self, S, verify_at, restart_at, done_at):
        from paper_2510_23221_b200 import dd

        self.dd = dd
        self.S = S
        self.verify_at, self.restart_at, self.done_at = verify_at, restart_at, done_at
        self.cmd, self.sa, self.m, self.iters = 0, S, 0, 0
        self.log = []

    def step(self, kind, m):
        dd = self.dd
        gated = bool(kind & dd.GATED)
        kind &= ~dd.GATED
        if gated and self.cmd != dd.CMD_PUPDATE:
            return
        if kind in (dd.READ, dd.READ_ASYNC):
            return
        self.log.append((kind, m if kind == dd.CTL_UPDATE else 0))
        if kind == dd.CTL_INIT:
            self.cmd, self.sa = dd.CMD_PUPDATE, self.S
        elif kind == dd.CTL_UPDATE:
            self.m = self.iters = m
            self.cmd = dd.CMD_VERIFY if m in self.verify_at else dd.CMD_PUPDATE
        elif kind == dd.CTL_VERIFY:
            if self.m in self.done_at:
                self.cmd, self.sa = dd.CMD_DONE, 0
            elif self.m in self.restart_at:
                self.cmd = dd.CMD_RESTART
            else:
                self.cmd, self.sa = dd.CMD_PUPDATE, self.sa - 1
        elif kind == dd.CTL_RESTART:
            self.cmd = dd.CMD_PUPDATE


def _run_fake_loop(monkeypatch, lookahead, deferred, max_iter, verify_at, restart_at, done_at):
    import ctypes as C
    from types import SimpleNamespace

    import paper_2510_23221_b200 as bk_real
    from paper_2510_23221_b200 import dd

    S = 16
    dev = _FakeDevice(S, verify_at, restart_at, done_at)

    class Lib:
        def bk_dd_deferred_x(self, h, S_):
            return int(deferred)

    fbk = SimpleNamespace(_load=lambda: Lib(), _Report=bk_real._Report,
                          SolveReport=bk_real.SolveReport)

    class Slab:
        bk = fbk
        op = SimpleNamespace(h=None)

        def __init__(self):
            self.S = S

        def step(self, kind, cfg_c, m=0, report=None):
            dev.step(kind, m)
            if kind == dd.CTL_FINAL and report is not None:
                report._obj.iterations = dev.iters
            return dev.cmd, dev.sa

    class Slots:
        def __init__(self, n):
            self.words = {}

        def post(self, slabs, cfg_c, m):
            self.words[m & 1] = (dev.cmd, dev.sa)  # the stream reaches the copy now

        def wait(self, m):
            return self.words[m & 1]

    class Comm:
        def allreduce(self, slabs, count):
            pass

        def halo(self, slabs, name):
            pass

    monkeypatch.setattr(dd, "_on_torch_stream", lambda slabs: None)
    monkeypatch.setattr(dd, "_ControlSlots", Slots)
    cfg = SimpleNamespace(max_iter=max_iter, _c=lambda: None)
    rep = dd.dd_block_cg([Slab()], Comm(), cfg, lookahead=lookahead)
    return dev.log, rep.iterations


@pytest.mark.parametrize("deferred", [True, False])
@pytest.mark.parametrize("script", [
    (40, {7, 19, 33}, {19}, {33}),      # verify, restart, done
    (12, {5}, set(), set()),            # iteration cap reached
    (12, {12}, set(), set()),           # verification on the last allowed iteration
    (30, {1, 2, 3}, {2}, {3}),          # back-to-back verifications
    (1, set(), set(), set()),           # a single iteration
])
def test_lookahead_loop_runs_the_synchronous_steps(monkeypatch, deferred, script):
    """dd_block_cg(lookahead=True) enqueues iteration m + 1 as BK_DD_GATED steps
    before reading m's control word; the steps that actually execute (gated
    ones are skipped while a verification is pending) are exactly those of the
    synchronous loop, in the same order, with the same iteration count."""
    max_iter, v, r, d = script
    sync_log, sync_it = _run_fake_loop(monkeypatch, False, deferred, max_iter, v, r, d)
    look_log, look_it = _run_fake_loop(monkeypatch, True, deferred, max_iter, v, r, d)
    assert look_log == sync_log
    assert look_it == sync_it
