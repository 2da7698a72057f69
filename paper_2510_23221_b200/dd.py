"""y-slab domain decomposition of the block-CG basis solve (BASELINE config 5).

The grid's y rows are split into contiguous slabs, one per rank (GPU). Every
rank assembles the GLOBAL operator (identical bits everywhere) and keeps its
slab of the block vectors in the slab-local layout nx x (nyl + 2) x nz x S with
one ghost row on each y side. The per-phase kernels (C ABI ``bk_dd_step``) run
in lockstep; between phases the driver

* all-reduces the s x s Gram partials (``red``) after every sweep — the only
  reductions of the algorithm (2 per iteration, <= S*S + S doubles), and
* refreshes the ghost rows of P before the stencil sweep (and of X before the
  rare true-residual / restart sweeps): one row per z-plane and neighbour.

Communicators:

* ``TorchComm`` — one slab per process, ``torch.distributed`` (NCCL on GPUs:
  all_reduce for the Gram data, batched isend/irecv for the halo rows over
  NVLink), rank r owns slab r.
* ``LocalComm`` — several virtual slabs in ONE process on one GPU: the
  all-reduce is a fixed-order sum of the slabs' ``red`` buffers and the halo a
  device copy. Kernels never wait on each other (phases are separate
  launches), so this is how the decomposition is validated on a single GPU.

The control decisions (convergence, freeze, restart) are computed by every
rank's control kernel from the same all-reduced data, so they agree.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

INIT_SWEEP, CTL_INIT, SPMM, CTL_ALPHA, UPDATE, CTL_UPDATE, TRUE_RES, CTL_VERIFY, \
    RESTART_SWEEP, CTL_RESTART, PUPDATE, CTL_FINAL, READ, UPDATE_D, PUPDATE_X, APPLY_X, \
    READ_ASYNC = range(17)
GATED = 0x100  # BK_DD_GATED: the kernels run only while no verification is pending
CMD_PUPDATE, CMD_VERIFY, CMD_RESTART, CMD_DONE = range(4)


def partition_rows(ny: int, world: int) -> List[tuple]:
    """Contiguous balanced y-slabs: [(y0, nyl)] for ranks 0..world-1."""
    if world < 1 or world > ny:
        raise ValueError("need 1 <= world <= ny")
    out = []
    for r in range(world):
        lo = r * ny // world
        hi = (r + 1) * ny // world
        out.append((lo, hi - lo))
    return out


def kernel_width(s: int) -> int:
    return 16 if s <= 16 else 32 if s <= 32 else 64


class _Bufs(C.Structure):
    _fields_ = [("B", C.c_void_p), ("X", C.c_void_p), ("R", C.c_void_p), ("P", C.c_void_p),
                ("W", C.c_void_p), ("part", C.c_void_p), ("red", C.c_void_p),
                ("ctl", C.c_void_p), ("nb", C.c_int)]


@dataclass
class Slab:
    """One rank's share: rows [y0, y0 + nyl) of the global grid."""
    bk: object
    ctx: object
    op: object
    y0: int
    nyl: int
    S: int
    B: object = None
    X: object = None
    R: object = None
    P: object = None
    W: object = None
    part: object = None
    red: object = None
    ctl: object = None
    nb: int = 0

    def allocate(self):
        import torch

        lib = self.bk._load()
        le, nb, pe, re_, cb = C.c_int64(), C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        self.bk._raise(lib.bk_dd_sizes(self.ctx.h, self.op.h, self.nyl, self.S, C.byref(le),
                                       C.byref(nb), C.byref(pe), C.byref(re_), C.byref(cb)),
                       self.ctx.h, "dd_sizes")
        dev = torch.device("cuda", self.ctx.device)
        shape = (self.op.grid.nz, self.nyl + 2, self.op.grid.nx, self.S)
        z = lambda: torch.zeros(shape, dtype=torch.float64, device=dev)  # noqa: E731
        self.B, self.X, self.R, self.P, self.W = z(), z(), z(), z(), z()
        self.part = torch.zeros(pe.value, dtype=torch.float64, device=dev)
        self.red = torch.zeros(re_.value, dtype=torch.float64, device=dev)
        self.ctl = torch.zeros(cb.value, dtype=torch.uint8, device=dev)
        self.nb = nb.value
        self._bufs = _Bufs(self.B.data_ptr(), self.X.data_ptr(), self.R.data_ptr(),
                           self.P.data_ptr(), self.W.data_ptr(), self.part.data_ptr(),
                           self.red.data_ptr(), self.ctl.data_ptr(), self.nb)
        return self

    def load_rhs(self, B_global):
        """Pack this slab's rows of a global n x S device block into B."""
        lib = self.bk._load()
        self.bk._raise(lib.bk_dd_pack(self.ctx.h, self.op.h, self.y0, self.nyl, self.S,
                                      C.c_void_p(B_global.data_ptr()),
                                      C.c_void_p(self.B.data_ptr()), 1), self.ctx.h, "dd_pack")

    def store_x(self, X_global):
        lib = self.bk._load()
        self.bk._raise(lib.bk_dd_pack(self.ctx.h, self.op.h, self.y0, self.nyl, self.S,
                                      C.c_void_p(X_global.data_ptr()),
                                      C.c_void_p(self.X.data_ptr()), 0), self.ctx.h, "dd_pack")

    def load_x(self, X_global):
        """Pack this slab's rows of a global n x S device block into X."""
        lib = self.bk._load()
        self.bk._raise(lib.bk_dd_pack(self.ctx.h, self.op.h, self.y0, self.nyl, self.S,
                                      C.c_void_p(X_global.data_ptr()),
                                      C.c_void_p(self.X.data_ptr()), 1), self.ctx.h, "dd_pack")

    def combine_action(self, coef, T, Q, nd):
        """Slab-local combine + operator action (bk_dd_combine_action) of every
        sample in coef (s x N device tensor) on this slab's rows; X's ghost rows
        must hold the neighbours' edge rows (one X halo exchange after the
        solve). T, Q: N x (nx nyl nz) device; nd: N x 2 residual partials."""
        lib = self.bk._load()
        s, N = int(coef.shape[0]), int(coef.shape[1])
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        self.bk._raise(lib.bk_dd_combine_action(self.ctx.h, self.op.h, self.y0, self.nyl, self.S,
                                                C.c_void_p(self.X.data_ptr()), s, ptr(coef), N,
                                                ptr(T), ptr(Q), ptr(nd)),
                       self.ctx.h, "dd_combine_action")

    def cells(self) -> int:
        return self.op.grid.nx * self.nyl * self.op.grid.nz

    def step(self, kind, cfg_c, m=0, report=None):
        lib = self.bk._load()
        cmd, sa = C.c_int(-1), C.c_int(-1)
        st = lib.bk_dd_step(self.ctx.h, self.op.h, self.y0, self.nyl, self.S,
                            C.byref(self._bufs), C.byref(cfg_c), kind, m, C.byref(cmd),
                            C.byref(sa), report)
        self.bk._raise(st, self.ctx.h, f"dd_step({kind})")
        return cmd.value, sa.value


def _red_count(kind: int, S: int) -> int:
    kind &= ~GATED
    return {INIT_SWEEP: S * S + S, SPMM: S * S, UPDATE: S * S + S, UPDATE_D: S * S + S,
            TRUE_RES: S, RESTART_SWEEP: S * S + S}[kind]


class LocalComm:
    """Virtual ranks in one process (one GPU): fixed-order sums and device copies."""

    def sum(self, tensors):
        """Sum one tensor per slab in slab order; every slab gets the total."""
        total = tensors[0].clone()
        for t in tensors[1:]:
            total += t
        for t in tensors:
            t.copy_(total)

    def allreduce(self, slabs, count):
        total = slabs[0].red[:count].clone()
        for sl in slabs[1:]:
            total += sl.red[:count]
        for sl in slabs:
            sl.red[:count].copy_(total)

    def halo(self, slabs, name):
        for r, sl in enumerate(slabs):
            v = getattr(sl, name)
            if r > 0:  # ghost row 0 <- last interior row of the slab below
                v[:, 0].copy_(getattr(slabs[r - 1], name)[:, slabs[r - 1].nyl])
            if r + 1 < len(slabs):  # ghost row nyl+1 <- first interior row above
                v[:, sl.nyl + 1].copy_(getattr(slabs[r + 1], name)[:, 1])


class TorchComm:
    """One slab per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce(self, slabs, count):
        (sl,) = slabs
        buf = sl.red[:count]
        self.dist.all_reduce(buf, op=self.dist.ReduceOp.SUM, group=self.group)

    def sum(self, tensors):
        (t,) = tensors
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def halo(self, slabs, name):
        (sl,) = slabs
        halo_exchange(getattr(sl, name), sl.nyl, self.rank, self.world, self.dist, self.group)


def halo_exchange(v, nyl, rank, world, dist, group=None):
    """v: (nz, nyl + 2, nx, S). Sends interior rows 1 and nyl to the neighbours,
    receives their boundary rows into ghost rows nyl + 1 and 0."""
    ops, recv = [], []
    if rank > 0:
        send_lo = v[:, 1].contiguous()
        recv_lo = torch_empty_like(send_lo)
        ops.append(dist.P2POp(dist.isend, send_lo, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_lo, rank - 1, group))
        recv.append((0, recv_lo))
    if rank + 1 < world:
        send_hi = v[:, nyl].contiguous()
        recv_hi = torch_empty_like(send_hi)
        ops.append(dist.P2POp(dist.isend, send_hi, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_hi, rank + 1, group))
        recv.append((nyl + 1, recv_hi))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for row, buf in recv:
        v[:, row].copy_(buf)


def torch_empty_like(t):
    import torch

    return torch.empty_like(t)


def _on_torch_stream(slabs):
    """The slab steps interleave library kernels with torch ops on the same
    buffers (halo copies, partial sums, zero fills): launch them on torch's
    current stream so they are ordered (a context's own stream is
    non-blocking with respect to torch's)."""
    import torch

    cs = torch.cuda.current_stream().cuda_stream
    for sl in slabs:
        sl.ctx.set_stream(cs)


class _ControlSlots:
    """Pinned host words for BK_DD_READ_ASYNC: two slots (iterations m and
    m + 1 in flight), each (cmd, sa) per slab plus the event that marks the
    copies done."""

    def __init__(self, nslabs):
        import torch

        self.words = [torch.zeros((nslabs, 2), dtype=torch.int32).pin_memory() for _ in range(2)]
        self.events = [None, None]

    def post(self, slabs, cfg_c, m):
        import torch

        w = self.words[m & 1]
        for i, sl in enumerate(slabs):
            lib = sl.bk._load()
            ptr = w.data_ptr() + 8 * i
            st = lib.bk_dd_step(sl.ctx.h, sl.op.h, sl.y0, sl.nyl, sl.S, C.byref(sl._bufs),
                                C.byref(cfg_c), READ_ASYNC, m, C.c_void_p(ptr),
                                C.c_void_p(ptr + 4), None)
            sl.bk._raise(st, sl.ctx.h, "dd_step(READ_ASYNC)")
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.events[m & 1] = ev

    def wait(self, m):
        self.events[m & 1].synchronize()
        vals = [tuple(int(v) for v in row) for row in self.words[m & 1].tolist()]
        assert all(v == vals[0] for v in vals), "ranks disagree on control state"
        return vals[0]


def dd_block_cg(slabs, comm, cfg, report_arrays=True, lookahead=True):
    """Run the decomposed block CG over `slabs` (lockstep). Returns the report
    of slab 0 (every rank's control state is identical).

    lookahead: iteration m + 1 is enqueued (BK_DD_GATED kernels, halo and
    all-reduces) before the host waits for iteration m's control word, read
    asynchronously into pinned memory — the device never drains between
    iterations. A verification due at m turns the enqueued m + 1 into no-ops
    (the gate), the host runs the verification and re-issues m + 1: the same
    kernel sequence on the same data as the synchronous loop (lookahead=False),
    so bitwise the same X."""
    bk = slabs[0].bk
    S = slabs[0].S
    cfg_c = cfg._c()
    _on_torch_stream(slabs)

    def all_step(kind, m=0):
        out = None
        for sl in slabs:
            out = sl.step(kind, cfg_c, m)
        if kind & ~GATED in (INIT_SWEEP, SPMM, UPDATE, UPDATE_D, TRUE_RES, RESTART_SWEEP):
            comm.allreduce(slabs, _red_count(kind, S))
        return out

    def read():
        vals = [sl.step(READ, cfg_c) for sl in slabs]
        assert all(v == vals[0] for v in vals), "ranks disagree on control state"
        return vals[0]

    # S = 64 on 16-aligned x: the single-GPU engine's warp-specialised sweeps
    # with X += P alpha deferred into the P update (bk_dd_deferred_x)
    lib = bk._load()
    deferred = bool(lib.bk_dd_deferred_x(slabs[0].op.h, S))
    all_step(INIT_SWEEP)
    all_step(CTL_INIT)
    cmd, sa = read()
    if lookahead:
        _pipelined_iterations(slabs, comm, cfg, cfg_c, all_step, read, deferred, sa)
    else:
        _synchronous_iterations(slabs, comm, cfg, all_step, read, deferred, sa)
    _, sa = read()
    if sa > 0:
        comm.halo(slabs, "X")
        all_step(TRUE_RES)
    res = np.zeros(S, np.float64)
    conv = np.zeros(S, np.int8)
    rep = bk._Report(0, 0, 0.0, res.ctypes.data_as(C.c_void_p), conv.ctypes.data_as(C.c_void_p))
    for i, sl in enumerate(slabs):
        sl.step(CTL_FINAL, cfg_c, 0, C.byref(rep) if i == 0 else None)
    return bk.SolveReport(iterations=rep.iterations, final_rel_residual=res,
                          converged=conv.astype(bool), wall_time=0.0,
                          matvec_count=rep.matvec_count)


def _verify(slabs, comm, all_step, read, deferred):
    """True-residual verification after iteration m flagged columns
    (solvers.cpp:582-634). Returns the control word after it."""
    if deferred:
        all_step(APPLY_X)
    comm.halo(slabs, "X")
    all_step(TRUE_RES)
    all_step(CTL_VERIFY)
    return read()


def _pipelined_iterations(slabs, comm, cfg, cfg_c, all_step, read, deferred, sa):
    slots = _ControlSlots(len(slabs))

    def issue(m):
        comm.halo(slabs, "P")
        all_step(SPMM | GATED)
        all_step(CTL_ALPHA | GATED)
        all_step((UPDATE_D if deferred else UPDATE) | GATED)
        all_step(CTL_UPDATE | GATED, m)
        all_step((PUPDATE_X if deferred else PUPDATE) | GATED)
        slots.post(slabs, cfg_c, m)

    m = 1
    if m > cfg.max_iter or sa <= 0:
        return
    issue(m)
    while True:
        ahead = m + 1 <= cfg.max_iter
        if ahead:
            issue(m + 1)
        cmd, _ = slots.wait(m)
        if cmd == CMD_PUPDATE:  # iteration m closed with its P update
            if not ahead:
                return
            m += 1
            continue
        # verification due at m: the enqueued m + 1 ran as no-ops
        cmd, sa = _verify(slabs, comm, all_step, read, deferred)
        if cmd == CMD_DONE:
            return
        if cmd == CMD_RESTART:
            all_step(RESTART_SWEEP)
            all_step(CTL_RESTART)
        else:
            all_step(PUPDATE)
        m += 1
        if m > cfg.max_iter or sa <= 0:
            return
        issue(m)


def _synchronous_iterations(slabs, comm, cfg, all_step, read, deferred, sa):
    m = 1
    while m <= cfg.max_iter and sa > 0:
        comm.halo(slabs, "P")
        all_step(SPMM)
        all_step(CTL_ALPHA)
        all_step(UPDATE_D if deferred else UPDATE)
        all_step(CTL_UPDATE, m)
        cmd, sa = read()
        if cmd == CMD_VERIFY:
            cmd, sa = _verify(slabs, comm, all_step, read, deferred)
            if cmd == CMD_DONE:
                break
            if cmd == CMD_RESTART:
                all_step(RESTART_SWEEP)
                all_step(CTL_RESTART)
                m += 1
                continue
            all_step(PUPDATE)
        else:
            all_step(PUPDATE_X if deferred else PUPDATE)
        m += 1


def make_slabs(bk, ctx, op, s: int, parts):
    S = kernel_width(s)
    return [Slab(bk, ctx, op, y0, nyl, S).allocate() for (y0, nyl) in parts]


def solve_decomposed(bk, ctx, op, B_global, cfg, parts, comm=None, X_global=None, lookahead=True):
    """Convenience: virtual (LocalComm) decomposition of one GPU's solve.
    B_global: n x S device tensor. Returns (X_global, report)."""
    import torch

    S = int(B_global.shape[1])
    if S not in (16, 32, 64):
        raise bk.DimensionMismatchError("decomposed solve: B must be n x 16/32/64 (zero-pad)")
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    slabs = make_slabs(bk, ctx, op, S, parts)
    for sl in slabs:
        sl.load_rhs(B_global)
    rep = dd_block_cg(slabs, comm or LocalComm(), cfg, lookahead=lookahead)
    if X_global is None:
        X_global = torch.empty_like(B_global)
    for sl in slabs:
        sl.store_x(X_global)
    return X_global, rep


def slab_outputs(slabs, comm, coef, T, Q, resid, halo=True):
    """After the decomposed solve: ONE halo exchange of X's edge rows, then
    every slab forms all samples of coef on its own rows (no gather of X);
    the per-sample residual partials are summed across slabs (N x 2 doubles)
    and finished on each rank. T, Q, resid: one tensor per slab (T[i], Q[i]:
    N x slab cells; resid[i]: N, identical on every slab afterwards)."""
    import torch

    _on_torch_stream(slabs)
    if halo:  # once per solve; later sample chunks reuse the ghost rows
        comm.halo(slabs, "X")
    N = int(coef.shape[1])
    nds = []
    for sl, t, q in zip(slabs, T, Q):
        nd = torch.zeros((N, 2), dtype=torch.float64, device=t.device)
        sl.combine_action(coef, t, q, nd)
        nds.append(nd)
    comm.sum(nds)
    lib = slabs[0].bk._load()
    for sl, nd, r in zip(slabs, nds, resid):
        slabs[0].bk._raise(lib.bk_dd_resid_from_nd(sl.ctx.h, C.c_void_p(nd.data_ptr()), N,
                                                   C.c_void_p(r.data_ptr())), sl.ctx.h,
                           "dd_resid_from_nd")

