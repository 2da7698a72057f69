"""bk_generate_stream: the per-chip loop of generate_blockoa (pipeline.cpp:
365-597) with the samples drained chunk by chunk to a host sink while the next
chip solves. Every sample the sink sees must be bitwise what bk_generate_chip
writes for the same chip (same kernels, same order), every sample exactly
once, in chip / sample order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-12


def cfg():
    import paper_2510_23221_b200 as bk
    return bk.SolverConfig(TOL, 100000, "jacobi")


@pytest.mark.parametrize("case,chunk", [((3, 24, 20, 8, 32, 37), 8), ((1, 40, 32, 1, 8, 50), 16),
                                        ((5, 16, 16, 16, 64, 21), 0)])
def test_stream_matches_generate_chip(bk, ctx, case, chunk):
    chips = [bk.synth_chip(*case, chip_id=c) for c in range(3)]
    n, N = chips[0].grid.cell_count(), case[-1]
    got_T = [np.full((N, n), np.nan) for _ in chips]
    got_Q = [np.full((N, n), np.nan) for _ in chips]
    got_R = [np.full(N, np.nan) for _ in chips]
    order = []

    def sink(chip, j0, T, Q, R):
        m = T.shape[0]
        assert np.isnan(got_T[chip][j0:j0 + m]).all()  # each sample exactly once
        got_T[chip][j0:j0 + m] = T
        got_Q[chip][j0:j0 + m] = Q
        got_R[chip][j0:j0 + m] = R
        order.append((chip, j0))

    reps, tim = bk.generate_stream(chips, cfg(), sink=sink, chunk=chunk, ctx=ctx)
    assert order == sorted(order)
    for c, ch in enumerate(chips):
        T, Q, R, rep, _ = bk.generate_chip(ch.grid, ch.k, ch.bc, ch.q_basis, ch.coef, cfg(),
                                           ctx=ctx)
        assert reps[c].iterations == rep.iterations
        assert np.array_equal(got_T[c], T) and np.array_equal(got_Q[c], Q)
        assert np.array_equal(got_R[c], R)
    assert tim.iterations_total == sum(r.iterations for r in reps)


def test_stream_device_inputs_and_no_sink(bk, ctx):
    import torch

    dev = torch.device("cuda", 0)
    from types import SimpleNamespace
    ch = bk.synth_chip(2, 48, 40, 1, 16, 33, chip_id=3)
    d = SimpleNamespace(grid=ch.grid, bc=ch.bc, k=torch.from_numpy(ch.k).to(dev),
                        q_basis=torch.from_numpy(ch.q_basis).to(dev),
                        coef=torch.from_numpy(ch.coef).to(dev))
    reps, _ = bk.generate_stream([d, d], cfg(), sink=None, chunk=16, ctx=ctx)
    assert all(r.all_converged() for r in reps)


def test_stream_sink_abort(bk, ctx):
    ch = bk.synth_chip(1, 32, 32, 1, 8, 40, chip_id=1)
    seen = []

    def sink(chip, j0, T, Q, R):
        seen.append(j0)
        return j0 >= 16  # abort on the second chunk

    with pytest.raises(bk.IoError):
        bk.generate_stream([ch, ch], cfg(), sink=sink, chunk=16, ctx=ctx)
    assert seen[:2] == [0, 16]
    # the context stays usable
    reps, _ = bk.generate_stream([ch], cfg(), sink=None, chunk=16, ctx=ctx)
    assert reps[0].all_converged()
