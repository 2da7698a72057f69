"""CPU tests of the reference-semantics generator's host side:
the chip floorplan model (build_floorplans / sample_power / rasterize_*,
chip.cpp:112-306) and the sample weights (draw_weights, pipeline.cpp:136-152)
are bit-exact restatements, pinned against the reference build and against
the committed golden (tests/golden/make_golden_blockoa.py)."""
import numpy as np
import pytest

from conftest import golden


def test_default_chip_matches_reference_spec(bk):
    c = bk.ChipSpec.default_chip()
    assert c.extent == (10e-3, 10e-3, 0.51e-3)
    assert [r for *_, r in c.layers] == ["tim", "cache", "tim", "cache", "tim", "core"]
    assert abs(c.layers[-1][1] - 0.51e-3) < 1e-18
    assert (c.core_blocks, c.high_power, c.caches_per_layer, c.tsv_count) == (156, 6, 2, 12)
    cfg = bk.GenerationConfig.default_run_config()
    assert (cfg.grid, cfg.n_data, cfg.n_basis, cfg.n_k, cfg.eta()) == ((24, 24, 12), 500, 50, 5, 10)


def test_chip_fields_match_golden_digests(bk):
    d = golden("chip_default.npz")
    grid = tuple(d["grid"].tolist())
    k, q = bk.chip_fields(bk.ChipSpec.default_chip(), grid, int(d["n_k"]),
                          int(d["n_basis"]) // int(d["n_k"]), int(d["seed"]))
    g = bk.GridSpec(*grid)
    assert [bk.field_digest(f, g) for f in k] == d["k_digest"].tolist()
    assert [bk.field_digest(f, g) for f in q] == d["q_digest"].tolist()
    assert np.array_equal(bk.draw_weights(int(d["n_basis"]), int(d["seed"]), 4), d["weights"])


@pytest.mark.parametrize("grid,n_k,eta,seed", [((24, 24, 12), 5, 10, 1), ((17, 13, 9), 3, 4, 7),
                                               ((96, 80, 24), 2, 3, 11), ((8, 8, 3), 4, 1, 2)])
def test_chip_fields_bitwise_vs_reference(bk, reference, grid, n_k, eta, seed):
    chip = bk.ChipSpec.default_chip()
    k, q = bk.chip_fields(chip, grid, n_k, eta, seed)
    kr, qr = reference.chip_fields(grid, n_k, eta, seed)
    assert np.array_equal(k, kr) and np.array_equal(q, qr)
    assert (q > 0).any()
    if grid[2] >= 12:  # the TIM layers are resolved
        assert len(np.unique(k)) >= 2


def test_weights_bitwise_vs_reference(bk, reference):
    for n_basis, seed in ((50, 1), (7, 123), (64, 9)):
        w = bk.draw_weights(n_basis, seed, 40)
        assert np.array_equal(w, reference.draw_weights(n_basis, seed, 40))
        assert np.allclose(w.sum(axis=1), 1.0, atol=1e-9)


def test_chip_spec_errors(bk):
    chip = bk.ChipSpec.default_chip()
    bad = bk.ChipSpec(**{**chip.__dict__, "high_power": chip.core_blocks + 1})
    with pytest.raises(bk.InvalidSpecError):
        bk.chip_fields(bad, (8, 8, 4), 1, 1, 1)
    with pytest.raises(bk.InvalidSpecError):
        bk.chip_fields(chip, (8, 8, 4), 0, 1, 1)
    nocore = bk.ChipSpec(**{**chip.__dict__, "layers": [(0.0, 0.51e-3, 150.0, "cache")]})
    with pytest.raises(bk.InvalidSpecError):
        bk.chip_fields(nocore, (8, 8, 4), 1, 1, 1)
