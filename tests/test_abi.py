"""CPU tests of the product boundary: the C-ABI library loads and exports every
symbol include/blockoa_b200.h declares, the host-side input synthesis is
deterministic and pinned, and the product never routes through oracle/."""
import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "blockoa_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(bk_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("bk_create", "bk_assemble", "bk_apply_block", "bk_block_cg", "bk_combine_action",
              "bk_generate_chip", "bk_rhs_from_power", "bk_power_from_rhs", "bk_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(bk):
    lib = ctypes.CDLL(bk.library_path())
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.bk_abi_version() == 1


def test_library_is_sm100a(bk):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bk.library_path()],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu(bk):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bk.DeviceError):
        bk.Context(0)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2510_23221_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "libblockoa_ref" not in txt, f


@pytest.mark.parametrize("name", ["c1_full", "c2_reduced", "c3_reduced", "c5_reduced"])
def test_synth_inputs_pinned(bk, name):
    d = golden(f"{name}.npz")
    cfg, (nx, ny, nz, s, N) = int(d["config"]), d["shape"].tolist()
    inp = bk.synth_chip(cfg, nx, ny, nz, s, N)
    h = hashlib.sha256()
    for a in (inp.k, inp.q_basis, inp.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(d["input_sha256"])


def test_synth_c2_full_pinned(bk):
    d = golden("c2_full_meta.npz")
    inp = bk.synth_chip(*bk.CONFIGS[2])
    h = hashlib.sha256()
    for a in (inp.k, inp.q_basis, inp.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(d["input_sha256"])


def test_synth_configs_shapes_and_pins(bk):
    for cfg, shape in bk.CONFIGS.items():
        if cfg == 5:
            shape = (5, 64, 64, 16, 64, 10)  # reduced: same generator, smaller plane
        inp = bk.synth_chip(*shape)
        _, nx, ny, nz, s, N = shape
        n = nx * ny * nz
        assert inp.k.shape == (n,) and inp.q_basis.shape == (n, s) and inp.coef.shape == (s, N)
        assert np.all(inp.k > 0) and np.all(inp.q_basis >= 0)
        assert np.all((inp.coef >= 0) & (inp.coef < 1))
        kinds = [type(f).__name__ for f in inp.bc.faces]
        assert kinds[:4] == ["Adiabatic"] * 4 and kinds[5] == "Robin"
        assert all(f.u_inf == 0.0 for f in inp.bc.faces if type(f).__name__ == "Robin")
        if cfg == 4:
            assert inp.grid.dz is not None and np.all((inp.grid.dz >= 50e-6) &
                                                      (inp.grid.dz <= 500e-6))
        a = bk.synth_chip(*shape, chip_id=3)
        assert not np.array_equal(a.q_basis, inp.q_basis)  # chips differ by seed


def test_cg_error_bound_product(bk):
    assert bk.cg_error_bound(100, 1, 1) == pytest.approx(1.6363636363636365, rel=1e-15)
    assert bk.cg_error_bound(1, 5, 3) == 0.0
    with pytest.raises(bk.InvalidKappaError):
        bk.cg_error_bound(0.5, 1, 1)
