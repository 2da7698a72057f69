import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def bk():
    import paper_2510_23221_b200 as bk

    bk._load()
    return bk


@pytest.fixture(scope="session")
def ctx(bk):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test on a box without CUDA")
    return bk.Context(0)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def grid_tuple(g):
    return (g.nx, g.ny, g.nz, g.lx, g.ly, g.lz)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
