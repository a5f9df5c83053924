"""Shared fixtures.  `-m gpu` tests need a B200 and the built sm_100a library;
everything else runs on CPU (oracle pinning, host logic, ABI exports)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and paper_1811_02761_b200/_build/libg2.so")
    config.addinivalue_line("markers", "slow: larger parity sizes")


@pytest.fixture(scope="session")
def oracle():
    from oracle.refpy import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.refpy import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libgravitree_ref.so not built (needs /root/reference at build time)")
    return Ref()


def load_golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing")
    return dict(np.load(path))


def plummer(n, seed=1, a=1.0, r_cut=20.0):
    """Plummer positions by inverse CDF (numpy), equal masses 1/n, zero velocity."""
    rng = np.random.default_rng(seed)
    fcut = r_cut ** 3 / (r_cut ** 2 + a * a) ** 1.5
    u = rng.uniform(0, 1, n) * fcut
    u23 = np.cbrt(u) ** 2
    r = a * np.sqrt(u23 / (1.0 - u23))
    d = rng.normal(size=(n, 3))
    pos = r[:, None] * d / np.linalg.norm(d, axis=1)[:, None]
    return np.full(n, 1.0 / n), pos, np.zeros((n, 3))


def random_cloud(n, seed, half=1.0):
    """test_support.hpp:14-23 analogue: uniform cube, masses in [0.5, 1.5]."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0.5, 1.5, n), rng.uniform(-half, half, (n, 3)), rng.uniform(-0.1, 0.1, (n, 3))
