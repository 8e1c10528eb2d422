"""Shared fixtures.  `gpu` tests need a B200 and the in-tree CUDA library; the
rest run on CPU (oracle vs reference goldens, host logic, ABI surface, gloo)."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

SEVEN_EDGES = [(0, 1), (1, 2), (1, 3), (2, 3), (3, 4), (3, 5), (4, 5), (5, 6)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libfcref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def seven():
    from paper_2506_04045_b200 import SparseSimilarity
    return SparseSimilarity.build_similarity(7, SEVEN_EDGES)


def random_graph(n, avg_deg, seed, weighted=False):
    """Random symmetric A+I similarity (optionally with symmetric random weights)."""
    from paper_2506_04045_b200 import SparseSimilarity
    rng = np.random.default_rng(seed)
    m = max(1, int(n * avg_deg / 2))
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    k = u != v
    e = np.unique(np.sort(np.stack([u[k], v[k]], 1), 1), axis=0) if k.any() else np.zeros((0, 2), np.int64)
    if not weighted:
        return SparseSimilarity.build_similarity(n, e)
    w = rng.uniform(0.1, 2.0, size=len(e))
    d = rng.uniform(0.5, 1.5, size=n)
    ids = np.arange(n)
    t = np.concatenate([np.stack([ids, ids, d], 1), np.stack([e[:, 0], e[:, 1], w], 1),
                        np.stack([e[:, 1], e[:, 0], w], 1)])
    return SparseSimilarity.from_triplets(n, t)


@pytest.fixture(scope="session")
def ctx():
    """The CUDA context of the gpu tests (fails loudly if the library is missing)."""
    from paper_2506_04045_b200 import capi, api
    c = capi.Context(0)
    api.set_default_context(c)
    yield c
    api.set_default_context(None)
    c.close()
