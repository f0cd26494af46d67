import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); the parity tests proper")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def _has_gpu():
    # the driver API directly: cheap, and no torch import at collection time
    import ctypes

    try:
        cu = ctypes.CDLL("libcuda.so.1")
    except OSError:
        return False
    if cu.cuInit(0) != 0:
        return False
    n = ctypes.c_int(0)
    return cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle

    lib = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        import subprocess

        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"])
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_PATH, RefLib

    if not os.path.exists(REF_PATH):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return RefLib()


@pytest.fixture(scope="session")
def im():
    import paper_2208_00613_b200 as im

    return im


def csr_of(g):
    """product Graph -> oracle CSR"""
    from oracle.oracle import CSR

    off, tgt, pr, _ = g.arrays()
    return CSR(int(off.size - 1), off, tgt, pr)


def make_csr(n, edges):
    """(u, v, p) triples -> oracle CSR in the given order per source (test_util.hpp:26-45)"""
    from oracle.oracle import CSR

    adj = [[] for _ in range(n)]
    for u, v, p in edges:
        adj[u].append((v, p))
    off = np.zeros(n + 1, np.uint64)
    tgt, pr = [], []
    for u in range(n):
        off[u + 1] = off[u] + len(adj[u])
        for v, p in adj[u]:
            tgt.append(v)
            pr.append(p)
    return CSR(n, off, np.array(tgt, np.uint32), np.array(pr, np.float64))


def random_graph(rng, n, m):
    """test_util.hpp:48-67: random simple directed graph, weights 0 (assign later)."""
    seen = set()
    edges = []
    for _ in range(m):
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        edges.append((u, v, 0.0))
    if not edges:
        edges.append((0, 1, 0.0))
    return make_csr(n, edges)


def random_sets(rng, n, count, max_size):
    """test_util.hpp:152-166"""
    sets = []
    for _ in range(count):
        target = int(rng.integers(1, max_size + 1))
        s, used = [], set()
        while len(s) < target and len(s) < n:
            v = int(rng.integers(0, n))
            if v not in used:
                used.add(v)
                s.append(v)
        sets.append(s)
    return sets


def sets_csr(sets):
    off = np.zeros(len(sets) + 1, np.uint64)
    for i, s in enumerate(sets):
        off[i + 1] = off[i] + len(s)
    mem = np.array([v for s in sets for v in s], np.uint32)
    return off, mem
