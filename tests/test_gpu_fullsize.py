"""BASELINE configs 4 and 5 at full size: properties that hold whatever the
size -- a bit-exact window of the full c4 graph against the oracle, and cross-mode equality
of complete IMM runs (the greedy is one function of the sets, so the Huffman store, the raw
pool and the per-set hybrid store must give the same seeds, marginals and coverage)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4_graph(im):
    dg = im.DeviceGraph.generate_rmat(22, 24, 0.57, 0.19, 0.19, 3, weights="wc")
    return dg


def test_c4_sample_window_matches_oracle(im, orc, c4_graph):
    # 1,500 samples from deep inside the c4 workload (global indices 12,000,000 +): the full
    # 4.2 M-vertex / 97 M-edge reverse CSR, downloaded, sampled by the oracle
    from oracle.oracle import CSR
    from test_gpu_parity import assert_same_sets

    dg = c4_graph
    row, col, pr = dg.download(probs=True)
    gt = CSR(dg.n, row, col, pr)
    first = 12_000_000
    a = orc.sample_block(gt, 1500, first, 42)
    pool = im.Pool(dg.device)
    pool.sample(dg, 1500, first, 42)
    off, mem = pool.read()
    assert_same_sets(a[0], a[1], off, mem)


def test_c4_full_run_cross_mode(im, c4_graph):
    # config 4 exactly (k=100, eps=0.13, 8 blocks, seed 42): theta = 17,794,633 sets
    kw = dict(epsilon=0.13, blocks=8, seed=42)
    h = im.run_device(c4_graph, 100, mode="huffman", **kw)
    r = im.run_device(c4_graph, 100, mode="raw", **kw)
    assert h["theta"] == r["theta"] == 17_794_633
    for key in ("seeds", "marginal", "coverage"):
        assert h[key] == r[key], key
    assert h["compression_ratio"] > 1.5 and h["uncoded_vertex_fraction"] < 0.5


def test_c5_full_run_cross_mode(im):
    # config 5 exactly (R-MAT 25, EF 42, 1.37 B edges generated in HBM; k=50): the per-set
    # hybrid store (what config 5 names) equals the Huffman store (no set above n/32) and
    # the raw greedy
    dg = im.DeviceGraph.generate_rmat(25, 42, 0.57, 0.19, 0.19, 4, weights="wc")
    kw = dict(epsilon=0.5, blocks=8, seed=42)
    y = im.run_device(dg, 50, mode="hybrid", **kw)
    h = im.run_device(dg, 50, mode="huffman", **kw)
    r = im.run_device(dg, 50, mode="raw", **kw)
    assert y["dense_sets"] == 0
    assert y["theta"] == h["theta"] == r["theta"]
    for key in ("seeds", "marginal", "coverage"):
        assert y[key] == h[key] == r[key], key
    assert y["encoded_bytes"] == h["encoded_bytes"] and y["compression_ratio"] == h["compression_ratio"]
