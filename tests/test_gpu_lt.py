"""LT extension (config 3's diffusion model; no reference counterpart -- SPEC.md:8): the
device against the builder's oracle contract oc_sample_lt / oc_run_lt (self-pinned)."""
import numpy as np
import pytest

from conftest import csr_of

pytestmark = pytest.mark.gpu


def test_lt_weights_generated_in_hbm(im, orc):
    # immx_graph_set_lt_random == host lt_weights + the same cumulative walk table
    g = im.generate_rmat(12, 8, 0.57, 0.19, 0.19, 2)
    im.assign_weights_f32(g, "wc")
    gt = im.transpose(g)
    w = im.lt_weights(gt, 9)
    gtc = csr_of(gt)
    a = orc.sample_block_lt(gtc, w, 3000, 0, 42)
    dg = im.DeviceGraph.generate_rmat(12, 8, 0.57, 0.19, 0.19, 2, weights="wc")
    dg.set_lt_random(9)
    pool = im.Pool(dg.device)
    pool.sample(dg, 3000, 0, 42, model=1)
    off, mem = pool.read()
    assert np.array_equal(a[0], off) and np.array_equal(a[1], mem)


@pytest.mark.parametrize("mode", ["huffman", "raw", "bitmap"])
def test_lt_full_run_matches_oracle(im, orc, mode):
    g = im.generate_rmat(11, 8, 0.57, 0.19, 0.19, 2)
    im.assign_weights_f32(g, "wc")
    w = im.lt_weights(im.transpose(g), 5)
    got = im.run(g, 8, epsilon=0.5, blocks=4, mode=mode, seed=42, diffusion="lt", lt_weights=w)
    want = orc.run(csr_of(g), 8, 0.5, 4, mode, 42, 1, lt_weights=w)
    assert got["seeds"] == want["seeds"] and got["marginal"] == want["marginal"]
    assert got["coverage"] == want["coverage"]
    for key in ("theta", "encoded_bytes", "compression_ratio", "peak_bytes"):
        assert got["stats"][key] == want[key], key


def test_lt_c3_shape_samples(im, orc):
    # config 3 graph shape (R-MAT 20, EF 16, seed 2) with generator LT weights: a window of walks
    dg = im.DeviceGraph.generate_rmat(20, 16, 0.57, 0.19, 0.19, 2, weights="wc")
    dg.set_lt_random(3)
    row, col, _ = dg.download(probs=False)
    from oracle.oracle import CSR
    gt = im.Graph.from_csr(dg.n, row, col, np.zeros(dg.m))
    w = im.lt_weights(gt, 3)
    a = orc.sample_block_lt(CSR(dg.n, row, col, np.zeros(dg.m)), w, 20000, 0, 42)
    pool = im.Pool(dg.device)
    pool.sample(dg, 20000, 0, 42, model=1)
    off, mem = pool.read()
    assert np.array_equal(a[0], off) and np.array_equal(a[1], mem)
    sizes = np.diff(off.astype(np.int64))
    assert sizes.max() <= dg.n // 32  # the hybrid store degenerates to Huffman on this shape
