"""The sampler's long-row path (rows of degree >= IMMX_LONG_MIN run alone, in slabs) against
the oracle: the threshold is forced low so every visited-set tier, probability mode and
special threshold goes through it, plus the exact-coin (tie) path.  Bit-exact sets in visit
order and edge counts (sampler.cpp:14-45)."""
import numpy as np
import pytest

from conftest import csr_of, random_graph
from test_gpu_parity import assert_same_sets, sample_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 33, 300])
def long_min(request, monkeypatch):
    monkeypatch.setenv("IMMX_LONG_MIN", str(request.param))
    return request.param


@pytest.mark.parametrize("model,p", [("wc", 0.0), ("uniform", 0.1), ("uniform", 0.5), ("uniform", 1.0),
                                     ("uniform", 0.0),
                                     # thresholds whose high word is outside [2, 2^32 - 2]: the coin
                                     # loop's running maximum cannot flag them, every draw goes
                                     # through the full 64-bit test
                                     ("uniform", 1.0 - 1e-12), ("uniform", 1e-12), ("uniform", 3e-10)])
def test_long_rows_random_graphs(im, orc, long_min, model, p):
    rng = np.random.default_rng(21)
    for trial in range(4):
        g = orc.assign_weights(random_graph(rng, 60 + 50 * trial, 1500 + 900 * trial), model, p)
        gt = orc.transpose(g)
        a = orc.sample_block(gt, 600, 7 * trial, 99 + trial)
        b = sample_dev(im, gt, 600, 7 * trial, 99 + trial)
        assert_same_sets(a[0], a[1], b[0], b[1])
        assert b[2]["edges"] == a[2]


def test_long_rows_rmat_bitmap_tier(im, orc, long_min):
    # scale 16 (bitmap tier), hub rows of thousands of edges
    g = im.generate_rmat(16, 16, 0.57, 0.19, 0.19, 3)
    im.assign_weights_f32(g, "uniform", 0.02)
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 1500, 100, 5)
    b = sample_dev(im, gt, 1500, 100, 5)
    assert_same_sets(a[0], a[1], b[0], b[1])
    assert b[2]["edges"] == a[2]


@pytest.mark.parametrize("p", [0.006, 0.1, 1.0, 0.0])
def test_long_rows_hash_promotion_and_global_tiers(im, orc, long_min, p):
    # n = 2^20: hash tier, promotion slots (p = 0.006), sets beyond a slot (p = 0.1), rows that
    # join without a draw (p = 1) and rows that never draw (p = 0).  (The long-row path is
    # compiled for these tiers only: the bitmap tiers of small graphs run the general path.)
    g = im.generate_rmat(20, 8, 0.57, 0.19, 0.19, 11)
    im.assign_weights_f32(g, "uniform", p)
    gt = orc.transpose(csr_of(g))
    cnt = 300 if p < 0.05 else (24 if p < 1.0 else 6)
    a = orc.sample_block(gt, cnt, 0, 5)
    b = sample_dev(im, gt, cnt, 0, 5)
    assert_same_sets(a[0], a[1], b[0], b[1])


def test_long_rows_weighted_cascade_hubs(im, orc, long_min):
    # per-row thresholds (WC), scale 20: the c4/c5 shape in small
    g = im.generate_rmat(20, 16, 0.57, 0.19, 0.19, 4)
    im.assign_weights_f32(g, "wc")
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 800, 5000, 42)
    b = sample_dev(im, gt, 800, 5000, 42)
    assert_same_sets(a[0], a[1], b[0], b[1])
    assert b[2]["edges"] == a[2]


def test_long_rows_exact_coin_path(im, orc, long_min, monkeypatch):
    monkeypatch.setenv("IMMX_EXACT_COINS", "1")
    g = im.generate_rmat(16, 16, 0.57, 0.19, 0.19, 3)
    im.assign_weights_f32(g, "wc")
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 1000, 0, 8)
    b = sample_dev(im, gt, 1000, 0, 8)
    assert_same_sets(a[0], a[1], b[0], b[1])
