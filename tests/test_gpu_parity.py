"""Parity of the sm_100a path (through the C-ABI) against the C restatement oracle.

Bit-exact for every integer/byte output: RRR sets (members in visit order), theta and the
estimation plan, Huffman codes, encoded bitstreams and copy buffers, seeds, marginals,
coverage (exact doubles: covered/theta), the memory ledger and compression ratio."""
import numpy as np
import pytest

from conftest import csr_of, make_csr, random_graph, random_sets, sets_csr

pytestmark = pytest.mark.gpu


def to_product(im, csr):
    return im.Graph.from_csr(csr.n, csr.off, csr.tgt, csr.prob)


def dev_gt(im, csr_t):
    return im.DeviceGraph.from_arrays(csr_t.n, np.ascontiguousarray(csr_t.off, np.uint64),
                                      np.ascontiguousarray(csr_t.tgt, np.uint32),
                                      np.ascontiguousarray(csr_t.prob, np.float64), True)


def sample_dev(im, csr_t, count, first=0, seed=42):
    dg = dev_gt(im, csr_t)
    pool = im.Pool(dg.device)
    pool.sample(dg, count, first, seed)
    off, mem = pool.read()
    return off, mem, pool.info()


def assert_same_sets(a_off, a_mem, b_off, b_mem):
    assert np.array_equal(np.asarray(a_off, np.uint64), np.asarray(b_off, np.uint64))
    assert np.array_equal(np.asarray(a_mem, np.uint32), np.asarray(b_mem, np.uint32))


# ------------------------------------------------------------------ sampling
def test_chain_and_singletons(im, orc):
    gt = make_csr(3, [(2, 1, 1.0), (1, 0, 1.0)])
    assert im.sample_rrr(to_product(im, gt), 2, 123) == [2, 1, 0]
    edges = [(u, v, 0.0) for u in range(5) for v in range(5) if u != v]
    g0 = orc.transpose(make_csr(5, edges))
    off, mem, _ = sample_dev(im, g0, 50, 0, 5)
    assert np.all(np.diff(off.astype(np.int64)) == 1)


@pytest.mark.parametrize("model,p", [("wc", 0.0), ("uniform", 0.1), ("uniform", 0.5), ("uniform", 1.0)])
def test_sample_block_random_graphs(im, orc, model, p):
    rng = np.random.default_rng(8)
    for trial in range(6):
        g = orc.assign_weights(random_graph(rng, 50 + 40 * trial, 400 + 300 * trial), model, p)
        gt = orc.transpose(g)
        a = orc.sample_block(gt, 700, 13 * trial, 1234 + trial)
        b = sample_dev(im, gt, 700, 13 * trial, 1234 + trial)
        assert_same_sets(a[0], a[1], b[0], b[1])
        assert b[2]["edges"] == a[2]


def test_sample_mixed_probabilities(im, orc):
    # per-edge probabilities (EDGE threshold mode), p<=0, p>=1 and tiny p mixed
    rng = np.random.default_rng(3)
    g = random_graph(rng, 200, 3000)
    pr = rng.choice([0.0, 1.0, 1e-12, 0.3, 0.7, 0.999], size=g.m)
    from oracle.oracle import CSR
    g = CSR(g.n, g.off, g.tgt, pr.astype(np.float64))
    gt = orc.transpose(g)
    a = orc.sample_block(gt, 2000, 0, 9)
    b = sample_dev(im, gt, 2000, 0, 9)
    assert_same_sets(a[0], a[1], b[0], b[1])


def test_sample_duplicate_edges(im, orc):
    # Gt rows with repeated targets (a multigraph): exercises the match.any window path
    rng = np.random.default_rng(5)
    edges = []
    for _ in range(4000):
        u, v = int(rng.integers(0, 120)), int(rng.integers(0, 120))
        if u != v:
            edges.append((u, v, float(rng.choice([0.2, 0.5, 1.0]))))
    g = make_csr(120, edges)
    gt = orc.transpose(g)
    a = orc.sample_block(gt, 1500, 0, 77)
    b = sample_dev(im, gt, 1500, 0, 77)
    assert_same_sets(a[0], a[1], b[0], b[1])


@pytest.mark.parametrize("p,lo,hi", [(0.006, 4096, 16384), (0.01, 16384, 1 << 30)])
def test_sample_hash_tiers(im, orc, p, lo, hi):
    # n = 2^20 > 2^19: the visited set is a shared-memory hash (tier 1: 4,096 members);
    # p near the giant-component threshold makes some sets grow past it: they continue in a
    # promotion slot (the no-promotion restarts are covered below)
    g = im.generate_rmat(20, 8, 0.57, 0.19, 0.19, 11)
    im.assign_weights_f32(g, "uniform", p)
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 600, 0, 5)
    b = sample_dev(im, gt, 600, 0, 5)
    assert_same_sets(a[0], a[1], b[0], b[1])
    sizes = np.diff(a[0].astype(np.int64))
    assert ((sizes > lo) & (sizes <= hi)).sum() >= 3


def test_sample_beyond_promotion_slot(im, orc):
    # p = 0.1 on n = 2^20: sets of ~164 K members outgrow a promotion slot's 2^17-member queue
    # and finish on the per-CTA global-bitmap tier
    g = im.generate_rmat(20, 8, 0.57, 0.19, 0.19, 11)
    im.assign_weights_f32(g, "uniform", 0.1)
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 40, 0, 5)
    b = sample_dev(im, gt, 40, 0, 5)
    assert_same_sets(a[0], a[1], b[0], b[1])
    assert (np.diff(a[0].astype(np.int64)) > (1 << 17)).sum() >= 3


def test_sample_tiers_without_promotion(tmp_path):
    # IMMX_NO_PROMOTE=1: overflowing samples restart on the 128 KB hash tier and the global
    # bitmap instead of continuing in a slot (a separate process: the switch is read once)
    import subprocess
    import sys

    code = (
        "import sys; sys.path[:0] = ['tests', '.']\n"
        "import numpy as np, paper_2208_00613_b200 as im\n"
        "from oracle.oracle import Oracle\n"
        "from conftest import csr_of\n"
        "from test_gpu_parity import sample_dev, assert_same_sets\n"
        "orc = Oracle()\n"
        "g = im.generate_rmat(20, 8, 0.57, 0.19, 0.19, 11)\n"
        "for p in (0.006, 0.01):\n"
        "    im.assign_weights_f32(g, 'uniform', p)\n"
        "    gt = orc.transpose(csr_of(g))\n"
        "    a = orc.sample_block(gt, 600, 0, 5)\n"
        "    b = sample_dev(im, gt, 600, 0, 5)\n"
        "    assert_same_sets(a[0], a[1], b[0], b[1])\n"
        "print('ok')\n")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IMMX_NO_PROMOTE="1")
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stderr[-2000:]


def test_sample_rooted(im, orc):
    rng = np.random.default_rng(2)
    g = orc.assign_weights(random_graph(rng, 80, 600), "wc")
    gt = orc.transpose(g)
    pg = to_product(im, gt)
    for root in range(0, 80, 9):
        assert im.sample_rrr(pg, root, 1000 + root) == orc.sample_rrr(gt, root, 1000 + root)


def test_c1_samples(im, orc):
    g = im.generate_er(10000, 100000, 0)
    im.assign_weights_f32(g, "wc")
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 20000, 0, 42)
    b = sample_dev(im, gt, 20000, 0, 42)
    assert_same_sets(a[0], a[1], b[0], b[1])


def test_c2_samples_subset(im, orc):
    # config 2 graph (R-MAT 18, p = fl32(0.01)): a window of samples incl. giant ones
    g = im.generate_rmat(18, 16, 0.57, 0.19, 0.19, 1)
    im.assign_weights_f32(g, "uniform", 0.01)
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 300, 1000, 42)
    b = sample_dev(im, gt, 300, 1000, 42)
    assert_same_sets(a[0], a[1], b[0], b[1])
    assert np.diff(a[0].astype(np.int64)).max() > 5000


# ------------------------------------------------------------------ device transpose
def test_device_transpose_matches(im, orc):
    # the forward upload transposes on the device; sampling on it equals sampling on the
    # host transpose (same Gt row order, graph.cpp:125-144)
    g = orc.assign_weights(random_graph(np.random.default_rng(4), 500, 6000), "wc")
    gt = orc.transpose(g)
    dg_f = im.DeviceGraph.from_arrays(g.n, g.off, g.tgt, g.prob, False)
    pool = im.Pool(dg_f.device)
    pool.sample(dg_f, 3000, 0, 42)
    off, mem = pool.read()
    a = orc.sample_block(gt, 3000, 0, 42)
    assert_same_sets(a[0], a[1], off, mem)
    assert dg_f.prob_mode == "row"


# ------------------------------------------------------------------ theta / selection
def test_estimate_theta(im, orc):
    rng = np.random.default_rng(31)
    for trial in range(5):
        g = orc.assign_weights(random_graph(rng, 60 + 30 * trial, 300 + 200 * trial), "wc")
        gt = orc.transpose(g)
        assert im.estimate_theta(to_product(im, gt), 4, 0.5, trial) == orc.estimate_theta(gt, 4, 0.5, trial)
    edges = [(u, v, 1.0) for u in range(4) for v in range(4) if u != v]
    gt = orc.transpose(make_csr(4, edges))
    assert im.estimate_theta(to_product(im, gt), 1, 0.5, 42) == orc.estimate_theta(gt, 1, 0.5, 42)


def test_select_raw_examples(im, orc):
    assert im.select_raw([[1, 2], [1, 3], [4]], 5, 2)["seeds"] == [1, 4]
    assert im.select_raw([[2], [1]], 3, 1)["seeds"] == [1]
    s = im.select_raw([[1], [1]], 5, 3)
    assert s["seeds"] == [1, 0, 2] and s["padded"] == 2 and s["marginal"] == [2, 0, 0]
    rng = np.random.default_rng(41)
    for trial in range(30):
        n = 5 + trial % 26
        sets = random_sets(rng, n, 3 + trial % 48, 6)
        k = 1 + trial % min(10, n - 1)
        off, mem = sets_csr(sets)
        assert im.select_raw(sets, n, k) == orc.select_raw(off, mem, n, k)
    with pytest.raises(ValueError):
        im.select_raw([[1]], 5, 5)


def test_table_argmax(im):
    assert im.table_argmax([3, 9, 9, 2]) == 1
    assert im.table_argmax([0, 0, 0]) == 0
    assert im.table_argmax([0, 5, 0, 7, 7]) == 3


# ------------------------------------------------------------------ huffman
def test_codebook_and_bitstream(im, orc):
    sets = [[0, 1], [0, 2], [0], [3, 0]]
    cb = im.build_codebook(sets, 4)
    ocb = orc.codebook_from_sets(sets, 4)
    assert cb.lens.tolist() == ocb.lens.tolist() and cb.bits.tolist() == ocb.bits.tolist()
    enc = im.encode_rrr(cb, [1, 0], top=0)
    assert im.decode_find(cb, enc, 0) == (True, [0])
    found, dec = im.decode_find(cb, enc, 3)
    assert not found and sorted(dec) == [0, 1]
    kat = im.codebook_from_counts([2, 1, 1])
    e = im.encode_rrr(kat, [1, 0, 2], 0)
    assert e.bit_length == 5 and e.bits == bytes([0b01011000]) and e.copied == []


def test_corrupt_payload_raises(im):
    cb = im.codebook_from_counts([5, 2, 1])
    enc = im.encode_rrr(cb, [1, 2])
    bad = im.EncodedRrr(enc.bits, 3, enc.copied)
    with pytest.raises(RuntimeError):
        im.decode_find(cb, bad, 0)
    lying = im.EncodedRrr(enc.bits, 64, enc.copied)
    with pytest.raises(RuntimeError):
        im.decode_find(cb, lying, 0)


def test_encode_random_sets(im, orc):
    rng = np.random.default_rng(77)
    for _ in range(20):
        n = 60
        warm = random_sets(rng, n, 40, 12)
        cb = im.build_codebook(warm, n)
        ocb = orc.codebook_from_sets(warm, n)
        for members in random_sets(rng, n, 10, 12):
            top = int(rng.integers(0, n))
            e = im.encode_rrr(cb, members, top)
            data, bl, cp = ocb.encode(members, top)
            assert (e.bits, e.bit_length, e.copied) == (data, bl, cp)
            assert im.decode_find(cb, e, top) == ocb.decode_find(data, bl, cp, top)
            assert im.decode_find(cb, e, n + 1) == ocb.decode_find(data, bl, cp, n + 1)


def test_bitmap_examples(im, orc):
    sets = [[0, 2], [0, 1, 3], [1, 2, 4], [3, 4], [0, 2, 4], [0, 1, 3]]
    bm = im.encode_bitmap(sets, 5)
    assert bm.popcount_row(0) == 4
    assert bm.row_bits(4) == [0, 0, 1, 1, 1, 0]
    snap = bm.snapshot_row(0)
    pops = [bm.subtract_snapshot(v, snap) for v in range(5)]
    assert pops == [0, 1, 1, 1, 2]
    assert bm.row_bits(4) == [0, 0, 1, 1, 0, 0]
    assert bm.byte_size() == 5 * 32 // 8
    assert im.select_bitmap(im.encode_bitmap(sets, 5), 2)["seeds"] == [0, 4]
    with pytest.raises(IndexError):
        im.encode_bitmap([[7]], 5)


# ------------------------------------------------------------------ full pipeline
def _cmp_run(im, orc, g_csr, k, eps, blocks, mode, seed, workers=1):
    pg = to_product(im, g_csr)
    r = im.run(pg, k, epsilon=eps, blocks=blocks, mode=mode, seed=seed, workers=workers)
    o = orc.run(g_csr, k, eps, blocks, mode, seed, workers)
    st = r["stats"]
    assert r["seeds"] == o["seeds"]
    assert r["marginal"] == o["marginal"]
    assert r["coverage"] == o["coverage"]
    assert r["padded"] == o["padded"]
    for key in ("theta", "raw_bytes", "encoded_bytes", "peak_bytes", "compression_ratio", "skewness", "density",
                "uncoded_vertex_fraction", "mode"):
        assert st[key] == o[key], key
    assert st["plan"]["exit_iteration"] == o["exit_iteration"]
    assert st["plan"]["estimation_samples"] == o["estimation_samples"]
    assert st["plan"]["covered_fraction"] == o["covered_fraction"]
    assert [b["sets"] for b in st["blocks"]] == o["block_sets"]
    assert [b["encoded_bytes"] for b in st["blocks"]] == o["block_enc"]
    return r, o


@pytest.mark.parametrize("mode", ["huffman", "bitmap", "raw", "auto"])
def test_run_modes(im, orc, mode):
    rng = np.random.default_rng(12)
    for trial in range(3):
        g = orc.assign_weights(random_graph(rng, 40 + 20 * trial, 300 + 100 * trial), "wc")
        _cmp_run(im, orc, g, 5, 0.5, 4, mode, 100 + trial, workers=1 + trial)


def test_run_smoke_graph(im, orc):
    lines = [f"0 {i}" for i in range(1, 7)] + [f"7 {i}" for i in range(8, 13)] + ["3 7"]
    g = im.load_edge_list_text("\n".join(lines) + "\n")
    im.assign_weights(g, "wc")
    seeds = {}
    for mode in ("raw", "huffman", "bitmap"):
        out = im.run(g, 2, mode=mode, seed=11, blocks=4)
        seeds[mode] = out["seed_ids"]
        assert out["stats"]["mode"] == mode
        assert 0.0 < out["stats"]["seeds"][-1]["cumulative"] <= 1.0
    assert seeds["raw"] == seeds["huffman"] == seeds["bitmap"]


def test_run_c1_full(im, orc):
    # BASELINE config 1 end to end: ER 10k/100k, fl32 WC, k=10, eps=0.5, 10 blocks, huffman
    g = im.generate_er(10000, 100000, 0)
    im.assign_weights_f32(g, "wc")
    r, o = _cmp_run(im, orc, csr_of(g), 10, 0.5, 10, "huffman", 42, workers=8)
    rel = abs(r["coverage"][-1] * g.n - o["coverage"][-1] * g.n) / (o["coverage"][-1] * g.n)
    assert rel <= 1e-6


def test_run_reuse_equals_resample(im, orc):
    g = im.generate_er(2000, 16000, 3)
    im.assign_weights_f32(g, "wc")
    a = im.run(g, 5, epsilon=0.5, blocks=4, mode="huffman", seed=7, reuse_pool=True)
    b = im.run(g, 5, epsilon=0.5, blocks=4, mode="huffman", seed=7, reuse_pool=False)
    for key in ("seeds", "marginal", "coverage"):
        assert a[key] == b[key]
    for key in ("theta", "encoded_bytes", "peak_bytes", "compression_ratio"):
        assert a["stats"][key] == b["stats"][key]


# ------------------------------------------------------------------ LT (self-pinned)
def test_lt_walk(im, orc):
    g = im.generate_er(3000, 20000, 5)
    gt = im.transpose(g)
    w = im.lt_weights(gt, 9)
    gtc = csr_of(gt)
    a = orc.sample_block_lt(gtc, w, 2000, 0, 42)
    dg = im.DeviceGraph(gt, transposed=True, lt_weights=w)
    pool = im.Pool(dg.device)
    pool.sample(dg, 2000, 0, 42, model=1)
    off, mem = pool.read()
    assert_same_sets(a[0], a[1], off, mem)


# ------------------------------------------------------------------ device generator
@pytest.mark.parametrize("weights,p", [("wc", 0.0), ("uniform", 0.01)])
def test_device_rmat_equals_host(im, orc, weights, p):
    # the in-HBM generator emits exactly transpose(host generator) with the same weights
    for scale, ef, seed in ((10, 8, 3), (14, 16, 1)):
        h = im.generate_rmat(scale, ef, 0.57, 0.19, 0.19, seed)
        im.assign_weights_f32(h, weights, p)
        ht = csr_of(im.transpose(h))
        dg = im.DeviceGraph.generate_rmat(scale, ef, 0.57, 0.19, 0.19, seed, weights=weights, p=p)
        row, col, pr = dg.download()
        assert np.array_equal(row, ht.off) and np.array_equal(col, ht.tgt) and np.array_equal(pr, ht.prob)
        pool = im.Pool(dg.device)
        pool.sample(dg, 500, 0, 42)
        off, mem = pool.read()
        a = orc.sample_block(ht, 500, 0, 42)
        assert_same_sets(a[0], a[1], off, mem)


def test_device_rmat_c2_matches_golden_graph(im):
    import hashlib
    import json
    import os
    from conftest import GOLDEN

    g = json.load(open(os.path.join(GOLDEN, "golden.json")))["cases"]["c2"]
    dg = im.DeviceGraph.generate_rmat(18, 16, 0.57, 0.19, 0.19, 1, weights="uniform", p=0.01)
    for w in g["windows"]:
        pool = im.Pool(dg.device)
        pool.sample(dg, w["count"], w["first"], 42)
        off, mem = pool.read()
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(off).tobytes())
        h.update(np.ascontiguousarray(mem).tobytes())
        assert h.hexdigest() == w["sha"]


@pytest.fixture
def exact_coins(monkeypatch):
    # IMMX_EXACT_COINS=1 routes every coin through the rare exact path (the one taken when the
    # draw's high word sits within one of the threshold's): bit-exact either way
    monkeypatch.setenv("IMMX_EXACT_COINS", "1")


@pytest.mark.parametrize("model,p", [("wc", 0.0), ("uniform", 0.1), ("uniform", 0.6)])
def test_sample_exact_coin_path(im, orc, exact_coins, model, p):
    rng = np.random.default_rng(21)
    for trial in range(3):
        g = orc.assign_weights(random_graph(rng, 120 + 60 * trial, 900 + 400 * trial), model, p)
        gt = orc.transpose(g)
        a = orc.sample_block(gt, 600, 7 * trial, 77 + trial)
        b = sample_dev(im, gt, 600, 7 * trial, 77 + trial)
        assert_same_sets(a[0], a[1], b[0], b[1])


def test_c2_samples_exact_coin_path(im, orc, exact_coins):
    g = im.generate_rmat(18, 16, 0.57, 0.19, 0.19, 1)
    im.assign_weights_f32(g, "uniform", 0.01)
    gt = orc.transpose(csr_of(g))
    a = orc.sample_block(gt, 120, 1000, 42)
    b = sample_dev(im, gt, 120, 1000, 42)
    assert_same_sets(a[0], a[1], b[0], b[1])



def test_sample_exact_coin_path_per_edge(im, orc, exact_coins):
    # per-edge thresholds: the exact path re-derives each position's threshold from its row
    rng = np.random.default_rng(13)
    g = random_graph(rng, 300, 5000)
    pr = rng.choice([0.0, 1.0, 1e-12, 0.3, 0.7, 0.999], size=g.m)
    from oracle.oracle import CSR
    g = CSR(g.n, g.off, g.tgt, pr.astype(np.float64))
    gt = orc.transpose(g)
    a = orc.sample_block(gt, 1500, 0, 11)
    b = sample_dev(im, gt, 1500, 0, 11)
    assert_same_sets(a[0], a[1], b[0], b[1])
