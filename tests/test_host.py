"""CPU tests of the product's host side: the C-ABI library loads and exports every symbol of
include/immx_b200.h, the ctypes binding matches the header, and the host-only logic
(ingestion, transpose, weights, cache, theta, characterization, the Huffman tree, the
generators) matches the reference semantics.  No compute call needs a GPU here; device
calls must fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, csr_of, random_graph

HEADER = os.path.join(ROOT, "include", "immx_b200.h")
LIB = os.path.join(ROOT, "paper_2208_00613_b200", "libimmx_b200.so")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"IMMX_API\s+[\w\s\*]+?\b(immx_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 60
    lib = ctypes.CDLL(LIB)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2208_00613_b200 import _capi

    assert sorted(_capi.SIGNATURES) == header_functions()


def test_device_calls_fail_loudly_without_gpu(im):
    from conftest import HAS_GPU

    if HAS_GPU:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        im.Device(0)


def test_theta(im):
    assert im.theta_bound(100, 1, 0.5, 1) == 229
    assert im.theta_bound_real(1000, 5, 0.3, 3) == 2 * im.theta_bound_real(1000, 5, 0.3, 2)
    for args in ((10, 10, 0.5, 1), (10, 0, 0.5, 1), (1, 1, 0.5, 1), (10, 1, 0.0, 1), (10, 1, 0.5, 0)):
        with pytest.raises(ValueError):
            im.theta_bound(*args)


def test_theta_matches_oracle(im, orc):
    for n in (10, 100, 5000, 1000000, 33554432):
        for k in (1, 5, 9, 50, 100):
            if k >= n:
                continue
            for eps in (0.13, 0.5):
                for i in (1, 4, 7):
                    assert im.theta_bound_real(n, k, eps, i) == orc.theta_bound_real(n, k, eps, i)
                    assert im.theta_bound(n, k, eps, i) == orc.theta_bound(n, k, eps, i)


def test_characterize(im, orc):
    assert im.skewness([1, 1, 1, 10]) == pytest.approx(1.1547, abs=1e-4)
    assert im.density([5, 5], 10) == 0.5
    assert im.choose_encoding(11.46, 0.00261) == "huffman"
    assert im.choose_encoding(-1.43, 0.6601) == "bitmap"
    assert im.choose_encoding(-0.5, 0.01) == "raw"
    rng = np.random.default_rng(99)
    for _ in range(100):
        s = rng.integers(1, 200, rng.integers(2, 400)).astype(np.uint32)
        assert im.skewness(s) == orc.skewness(s)
        assert im.density(s, 200) == orc.density(s, s.size and 200)
    with pytest.raises(ValueError):
        im.skewness([3])


def test_codebook_matches_oracle(im, orc):
    rng = np.random.default_rng(12)
    for trial in range(60):
        f = rng.integers(0, 501, 40 + trial)
        f[0] = 1
        a, b = im.codebook_from_counts(f), orc.codebook(f)
        assert a.lens.tolist() == b.lens.tolist() and a.bits.tolist() == b.bits.tolist()
        assert a.coded_vertices == b.coded_vertices
    # tie-heavy alphabets (the linear merge orders equal-frequency merged nodes by min id)
    for trial in range(20):
        f = rng.integers(0, 4, 3000 + 97 * trial)
        f[rng.integers(0, f.size, 5)] = rng.integers(50, 5000, 5)
        a, b = im.codebook_from_counts(f), orc.codebook(f)
        assert a.lens.tolist() == b.lens.tolist() and a.bits.tolist() == b.bits.tolist()
    # a skewed alphabet with deep codes
    f = (2 ** np.arange(40)).astype(np.uint64)
    assert im.codebook_from_counts(f).lens.tolist() == orc.codebook(f).lens.tolist()
    f = (2 ** np.arange(63)).astype(np.uint64)
    assert im.codebook_from_counts(f).bits.tolist() == orc.codebook(f).bits.tolist()
    fib = [1, 1]
    while len(fib) < 70:
        fib.append(fib[-1] + fib[-2])
    with pytest.raises(RuntimeError):
        im.codebook_from_counts(np.array(fib, dtype=np.uint64))
    with pytest.raises(RuntimeError):
        im.codebook_from_counts([0, 0, 0])
    assert im.codebook_from_counts([5, 2, 1]).dump() == "0 1 1\n1 2 01\n2 2 00\n"


def test_loader_semantics(im):
    # graph.cpp:24-117: comments, weights, self-loop keeps the vertex, first-seen ids, dedup
    txt = "# c\n10 20\n20 30 0.5\n10 20 0.9\n40 40\n\n30 10\n"
    g = im.load_edge_list_text(txt, directed=True)
    assert g.n == 4 and g.m == 3
    assert list(g.original_ids) == [10, 20, 30, 40]
    off, tgt, pr, _ = g.arrays()
    assert off.tolist() == [0, 1, 2, 3, 3] and tgt.tolist() == [1, 2, 0] and pr.tolist() == [1.0, 0.5, 1.0]
    u = im.load_edge_list_text("0 1\n1 2\n")
    assert u.m == 4
    for bad in ("0\n", "0 1 2 3\n", "a b\n", "0 1 -1\n", "0 1 x\n"):
        with pytest.raises(RuntimeError, match="line 1"):
            im.load_edge_list_text(bad)
    with pytest.raises(RuntimeError):
        im.load_edge_list_text("# only\n")
    with pytest.raises(RuntimeError):
        im.load_edge_list("/nonexistent/file.txt")


def test_transpose_and_weights_match_oracle(im, orc):
    rng = np.random.default_rng(4)
    for _ in range(10):
        c = random_graph(rng, 40, 300)
        g = im.Graph.from_csr(c.n, c.off, c.tgt, c.prob)
        im.assign_weights(g, "wc")
        ow = orc.assign_weights(c, "wc")
        assert np.array_equal(g.probs, ow.prob)
        t, ot = csr_of(im.transpose(g)), orc.transpose(ow)
        assert np.array_equal(t.off, ot.off) and np.array_equal(t.tgt, ot.tgt) and np.array_equal(t.prob, ot.prob)
    g = im.Graph.from_csr(3, [0, 1, 2, 2], [1, 2], [0.0, 0.0])
    im.assign_weights(g, "uniform", 0.1)
    assert g.probs.tolist() == [0.1, 0.1]
    with pytest.raises(ValueError):
        im.assign_weights(g, "uniform", 1.5)
    with pytest.raises(ValueError):
        im.assign_weights(g, "lt")
    im.assign_weights_f32(g, "uniform", 0.01)
    assert g.probs.tolist() == [float(np.float32(0.01))] * 2


def test_cache_round_trip(im, tmp_path):
    g = im.generate_er(50, 300, 1)
    im.assign_weights(g, "wc")
    p = str(tmp_path / "g.bin")
    im.save_graph_cache(g, p)
    r = im.load_graph_cache(p)
    for a, b in zip(g.arrays()[:3], r.arrays()[:3]):
        assert np.array_equal(a, b)
    assert open(p, "rb").read(6) == b"IMMXG1"
    bad = tmp_path / "x.bin"
    bad.write_bytes(b"something else entirely")
    with pytest.raises(RuntimeError):
        im.load_graph_cache(str(bad))
    with pytest.raises(RuntimeError):
        im.load_graph_cache(str(tmp_path / "missing.bin"))


def test_generators_deterministic(im):
    a, b = im.generate_rmat(12, 8, 0.57, 0.19, 0.19, 5), im.generate_rmat(12, 8, 0.57, 0.19, 0.19, 5)
    for x, y in zip(a.arrays()[:2], b.arrays()[:2]):
        assert np.array_equal(x, y)
    off, tgt, _, _ = a.arrays()
    assert a.n == 4096 and a.m <= 8 * 4096
    for u in range(a.n):  # rows sorted, distinct, no self-loops
        row = tgt[off[u]:off[u + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0) and not np.any(row == u)
    e = im.generate_er(1000, 5000, 2)
    assert e.m == 5000
    c = im.generate_rmat(12, 8, 0.57, 0.19, 0.19, 6)
    assert not np.array_equal(c.arrays()[1][:100], tgt[:100])


def test_lt_weights_normalised(im):
    g = im.generate_er(200, 2000, 3)
    gt = im.transpose(g)
    w = im.lt_weights(gt, 9)
    off = gt.offsets
    for v in range(gt.n):
        if off[v + 1] > off[v]:
            assert abs(float(w[off[v]:off[v + 1]].astype(np.float64).sum()) - 1.0) < 1e-5
    assert np.all(w > 0)


def test_merged_argmax_multiworker_refused(im):
    """select.cpp:71-74: merged_argmax with > 1 worker is the reference's per-chunk heuristic;
    the device path selects exactly, so the flag is refused instead of silently ignored."""
    g = im.generate_er(50, 300, 1)
    im.assign_weights_f32(g, "wc")
    with pytest.raises(ValueError, match="merged_argmax"):
        im.run(g, 3, merged_argmax=True, workers=4)
    with pytest.raises(ValueError, match="merged_argmax"):
        im.select_raw([[0, 1], [2]], 5, 1, workers=2, merged_argmax=True)
