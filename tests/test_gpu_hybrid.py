"""Per-set hybrid store (builder extension with no reference counterpart):
the device against the oracle's hybrid contract (oracle/immx_oracle.c, oc_store / mode 3),
which is itself pinned to the Huffman and raw modes in tests/test_oracle_kat.py."""
import numpy as np
import pytest

from conftest import csr_of, random_graph
from test_gpu_parity import _cmp_run, to_product

pytestmark = pytest.mark.gpu


def _uniform(g, p):
    from oracle.oracle import CSR
    return CSR(g.n, g.off, g.tgt, np.full(g.m, p, np.float64))


@pytest.mark.parametrize("trial", range(3))
def test_hybrid_run_matches_oracle(im, orc, trial):
    rng = np.random.default_rng(5 + trial)
    g = _uniform(random_graph(rng, 300 + 50 * trial, 3000), 0.3)
    r, o = _cmp_run(im, orc, g, 6, 0.5, 4, "hybrid", 7 + trial, workers=2)
    assert r["stats"]["device"]["dense_sets"] == o["dense_sets"] > 0
    # the same greedy as raw mode
    raw = orc.run(g, 6, 0.5, 4, "raw", 7 + trial)
    assert r["seeds"] == raw["seeds"] and r["coverage"] == raw["coverage"]


def test_hybrid_store_bytes(im, orc):
    rng = np.random.default_rng(21)
    g = _uniform(random_graph(rng, 333, 3000), 0.25)
    o = orc.run(g, 5, 0.5, 4, "hybrid", 9, want_store=True)
    dg = im.DeviceGraph(to_product(im, g), transposed=False)
    r = im.run_device(dg, 5, epsilon=0.5, blocks=4, mode="hybrid", seed=9, keep=True)
    assert r["dense_sets"] == o["dense_sets"] > 0
    bo, by, bl, co, cp = r["_store"].read(0, r["theta"])
    st = o["store"]
    assert np.array_equal(bo, st["enc_off"]) and np.array_equal(bl, st["bit_length"])
    assert by.tobytes() == st["bytes"].tobytes()
    assert np.array_equal(co, st["cp_off"]) and np.array_equal(cp, st["copied"])
    # decode_find on a bitmap set is a bit test
    j = int(np.nonzero(bl == np.iinfo(np.uint64).max)[0][0])
    bm = np.frombuffer(by[int(bo[j]):int(bo[j + 1])].tobytes(), "<u4")
    bits = (bm[np.arange(g.n) // 32] >> (np.arange(g.n) % 32)) & 1
    assert r["_store"].decode_find(j, int(np.nonzero(bits)[0][0])) == (True, [])
    assert r["_store"].decode_find(j, int(np.nonzero(bits == 0)[0][0])) == (False, [])


def test_hybrid_degenerates_to_huffman(im, orc):
    # no set above n/32 (the c3 / c5 shapes): hybrid == Huffman, byte for byte
    g = im.generate_er(3000, 4000, 4)
    im.assign_weights_f32(g, "wc")
    a = im.run(g, 5, epsilon=0.5, blocks=4, mode="hybrid", seed=3)
    b = im.run(g, 5, epsilon=0.5, blocks=4, mode="huffman", seed=3)
    assert a["stats"]["device"]["dense_sets"] == 0
    for key in ("seeds", "marginal", "coverage"):
        assert a[key] == b[key]
    for key in ("theta", "encoded_bytes", "compression_ratio", "peak_bytes"):
        assert a["stats"][key] == b["stats"][key]
    o = orc.run(csr_of(g), 5, 0.5, 4, "hybrid", 3)
    assert a["seeds"] == o["seeds"] and a["stats"]["encoded_bytes"] == o["encoded_bytes"]
