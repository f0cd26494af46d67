"""The decode table built on the device from the codes (lut_dev.cu) against the host builder
(codebook.cpp build_decode_lut, from the tree) and the oracle.

Both tables decode the same prefix code, so every result of a Huffman run -- seeds, marginals,
coverage, the decode-buffer ledger -- must equal the oracle's whichever builder ran and
whatever the table widths (IMMX_LUT_ROOT / IMMX_LUT_SUB: 3 / 2 forces five and more levels on
these small alphabets; 16 / 12 is the default).  Stored sets are also decoded one by one
through the run's own table and compared with the raw sets."""
import numpy as np
import pytest

from conftest import random_graph
from test_gpu_parity import _cmp_run, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[("0", None, None), ("1", None, None), ("0", "3", "2"), ("1", "3", "2"), ("0", "5", "1")])
def lut_mode(request, monkeypatch):
    host, root, sub = request.param
    monkeypatch.setenv("IMMX_LUT_HOST", host)
    if root:
        monkeypatch.setenv("IMMX_LUT_ROOT", root)
        monkeypatch.setenv("IMMX_LUT_SUB", sub)
    return request.param


def test_runs_equal_oracle(im, orc, lut_mode):
    rng = np.random.default_rng(41)
    for trial in range(3):
        g = orc.assign_weights(random_graph(rng, 200 + 300 * trial, 1500 + 3000 * trial), "wc")
        _cmp_run(im, orc, g, 6, 0.5, 4, "huffman", 19 + trial, workers=1)


def test_stored_sets_decode_to_their_members(im, orc, lut_mode):
    rng = np.random.default_rng(43)
    g = orc.assign_weights(random_graph(rng, 700, 9000), "wc")
    dg = im.DeviceGraph(to_product(im, g), transposed=False)
    r = im.run_device(dg, 5, epsilon=0.5, blocks=4, mode="huffman", seed=5, keep=True)
    st = r["_store"]
    _, lens = st.codebook(g.n)
    pool = im.Pool(dg.device)
    pool.sample(dg, 400, 0, 5)
    off, mem = pool.read()
    for j in range(400):
        members = mem[int(off[j]):int(off[j + 1])]
        codable = sorted(int(v) for v in members if lens[v])
        found, dec = st.decode_find(j, g.n + 7)  # no such vertex: the whole stream is decoded
        assert not found and sorted(dec) == codable
        v = int(members[-1])
        found, dec = st.decode_find(j, v)
        assert found and (not lens[v] or dec[-1] == v)


def test_single_symbol_and_tiny_alphabets(im, orc, lut_mode):
    # a star: every RRR set is {leaf} or {leaf, hub}-like; alphabets of 1-3 symbols in block 1
    for n in (2, 3, 5):
        edges = [(0, v, 1.0) for v in range(1, n)]
        from conftest import make_csr
        g = make_csr(n, edges)
        _cmp_run(im, orc, g, 1, 0.5, 2, "huffman", 3, workers=1)
