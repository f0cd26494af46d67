"""select_huffman's member-signature filter (select.cu k_sig_filter; a side index of the store).

Each stored set carries a 64-bit signature of its members; a greedy round decodes only the
live sets whose signature holds the pick's bits.  The filter must not change any result: for
IMMX_SIG_K = 0 (no signatures: every live set is decoded, the reference's loop,
select.cpp:186-214), 1, 2 (default) and 3 bits per member the run equals the oracle in seeds,
marginals, coverage, the ledger peak (its decode buffers count the codewords each set would
decode, huffman.cpp:148-157) and the encoded bytes.  Sets appended from host bytes (members
unknown to the device) take part in every round."""
import numpy as np
import pytest

from conftest import random_graph, random_sets, sets_csr
from test_gpu_parity import _cmp_run, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[0, 1, 2, 3])
def sig_k(request, monkeypatch):
    monkeypatch.setenv("IMMX_SIG_K", str(request.param))
    return request.param


@pytest.mark.parametrize("mode", ["huffman", "hybrid"])
def test_run_equals_oracle_for_every_signature_width(im, orc, sig_k, mode):
    rng = np.random.default_rng(5)
    for trial in range(2):
        g = orc.assign_weights(random_graph(rng, 400 + 150 * trial, 4000 + 1500 * trial), "wc")
        if mode == "hybrid":
            o = orc.run(g, 8, 0.5, 4, "hybrid", 31 + trial)
            dg = im.DeviceGraph(to_product(im, g), transposed=False)
            r = im.run_device(dg, 8, epsilon=0.5, blocks=4, mode="hybrid", seed=31 + trial)
            for key in ("seeds", "marginal", "coverage", "padded"):
                assert r[key] == o[key], key
            assert r["encoded_bytes"] == o["encoded_bytes"] and r["peak_bytes"] == o["peak_bytes"]
        else:
            _cmp_run(im, orc, g, 8, 0.5, 4, "huffman", 31 + trial, workers=2)


def test_long_sets_and_uncoded_members(im, orc, sig_k):
    # sets beyond one decode segment (64 codewords) and members without a code (copied): the
    # filter lists every segment of a candidate and the copied members still decide a hit
    rng = np.random.default_rng(9)
    n = 3000
    warm = random_sets(rng, n // 2, 60, 300)           # the codebook knows half the vertices
    sets = random_sets(rng, n, 400, 300) + random_sets(rng, n, 300, 6)
    cb = im.build_codebook(warm, n)
    ocb = orc.codebook_from_sets(warm, n)
    off, mem = sets_csr(sets)
    top = int(np.bincount(mem, minlength=n).argmax())
    ost = ocb.store(off, mem, top)
    hist = np.bincount(mem, minlength=n).astype(np.uint64)
    want = ost.select(hist, 12)
    st = im.Store(cb)
    pool = im.Pool(st.device)
    pool.upload(sets)
    st.encode(pool, 0, len(sets), top)
    got = im.select_huffman(cb, st, hist, 12)
    assert got == want


def test_host_appended_sets_pass_every_round(im, orc, sig_k):
    rng = np.random.default_rng(3)
    n = 200
    sets = random_sets(rng, n, 150, 20)
    cb = im.build_codebook(sets, n)
    ocb = orc.codebook_from_sets(sets, n)
    off, mem = sets_csr(sets)
    hist = np.bincount(mem, minlength=n).astype(np.uint64)
    want = ocb.store(off, mem, None).select(hist, 6)
    st = im.Store(cb)
    for members in sets:
        data, bl, cp = ocb.encode(members, None)
        st.append(data, bl, cp)
    assert im.select_huffman(cb, st, hist, 6) == want
