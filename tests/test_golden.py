"""The oracle against golden vectors the REFERENCE produced (tests/golden/make_golden.py ran
oracle/_ref, the unmodified reference compiled from its sources).  CPU only: this pins the
checker; tests/test_gpu_golden.py holds the device to the same vectors."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, csr_of

with open(os.path.join(GOLDEN, "golden.json")) as f:
    G = json.load(f)["cases"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def small_graph():
    from oracle.oracle import CSR

    z = np.load(os.path.join(GOLDEN, "small.npz"))
    return CSR(300, z["off"], z["tgt"], z["prob"])


def test_small_graph_inputs(orc):
    g = small_graph()
    assert sha(g.off, g.tgt, g.prob) == G["small"]["graph_sha"]
    gt = orc.transpose(g)
    assert sha(gt.off, gt.tgt, gt.prob) == G["small"]["gt_sha"]


def test_small_samples(orc):
    gt = orc.transpose(small_graph())
    for key, (first, count) in (("sample_0_2000_seed42", (0, 2000)), ("sample_12345_500_seed42", (12345, 500))):
        off, mem, _ = orc.sample_block(gt, count, first, 42)
        assert off.tolist() == G["small"][key]["offsets"]
        assert mem.tolist() == G["small"][key]["members"]


def test_small_estimate_theta(orc):
    gt = orc.transpose(small_graph())
    assert orc.estimate_theta(gt, 5, 0.5, 3) == G["small"]["estimate_theta_k5_eps05_seed3"]


@pytest.mark.parametrize("mode", ["huffman", "bitmap", "raw", "auto"])
def test_small_runs(orc, mode):
    want = G["small"]["run_k5_eps05_b4_seed11_w2"][mode]
    got = orc.run(small_graph(), 5, 0.5, 4, mode, 11, 2)
    assert got["seeds"] == want["seeds"] and got["marginal"] == want["marginal"]
    assert got["coverage"] == want["coverage"] and got["padded"] == want["padded"]
    for k, v in want["stats"].items():
        assert got[k] == v, k
    for k, v in want["plan"].items():
        assert got[k] == v, k
    assert got["block_sets"] == [b["sets"] for b in want["blocks"]]
    assert got["block_enc"] == [b["encoded_bytes"] for b in want["blocks"]]


def test_huffman_small(orc):
    h = G["huffman_small"]
    gt = orc.transpose(small_graph())
    off, mem, _ = orc.sample_block(gt, 500, 0, 42)
    sets = [mem[off[j]:off[j + 1]].tolist() for j in range(500)]
    cb = orc.codebook_from_sets(sets, 300)
    dump = "".join(f"{v} {int(cb.lens[v])} {cb.code(v)}\n" for v in range(300) if cb.lens[v])
    assert dump == h["codebook_dump"] and cb.coded_vertices == h["coded_vertices"]
    for s, e in zip(sets[:200], h["encoded"]):
        data, bl, cp = cb.encode(s, h["top"])
        assert (data.hex(), bl, cp) == (e["bits"], e["bit_length"], e["copied"])


def test_c1_reference_run(orc, im):
    c1 = G["c1"]
    g = im.generate_er(10000, 100000, 0)
    im.assign_weights_f32(g, "wc")
    csr = csr_of(g)
    assert sha(csr.off, csr.tgt, csr.prob) == c1["graph_sha"]
    got = orc.run(csr, 10, 0.5, 10, "huffman", 42, 8)
    assert got["seeds"] == c1["seeds"] and got["marginal"] == c1["marginal"] and got["coverage"] == c1["coverage"]
    for k, v in c1["stats"].items():
        assert got[k] == v, k
    for k, v in c1["plan"].items():
        assert got[k] == v, k
    off, mem, _ = orc.sample_block(orc.transpose(csr), 5000, 0, 42)
    assert sha(off, mem) == c1["sample_0_5000_sha"]


def test_c2_windows(orc, im):
    c2 = G["c2"]
    g = im.generate_rmat(18, 16, 0.57, 0.19, 0.19, 1)
    im.assign_weights_f32(g, "uniform", 0.01)
    csr = csr_of(g)
    assert sha(csr.off, csr.tgt, csr.prob) == c2["graph_sha"]
    gt = orc.transpose(csr)
    w = c2["windows"][0]  # one window keeps the CPU suite short; the GPU suite checks all
    off, mem, _ = orc.sample_block(gt, w["count"], w["first"], 42)
    assert sha(off, mem) == w["sha"]
