"""Bit-exact parity at the BASELINE configs against the UNMODIFIED reference.

Goldens: tests/golden/<config>_run.json, written by tests/golden/make_config_golden.py from
oracle/_ref (the reference compiled from its sources, OpenMP) on the graphs of
oracle/gen_graph.c.  For each config the device must reproduce:

* the graph: SHA-256 of G^T (row offsets, column ids) -- the device generator (c2..c5) or
  the host generator + device transpose (c1) against the CPU generator;
* the full run (pipeline.cpp:47-178): seeds, marginals, coverage, padding, theta plan,
  characterization, block stats, raw/encoded bytes, compression ratio, ledger peak, uncoded
  fraction.  c5 runs the per-set hybrid store, which must hold no dense set and then IS the
  Huffman store, so it is compared with the reference's Huffman run;
* block 1 as the reference's public functions compute it: the histogram, the Huffman
  codebook (bits and lengths of every vertex), the encode `top`, and the encoded bitstreams,
  bit lengths and copy buffers of a window of sets -- read back from the run's own store;
* raw sample windows at the start of block 1 and at the end of [0, theta).

Each config is skipped until its golden exists (c4/c5 take 1-2 h of reference CPU time).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CONFIGS = {
    "c1": dict(gen=("er", 10000, 100000, 0), weights=("wc", 0.0), k=10, eps=0.5, blocks=10, mode="huffman"),
    "c2": dict(gen=("rmat", 18, 16, 1), weights=("uniform", 0.01), k=50, eps=0.5, blocks=8, mode="huffman"),
    "c4": dict(gen=("rmat", 22, 24, 3), weights=("wc", 0.0), k=100, eps=0.13, blocks=8, mode="huffman"),
    "c5": dict(gen=("rmat", 25, 42, 4), weights=("wc", 0.0), k=50, eps=0.5, blocks=8, mode="hybrid"),
}


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def golden(name):
    path = os.path.join(GOLDEN, f"{name}_run.json")
    if not os.path.exists(path):
        pytest.skip(f"{name}_run.json not generated yet (tests/golden/make_config_golden.py {name})")
    with open(path) as f:
        return json.load(f)


def device_graph(im, cfg):
    gen, (model, p) = cfg["gen"], cfg["weights"]
    if gen[0] == "rmat":
        return im.DeviceGraph.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], weights=model, p=p)
    g = im.generate_er(*gen[1:])
    im.assign_weights_f32(g, model, p)
    return im.DeviceGraph(g, transposed=False)  # transposed on the device


_CACHE = {}


def config_run(im, name):
    """(golden, device graph, run result with its store) -- one run per config per session."""
    if name not in _CACHE:
        _CACHE.clear()  # one large config resident at a time
        gd = golden(name)
        cfg = CONFIGS[name]
        dg = device_graph(im, cfg)
        # the golden's worker count: the reference's selection ledger (per-worker frequency
        # tables and decode buffers, select.cpp:75-79, :218-223) depends on it
        r = im.run_device(dg, cfg["k"], epsilon=cfg["eps"], blocks=cfg["blocks"], mode=cfg["mode"], seed=42,
                          workers=gd["workers"], keep=True)
        _CACHE[name] = (gd, dg, r)
    return _CACHE[name]


@pytest.mark.parametrize("name", list(CONFIGS))
def test_graph_equals_reference_generator(im, name):
    gd, dg, _ = config_run(im, name)
    off, tgt, _ = dg.download(probs=False)
    assert (off.size - 1, tgt.size) == (gd["graph"]["n"], gd["graph"]["m"])
    assert sha(off, tgt) == gd["graph"]["gt_sha"]


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_run_equals_reference(im, name):
    gd, dg, r = config_run(im, name)
    ref = gd["run"]
    assert r["seeds"] == ref["seeds"]
    assert r["marginal"] == ref["marginal"]
    assert r["coverage"] == ref["coverage"]  # covered / theta in FP64: exact
    assert r["padded"] == ref["padded"]
    st = ref["stats"]
    assert r["theta"] == st["theta"]
    assert r["estimation_samples"] == ref["plan"]["estimation_samples"]
    assert r["exit_iteration"] == ref["plan"]["exit_iteration"]
    assert r["covered_fraction"] == ref["plan"]["covered_fraction"]
    assert r["skewness"] == st["skewness"] and r["density"] == st["density"]
    if CONFIGS[name]["mode"] == "hybrid":
        assert r["dense_sets"] == 0  # no set above n/32: the hybrid store is the Huffman store
    else:
        assert r["mode"] == st["mode"]
    for key in ("raw_bytes", "encoded_bytes", "compression_ratio", "peak_bytes", "uncoded_vertex_fraction"):
        assert r[key] == st[key], key
    assert [{"sets": s, "raw_bytes": a, "encoded_bytes": e}
            for s, a, e in zip(r["block_sets"], r["block_raw"], r["block_enc"])] == ref["blocks"]
    # influence estimate = coverage x n, within the north star's 1e-6 relative (exact here)
    n = gd["graph"]["n"]
    assert abs(r["coverage"][-1] * n - ref["coverage"][-1] * n) <= 1e-6 * ref["coverage"][-1] * n


@pytest.mark.parametrize("name", list(CONFIGS))
def test_block1_codebook_and_bitstreams_equal_reference(im, name):
    gd, dg, r = config_run(im, name)
    b1 = gd["block1"]
    n = gd["graph"]["n"]
    store = r["_store"]
    bits, lens = store.codebook(n)
    assert int((lens > 0).sum()) == b1["coded"] == r["coded_vertices"]
    assert int(lens.max()) == b1["max_code_len"]
    assert sha(bits, lens) == b1["codebook_sha"]
    lo, hi = b1["window"]
    bo, by, bl, co, cp = store.read(lo, hi)
    assert int(bo[-1]) == b1["enc_bytes"] and int(co[-1]) == b1["enc_copied"]
    assert sha(bo, by, bl, co, cp) == b1["enc_sha"]


@pytest.mark.parametrize("name", list(CONFIGS))
def test_block1_histogram_top_and_windows_equal_reference(im, name):
    gd, dg, r = config_run(im, name)
    b1 = gd["block1"]
    n = gd["graph"]["n"]
    pool = im.Pool(dg.device)
    pool.sample(dg, b1["per_block"], 0, 42)
    hist = pool.histogram(n)
    assert int(hist.sum()) == b1["members"]
    assert sha(hist) == b1["hist_sha"]
    assert int(np.argmax(hist)) == b1["top"]  # table_argmax: lowest id among the maxima
    lo, hi = b1["window"]
    off, mem = pool.read(lo, hi)
    assert sha(off, mem) == b1["raw_sha"]
    del pool
    tw = gd["tail_window"]
    pool = im.Pool(dg.device)
    pool.sample(dg, tw["count"], tw["first"], 42)
    off, mem = pool.read()
    assert int(mem.size) == tw["members"]
    assert sha(off, mem) == tw["sha"]


def test_c3_lt_full_run_equals_oracle(im, orc):
    """c3 (LT) has no reference counterpart: the device's full hybrid LT IMM run
    against the C restatement's (oc_run_lt), both on the generator's graph and weights."""
    g = orc.generate(("rmat", 20, 16, 2), ("wc", 0.0), reverse=False)
    gt, w = orc.generate(("rmat", 20, 16, 2), ("wc", 0.0), reverse=True, lt_seed=3)
    want = orc.run(g, 100, 0.5, 8, "hybrid", 42, lt_weights=w)
    dg = im.DeviceGraph.generate_rmat(20, 16, 0.57, 0.19, 0.19, 2, weights="wc")
    dg.set_lt_random(3)
    got = im.run_device(dg, 100, epsilon=0.5, blocks=8, mode="hybrid", seed=42, model=1)
    for key in ("seeds", "marginal", "coverage", "padded", "theta", "estimation_samples", "exit_iteration",
                "covered_fraction", "skewness", "density", "raw_bytes", "encoded_bytes", "peak_bytes",
                "coded_vertices", "dense_sets", "compression_ratio", "uncoded_vertex_fraction", "block_sets",
                "block_raw", "block_enc"):
        assert got[key] == want[key], key


def test_c5_sample_window_equals_oracle(im, orc):
    """A window of c5 samples against the C restatement on the device's own G^T (the
    reference golden's windows are checked above; this pins the oracle at c5 scale too)."""
    dg = im.DeviceGraph.generate_rmat(25, 42, 0.57, 0.19, 0.19, 4, weights="wc")
    off, tgt, pr = dg.download()
    from oracle.oracle import CSR

    gt = CSR(int(off.size - 1), off, tgt, pr)
    first, count = 1_500_000, 300
    pool = im.Pool(dg.device)
    pool.sample(dg, count, first, 42)
    got = pool.read()
    want = orc.sample_block(gt, count, first, 42)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_run_releases_raw_sets_and_reports_device_memory():
    """pipeline.cpp:129-133: raw blocks are dropped once encoded.  After a Huffman run only the
    graph and the compressed store stay in use; the high-water mark is reported.  (A fresh
    process: the in-use figure is process-wide.)"""
    import subprocess
    import sys

    from conftest import ROOT

    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "mem_probe.py"), "16"], capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    runs = [eval(line.split(" ", 1)[1]) for line in out.stdout.strip().splitlines()]
    for r in runs:
        assert r["device_graph_bytes"] > 0 and r["device_store_bytes"] > 0
        assert r["device_peak_bytes"] > r["device_resident_bytes"] > 0
        # resident = graph + store (+ the store's codes / decode table and per-device scalars)
        assert r["device_resident_bytes"] <= r["device_graph_bytes"] + 2 * r["device_store_bytes"] + (16 << 20)
    # repeated runs neither leak nor grow
    assert runs[2]["device_resident_bytes"] == runs[1]["device_resident_bytes"]


def test_second_device_context_refused(im):
    """One immx_device per process: the allocation stream is the context's work stream."""
    im.default_device()
    with pytest.raises(RuntimeError, match="one immx_device per process"):
        im.Device(0)
