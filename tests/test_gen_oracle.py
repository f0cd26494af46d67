"""oracle/gen_graph.c (the CPU statement of the config graphs the bench's reference arm and
the golden scripts use) against the product's host generator, and the reference arm's
isolation from the product library.  CPU only."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


CASES = [(("er", 10000, 100000, 0), ("wc", 0.0)), (("er", 300, 3000, 7), ("uniform", 0.1)),
         (("rmat", 10, 8, 5), ("wc", 0.0)), (("rmat", 14, 16, 7), ("uniform", 0.01)),
         (("rmat", 18, 16, 1), ("uniform", 0.01))]


@pytest.mark.parametrize("gen,weights", CASES)
def test_generator_equals_product_host_generator(orc, im, gen, weights):
    h = im.generate_er(*gen[1:]) if gen[0] == "er" else im.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3])
    im.assign_weights_f32(h, *weights)
    off, tgt, pr, _ = h.arrays()
    g = orc.generate(gen, weights, reverse=False)
    assert np.array_equal(g.off, off) and np.array_equal(g.tgt, tgt) and np.array_equal(g.prob, pr)
    t = im.transpose(h)
    toff, ttgt, tpr, _ = t.arrays()
    gt = orc.generate(gen, weights, reverse=True)
    assert np.array_equal(gt.off, toff) and np.array_equal(gt.tgt, ttgt) and np.array_equal(gt.prob, tpr)


def test_lt_weights_equal_product(orc, im):
    gen = ("rmat", 14, 16, 2)
    h = im.transpose(im.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2))
    want = im.lt_weights(h, 3)
    gt, w = orc.generate(gen, ("wc", 0.0), reverse=True, lt_seed=3)
    assert np.array_equal(w, want)
    # normalised per row (rows with in-edges sum to ~1 in f32)
    s = np.add.reduceat(w.astype(np.float64), gt.off[:-1][np.diff(gt.off) > 0].astype(np.int64))
    assert np.allclose(s, 1.0, atol=1e-5)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_golden_graph_sha(orc, name):
    path = os.path.join(GOLDEN, f"{name}_run.json")
    if not os.path.exists(path):
        pytest.skip(f"{name}_run.json not generated")
    gd = json.load(open(path))
    cfg = {"c1": (("er", 10000, 100000, 0), ("wc", 0.0)), "c2": (("rmat", 18, 16, 1), ("uniform", 0.01))}[name]
    gt = orc.generate(*cfg, reverse=True)
    assert (gt.n, gt.m) == (gd["graph"]["n"], gd["graph"]["m"])
    assert _sha(gt.off, gt.tgt) == gd["graph"]["gt_sha"]


def test_reference_arm_never_maps_product_library():
    """bench.py --impl reference must run the reference (oracle/_ref) with no product code."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libimmx_ref.so")):
        pytest.skip("oracle/_ref not built")
    code = ("import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', "
            "'--warmup', '3', '--ref-samples', '2000']; import bench; bench.main(); "
            "maps = open('/proc/self/maps').read(); print('MAPPED', 'libimmx_b200' in maps, "
            "'paper_2208_00613_b200' in sys.modules)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["workload"] == "c1"
    assert lines[-1] == "MAPPED False False"
