"""The drop-in boundary, exercised: the reference's OWN pybind module (proj/bindings/module.cpp)
rebuilt by integration/Makefile with integration/immx_b200_glue.cpp in place of sampler.cpp,
select.cpp and pipeline.cpp, so its sample_rrr / sample_block / estimate_theta / select_raw /
run execute on the GPU through libimmx_b200.so.  Its outputs must equal the UNMODIFIED
reference's goldens (tests/golden/, from oracle/_ref)."""
import glob
import importlib.util
import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

G = json.load(open(os.path.join(GOLDEN, "golden.json")))["cases"]


@pytest.fixture(scope="module")
def core():
    cands = glob.glob(os.path.join(ROOT, "integration", "_build", "immx_b200_ref", "_core*.so"))
    if not cands:
        pytest.skip("integration module not built (make -C integration; needs /root/reference)")
    spec = importlib.util.spec_from_file_location("_core", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    # the glue must be what runs: the module links the product library, not the reference's hot path
    maps = open("/proc/self/maps").read()
    assert "libimmx_b200.so" in maps
    return mod


def cache_graph(core, tmp_path, off, tgt, prob, name="g.bin"):
    """A forward graph into the reference's IMMXG1 cache format (graph.hpp:41-43), loaded by the
    module's own load_graph_cache."""
    n, m = off.size - 1, tgt.size
    path = str(tmp_path / name)
    with open(path, "wb") as f:
        f.write(b"IMMXG1")
        f.write(struct.pack("<QQ", n, m))
        f.write(np.ascontiguousarray(off, np.uint64).tobytes())
        f.write(np.ascontiguousarray(tgt, np.uint32).tobytes())
        f.write(np.ascontiguousarray(prob, np.float64).tobytes())
    return core.load_graph_cache(path)


@pytest.fixture(scope="module")
def small(core, tmp_path_factory):
    z = np.load(os.path.join(GOLDEN, "small.npz"))
    g = cache_graph(core, tmp_path_factory.mktemp("g"), z["off"], z["tgt"], z["prob"])
    return g, core.transpose(g)


def csr(sets):
    off = np.zeros(len(sets) + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in sets])
    return off.tolist(), [v for s in sets for v in s]


def test_sample_block_equals_reference(core, small):
    _, gt = small
    for key, (count, first) in (("sample_0_2000_seed42", (2000, 0)), ("sample_12345_500_seed42", (500, 12345))):
        sets = core.sample_block(gt, count, first, 1, 42, 4)
        off, mem = csr(sets)
        assert off == G["small"][key]["offsets"] and mem == G["small"][key]["members"]


def test_estimate_theta_equals_reference(core, small):
    _, gt = small
    assert core.estimate_theta(gt, 5, 0.5, 3, 2) == G["small"]["estimate_theta_k5_eps05_seed3"]


@pytest.mark.parametrize("mode", ["huffman", "bitmap", "raw", "auto"])
def test_run_equals_reference(core, small, mode):
    g, _ = small
    want = G["small"]["run_k5_eps05_b4_seed11_w2"][mode]
    out = core.run(g, 5, 0.5, 4, mode, 11, 2, False)
    st = json.loads(out["stats_json"])
    assert (out["seeds"], out["marginal"], out["coverage"], out["padded"]) == \
        (want["seeds"], want["marginal"], want["coverage"], want["padded"])
    assert {k: st[k] for k in want["stats"]} == want["stats"]
    assert {k: st["plan"][k] for k in want["plan"]} == want["plan"]
    assert st["blocks"] == want["blocks"]


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_run_equals_reference(core, orc, tmp_path, name):
    path = os.path.join(GOLDEN, f"{name}_run.json")
    gd = json.load(open(path))
    gen, weights = {"c1": (("er", 10000, 100000, 0), ("wc", 0.0)),
                    "c2": (("rmat", 18, 16, 1), ("uniform", 0.01))}[name]
    fg = orc.generate(gen, weights, reverse=False)
    g = cache_graph(core, tmp_path, fg.off, fg.tgt, fg.prob)
    out = core.run(g, gd["k"], gd["epsilon"], gd["blocks"], gd["mode"], 42, 8, False)
    st = json.loads(out["stats_json"])
    ref = gd["run"]
    assert out["seeds"] == ref["seeds"] and out["marginal"] == ref["marginal"]
    assert out["coverage"] == ref["coverage"] and out["padded"] == ref["padded"]
    assert {k: st[k] for k in ref["stats"]} == ref["stats"]
    assert {k: st["plan"][k] for k in ref["plan"]} == ref["plan"]
    assert st["blocks"] == ref["blocks"]


def test_sample_rrr_and_select_raw_equal_oracle(core, orc, small):
    _, gt = small
    from oracle.oracle import CSR

    z = np.load(os.path.join(GOLDEN, "small.npz"))
    ogt = orc.transpose(CSR(300, z["off"], z["tgt"], z["prob"]))
    for root, seed in ((0, 1), (17, 99), (299, 12345)):
        assert core.sample_rrr(gt, root, seed) == orc.sample_rrr(ogt, root, seed)
    sets = core.sample_block(gt, 700, 0, 1, 7, 1)
    off, mem = csr(sets)
    want = orc.select_raw(np.array(off, np.uint64), np.array(mem, np.uint32), 300, 6)
    got = core.select_raw(sets, 300, 6, 4, False)
    assert (got["seeds"], got["marginal"], got["coverage"], got["padded"]) == \
        (want["seeds"], want["marginal"], want["coverage"], want["padded"])
    with pytest.raises(ValueError, match="merged_argmax"):
        core.select_raw(sets, 300, 6, 4, True)
    assert core.table_argmax([3, 9, 9, 1]) == 1
    assert core.merged_argmax([[5, 0, 1], [0, 4, 4]]) == 0
