"""Look-ahead sampling in the theta estimation (capi.cu estimate_theta_dev).

The device may draw the sets of several estimation iterations in one launch when the last
measured covered fraction says the iterations in between cannot exit (sampler.cpp:106-161
draws them one iteration at a time).  Every exit test still runs on exactly its first theta_i
sets, so the plan and every run result are the reference's whatever was drawn ahead:
IMMX_LOOKAHEAD=0 (off), the default margin, and "force" (always two iterations ahead -- the
pool then holds more sets than theta, in every store mode) must all equal the oracle."""
import numpy as np
import pytest

from conftest import random_graph
from test_gpu_parity import _cmp_run, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["0", "1.25", "force"])
def lookahead(request, monkeypatch):
    monkeypatch.setenv("IMMX_LOOKAHEAD", request.param)
    return request.param


def test_estimate_theta_plan(im, orc, lookahead):
    rng = np.random.default_rng(17)
    for trial in range(3):
        g = orc.assign_weights(random_graph(rng, 300 + 200 * trial, 2500 + 2500 * trial), "wc")
        gt = orc.transpose(g)
        want = orc.estimate_theta(gt, 4 + trial, 0.4, 7 + trial)
        got = im.estimate_theta(to_product(im, gt), 4 + trial, 0.4, 7 + trial)
        assert got == want


@pytest.mark.parametrize("mode", ["raw", "huffman", "bitmap", "hybrid"])
def test_runs_equal_oracle(im, orc, lookahead, mode):
    rng = np.random.default_rng(23)
    for trial in range(2):
        g = orc.assign_weights(random_graph(rng, 250 + 250 * trial, 2000 + 3000 * trial), "wc")
        if mode == "hybrid":
            o = orc.run(g, 6, 0.5, 4, "hybrid", 3 + trial)
            dg = im.DeviceGraph(to_product(im, g), transposed=False)
            r = im.run_device(dg, 6, epsilon=0.5, blocks=4, mode="hybrid", seed=3 + trial)
            for key in ("seeds", "marginal", "coverage", "padded", "theta", "encoded_bytes", "peak_bytes"):
                assert r[key] == o[key], key
            assert r["exit_iteration"] == o["exit_iteration"]
            assert r["estimation_samples"] == o["estimation_samples"]
        else:
            _cmp_run(im, orc, g, 6, 0.5, 4, mode, 3 + trial, workers=1 + trial)


def test_forced_lookahead_draws_past_theta(im, orc, monkeypatch):
    # the forced mode really leaves more sets in the pool than the run uses
    monkeypatch.setenv("IMMX_LOOKAHEAD", "force")
    rng = np.random.default_rng(29)
    g = orc.assign_weights(random_graph(rng, 400, 4000), "wc")
    o = orc.run(g, 5, 0.5, 4, "huffman", 11)
    dg = im.DeviceGraph(to_product(im, g), transposed=False)
    r = im.run_device(dg, 5, epsilon=0.5, blocks=4, mode="huffman", seed=11)
    assert r["seeds"] == o["seeds"] and r["theta"] == o["theta"]
    assert r["samples_drawn"] >= r["theta"]


@pytest.mark.parametrize("mode", ["raw", "huffman", "hybrid"])
def test_pilot_and_remembered_fraction(im, orc, monkeypatch, mode):
    """Iteration 1's look-ahead guess: a pilot's greedy coverage on a cold graph, the last
    estimation's covered fraction on a graph this device has run before (same k, epsilon).
    Both only choose how many sets a launch draws; plan and results stay the oracle's."""
    monkeypatch.setenv("IMMX_LOOKAHEAD", "1.25")
    monkeypatch.setenv("IMMX_LA_PILOT", "64")
    rng = np.random.default_rng(31)
    g = orc.assign_weights(random_graph(rng, 600, 6000), "wc")
    o = orc.run(g, 5, 0.5, 4, mode, 13)
    dg = im.DeviceGraph(to_product(im, g), transposed=False)
    drawn = []
    for rep in range(3):  # rep 0: pilot; rep 1, 2: the remembered fraction
        r = im.run_device(dg, 5, epsilon=0.5, blocks=4, mode=mode, seed=13)
        for key in ("seeds", "marginal", "coverage", "padded", "theta", "encoded_bytes", "peak_bytes"):
            assert r[key] == o[key], (rep, key)
        assert r["exit_iteration"] == o["exit_iteration"]
        assert r["estimation_samples"] == o["estimation_samples"]
        drawn.append(r["samples_drawn"])
    assert drawn[1] == drawn[2]
    # another k on the same graph: no remembered fraction for it, the pilot again
    o2 = orc.run(g, 9, 0.5, 4, mode, 13)
    r2 = im.run_device(dg, 9, epsilon=0.5, blocks=4, mode=mode, seed=13)
    assert r2["seeds"] == o2["seeds"] and r2["theta"] == o2["theta"] and r2["coverage"] == o2["coverage"]
    monkeypatch.setenv("IMMX_LA_PILOT", "0")
    r3 = im.run_device(dg, 5, epsilon=0.5, blocks=4, mode=mode, seed=13)
    assert r3["seeds"] == o["seeds"] and r3["theta"] == o["theta"]
