"""immx_graph_upload_model: the probabilities come from a weight model applied on the device
(assign_weights, graph.cpp:146-157, float32 values) instead of per-edge f64 arrays.  The device
graph -- CSR, probability mode, thresholds -- and the samples must equal the per-edge upload of
the same graph with assign_weights_f32 on the host."""
import numpy as np
import pytest

from conftest import csr_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,p", [("wc", 0.0), ("uniform", 0.01), ("uniform", 1.0), ("uniform", 0.0)])
@pytest.mark.parametrize("transposed", [False, True])
def test_model_upload_equals_per_edge_upload(im, orc, model, p, transposed):
    g = im.generate_rmat(12, 8, 0.57, 0.19, 0.19, 5)
    im.assign_weights_f32(g, model, p)
    off, tgt, pr, _ = g.arrays()
    if transposed:
        gt = orc.transpose(csr_of(g))
        off, tgt, pr = gt.off, gt.tgt, gt.prob
    a = im.DeviceGraph.from_arrays(int(off.size - 1), off, tgt, pr, transposed)
    b = im.DeviceGraph.from_arrays(int(off.size - 1), off, tgt, None, transposed, weights=model, p=p)
    ra, ca, pa = a.download()
    rb, cb, pb = b.download()
    assert np.array_equal(ra, rb) and np.array_equal(ca, cb) and np.array_equal(pa, pb)
    assert a.prob_mode == b.prob_mode
    pa_ = im.Pool(a.device)
    pa_.sample(a, 500, 0, 42)
    pb_ = im.Pool(b.device)
    pb_.sample(b, 500, 0, 42)
    for x, y in zip(pa_.read(), pb_.read()):
        assert np.array_equal(x, y)


def test_model_upload_rejects_bad_arguments(im):
    off = np.array([0, 1, 1], np.uint64)
    tgt = np.array([1], np.uint32)
    with pytest.raises(ValueError):
        im.DeviceGraph.from_arrays(2, off, tgt, None, False, weights="uniform", p=1.5)
    with pytest.raises(ValueError):
        im.DeviceGraph.from_arrays(2, off, tgt, None, False, weights="lt")


@pytest.mark.parametrize("kind", ["sorted", "repeats", "unsorted", "repeat_at_row_end", "descent_only_across_rows"])
def test_model_upload_row_order_detection(im, orc, monkeypatch, kind):
    """The model upload finds "some row is not strictly increasing" by counting descents over all
    adjacent edge pairs and over the row-straddling ones (device_graph.cu k_edge_descents /
    k_row_bounds); the per-edge upload scans row by row.  With the long-row path forced onto
    every row (it requires distinct targets per row and is switched off otherwise), samples from
    both uploads must agree with each other and with the oracle."""
    monkeypatch.setenv("IMMX_LONG_MIN", "1")
    rng = np.random.default_rng(5)
    n = 300
    rows = []
    for v in range(n):
        d = int(rng.integers(0, 12))
        rows.append(np.sort(rng.choice(n, size=d, replace=False)).astype(np.uint32))
    if kind == "repeats":
        rows[7] = np.array([3, 9, 9, 20], np.uint32)
    elif kind == "unsorted":
        rows[11] = np.array([40, 12, 77], np.uint32)
    elif kind == "repeat_at_row_end":
        rows[n - 1] = np.array([5, 8, 8], np.uint32)
    elif kind == "descent_only_across_rows":  # strictly increasing rows; row v ends above row v+1's start
        rows[20] = np.array([100, 200, 299], np.uint32)
        rows[21] = np.array([0, 1], np.uint32)
        rows[22] = np.array([], np.uint32)  # an empty row between two straddling ones
        rows[23] = np.array([0, 250], np.uint32)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([r.size for r in rows])
    tgt = np.concatenate(rows).astype(np.uint32)
    pr = np.full(tgt.size, float(np.float32(0.3)), np.float64)
    a = im.DeviceGraph.from_arrays(n, off, tgt, pr, True)
    b = im.DeviceGraph.from_arrays(n, off, tgt, None, True, weights="uniform", p=0.3)
    pa_ = im.Pool(a.device)
    pa_.sample(a, 800, 0, 7)
    pb_ = im.Pool(b.device)
    pb_.sample(b, 800, 0, 7)
    for x, y in zip(pa_.read(), pb_.read()):
        assert np.array_equal(x, y)
    from oracle.oracle import CSR  # the oracle on the same reverse CSR

    want = orc.sample_block(CSR(n, off, tgt, pr), 800, 0, 7)
    got = pb_.read()
    assert np.array_equal(want[0], got[0]) and np.array_equal(want[1], got[1])
