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
