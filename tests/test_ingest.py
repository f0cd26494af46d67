"""Host ingestion (graph_host.cpp, out of the hot path) against the reference's own parser,
transpose, weights and cache (the reference's pybind module built from its sources,
oracle/_ref/immx_ref) on fuzzed edge lists: comments, blank lines, CR line ends, self-loops,
duplicate edges, weights, undirected input and malformed lines.  CPU only."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def refcore():
    from oracle.oracle import load_ref_core

    core = load_ref_core()
    if core is None:
        pytest.skip("reference pybind module not built (make -C oracle ref)")
    return core


def fuzz_text(rng, n_lines):
    ids = rng.integers(0, 10 ** rng.integers(1, 12), size=rng.integers(3, 40)).tolist()
    lines = []
    for _ in range(n_lines):
        r = rng.random()
        if r < 0.05:
            lines.append("# comment " + str(rng.integers(0, 9)))
        elif r < 0.08:
            lines.append(" " * int(rng.integers(0, 3)))
        else:
            a, b = (ids[int(rng.integers(0, len(ids)))] for _ in range(2))
            sep = [" ", "\t", "  ", " \t"][int(rng.integers(0, 4))]
            line = f"{a}{sep}{b}"
            if rng.random() < 0.4:
                line += f"{sep}{rng.choice(['0.5', '1', '0.125', '3e-3', '2.0'])}"
            if rng.random() < 0.1:
                line += "\r"
            if rng.random() < 0.1:
                line = "  " + line
            lines.append(line)
    return "\n".join(lines) + ("\n" if rng.random() < 0.5 else "")


def same_graph(ours, ref):
    off, tgt, pr, ids = ours.arrays()
    assert off.tolist() == list(ref.offsets)
    assert tgt.tolist() == list(ref.targets)
    assert pr.tolist() == list(ref.probs)
    assert ids.tolist() == list(ref.original_ids)


@pytest.mark.parametrize("directed", [True, False])
def test_parser_equals_reference(im, refcore, directed):
    rng = np.random.default_rng(4 if directed else 5)
    for trial in range(60):
        text = fuzz_text(rng, int(rng.integers(1, 120)))
        try:
            want = refcore.load_edge_list_text(text, directed)
        except RuntimeError as e:
            with pytest.raises(RuntimeError) as got:
                im.load_edge_list_text(text, directed=directed)
            assert str(got.value) == str(e)
            continue
        ours = im.load_edge_list_text(text, directed=directed)
        same_graph(ours, want)
        same_graph(im.transpose(ours), refcore.transpose(want))
        im.assign_weights(ours, "wc")
        refcore.assign_weights(want, "wc", 0.1)
        same_graph(ours, want)


@pytest.mark.parametrize("bad", ["1", "1 2 3 4", "a b", "1 -2", "1 2 x", "1 2 -0.5", "1 2 inf", "1 2 nan",
                                 "99999999999999999999 1", "1 2 1e999", "+1 2", "0x1 2", "1 2 0.5x"])
def test_malformed_lines_match_reference(im, refcore, bad):
    # the same exception class and message (an id past 2^64-1 is the reference's uncaught
    # std::out_of_range "stoull" -> IndexError)
    text = f"0 1\n# c\n{bad}\n"
    with pytest.raises((RuntimeError, IndexError)) as want:
        refcore.load_edge_list_text(text, True)
    with pytest.raises(want.type) as got:
        im.load_edge_list_text(text, directed=True)
    assert str(got.value) == str(want.value)


def test_cache_round_trip_with_reference(im, refcore, tmp_path):
    rng = np.random.default_rng(9)
    text = fuzz_text(rng, 300)
    ours = im.load_edge_list_text(text, directed=True)
    im.assign_weights(ours, "uniform", 0.25)
    p = str(tmp_path / "g.bin")
    im.save_graph_cache(ours, p)
    back = refcore.load_graph_cache(p)
    off, tgt, pr, _ = ours.arrays()
    assert list(back.offsets) == off.tolist() and list(back.targets) == tgt.tolist()
    assert list(back.probs) == pr.tolist()
    q = str(tmp_path / "r.bin")
    refcore.save_graph_cache(back, q)
    again = im.load_graph_cache(q)
    assert [a.tolist() for a in again.arrays()[:3]] == [off.tolist(), tgt.tolist(), pr.tolist()]
