"""The command line (proj/tests/test_cli.cpp): flags, exit codes, outputs.  Usage and input
errors are host-side (CPU); the end-to-end cases run the B200 path (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(args, cwd):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    p = subprocess.run([sys.executable, "-m", "paper_2208_00613_b200"] + args.split(), cwd=cwd, env=env,
                       capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def write_demo_graph(path):
    # test_cli.cpp:35-42: two communities with a hub in each
    lines = ["# demo"] + [f"0 {i}" for i in range(1, 7)] + [f"7 {i}" for i in range(8, 14)] + ["3 7", "10 0"]
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def test_missing_required_flag_exits_2(tmp_path):
    write_demo_graph(tmp_path / "demo.txt")
    assert run_cli("--input demo.txt", tmp_path)[0] == 2
    assert run_cli("--k 2", tmp_path)[0] == 2
    assert run_cli("--input demo.txt --k 2 --mode zstd", tmp_path)[0] == 2
    assert run_cli("--input demo.txt --k 2 --blocks 1", tmp_path)[0] == 2
    assert run_cli("--input demo.txt --k 2 --p 1.5", tmp_path)[0] == 2
    assert run_cli("--help", tmp_path)[0] == 0


def test_runtime_failures_exit_1(tmp_path):
    rc, _, err = run_cli("--input no_such_file.txt --k 2", tmp_path)
    assert rc == 1 and err.startswith("error: ")
    (tmp_path / "bad.txt").write_text("0 1\nbroken line here\n")
    assert run_cli("--input bad.txt --k 2", tmp_path)[0] == 1


@pytest.mark.gpu
def test_end_to_end_run_writes_seeds_and_stats(tmp_path):
    write_demo_graph(tmp_path / "demo.txt")
    rc, out, err = run_cli("--input demo.txt --k 2 --epsilon 0.5 --seed 42 --seeds-out seeds.txt "
                           "--stats-json stats.json", tmp_path)
    assert rc == 0, err
    assert len((tmp_path / "seeds.txt").read_text().splitlines()) == 2
    stats = json.loads((tmp_path / "stats.json").read_text())
    assert stats["n"] == 14 and len(stats["seeds"]) == 2
    assert isinstance(stats["compression_ratio"], float) and stats["plan"]["rng_seed"] == 42
    assert list(stats) == ["n", "m", "theta", "skewness", "density", "mode", "mode_override", "phase_seconds",
                           "raw_bytes", "encoded_bytes", "compression_ratio", "peak_bytes", "padded_seeds",
                           "uncoded_vertex_fraction", "blocks", "seeds", "plan", "original_ids", "rss_bytes"]
    assert out.startswith("n=14 m=") and "\nseeds:" in out and "coverage=" in out


@pytest.mark.gpu
def test_seeds_reported_as_original_ids(tmp_path):
    (tmp_path / "sparse.txt").write_text("1000 2000\n1000 3000\n1000 4000\n")
    assert run_cli("--input sparse.txt --k 1 --seed 1 --seeds-out seeds.txt --stats-json stats.json",
                   tmp_path)[0] == 0
    assert (tmp_path / "seeds.txt").read_text() == "1000\n"
    stats = json.loads((tmp_path / "stats.json").read_text())
    assert stats["seeds"][0]["id"] == 1000 and stats["original_ids"][0] == 1000


@pytest.mark.gpu
def test_forced_mode_is_honored(tmp_path):
    write_demo_graph(tmp_path / "demo.txt")
    assert run_cli("--input demo.txt --k 2 --mode bitmap --seed 9 --stats-json stats.json", tmp_path)[0] == 0
    assert json.loads((tmp_path / "stats.json").read_text())["mode"] == "bitmap"


@pytest.mark.gpu
def test_identical_across_worker_counts(tmp_path):
    write_demo_graph(tmp_path / "demo.txt")
    outs = set()
    for w in (1, 2, 4):
        assert run_cli(f"--input demo.txt --k 3 --seed 5 --workers {w} --seeds-out seeds.txt", tmp_path)[0] == 0
        outs.add((tmp_path / "seeds.txt").read_text())
    assert len(outs) == 1


@pytest.mark.gpu
def test_binary_cache_round_trip(tmp_path):
    write_demo_graph(tmp_path / "demo.txt")
    assert run_cli("--input demo.txt --k 2 --seed 3 --save-binary cache.bin --seeds-out a.txt", tmp_path)[0] == 0
    assert run_cli("--input cache.bin --format binary --k 2 --seed 3 --seeds-out b.txt", tmp_path)[0] == 0
    assert (tmp_path / "a.txt").read_text() == (tmp_path / "b.txt").read_text()


@pytest.mark.gpu
def test_uniform_weight_model_flag(tmp_path):
    write_demo_graph(tmp_path / "demo.txt")
    assert run_cli("--input demo.txt --k 1 --weight-model uniform --p 1.0 --stats-json stats.json", tmp_path)[0] == 0
    assert json.loads((tmp_path / "stats.json").read_text())["seeds"][0]["cumulative"] > 0.0


@pytest.mark.gpu
def test_cli_matches_reference_stats_schema_values(tmp_path, orc):
    # the same run through the oracle: seeds and the deterministic stats fields agree
    from conftest import csr_of
    import paper_2208_00613_b200 as immx

    write_demo_graph(tmp_path / "demo.txt")
    assert run_cli("--input demo.txt --k 2 --seed 42 --stats-json stats.json", tmp_path)[0] == 0
    stats = json.loads((tmp_path / "stats.json").read_text())
    g = immx.load_edge_list(str(tmp_path / "demo.txt"))
    immx.assign_weights(g, "wc")
    o = orc.run(csr_of(g), 2, 0.5, 8, "auto", 42)
    assert [s["id"] for s in stats["seeds"]] == [int(g.original_ids[v]) for v in o["seeds"]]
    for key in ("theta", "raw_bytes", "encoded_bytes", "compression_ratio", "peak_bytes", "mode"):
        assert stats[key] == o[key], key
