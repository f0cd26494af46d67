"""The ``immx`` command line (proj/tools/immx_main.cpp) over the B200 path.

  python -m paper_2208_00613_b200 --input G --k K [--format edgelist|binary] [--directed]
      [--weight-model wc|uniform] [--p P] [--epsilon E] [--blocks B] [--mode M] [--workers W]
      [--seed S] [--stats-json F] [--seeds-out F] [--save-binary F]

Same flags, defaults and exit codes as the reference: 0 success, 2 usage error (argparse),
1 runtime error ("error: ..." on stderr).  Extensions (no reference counterpart): ``--mode
hybrid`` and ``--diffusion lt [--lt-seed N]``.
"""
import argparse
import os
import sys


def _range(lo, hi, kind):
    def check(text):
        try:
            x = kind(text)
        except ValueError:
            raise argparse.ArgumentTypeError(f"{text!r} is not a valid {kind.__name__}")
        if not lo <= x <= hi:
            raise argparse.ArgumentTypeError(f"{x} not in [{lo} - {hi}]")
        return x

    return check


def parser():
    ap = argparse.ArgumentParser(prog="immx", description="IMM influence maximization over Huffman- or "
                                 "bitmap-encoded RRR sets (B200 path)")
    ap.add_argument("--input", required=True, help="input graph path")
    ap.add_argument("--format", default="edgelist", choices=["edgelist", "binary"], help="input format")
    ap.add_argument("--directed", action="store_true", help="treat edge list lines as directed edges")
    ap.add_argument("--weight-model", default="wc", choices=["wc", "uniform"], help="edge probability model")
    ap.add_argument("--p", type=_range(0.0, 1.0, float), default=0.1, help="probability for --weight-model uniform")
    ap.add_argument("--k", type=_range(0, 2 ** 32 - 1, int), required=True, help="number of seeds")
    ap.add_argument("--epsilon", type=float, default=0.5, help="approximation factor")
    ap.add_argument("--blocks", type=_range(2, 1000000, int), default=8,
                    help="sampling blocks (block 1 is the warm-up)")
    ap.add_argument("--mode", default="auto", choices=["auto", "huffman", "bitmap", "raw", "hybrid"],
                    help="encoding mode (hybrid: extension)")
    ap.add_argument("--workers", type=int, default=int(os.environ.get("IMMX_WORKERS", "1") or 1),
                    help="worker count (env IMMX_WORKERS sets the default)")
    ap.add_argument("--seed", type=_range(0, 2 ** 64 - 1, int), default=42,
                    help="rng seed; all randomness flows from it")
    ap.add_argument("--stats-json", default="", help="write run stats as JSON here")
    ap.add_argument("--seeds-out", default="", help="write seed ids here, one per line")
    ap.add_argument("--save-binary", default="", help="write the parsed graph as an IMMXG1 cache")
    ap.add_argument("--diffusion", default="ic", choices=["ic", "lt"], help="diffusion model (lt: extension)")
    ap.add_argument("--lt-seed", type=int, default=0, help="LT in-weight generator seed (extension)")
    return ap


def main(argv=None):
    args = parser().parse_args(argv)  # usage errors exit 2
    try:
        import paper_2208_00613_b200 as immx

        g = immx.load_graph_cache(args.input) if args.format == "binary" else immx.load_edge_list(
            args.input, args.directed)
        if args.save_binary:
            immx.save_graph_cache(g, args.save_binary)
        immx.assign_weights(g, args.weight_model, args.p)
        out = immx.run(g, args.k, epsilon=args.epsilon, blocks=args.blocks, mode=args.mode, seed=args.seed,
                       workers=args.workers, diffusion=args.diffusion, lt_seed=args.lt_seed)
        st = out["stats"]
        if args.seeds_out:
            immx.write_seeds(st, args.seeds_out)
        if args.stats_json:
            immx.write_stats(st, args.stats_json)
        print(f"n={st['n']} m={st['m']} theta={st['theta']} mode={st['mode']}"
              f"{' (override)' if st['mode_override'] else ''} S={st['skewness']:g} D={st['density']:g}"
              f" compression={st['compression_ratio']:g} peak_bytes={st['peak_bytes']}")
        print("seeds:" + "".join(f" {i}" for i in out["seed_ids"]))
        cov = out["coverage"][-1] if out["coverage"] else 0.0
        print(f"coverage={cov:g} time={st['phase_seconds']['total']:g}s")
        return 0
    except Exception as e:  # runtime failures exit 1 (immx_main.cpp:90-93)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
