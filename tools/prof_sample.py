"""Profiling driver: one warm-up and one measured sampler launch on a BASELINE config graph.

  python tools/prof_sample.py [--config c2] [--count 30000] [--first 0]

Prints the device time (CUDA events, library stream) and algorithmic GB/s of the second
launch; under ncu capture it with -k regex:rrr_kernel -s <launches of the warm-up>."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2208_00613_b200 as im  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--count", type=int, default=30000)
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    t = time.time()
    dev = im.default_device()
    if cfg.get("device_gen"):
        gen = cfg["gen"]
        dg = im.DeviceGraph.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], weights=cfg["weights"][0],
                                          p=cfg["weights"][1], device=dev)
        dev.synchronize()
        print(f"device graph n={dg.n} m={dg.m} in {time.time() - t:.1f}s", flush=True)
    else:
        g = bench.make_graph(im, cfg)
        print(f"graph {g} in {time.time() - t:.1f}s", flush=True)
        dg = im.DeviceGraph(g, transposed=False, device=dev)
    model = 0
    if "lt_seed" in cfg:  # c3: LT walks (weights generated in HBM)
        dg.set_lt_random(cfg["lt_seed"])
        model = 1
    print("prob mode", dg.prob_mode, "model", "LT" if model else "IC", flush=True)
    for rep in range(a.reps):
        pool = im.Pool(dev)
        pool.sample(dg, 2048, a.first, 42, model)  # pilot: sizes the arena, so the measured batch is one launch
        dev.synchronize()
        dev.profile(True)
        dev.reset_stats()
        t = time.time()
        pool.sample(dg, a.count, a.first + 2048, 42, model)
        dev.synchronize()
        wall = time.time() - t
        st = dev.kernel_stats("sample")
        info = pool.info()
        gbs = st["bytes"] / (st["ms"] / 1e3) / 1e9 if st["ms"] else 0
        print(f"rep {rep}: {a.count} samples wall {wall*1e3:.1f} ms, kernel {st['ms']:.1f} ms in {st['launches']} "
              f"launches, {gbs:.1f} GB/s alg, members {info['members']}, edges {info['edges']}, "
              f"{info['edges'] / (st['ms'] / 1e3) / 1e9:.2f} Gedges/s", flush=True)


if __name__ == "__main__":
    main()
