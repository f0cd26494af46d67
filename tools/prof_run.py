"""Back-to-back IMM runs on a device-resident graph: wall vs the run's own phase clock.
  python tools/prof_run.py [--config c2] [--reps 5]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2208_00613_b200 as im  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--profile", type=int, default=0)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
g = bench.make_graph(im, cfg)
dev = im.default_device()
dg = im.DeviceGraph(g, transposed=False, device=dev)
dev.profile(bool(a.profile))
for r in range(a.reps):
    dev.reset_stats()
    t = time.perf_counter()
    out = im.run_device(dg, cfg["k"], epsilon=cfg["eps"], blocks=cfg["blocks"], mode=cfg["mode"], seed=42)
    wall = time.perf_counter() - t
    st = {k: dev.kernel_stats(k) for k in ("sample", "encode", "hselect")}
    print(f"rep {r}: wall {wall:.3f}s phases {out['phase_seconds']} theta {out['theta']} drawn {out['samples_drawn']} "
          f"sample_ms {st['sample']['ms']:.0f} enc_ms {st['encode']['ms']:.0f} hsel_ms {st['hselect']['ms']:.0f}",
          flush=True)
