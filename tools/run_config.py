"""One IMM run of a BASELINE config on a device-generated or host-generated graph (dev tooling).
  python tools/run_config.py --config c5 [--reps 1]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2208_00613_b200 as im  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dev = im.default_device()
t = time.perf_counter()
if cfg.get("device_gen"):
    gen = cfg["gen"]
    dg = im.DeviceGraph.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], weights=cfg["weights"][0],
                                      p=cfg["weights"][1], device=dev)
else:
    dg = im.DeviceGraph(bench.make_graph(im, cfg), transposed=False, device=dev)
model = 0
if "lt_seed" in cfg:
    dg.set_lt_random(cfg["lt_seed"])
    model = 1
dev.synchronize()
print(f"graph n={dg.n} m={dg.m} built in {time.perf_counter() - t:.2f}s", flush=True)
dev.profile(True)
for r in range(a.reps):
    dev.reset_stats()
    t = time.perf_counter()
    out = im.run_device(dg, cfg["k"], epsilon=cfg["eps"], blocks=cfg["blocks"], mode=cfg["mode"], seed=42, model=model)
    wall = time.perf_counter() - t
    st = dev.kernel_stats("sample")
    print(f"rep {r}: wall {wall:.2f}s theta {out['theta']} exit {out['exit_iteration']} est {out['estimation_samples']} "
          f"phases {out['phase_seconds']} ratio {out['compression_ratio']:.3f} store {out['device_store_bytes']/1e9:.2f} GB "
          f"edges {out['edges_scanned']:.3e} sample_ms {st['ms']:.0f} ({out['edges_scanned'] / (st['ms'] / 1e3) / 1e9:.1f} "
          f"Gedges/s) seeds {out['seeds'][:6]} cov {out['coverage'][-1]:.5f} dense {out['dense_sets']} host {out['host_seconds']}", flush=True)
