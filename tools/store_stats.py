"""Per-set copied (uncodable) member counts of a config's Huffman store (dev tooling)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import bench
import paper_2208_00613_b200 as im

cfg = bench.CONFIGS[sys.argv[1]]
dev = im.default_device()
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
r = im.run_device(dg, cfg["k"], epsilon=cfg["eps"], blocks=cfg["blocks"], mode=cfg["mode"], seed=42, model=model,
                  keep=True)
bo, by, bl, co, cp = r["_store"].read(0, r["theta"])
nc = np.diff(co.astype(np.int64))
print("theta", r["theta"], "uncoded frac", r["uncoded_vertex_fraction"], "copied total", nc.sum(),
      "max", nc.max(), "p99", np.percentile(nc, 99), "sets>32", (nc > 32).sum(), "sets>128", (nc > 128).sum())
