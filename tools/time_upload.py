"""Time of the e2e leg's graph upload alone (config 5: 5.74 GB of pinned CSR) -- dev tooling."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2208_00613_b200 as im
import bench

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dev = im.default_device(0)
gen = cfg["gen"]
dg = im.DeviceGraph.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], weights=cfg["weights"][0], p=cfg["weights"][1], device=dev)
off, tgt, _ = dg.download(probs=False)
n = int(off.size - 1)
p_off, p_tgt = bench.pinned_copy(off), bench.pinned_copy(tgt)
nbytes = p_off.nbytes + p_tgt.nbytes
for rep in range(4):
    dev.synchronize(); t0 = time.perf_counter()
    g = im.DeviceGraph.from_arrays(n, p_off, p_tgt, None, True, device=dev, weights=cfg["weights"][0], p=cfg["weights"][1])
    dev.synchronize(); t1 = time.perf_counter()
    del g
    dev.synchronize(); t2 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):.1f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s incl. setup kernels), free {1e3*(t2-t1):.1f} ms")
# raw copy rate of the same pinned buffer through torch
t = torch.empty(p_tgt.nbytes, dtype=torch.uint8, device="cuda")
src = torch.from_numpy(p_tgt.view(np.uint8))
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    t.copy_(src, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"torch copy {p_tgt.nbytes/1e9:.2f} GB: {1e3*(t1-t0):.1f} ms = {p_tgt.nbytes/(t1-t0)/1e9:.1f} GB/s (is_pinned={src.is_pinned()})")
