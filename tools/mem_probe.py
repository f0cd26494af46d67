"""Device memory of repeated runs (dev tooling): peak / resident per run."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_00613_b200 as im

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dg = im.DeviceGraph.generate_rmat(scale, 16, 0.57, 0.19, 0.19, 5, weights="wc")
for i in range(3):
    r = im.run_device(dg, 20, epsilon=0.5, blocks=8, mode="huffman", seed=42)
    print(i, {k: r[k] for k in ("theta", "device_peak_bytes", "device_resident_bytes", "device_graph_bytes",
                                "device_store_bytes", "estimation_samples")}, flush=True)
