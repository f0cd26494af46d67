"""Golden vector for the headline config: the UNMODIFIED reference (oracle/_ref, built from
/root/reference with OpenMP) runs the full config-2 IMM (R-MAT 18 / EF 16, seed 1, uniform
p = fl32(0.01), k = 50, eps = 0.5, 8 blocks, huffman, rng seed 42).  Takes ~15 min on 8
cores; run here once, the result is committed as tests/golden/c2_run.json.

  python tests/golden/make_c2_run_golden.py
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_2208_00613_b200 as im  # noqa: E402  (host generator only)
from oracle.oracle import CSR, RefLib  # noqa: E402
from make_golden import graph_arrays, sha  # noqa: E402


def main():
    ref = RefLib()
    g = im.generate_rmat(18, 16, 0.57, 0.19, 0.19, 1)
    im.assign_weights_f32(g, "uniform", 0.01)
    o, t, p = graph_arrays(g)
    rg = ref.graph(CSR(262144, o, t, p))
    t0 = time.time()
    r = rg.run(50, 0.5, 8, "huffman", 42, os.cpu_count() or 1)
    dt = time.time() - t0
    st = r["stats"]
    out = {"graph_sha": sha(o, t, p), "seeds": r["seeds"], "marginal": r["marginal"], "coverage": r["coverage"],
           "padded": r["padded"],
           "stats": {k: st[k] for k in ("theta", "skewness", "density", "mode", "raw_bytes", "encoded_bytes",
                                        "compression_ratio", "peak_bytes", "uncoded_vertex_fraction")},
           "plan": {k: st["plan"][k] for k in ("exit_iteration", "estimation_samples", "covered_fraction")},
           "blocks": st["blocks"],
           "reference_seconds": dt, "reference_threads": os.cpu_count() or 1,
           "reference_phase_seconds": st.get("phase_seconds")}
    with open(os.path.join(HERE, "c2_run.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote c2_run.json in", round(dt, 1), "s")


if __name__ == "__main__":
    main()
