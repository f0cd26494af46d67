"""Generate golden vectors from the REFERENCE itself (oracle/_ref, compiled from
/root/reference/proj sources by oracle/Makefile).  Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Writes tests/golden/golden.json (+ small.npz with the small graph).  The inputs come from
the product's deterministic host generators (input generation only); every OUTPUT here is
produced by the unmodified reference code (sample_block, estimate_theta, run, and the
pybind module's build_codebook / encode_rrr)."""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_2208_00613_b200 as im  # noqa: E402  (host generators only)
from oracle.oracle import CSR, RefLib, load_ref_core  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def graph_arrays(g):
    off, tgt, pr, _ = g.arrays()
    return off, tgt, pr


def main():
    ref = RefLib()
    core = load_ref_core()
    out = {"generated_by": "oracle/_ref (reference sources, unmodified)", "cases": {}}

    # ---- small graph: full outputs ----
    g = im.generate_er(300, 3000, 7)
    im.assign_weights_f32(g, "wc")
    off, tgt, pr = graph_arrays(g)
    np.savez_compressed(os.path.join(HERE, "small.npz"), off=off, tgt=tgt, prob=pr)
    rg = ref.graph(CSR(300, off, tgt, pr))
    rgt = rg.transpose()
    gt = rgt.csr()
    small = {"n": 300, "graph_sha": sha(off, tgt, pr), "gt_sha": sha(gt.off, gt.tgt, gt.prob)}
    so, sm = rgt.sample_block(2000, 0, 42, 4)
    small["sample_0_2000_seed42"] = {"offsets": so.tolist(), "members": sm.tolist()}
    so2, sm2 = rgt.sample_block(500, 12345, 42, 4)
    small["sample_12345_500_seed42"] = {"offsets": so2.tolist(), "members": sm2.tolist()}
    small["estimate_theta_k5_eps05_seed3"] = rgt.estimate_theta(5, 0.5, 3, 2)
    runs = {}
    for mode in ("huffman", "bitmap", "raw", "auto"):
        r = rg.run(5, 0.5, 4, mode, 11, 2)
        st = r["stats"]
        runs[mode] = {"seeds": r["seeds"], "marginal": r["marginal"], "coverage": r["coverage"],
                      "padded": r["padded"],
                      "stats": {k: st[k] for k in ("theta", "skewness", "density", "mode", "raw_bytes", "encoded_bytes",
                                                   "compression_ratio", "peak_bytes", "uncoded_vertex_fraction")},
                      "plan": {k: st["plan"][k] for k in ("exit_iteration", "estimation_samples", "covered_fraction")},
                      "blocks": st["blocks"]}
    small["run_k5_eps05_b4_seed11_w2"] = runs
    # uniform p graph
    gu = im.generate_er(300, 3000, 8)
    im.assign_weights_f32(gu, "uniform", 0.1)
    offu, tgtu, pru = graph_arrays(gu)
    rgu = ref.graph(CSR(300, offu, tgtu, pru)).transpose()
    sou, smu = rgu.sample_block(2000, 0, 42, 4)
    small["uniform01"] = {"graph_sha": sha(offu, tgtu, pru), "sample_sha": sha(sou, smu), "members": int(smu.size)}
    out["cases"]["small"] = small

    # ---- Huffman via the reference's pybind module (codebook + bitstreams) ----
    if core is not None:
        sets = [sm[so[j]:so[j + 1]].tolist() for j in range(500)]
        cb = core.build_codebook(sets, 300)
        dump = cb.dump()
        hist = np.bincount(np.concatenate([np.array(s) for s in sets]), minlength=300)
        top = int(np.argmax(hist))
        encs = []
        for s in sets[:200]:
            e = core.encode_rrr(cb, s, top)
            encs.append({"bits": e.bits.hex(), "bit_length": e.bit_length, "copied": list(e.copied)})
        out["cases"]["huffman_small"] = {"codebook_dump": dump, "top": top, "encoded": encs,
                                         "coded_vertices": cb.coded_vertices}

    # ---- config 1 (ER 10k/100k, fl32 WC): the full reference run ----
    g1 = im.generate_er(10000, 100000, 0)
    im.assign_weights_f32(g1, "wc")
    o1, t1, p1 = graph_arrays(g1)
    rg1 = ref.graph(CSR(10000, o1, t1, p1))
    r1 = rg1.run(10, 0.5, 10, "huffman", 42, 8)
    st = r1["stats"]
    c1 = {"graph_sha": sha(o1, t1, p1), "seeds": r1["seeds"], "marginal": r1["marginal"], "coverage": r1["coverage"],
          "stats": {k: st[k] for k in ("theta", "skewness", "density", "mode", "raw_bytes", "encoded_bytes",
                                       "compression_ratio", "peak_bytes", "uncoded_vertex_fraction")},
          "plan": {k: st["plan"][k] for k in ("exit_iteration", "estimation_samples", "covered_fraction")},
          "blocks": st["blocks"]}
    so1, sm1 = rg1.transpose().sample_block(5000, 0, 42, 8)
    c1["sample_0_5000_sha"] = sha(so1, sm1)
    out["cases"]["c1"] = c1

    # ---- config 2 graph (R-MAT 18, p = fl32(0.01)): sample windows incl. giant sets ----
    g2 = im.generate_rmat(18, 16, 0.57, 0.19, 0.19, 1)
    im.assign_weights_f32(g2, "uniform", 0.01)
    o2, t2, p2 = graph_arrays(g2)
    rgt2 = ref.graph(CSR(262144, o2, t2, p2)).transpose()
    c2 = {"graph_sha": sha(o2, t2, p2), "windows": []}
    for first, count in ((0, 400), (100000, 300), (1500000, 300)):
        so2_, sm2_ = rgt2.sample_block(count, first, 42, 8)
        sizes = np.diff(so2_.astype(np.int64))
        c2["windows"].append({"first": first, "count": count, "sha": sha(so2_, sm2_), "members": int(sm2_.size),
                              "max_size": int(sizes.max())})
    out["cases"]["c2"] = c2

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
