import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import random_graph
from oracle.oracle import Oracle, CSR
import paper_2208_00613_b200 as im
orc = Oracle()
rng = np.random.default_rng(5)
g = random_graph(rng, 300, 3000)
g = CSR(g.n, g.off, g.tgt, np.full(g.m, 0.3))
for mode in ("huffman", "hybrid"):
    r = im.run(im.Graph.from_csr(g.n, g.off, g.tgt, g.prob), 6, epsilon=0.5, blocks=4, mode=mode, seed=7, workers=2)
    o = orc.run(g, 6, 0.5, 4, mode, 7)
    print(mode, r["seeds"], r["marginal"], o["seeds"], o["marginal"], r["stats"]["device"]["dense_sets"], o["dense_sets"])
