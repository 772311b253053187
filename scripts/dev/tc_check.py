"""Dev check: tensor-core high-d path vs CUDA-core path vs oracle (small n)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
from oracle.pyoracle import Oracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 784
w = datasets.config("C5", n=n) if d == 784 else None
if w is None:
    p = np.random.default_rng(0).random((n, d)).astype(np.float32); sigma = 2.0
else:
    p, sigma = w.points, w.sigma
ds = F.Dataset(p)
k = F.Kernel(F.KernelFamily.gaussian, sigma)
t = time.time()
tri = F.sample_neighbors_counted(ds, k, np.arange(n), 8, 3)
print("gpu sample", time.time() - t, tri.shape, flush=True)
ref = Oracle().sample_counted(p.astype(np.float64), np.arange(n), 8, 3, sigma)["triples"]
print("triples equal:", np.array_equal(tri, ref), tri.shape, ref.shape)
g, rep, est = F.build_similarity_graph(ds, k, F.SparsifierConfig(rounds=8, seed=3), report=True, estimates=True)
print("edges", g.num_edges(), "evals", rep.kernel_evals, "tiled", rep.kde_tiled_evals, "tiled_s", rep.kde_tiled_seconds)
o = Oracle().build_graph(p.astype(np.float64), sigma, 8, seed=3)
print("graph equal:", np.array_equal(g.u, o["u"]) and np.array_equal(g.v, o["v"]),
      "g rel err", float(np.max(np.abs(est["g_i"] - o["g_full"][est["i"]]) / o["g_full"][est["i"]])))
