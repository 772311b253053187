"""One build_similarity_graph on a config (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = datasets.config(name)
ds = F.Dataset(w.points)
k = F.Kernel(F.KernelFamily.gaussian, w.sigma)
for _ in range(reps):
    g, rep = F.build_similarity_graph_device(ds, k, F.SparsifierConfig(rounds=w.rounds, seed=1))
print(name, "edges", g.num_edges, "launches", rep.gpu_launches)
