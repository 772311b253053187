"""Small builds through the round-2 kernels for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets  # noqa: E402

p, _ = datasets.make_moons(16000, 0.05, 11)   # 250-point nodes at level 6: two-deep rows + walks
ds = F.Dataset(p.astype(np.float32))
g, rep, _ = F.build_similarity_graph(ds, F.Kernel(F.KernelFamily.gaussian, 0.05),
                                     F.SparsifierConfig(rounds=8, seed=3), report=True)
print("d=2", g.num_edges(), rep.kde_root_performed_evals)
rng = np.random.default_rng(5)
p5 = rng.normal(size=(5000, 5)) * 0.5 + rng.integers(0, 3, size=(5000, 1))
ds5 = F.Dataset(p5.astype(np.float32))
g5, rep5, _ = F.build_similarity_graph(ds5, F.Kernel(F.KernelFamily.gaussian, 0.3),
                                       F.SparsifierConfig(rounds=8, seed=3), report=True)
print("d=5", g5.num_edges(), rep5.kde_root_performed_evals)
