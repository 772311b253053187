import numpy as np, torch
import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
for name in ["C3","C2","C4","C5"]:
    w = datasets.config(name)
    ds = F.Dataset(w.points)
    g = F.build_similarity_graph(ds, F.Kernel(F.KernelFamily.gaussian, w.sigma), F.SparsifierConfig(rounds=w.rounds, seed=1))
    u = np.asarray(g.u); c = np.bincount(u, minlength=ds.n)
    qs = np.percentile(c, [50, 90, 99, 99.9, 100])
    print(name, "edges", len(u), "rows", ds.n, "mean", c.mean(), "pcts", qs, ">256", (c>256).sum(), ">1024", (c>1024).sum(), "elems in >256 rows", c[c>256].sum(), flush=True)
