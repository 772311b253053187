"""Beyond the benchmark sizes: builds at n = 4M / 2M (moons) on one GPU."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
for n, sigma in ((4_000_000, 0.025), (2_000_000, 0.035)):
    p, lab = datasets.make_moons(n, 0.05, 1)
    ds = F.Dataset(p.astype(np.float32))
    k = F.Kernel(F.KernelFamily.gaussian, sigma)
    cfg = F.SparsifierConfig(rounds=64, seed=1)
    for it in range(2):
        t = time.time()
        g, rep = F.build_similarity_graph_device(ds, k, cfg)
        dt = time.time() - t
    print(n, f"{dt:.3f}s edges={g.num_edges} performed={rep.kernel_evals_performed:.3e} ties={rep.tie_verified_entries}", flush=True)
    try:
        labels = F.spectral_cluster(ds, 2, seed=7)
        from sklearn.metrics import adjusted_rand_score
        print("  ARI vs truth", adjusted_rand_score(lab, labels), flush=True)
    except F.InvalidConfig as exc:  # e.g. an outlier whose tickets all hit itself
        print("  spectral:", exc, flush=True)
    del ds
