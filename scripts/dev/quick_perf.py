"""Quick timing of the device build on the benchmark configs (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets

for name in sys.argv[1:] or ["C2"]:
    w = datasets.config(name)
    ds = F.Dataset(w.points)
    k = F.Kernel(F.KernelFamily.gaussian, w.sigma)
    cfg = F.SparsifierConfig(rounds=w.rounds, seed=1, dense_kde=os.environ.get("DENSE") == "1")
    for it in range(2):
        t = time.time()
        g, rep = F.build_similarity_graph_device(ds, k, cfg)
        dt = time.time() - t
        print(f"{name} it{it}: {dt:.3f}s edges={g.num_edges} evals={rep.kernel_evals:.3e} "
              f"tiled_evals={rep.kde_tiled_evals:.3e} performed={rep.kde_tiled_performed_evals:.3e} tiled_s={rep.kde_tiled_seconds:.3f} "
              f"({rep.kde_tiled_performed_evals/max(rep.kde_tiled_seconds,1e-9)/1e12:.3f} Tperf/s) "
              f"sample_s={rep.sampling_seconds:.3f} graph_s={rep.weighting_seconds:.3f} "
              f"tree_s={rep.estimator_build_seconds:.3f} levels={rep.levels} peak={rep.peak_entries} "
              f"launches={rep.gpu_launches} ties={rep.tie_verified_entries}", flush=True)
