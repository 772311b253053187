"""FSGG_TRACE per-level breakdown of the full C3 build and of one query shard.

    FSGG_TRACE=1 python scripts/trace_shard.py [--world 8 --rank 1]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets, parallel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--sigma", type=float, default=0.05)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=1)
a = ap.parse_args()
p, _ = datasets.make_moons(a.n, 0.05, 1)
ds = F.Dataset(p.astype(np.float32))
k = F.Kernel(F.KernelFamily.gaussian, a.sigma)
b = parallel.shard_bounds(a.n, a.world)
for label, cfg in (("full", F.SparsifierConfig(rounds=64, seed=1)),
                   (f"shard {a.rank}/{a.world}",
                    F.SparsifierConfig(rounds=64, seed=1, query_begin=b[a.rank],
                                       query_end=b[a.rank + 1]))):
    for it in range(2):
        print(f"==== {label} iteration {it}", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        if label == "full":
            F.build_similarity_graph_device(ds, k, cfg)
        else:
            parallel.sample_shard(ds, k, cfg)
        torch.cuda.synchronize()
        print(f"==== {label}: {(time.perf_counter() - t) * 1e3:.2f} ms", file=sys.stderr,
              flush=True)
