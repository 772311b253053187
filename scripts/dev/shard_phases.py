"""Wall time of each phase of one owner-mode C3 shard (rank r of N), after a
warm-up run: prepare, receive, sample_shard_routed (+ its report's phases)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets, parallel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=1)
ap.add_argument("--rank", type=int, default=0)
a = ap.parse_args()
p, _ = datasets.make_moons(1_000_000, 0.05, 1)
ds = F.Dataset(p.astype(np.float32))
k = F.Kernel(F.KernelFamily.gaussian, 0.05)
b = parallel.block_shard_bounds(ds, a.world, k)
cfg = F.SparsifierConfig(rounds=64, seed=1, query_begin=b[a.rank], query_end=b[a.rank + 1])
empty = torch.empty((0, parallel.RECORD_WORDS), dtype=torch.int32, device="cuda")


def tm(f):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3, r


for it in range(3):
    t1, _ = tm(lambda: parallel.prepare_root(ds, k, cfg))
    t2, _ = tm(lambda: parallel.receive_root(ds, empty))
    t3, (sh, rep, pr, cnt, g) = tm(lambda: parallel.sample_shard_routed(ds, k, cfg, b))
    print(f"it {it}: prepare {t1:.2f} receive {t2:.2f} sample_routed {t3:.2f} | report: "
          f"tree {rep.estimator_build_seconds * 1e3:.2f} sampling {rep.sampling_seconds * 1e3:.2f} "
          f"keys {rep.weighting_seconds * 1e3:.2f} total {rep.total_seconds * 1e3:.2f}", flush=True)
