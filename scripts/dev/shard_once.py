"""One owner-mode C3 shard (rank r of N) between cudaProfilerStart/Stop, for
an ncu launch list of exactly one shard descent:

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv python scripts/dev/shard_once.py --world 8
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets, parallel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=1)
ap.add_argument("--full", action="store_true", help="profile the full 1-GPU build instead")
a = ap.parse_args()
p, _ = datasets.make_moons(a.n, 0.05, 1)
ds = F.Dataset(p.astype(np.float32))
k = F.Kernel(F.KernelFamily.gaussian, 0.05)
if a.full:
    cfg = F.SparsifierConfig(rounds=64, seed=1)
    run = lambda: F.build_similarity_graph_device(ds, k, cfg)  # noqa: E731
else:
    b = parallel.block_shard_bounds(ds, a.world, k)
    cfg = F.SparsifierConfig(rounds=64, seed=1, query_begin=b[a.rank], query_end=b[a.rank + 1])

    def run():
        parallel.prepare_root(ds, k, cfg)
        parallel.receive_root(ds, torch.empty((0, parallel.RECORD_WORDS), dtype=torch.int32,
                                              device="cuda"))
        parallel.sample_shard(ds, k, cfg)
run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
