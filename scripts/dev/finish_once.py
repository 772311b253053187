"""Row-sharded finish of one rank (rank r of N, C3) between
cudaProfilerStart/Stop: fsgg_finish_graph on the keys routed to it,
fsgg_rows_transposed and fsgg_rows_degrees (lower contributions emulated)."""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import _native as N  # noqa: E402
from paper_2310_13870_b200 import datasets, parallel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=5)
a = ap.parse_args()
p, _ = datasets.make_moons(1_000_000, 0.05, 1)
ds = F.Dataset(p.astype(np.float32))
k = F.Kernel(F.KernelFamily.gaussian, 0.05)
b = parallel.shard_bounds(ds.n, a.world)
pairs, counts, gs = [], [], []
for r in range(a.world):
    cfg = F.SparsifierConfig(rounds=64, seed=1, query_begin=b[r], query_end=b[r + 1])
    _, _, pr, cnt, g = parallel.sample_shard_routed(ds, k, cfg, b)
    pairs.append(pr.clone())
    counts.append(cnt)
    gs.append(g.clone())
g_full = torch.cat(gs)
mine = torch.cat([torch.split(pairs[s], counts[s])[a.rank] for s in range(a.world)])
rb, re = b[a.rank], b[a.rank + 1]


def finish():
    graph, _ = parallel.finish_graph(ds, k, 64, g_full, mine)
    m = int(graph.num_edges)
    v = torch.empty(m, dtype=torch.int32, device="cuda")
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    N.check(N.lib().fsgg_rows_transposed(ds._h, C.c_void_p(v.data_ptr()), C.c_void_p(w.data_ptr())))
    deg = torch.empty(re - rb, dtype=torch.float64, device="cuda")
    # lower contributions: this rank's own transposed rows stand in (timing only)
    N.check(N.lib().fsgg_rows_degrees(ds._h, C.c_void_p(v.data_ptr()), C.c_void_p(w.data_ptr()),
                                      m // 8, rb, re, C.c_void_p(deg.data_ptr())))


for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    finish()
    torch.cuda.synchronize()
    print(f"finish wall {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
torch.cuda.profiler.start()
finish()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
