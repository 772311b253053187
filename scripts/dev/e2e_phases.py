"""e2e (host points in, CSR graph out) timing variants for C3: chunk counts
and a compute-only run (device build, no host copies)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets  # noqa: E402

w = datasets.config("C3")
ds = F.Dataset(w.points)
k = F.Kernel(F.KernelFamily.gaussian, w.sigma)
cfg = F.SparsifierConfig(rounds=w.rounds, seed=1)
pinned = torch.empty(w.points.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = w.points
hb = F.api.HostGraphBuffers()


def t(f, reps=4):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best


for chunks in ("0", "4", "8", "16"):
    os.environ["FSGG_E2E_CHUNKS"] = chunks
    def e2e():
        ds.upload_ptr(pinned.data_ptr())
        hb.build_into(ds, k, cfg, w.rounds)
    e2e()
    print(f"chunks={chunks}: e2e {t(e2e):.2f} ms", flush=True)
print(f"device build only: {t(lambda: F.build_similarity_graph_device(ds, k, cfg)):.2f} ms")
g, _ = F.build_similarity_graph_device(ds, k, cfg)
print(f"device build + fetch: {t(lambda: hb.fetch(ds, F.build_similarity_graph_device(ds, k, cfg)[0])):.2f} ms")
