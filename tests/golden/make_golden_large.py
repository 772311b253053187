"""Full-size golden checksums from the REFERENCE (exact backend).

Runs the reference's own code (oracle/_ref) at the BASELINE configs' full
sizes where that is affordable on the build host, and stores compact
fingerprints (counts, SHA-256 of the sorted edge arrays, weight samples)
plus query-subset triples for C3, whose full exact run would take hours.

    python tests/golden/make_golden_large.py [C2] [C3] [C3full] [C4] [C5]

FSG_GOLDEN_THREADS overrides the worker count (default: all host cores).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2310_13870_b200 import datasets  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def full_graph(ref, name):
    w = datasets.config(name)
    p64 = w.points.astype(np.float64)
    t0 = time.time()
    g = ref.build_graph(p64, w.sigma, w.rounds, seed=1, backend=0, want_estimates=False)
    dt = time.time() - t0
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(g["u"].size, size=min(20000, g["u"].size), replace=False))
    rep = {k: v for k, v in g["report"].items()}
    np.savez_compressed(os.path.join(OUT, f"{name.lower()}_full.npz"),
                        pick=pick, u=g["u"][pick], v=g["v"][pick], w=g["w"][pick],
                        degrees_sample=g["degrees"][:: max(1, w.n // 20000)])
    return {"n": w.n, "sigma": w.sigma, "rounds": w.rounds, "edge_count": int(g["u"].size),
            "sha_u": sha(g["u"]), "sha_v": sha(g["v"]), "total_weight": float(g["w"].sum()),
            "report": rep, "seconds": dt, "threads": ref.worker_count()}


def query_subset(ref, name, count=256):
    w = datasets.config(name)
    p64 = w.points.astype(np.float64)
    est = ref.estimator(p64, 0, w.sigma, 0)
    rng = np.random.default_rng(1)
    q = np.sort(rng.choice(w.n, size=count, replace=False)).astype(np.uint32)
    t0 = time.time()
    s = est.sample_counted(q, w.rounds, 1)
    g = est.eval(0, w.n, q)
    dt = time.time() - t0
    np.savez_compressed(os.path.join(OUT, f"{name.lower()}_queries.npz"), queries=q,
                        triples=s["triples"], g_full=g)
    return {"n": w.n, "queries": int(q.size), "triples": int(s["triples"].shape[0]),
            "seconds": dt}


def main():
    ref = Ref()
    ref.set_threads(int(os.environ.get("FSG_GOLDEN_THREADS", os.cpu_count() or 1)))
    which = sys.argv[1:] or ["C2", "C3"]
    path = os.path.join(OUT, "golden_large.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    for name in which:
        if name == "C3":
            meta["C3_queries"] = query_subset(ref, "C3")
        elif name == "C3full":  # the whole n = 1M exact graph (~2 h on 7 threads)
            meta["C3"] = full_graph(ref, "C3")
        else:
            meta[name] = full_graph(ref, name)
        print(name, json.dumps(meta.get(name) or meta.get(name + "_queries"))[:300], flush=True)
        json.dump(meta, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
