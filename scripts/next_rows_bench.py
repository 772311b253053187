"""Measurements for SURVEY.md §8f rows built this round (not the headline
bench): spectral clustering on the device graph and graph-file I/O, each
beside the reference's own implementation (oracle/_ref) on the same input.

Usage: python scripts/next_rows_bench.py [C2|C3] > profiles/r1_next_rows_<cfg>.json
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import datasets  # noqa: E402


def timed(fn, reps=3):
    best = None
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return out, best


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    w = datasets.config(name)
    ds = F.Dataset(w.points)
    k = F.Kernel(F.KernelFamily.gaussian, w.sigma)
    cfg = F.SparsifierConfig(rounds=w.rounds, seed=1)
    F.build_similarity_graph_device(ds, k, cfg)
    host = F.device_graph_to_host(ds)
    res = {"config": name, "n": w.n, "edges": host.num_edges()}

    # spectral clustering (k = 2 moons) on the device graph
    F.spectral_cluster(ds, 2, seed=7)  # warm-up
    (labels, rep), t = timed(lambda: F.spectral_cluster(ds, 2, seed=7, report=True), reps=2)
    truth = getattr(w, "labels", None)
    spec = {"seconds": t, "report": rep}
    if truth is not None:
        from sklearn.metrics import adjusted_rand_score
        spec["ari_vs_generator_labels"] = float(adjusted_rand_score(truth, labels))
    res["spectral_gpu"] = spec

    # graph files
    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "g.txt")
    _, t_write = timed(lambda: host.write_edge_list(path), reps=1)
    size = os.path.getsize(path)
    _, t_read = timed(lambda: F.read_edge_list(path), reps=1)
    res["text_io"] = {"write_seconds": t_write, "read_seconds": t_read, "bytes": size,
                      "threads": os.cpu_count()}

    try:
        from oracle.pyoracle import Ref
        if Ref.available and os.environ.get("FSGG_SKIP_REF") != "1":
            ref = Ref()
            ref.set_threads(os.cpu_count())
            p2 = os.path.join(tmp, "ref.txt")
            _, tw = timed(lambda: ref.save_edge_list(p2, host.n, host.u, host.v, host.w), reps=1)
            same = open(p2, "rb").read() == open(path, "rb").read()
            _, tr = timed(lambda: ref.load_edge_list(p2), reps=1)
            res["text_io"]["reference"] = {"write_seconds": tw, "read_seconds": tr,
                                           "bytes_identical": same}
            if w.n <= 200000:
                t0 = time.perf_counter()
                rl = ref.spectral_cluster(host.n, host.u, host.v, host.w, 2, seed=7)
                ts = time.perf_counter() - t0
                from sklearn.metrics import adjusted_rand_score
                res["spectral_reference"] = {
                    "seconds": ts, "threads": ref.worker_count(),
                    "ari_gpu_vs_reference": float(adjusted_rand_score(rl, labels))}
    except Exception as exc:  # reported, not fatal
        res["reference_error"] = repr(exc)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
