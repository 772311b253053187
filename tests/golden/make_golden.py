"""Generate the golden fixtures from the REFERENCE implementation.

Runs the reference's own hot-path code (oracle/_ref/libfsgref.so, compiled in
place from /root/reference/proj by oracle/Makefile) on seeded inputs and
stores its outputs as small .npz files in tests/golden/. Must run where
/root/reference exists (this build container); the fixtures are committed
and travel to the GPU box, which never reads /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def case_points(ref: Ref, kind: str, n: int, seed: int):
    if kind == "blobs":
        p, lab = ref.make_blobs(n, [[-2.0, 0.0], [2.0, 0.0]], 0.5, seed)
    elif kind == "moons":
        p, lab = ref.make_moons(n, 0.05, seed)
    else:
        raise ValueError(kind)
    # the device consumes fp32; the reference sees the same values promoted
    return p.astype(np.float32), lab


CASES = [
    # name, generator, n, sigma, rounds, seed
    ("c1_blobs", "blobs", 2000, 0.5, 32, 1),
    ("moons4k", "moons", 4096, 0.1, 16, 3),
]


def main():
    ref = Ref()
    ref.set_threads(os.cpu_count() or 1)
    meta = {}
    for name, kind, n, sigma, rounds, seed in CASES:
        p32, lab = case_points(ref, kind, n, seed)
        p64 = p32.astype(np.float64)
        g = ref.build_graph(p64, sigma, rounds, seed=seed, backend=0)
        est = ref.estimator(p64, 0, sigma, 0)
        s = est.sample_counted(np.arange(n), rounds, seed, inline_range=0, record=True)
        gfull = est.eval(0, n, np.arange(n))
        rec = s["rec"]
        # deterministic subsample of the per-node sums (every 16th record)
        keep = np.arange(0, rec["sum"].size, 16)
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"),
            points=p32, labels=lab, sigma=sigma, rounds=rounds, seed=seed,
            triples=s["triples"], entries_per_level=np.array(s["entries_per_level"]),
            tickets_per_level=np.array(s["tickets_per_level"]),
            u=g["u"], v=g["v"], w=g["w"], degrees=g["degrees"],
            g_full=gfull, rec_first=rec["first"][keep], rec_last=rec["last"][keep],
            rec_query=rec["query"][keep], rec_sum=rec["sum"][keep])
        meta[name] = {k: v for k, v in g["report"].items() if not k.endswith("seconds")}
        meta[name].update(kind=kind, n=n, sigma=sigma, rounds=rounds, seed=seed,
                          records=int(rec["sum"].size), records_kept=int(keep.size))
        print(name, meta[name])

    # Reference known-answer values (restated from proj/tests/*.cpp) computed
    # by the reference itself.
    kat = {
        "default_epsilon_1024": ref.default_epsilon(1024),
        "default_epsilon_2": ref.default_epsilon(2),
        "rounds_for": {"1024": ref.rounds_for(1024), "1000": ref.rounds_for(1000),
                       "1024_C2": ref.rounds_for(1024, C_=2.0),
                       "1024_lambda_half": ref.rounds_for(1024, lam=0.5)},
        "kernel_exp_minus1": ref.kernel(0, 1.0, [0.0, 0.0], [1.0, 0.0]),
    }
    # reference generator outputs (first rows) to pin the product generators
    mp, _ = ref.make_moons(1000, 0.05, 1)
    bp, _ = ref.make_blobs(1000, [[-2.0, 0.0], [2.0, 0.0]], 0.5, 1)
    np.savez_compressed(os.path.join(OUT, "generators.npz"), moons1000=mp, blobs1000=bp)
    with open(os.path.join(OUT, "golden_meta.json"), "w") as f:
        json.dump({"cases": meta, "kat": kat}, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
