"""Per-node KDE sum fixtures from the REFERENCE for the descent's hot kernels.

SURVEY.md §8(c) protocol step 1: every (range, query) -> g the reference's
sampler asks its estimator for (proj/src/sampler.cpp:146-149, exact backend
proj/src/kde.cpp:38-49, ``inline_range=0`` so no sum bypasses the estimator),
recorded by oracle/ref/ref_driver.cpp's wrapper estimator, on inputs shaped
to drive the device kernels the benchmarked configs run:

* ``sums_image8k``  C4-shaped pixels (110 x 73 raster, d=5, sigma=0.2):
  contiguous queries -> the symmetric root (kde_sym.cu, 32 blocks of ~251
  points), root-row lookups, block lookups, tiled and direct levels;
* ``sums_gmm784``   C5-shaped mixture (n=3000, d=784, 10 components, sigma =
  median distance): the tcgen05 3xTF32 kernel (kde_tc.cu) at the root and the
  levels it serves, the CUDA-core high-d kernels below.

The moons4k / c1_blobs fixtures (make_golden.py) hold the same records for
d=2. Records are subsampled deterministically (every ``keep``-th). The points
are not stored: the fixture keeps the generator call and the SHA-256 of the
fp32 array, and the test regenerates and checks them (``points_for``).

    python tests/golden/make_golden_sums.py
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2310_13870_b200 import datasets  # noqa: E402  (input generation only)

OUT = os.path.dirname(os.path.abspath(__file__))


GEN = {
    "sums_image8k": ("image", (110, 73, 8, 0.03, 5), 0.2, 32, 5, 16),
    "sums_gmm784": ("gmm", (3000, 784, 10, 0.1, 7), None, 32, 7, 24),
}


def points_for(name):
    """(fp32 points, sigma, rounds, seed, keep) of a fixture."""
    kind, args, sigma, rounds, seed, keep = GEN[name]
    if kind == "image":
        p, _ = datasets.make_image_features(*args)
    else:
        p, _ = datasets.make_gmm(*args)
    p32 = p.astype(np.float32)
    if sigma is None:
        sigma = datasets.median_pairwise_distance(p32.astype(np.float64), 1000, args[-1])
    return p32, sigma, rounds, seed, keep


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Ref()
    ref.set_threads(int(os.environ.get("FSG_GOLDEN_THREADS", os.cpu_count() or 1)))
    for name in GEN:
        p32, sigma, rounds, seed, keep = points_for(name)
        n = p32.shape[0]
        p64 = p32.astype(np.float64)
        est = ref.estimator(p64, 0, sigma, 0)
        s = est.sample_counted(np.arange(n), rounds, seed, inline_range=0, record=True)
        rec = s["rec"]
        idx = np.arange(0, rec["sum"].size, keep)
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), points_sha=sha(p32), sigma=sigma,
            rounds=rounds, seed=seed, triples=s["triples"],
            entries_per_level=np.array(s["entries_per_level"]),
            rec_first=rec["first"][idx], rec_last=rec["last"][idx],
            rec_query=rec["query"][idx], rec_sum=rec["sum"][idx])
        print(name, n, p32.shape[1], f"sigma={sigma:.6g}", "records", rec["sum"].size,
              "kept", idx.size, "triples", s["triples"].shape[0], flush=True)


if __name__ == "__main__":
    main()
