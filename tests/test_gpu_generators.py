"""Device-side generators (csrc/datasets_dev.cu, §8f row 3) against the host
generators (csrc/datasets.cpp, bit-identical to proj/src/datasets.cpp:20-124
per test_oracle.py): every BASELINE config at full size.

* fp32 points (what the descent consumes) and labels: identical;
* fp64 points: the device's log/sin/cos are correctly rounded, glibc's are
  within 0.502 ulp, so a coordinate may differ in its last bits — bounded
  here in count (< 0.5%) and size (a few ulp of 1);
* a graph built from device-generated C2 points is the reference's
  (golden SHA-256 of the exact backend's edge list).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _check(dev, host_pts, host_lab):
    p32, p64, lab = dev
    assert np.array_equal(p32.cpu().numpy(), host_pts.astype(np.float32))
    assert np.array_equal(lab.cpu().numpy().astype(np.uint32), host_lab)
    d = p64.cpu().numpy()
    diff = d != host_pts
    assert diff.mean() < 0.005
    assert np.abs(d - host_pts).max() <= 8 * np.spacing(1.0)
    return float(diff.mean())


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_device_generator_matches_host(name):
    if name == "C1":
        c = [[-2.0, 0.0], [2.0, 0.0]]
        host = datasets.make_blobs(2000, c, 0.5, 1)
        dev = datasets.make_blobs_device(2000, c, 0.5, 1, fp64=True)
    elif name in ("C2", "C3"):
        n = 100_000 if name == "C2" else 1_000_000
        host = datasets.make_moons(n, 0.05, 1)
        dev = datasets.make_moons_device(n, 0.05, 1, fp64=True)
    elif name == "C4":
        host = datasets.make_image_features(481, 321, 8, 0.03, 1)
        dev = datasets.make_image_features_device(481, 321, 8, 0.03, 1, fp64=True)
    else:
        host = datasets.make_gmm(70_000, 784, 10, 0.1, 1)
        dev = datasets.make_gmm_device(70_000, 784, 10, 0.1, 1, fp64=True)
    frac = _check(dev, *host)
    print(f"{name}: fp64 coordinates differing in the last bits: {frac:.2e}")


def test_config_device_matches_config():
    for name in ("C1", "C4", "C5"):
        w = datasets.config(name)
        p, lab, sigma, rounds = datasets.config_device(name)
        assert np.array_equal(p.cpu().numpy(), w.points)
        assert sigma == w.sigma and rounds == w.rounds


def test_generator_edge_cases_and_errors():
    # odd n splits the moons n/2 outer, the rest inner; noise 0 is exact
    p32, p64, lab = datasets.make_moons_device(7, 0.0, 3, fp64=True)
    hp, hl = datasets.make_moons(7, 0.0, 3)
    assert np.array_equal(p64.cpu().numpy(), hp)
    assert np.array_equal(lab.cpu().numpy().astype(np.uint32), hl)
    # uneven blobs: the first n % k clusters hold one more point
    c = [[0.0, 0.0, 1.0], [5.0, 5.0, 5.0], [-3.0, 2.0, 0.5]]
    p32, p64, lab = datasets.make_blobs_device(11, c, 0.25, 9, fp64=True)
    hp, hl = datasets.make_blobs(11, c, 0.25, 9)
    assert np.array_equal(lab.cpu().numpy().astype(np.uint32), hl)
    assert np.array_equal(p32.cpu().numpy(), hp.astype(np.float32))
    # proj/src/datasets.cpp:33-34, 71-80
    with pytest.raises(F.InvalidConfig):
        datasets.make_moons_device(1, 0.1, 1)
    with pytest.raises(F.InvalidConfig):
        datasets.make_moons_device(10, -0.1, 1)
    with pytest.raises(F.InvalidConfig):
        datasets.make_blobs_device(1, c, 0.1, 1)
    with pytest.raises(F.InvalidConfig):
        datasets.make_gmm_device(5, 3, 10, 0.1, 1)


def test_graph_from_device_points_matches_reference_c2():
    meta = json.load(open(os.path.join(GOLDEN, "golden_large.json")))["C2"]
    p, _, sigma, rounds = datasets.config_device("C2")
    ds = F.Dataset(p)  # device tensor: no host round trip
    g = F.build_similarity_graph(ds, F.Kernel(F.KernelFamily.gaussian, sigma),
                                 F.SparsifierConfig(rounds=rounds, seed=1))
    assert g.num_edges() == meta["edge_count"]
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(g.u) == meta["sha_u"] and sha(g.v) == meta["sha_v"]
