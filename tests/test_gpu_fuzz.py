"""Randomised parity sweep: the device graph equals the plain-C oracle's
(pinned bit-for-bit to the reference, tests/test_oracle.py) edge for edge on
seeded random problems spanning every code path — dimension class (low-d
tiled/direct, mid-d CUDA-core, high-d tensor cores), kernel family, sizes on
either side of the symmetric-root and walk thresholds, clustered and uniform
data, index orders, L, seeds."""
import zlib

import numpy as np
import pytest

import paper_2310_13870_b200 as F

pytestmark = pytest.mark.gpu

FAMILIES = [F.KernelFamily.gaussian, F.KernelFamily.exponential, F.KernelFamily.laplacian]


def make_case(i):
    rng = np.random.default_rng(1000 + i)
    d = int(rng.choice([1, 2, 2, 3, 4, 5, 6, 8, 12, 20, 64, 130]))
    fam = FAMILIES[int(rng.integers(0, 3))]
    if d >= 64 and fam == F.KernelFamily.laplacian:
        fam = F.KernelFamily.gaussian  # laplacian high-d runs on CUDA cores; keep tc coverage
    n = int(rng.choice([2, 3, 17, 256, 700, 1500, 3300, 5000]))
    if d >= 64:
        n = min(n, 1500)
    clustered = rng.random() < 0.6
    if clustered:
        k = int(rng.integers(2, 6))
        centers = rng.random((k, d)) * 4
        lab = rng.integers(0, k, n)
        p = centers[lab] + rng.normal(0, 0.3, (n, d))
        if rng.random() < 0.7:
            p = p[np.argsort(lab, kind="stable")]
    else:
        p = rng.random((n, d))
    p = p.astype(np.float32)
    med = np.median(np.linalg.norm(p[rng.integers(0, n, 64)] - p[rng.integers(0, n, 64)], axis=1))
    sigma = float(max(med, 1e-3) * rng.choice([0.05, 0.2, 0.6, 1.5]))
    if fam != F.KernelFamily.gaussian:
        sigma *= 0.5
    L = int(rng.choice([1, 3, 8, 16]))
    seed = int(rng.integers(1, 1 << 30))
    return p, fam, sigma, L, seed


@pytest.mark.parametrize("i", range(64))
def test_random_graph_matches_oracle(oracle, i):
    p, fam, sigma, L, seed = make_case(i)
    n = p.shape[0]
    if n < 2:
        pytest.skip("n < 2")
    g, rep, est = F.build_similarity_graph(F.Dataset(p), F.Kernel(fam, sigma),
                                           F.SparsifierConfig(rounds=L, seed=seed), report=True,
                                           estimates=True)
    ref = oracle.build_graph(p.astype(np.float64), sigma, L, seed=seed, family=int(fam))
    info = f"n={n} d={p.shape[1]} fam={int(fam)} sigma={sigma:.4g} L={L} seed={seed}"
    assert np.array_equal(g.u, ref["u"]) and np.array_equal(g.v, ref["v"]), info
    if g.w.size:
        # weights inherit g_full's error: ~1e-6 on CUDA cores; on the tensor
        # cores (d >= 64) the fp32 accumulation inside the MMAs adds a bias
        # that grows with |x|^2 (measured up to 1.9e-5 on clustered d = 130
        # data with |x - mean|^2 ~ 170) — within the north star's 1e-4
        tol = 5e-5 if p.shape[1] >= 64 else 1e-5
        r = np.abs(g.w - ref["w"]) / ref["w"]
        assert r.max() <= tol, info
    assert rep.sampled_pairs == ref["report"]["sampled_pairs"], info
    assert rep.self_pairs_discarded == ref["report"]["self_pairs_discarded"], info
    assert rep.degenerate_draws == ref["report"]["degenerate_draws"], info


def _edge_case(name):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    if name == "identical-points":
        p = np.zeros((600, 2), np.float32)
        return p, F.KernelFamily.gaussian, 0.1, 8
    if name == "far-clusters":  # cross-cluster terms underflow: degenerate draws
        p = np.concatenate([rng.normal(0, 0.01, (400, 2)), rng.normal(50, 0.01, (400, 2))])
        return p.astype(np.float32), F.KernelFamily.gaussian, 0.05, 16
    if name == "tiny-sigma":  # almost every sum at the 1e-300 floor
        p = rng.random((3500, 2)).astype(np.float32)
        return p, F.KernelFamily.gaussian, 1e-4, 4
    if name == "huge-sigma":  # flat kernel: tickets spread uniformly
        p = rng.random((3500, 3)).astype(np.float32)
        return p, F.KernelFamily.gaussian, 1e3, 8
    if name == "duplicates":  # many exact duplicates among distinct points
        base = rng.random((50, 2))
        p = base[rng.integers(0, 50, 3400)].astype(np.float32)
        return p, F.KernelFamily.laplacian, 0.2, 8
    if name == "line-1d-large":
        p = np.sort(rng.random((20000, 1)), axis=0).astype(np.float32)
        return p, F.KernelFamily.exponential, 0.002, 8
    raise ValueError(name)


@pytest.mark.parametrize("name", ["identical-points", "far-clusters", "tiny-sigma", "huge-sigma",
                                  "duplicates", "line-1d-large"])
def test_edge_cases_match_oracle(oracle, name):
    p, fam, sigma, L = _edge_case(name)
    seed = 17
    g, rep, _ = F.build_similarity_graph(F.Dataset(p), F.Kernel(fam, sigma),
                                         F.SparsifierConfig(rounds=L, seed=seed), report=True,
                                         estimates=True)
    ref = oracle.build_graph(p.astype(np.float64), sigma, L, seed=seed, family=int(fam))
    assert np.array_equal(g.u, ref["u"]) and np.array_equal(g.v, ref["v"])
    if g.w.size:
        assert (np.abs(g.w - ref["w"]) / ref["w"]).max() <= 1e-5
    assert rep.sampled_pairs == ref["report"]["sampled_pairs"]
    assert rep.self_pairs_discarded == ref["report"]["self_pairs_discarded"]
    assert rep.degenerate_draws == ref["report"]["degenerate_draws"]
    assert rep.underflow_edges_discarded == ref["report"]["underflow_edges_discarded"]
