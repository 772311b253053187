"""Pins the C restatement (oracle/libfsgoracle.so) against the reference.

* always: against the committed golden fixtures, which the reference's own
  code produced (tests/golden/make_golden.py);
* when oracle/_ref is built (this container): against the reference itself
  on fresh random cases, bit for bit.
Also restates the reference's known-answer tests (proj/tests/*.cpp).
"""
import math

import numpy as np
import pytest

from conftest import load_golden

MASK = (1 << 64) - 1


def py_splitmix64(x):
    """Independent Python restatement of proj/include/fsg/rng.hpp:11-16."""
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def test_splitmix64_and_keyed_stream(oracle):
    for x in [0, 1, 2, 12345, 2**63, MASK]:
        assert oracle.splitmix64(x) == py_splitmix64(x)
    seed, tag, a, b = 7, 0x88B4F8A3C2D1E5F7, (3 << 32) | 9, 5
    k = py_splitmix64(seed)
    k = py_splitmix64(k ^ py_splitmix64(tag ^ 0x6A09E667F3BCC909))
    k = py_splitmix64(k ^ py_splitmix64(a ^ 0xBB67AE8584CAA73B))
    k = py_splitmix64(k ^ py_splitmix64(b ^ 0x3C6EF372FE94F82B))
    assert oracle.rng_key(seed, tag, a, b) == k
    for c in range(5):
        assert oracle.rng_double(k, c) == (py_splitmix64((k + c) & MASK) >> 11) * 2.0**-53


def test_binomial_is_bernoulli_trials(oracle):
    key = oracle.rng_key(1, 99, 0, 0)
    assert oracle.binomial(key, 10, 0.0) == 0 and oracle.binomial(key, 10, 1.0) == 10
    p = 0.3
    expect = sum(oracle.rng_double(key, c) < p for c in range(50))
    assert oracle.binomial(key, 50, p) == expect


def test_kernel_known_answers(oracle):
    # proj/tests/test_kernel.cpp:16-36
    assert oracle.kernel(0, 1.0, [0.3, -0.7], [0.3, -0.7]) == 1.0
    assert oracle.kernel(0, 1.0, [0, 0], [1, 0]) == pytest.approx(0.36787944117144233, rel=1e-14)
    assert oracle.kernel(2, 1.0, [0, 0], [3, 4]) == pytest.approx(math.exp(-7.0), rel=1e-14)
    assert oracle.kernel(1, 2.0, [0, 0], [3, 4]) == pytest.approx(math.exp(-2.5), rel=1e-14)


def test_kde_hand_values(oracle):
    # proj/tests/test_kde.cpp:25-37
    assert oracle.kde_exact(np.array([[0.4, 0.6]]), 0, 1, [0], 1.0)[0] == 1.0
    g = oracle.kde_exact(np.array([[0.0], [1.0]]), 0, 2, [0], 1.0)[0]
    assert g == pytest.approx(1.3678794411714423, rel=1e-15)


def test_rounds_for_and_epsilon(oracle):
    # proj/tests/test_sparsifier.cpp:34-46, proj/tests/test_kde.cpp:145-150
    assert oracle.rounds_for(1024) == 60
    assert oracle.rounds_for(1000) == 60
    assert oracle.rounds_for(1024, C_=2.0) == 120
    assert oracle.rounds_for(1024, lam=0.5) == 120
    assert oracle.rounds_for(1024, rounds=7) == 7
    assert oracle.default_epsilon(1024) == pytest.approx(1 / 60, rel=1e-12)
    assert oracle.default_epsilon(2) == pytest.approx(1 / 6, rel=1e-12)
    assert oracle.default_epsilon(100000, 1) == pytest.approx(1 / (6 * math.log(1e5)), rel=1e-12)


@pytest.mark.parametrize("name", ["c1_blobs", "moons4k"])
def test_oracle_matches_golden(oracle, name):
    g = load_golden(name)
    p = g["points"].astype(np.float64)
    n = p.shape[0]
    sigma, L, seed = float(g["sigma"]), int(g["rounds"]), int(g["seed"])
    s = oracle.sample_counted(p, np.arange(n), L, seed, sigma, record=True)
    assert np.array_equal(s["triples"], g["triples"])
    assert s["entries_per_level"] == g["entries_per_level"].tolist()
    assert s["tickets_per_level"] == g["tickets_per_level"].tolist()
    rec = s["rec"]
    keep = np.arange(0, rec["sum"].size, 16)
    assert np.array_equal(rec["first"][keep], g["rec_first"])
    assert np.array_equal(rec["query"][keep], g["rec_query"])
    assert np.array_equal(rec["sum"][keep], g["rec_sum"])
    b = oracle.build_graph(p, sigma, L, seed)
    for k in ("u", "v", "w", "degrees"):
        assert np.array_equal(b[k], g[k]), k
    assert np.array_equal(b["g_full"], g["g_full"])


def test_oracle_vs_reference_random(oracle, ref):
    rng = np.random.default_rng(0)
    for trial, (n, d, fam, sigma, L) in enumerate([(300, 2, 0, 0.2, 9), (257, 3, 1, 0.4, 5),
                                                    (200, 5, 2, 0.8, 7), (150, 1, 0, 0.05, 12),
                                                    (64, 16, 0, 1.5, 4)]):
        p = rng.random((n, d)).astype(np.float32).astype(np.float64)
        a = oracle.build_graph(p, sigma, L, seed=trial + 3, family=fam)
        b = ref.build_graph(p, sigma, L, seed=trial + 3, family=fam, backend=0)
        for k in ("u", "v", "w", "degrees"):
            assert np.array_equal(a[k], b[k]), (trial, k)
        # sampler with duplicate queries merged (proj/src/sampler.cpp:89-106)
        q = np.array([5, 1, 5, n - 1, 0, 5])
        sa = oracle.sample_counted(p, q, L, 11, sigma, family=fam)
        sb = ref.estimator(p, fam, sigma, 0).sample_counted(q, L, 11)
        assert np.array_equal(sa["triples"], sb["triples"])
        assert sa["entries_per_level"] == sb["entries_per_level"]
        # KdeEstimator::eval on arbitrary (non-node) ranges
        t = np.arange(0, n, 7)
        ka = oracle.kde_exact(p, 3, n - 2, t, sigma, family=fam)
        kb = ref.estimator(p, fam, sigma, 0).eval(3, n - 2, t)
        assert np.array_equal(ka, kb)


def test_oracle_chi_squared_gof(oracle):
    # proj/tests/test_sampler.cpp:95-130 on the restatement
    from scipy.stats import chi2 as chi2_dist
    n, rounds = 48, 120000
    p = oracle.random_dataset(n, 2, 29)
    for q in (0, 17, 40):
        k = np.array([oracle.kernel(0, 0.4, p[q], p[j]) for j in range(n)])
        expect = k / k.sum() * rounds
        tri = oracle.sample_counted(p, [q], rounds, 1000 + q, 0.4)["triples"]
        obs = np.zeros(n)
        obs[tri[:, 1]] = tri[:, 2]
        small = expect < 5
        stat = (((obs[~small] - expect[~small]) ** 2) / expect[~small]).sum()
        bins = int((~small).sum())
        if small.any():
            stat += (obs[small].sum() - expect[small].sum()) ** 2 / expect[small].sum()
            bins += 1
        assert stat <= chi2_dist.ppf(1 - 1e-3, bins - 1)


def test_oracle_ticket_conservation(oracle):
    # proj/tests/test_sampler.cpp:164-185
    n = 64
    p = oracle.random_dataset(n, 2, 5)
    s = oracle.sample_counted(p, np.arange(n), 37, 13, 0.3)
    assert len(s["tickets_per_level"]) == 7
    assert all(t == n * 37 for t in s["tickets_per_level"])
    assert s["entries_per_level"][0] == n
    assert int(s["triples"][:, 2].sum()) == n * 37


def test_oracle_rejects_invalid(oracle):
    from oracle.pyoracle import OracleError
    p = oracle.random_dataset(10, 2, 1)
    with pytest.raises(OracleError):
        oracle.sample_counted(p, [10], 1, 1, 1.0)
    with pytest.raises(OracleError):
        oracle.sample_counted(p, [1], 0, 1, 1.0)
    with pytest.raises(OracleError):
        oracle.kde_exact(p, 4, 2, [0], 1.0)
    with pytest.raises(OracleError):
        oracle.build_graph(p[:1], 1.0, 4)


def test_reference_spectral_module_on_eigen_standin(ref):
    """Pins the reference spectral module as built here (proj/src/spectral.cpp
    on oracle/ref/eigen_shim): its eigenvalues agree with scipy's dense
    solver on the same normalised Laplacian, and spectral_cluster recovers
    the two moons."""
    from paper_2310_13870_b200 import datasets
    from sklearn.metrics import adjusted_rand_score
    pts, truth = datasets.make_moons(3000, 0.05, 1)
    g = ref.build_graph(pts.astype(np.float32).astype(np.float64), 0.15, 32, seed=1,
                        want_estimates=False)
    n = 3000
    e = ref.smallest_eigenpairs(n, g["u"], g["v"], g["w"], 4)
    a = np.zeros((n, n))
    a[g["u"], g["v"]] = g["w"]
    a[g["v"], g["u"]] = g["w"]
    dinv = 1.0 / np.sqrt(a.sum(1))
    lap = np.eye(n) - dinv[:, None] * a * dinv[None, :]
    dense = np.linalg.eigvalsh(lap)[:4]
    np.testing.assert_allclose(e["eigenvalues"], dense, atol=1e-6)
    assert np.all(e["residuals"] < 1e-5)
    lab = ref.spectral_cluster(n, g["u"], g["v"], g["w"], 2, seed=7)
    assert adjusted_rand_score(truth, lab) > 0.99
