"""Spectral clustering on the device against the
reference's own spectral module (proj/src/spectral.cpp, compiled in place
into oracle/_ref on a stand-in for the absent Eigen headers).

Lanczos, Jacobi and k-means are floating-point iterations, so the bar is:
eigenvalues within 5e-6 absolute (the reference's convergence test is
|beta * s_{m,i}| <= tol = 1e-6), eigenvectors parallel to 1e-6, k-means on
identical rows bit-for-bit the same labels, and spectral labels ARI >= 0.99
(== 1 on the same graph)."""
import numpy as np
import pytest
from sklearn.metrics import adjusted_rand_score

import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
from paper_2310_13870_b200.api import WeightedGraph

pytestmark = pytest.mark.gpu


def ref_graph(ref, pts, sigma, L, backend=0):
    r = ref.build_graph(pts.astype(np.float64), sigma, L, seed=1, backend=backend,
                        want_estimates=False)
    n = pts.shape[0]
    u = r["u"]
    row_ptr = np.searchsorted(u, np.arange(n + 1), side="left").astype(np.uint64)
    return WeightedGraph(n=n, u=u, v=r["v"], w=r["w"], row_ptr=row_ptr, degrees=r["degrees"],
                         total_weight=float(r["report"]["total_weight"]))


CASES = {
    "blobs2k": lambda: (datasets.make_blobs(2000, np.array([[-2.0, 0.0], [2.0, 0.0]]), 0.5,
                                            1)[0], 0.5, 32),
    "moons4k": lambda: (datasets.make_moons(4000, 0.05, 1)[0], 0.1, 32),
    "blobs3_6k": lambda: (datasets.make_blobs(6000, np.array([[0.0, 0.0], [3.0, 0.0],
                                                              [0.0, 3.0]]), 0.6, 2)[0], 0.5, 16),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request, ref):
    pts, sigma, L = CASES[request.param]()
    p32 = pts.astype(np.float32)
    return request.param, p32, sigma, L, ref_graph(ref, p32, sigma, L)


def test_eigenpairs_match_reference(ref, case):
    name, p32, sigma, L, g = case
    q = 5
    r = ref.smallest_eigenpairs(g.n, g.u, g.v, g.w, q)
    e = F.smallest_eigenpairs(g, q)
    print(name, r["eigenvalues"], e.eigenvalues, r["matvecs"], e.matvecs)
    np.testing.assert_allclose(e.eigenvalues, r["eigenvalues"], atol=5e-6, rtol=0)
    assert np.all(e.residuals <= 1e-4)
    gaps = np.diff(r["eigenvalues"])
    for i in range(q):
        left = gaps[i - 1] if i > 0 else np.inf
        right = gaps[i] if i < q - 1 else np.inf
        if min(left, right) < 1e-4:  # (near-)degenerate: only the subspace is defined
            continue
        c = abs(float(np.dot(e.eigenvectors[i], r["eigenvectors"][i])))
        assert c >= 1 - 1e-6, (i, c)


def test_spectral_labels_same_graph(ref, case):
    name, p32, sigma, L, g = case
    k = 3 if name == "blobs3_6k" else 2
    lab_ref = ref.spectral_cluster(g.n, g.u, g.v, g.w, k, seed=7)
    lab_gpu, rep = F.spectral_cluster(g, k, seed=7, report=True)
    print(name, rep)
    assert adjusted_rand_score(lab_ref, lab_gpu) == 1.0


def test_spectral_end_to_end_vs_reference(ref, case):
    """The north-star check with both halves on each side: GPU graph + GPU
    spectral against reference graph + reference spectral."""
    name, p32, sigma, L, g = case
    k = 3 if name == "blobs3_6k" else 2
    ds = F.Dataset(p32)
    F.build_similarity_graph_device(ds, F.Kernel(F.KernelFamily.gaussian, sigma),
                                    F.SparsifierConfig(rounds=L, seed=1))
    lab_gpu = F.spectral_cluster(ds, k, seed=7)
    lab_ref = ref.spectral_cluster(g.n, g.u, g.v, g.w, k, seed=7)
    ari = adjusted_rand_score(lab_ref, lab_gpu)
    print(name, "ARI", ari)
    assert ari >= 0.99


def test_handle_and_host_graph_paths_agree(case):
    name, p32, sigma, L, g = case
    ds = F.Dataset(p32)
    F.build_similarity_graph_device(ds, F.Kernel(F.KernelFamily.gaussian, sigma),
                                    F.SparsifierConfig(rounds=L, seed=1))
    host = F.device_graph_to_host(ds)
    a = F.smallest_eigenpairs(ds, 3)
    b = F.smallest_eigenpairs(host, 3)
    assert a.eigenvalues.tobytes() == b.eigenvalues.tobytes()
    assert np.array_equal(F.spectral_cluster(ds, 2, seed=3), F.spectral_cluster(host, 2, seed=3))


@pytest.mark.parametrize("n,dim,k", [(5000, 3, 4), (3000, 2, 2), (20000, 5, 8)])
def test_kmeans_matches_reference(ref, n, dim, k):
    rng = np.random.default_rng(n + k)
    centers = rng.normal(0, 3, (k, dim))
    pts = centers[rng.integers(0, k, n)] + rng.normal(0, 1, (n, dim))
    lab_r, cost_r, it_r = ref.kmeans(pts, k, seed=11)
    lab_g, cost_g, it_g = F.kmeans(pts, k, F.KMeansOptions(seed=11))
    assert adjusted_rand_score(lab_r, lab_g) == 1.0
    assert np.array_equal(lab_r, lab_g)
    assert cost_g == pytest.approx(cost_r, rel=1e-10)
    assert it_g == it_r


def test_errors_match_reference(ref):
    from oracle.pyoracle import OracleError
    # isolated vertex 0 (NormalizedLaplacian, graph.cpp:150-158)
    u = np.array([1, 1, 2], np.uint32)
    v = np.array([2, 3, 3], np.uint32)
    w = np.array([1.0, 2.0, 3.0])
    deg = np.array([0.0, 3.0, 4.0, 5.0])
    g = WeightedGraph(n=4, u=u, v=v, w=w,
                      row_ptr=np.searchsorted(u, np.arange(5)).astype(np.uint64), degrees=deg,
                      total_weight=6.0)
    with pytest.raises(F.InvalidConfig):
        F.smallest_eigenpairs(g, 2)
    with pytest.raises(OracleError) as e:
        ref.smallest_eigenpairs(4, u, v, w, 2)
    assert e.value.code == 2
    pts, _ = datasets.make_moons(500, 0.05, 1)
    ds = F.Dataset(pts.astype(np.float32))
    F.build_similarity_graph_device(ds, F.Kernel(F.KernelFamily.gaussian, 0.3),
                                    F.SparsifierConfig(rounds=16, seed=1))
    with pytest.raises(F.InvalidConfig):
        F.spectral_cluster(ds, 1)
    with pytest.raises(F.InvalidConfig):
        F.smallest_eigenpairs(ds, 0)
    with pytest.raises(F.InvalidConfig):
        F.smallest_eigenpairs(ds, 501)
    # k-means with fewer distinct rows than k: DegenerateInput (exit 4)
    with pytest.raises(F.NumericError):
        F.kmeans(np.ones((10, 2)), 3)
    with pytest.raises(OracleError) as e:
        ref.kmeans(np.ones((10, 2)), 3)
    assert e.value.code == 4
