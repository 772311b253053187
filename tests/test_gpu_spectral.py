"""North-star check: spectral-clustering labels on the GPU graph agree with
those on the reference's graph (ARI >= 0.99), for the reference's exact
backend and for its default (auto -> FGT) backend.

Spectral clustering is the downstream consumer of the graph (reference:
proj/src/spectral.cpp:40-419: bottom-k eigenvectors of the normalised
Laplacian, row-normalised embedding, k-means). It is not on the hot path and
runs here with scipy/sklearn on both graphs identically.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import eigsh
from sklearn.cluster import KMeans
from sklearn.metrics import adjusted_rand_score

import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets

pytestmark = pytest.mark.gpu


def spectral_labels(n, u, v, w, k, seed=7):
    a = sp.coo_matrix((np.concatenate([w, w]), (np.concatenate([u, v]), np.concatenate([v, u]))),
                      shape=(n, n)).tocsr()
    deg = np.asarray(a.sum(1)).ravel()
    dinv = sp.diags(1.0 / np.sqrt(deg))
    m = dinv @ a @ dinv  # eigenvalues 1 - lambda(N)
    vals, vecs = eigsh(m, k=k, which="LA", tol=1e-8, v0=np.ones(n))
    emb = vecs / np.maximum(np.linalg.norm(vecs, axis=1, keepdims=True), 1e-300)
    return KMeans(n_clusters=k, n_init=10, random_state=seed).fit_predict(emb)


@pytest.mark.parametrize("ours", [F.KdeBackend.exact, F.KdeBackend.fast],
                         ids=["gpu-exact", "gpu-fast"])
@pytest.mark.parametrize("backend", [0, 2], ids=["ref-exact", "ref-auto-fgt"])
def test_spectral_ari_vs_reference_graph(ref, backend, ours):
    n, sigma, L = 20000, 0.1, 32
    pts, truth = datasets.make_moons(n, 0.05, 1)
    p32 = pts.astype(np.float32)
    g = F.build_similarity_graph(F.Dataset(p32), F.Kernel(F.KernelFamily.gaussian, sigma),
                                 F.SparsifierConfig(rounds=L, seed=1, kde_backend=ours))
    r = ref.build_graph(p32.astype(np.float64), sigma, L, seed=1, backend=backend,
                        want_estimates=False)
    lab_gpu = spectral_labels(n, g.u, g.v, g.w, 2)
    lab_ref = spectral_labels(n, r["u"], r["v"], r["w"], 2)
    ari = adjusted_rand_score(lab_ref, lab_gpu)
    print(f"gpu={ours.name} ref={r['report']['backend']}: ARI(gpu, ref) = {ari:.5f}, "
          f"ARI(gpu, truth) = {adjusted_rand_score(truth, lab_gpu):.5f}")
    assert ari >= 0.99
