"""The fast KDE backend (fsg::KdeBackend::fast,
proj/src/kde.cpp:104-129, kde_fast.cpp:153-656 in the reference).

The reference's fast backend is an FGT with a (1 +- eps) guarantee per sum.
The device analogue (include/fsgg.h, fsgg_config::kde_backend) keeps the
exact kernels and only widens the certified pruning budget: with
B = 19 + log2((depth + 1) / eps) bits, every level skips at most
eps_s = 2^(19 - B) <= eps / (depth + 1) of each node's mass; a query reaches
node N with probability g_N / g_full and one level's node masses add up to
g_full, so each level moves a query's sampling distribution by <= eps_s in
total variation, <= eps over the whole descent.

Checked here:
* every child sum the descent used (record mode) is within the budget of the
  reference's exact sum: g_ref - g_dev <= eps_s * g_full(q) + 2e-5 * g_ref
  (the skipped mass of any node is part of its level's total, which is
  <= eps_s * g_full(q));
* degrees (root sums) within (1 - eps_s) of exact;
* epsilon / backend reporting and the reference's autoselect rule;
* spectral labels of fast-backend graphs vs the reference's FGT and exact
  graphs: ARI >= 0.99 (tests/test_gpu_spectral.py).
"""
import math
import os

import numpy as np
import pytest

import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def budget(n, eps):
    depth = math.ceil(math.log2(n))
    bits = min(48.0, max(20.0, math.ceil(19.0 + math.log2((depth + 1) / eps))))
    return bits, 2.0 ** (19.0 - bits)


@pytest.mark.parametrize("eps", [0.0, 0.05], ids=["default-eps", "eps0.05"])
@pytest.mark.parametrize("name", ["moons4k", "c1_blobs"])
def test_fast_sums_within_certified_budget(name, eps):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    p32, sigma = z["points"], float(z["sigma"])
    rounds, seed = int(z["rounds"]), int(z["seed"])
    n = p32.shape[0]
    e = eps if eps > 0 else F.default_epsilon(n)
    bits, eps_s = budget(n, e)
    ds = F.Dataset(p32)
    k = F.Kernel(F.KernelFamily.gaussian, sigma)
    _, rep = F.sample_neighbors_counted_ex(ds, k, np.arange(n), rounds, seed, record_sums=True,
                                          kde_backend=F.KdeBackend.fast, epsilon=eps)
    r = rep.records
    keep = r["last"] - r["first"] >= 2
    r = r[keep]
    first = r["first"].astype(np.int64)
    last = r["last"].astype(np.int64)
    mid = first + (last - first) // 2
    q = r["query"].astype(np.int64)
    keys = np.concatenate([(first * (n + 1) + mid) * n + q, (mid * (n + 1) + last) * n + q])
    sums = np.concatenate([r["left"], r["right"]])
    order = np.argsort(keys)
    keys, sums = keys[order], sums[order]
    # the reference's records: its descent visits other (node, query) pairs
    # where the fast samples differ; compare the common ones
    want = (z["rec_first"].astype(np.int64) * (n + 1) + z["rec_last"]) * n + z["rec_query"]
    pos = np.minimum(np.searchsorted(keys, want), keys.size - 1)
    hit = keys[pos] == want
    assert hit.mean() > 0.5
    got, ref = sums[pos[hit]], z["rec_sum"][hit]
    gfull = z["g_full"][z["rec_query"][hit]]
    slack = eps_s * gfull + 2e-5 * ref
    assert np.all(ref - got <= slack), (ref - got - slack).max()
    assert np.all(got - ref <= 2e-5 * ref + 1e-300)
    skipped = np.maximum(ref - got, 0.0) / gfull
    print(f"{name} eps={e:.4g} B={bits:.0f}: {hit.sum()} common sums, max skipped/g_full "
          f"{skipped.max():.3e} (budget {eps_s:.3e})")


def test_fast_graph_degrees_and_report():
    w = datasets.config("C2")
    ds = F.Dataset(w.points)
    k = F.Kernel(F.KernelFamily.gaussian, w.sigma)
    ge, rep_e, est_e = F.build_similarity_graph(ds, k, F.SparsifierConfig(rounds=w.rounds),
                                                report=True, estimates=True)
    gf, rep_f, est_f = F.build_similarity_graph(
        ds, k, F.SparsifierConfig(rounds=w.rounds, kde_backend=F.KdeBackend.fast),
        report=True, estimates=True)
    eps = F.default_epsilon(w.n)
    assert rep_e.epsilon == 0.0 and "exact" in rep_e.backend
    assert rep_f.epsilon == pytest.approx(eps) and "fast" in rep_f.backend
    _, eps_s = budget(w.n, eps)
    # g_i of a shared edge's endpoint: the degree KDE of that point
    common = np.intersect1d(est_e["i"].astype(np.int64) << 32 | est_e["j"],
                            est_f["i"].astype(np.int64) << 32 | est_f["j"])
    assert common.size > 0.9 * ge.num_edges()
    ie = np.searchsorted(est_e["i"].astype(np.int64) << 32 | est_e["j"], common)
    jf = np.searchsorted(est_f["i"].astype(np.int64) << 32 | est_f["j"], common)
    ratio = est_f["g_i"][jf] / est_e["g_i"][ie]
    assert np.all(ratio >= 1 - eps_s - 2e-5) and np.all(ratio <= 1 + 2e-5)
    assert rep_f.kernel_evals_performed < rep_e.kernel_evals_performed
    print(f"C2 fast: {rep_f.kernel_evals_performed:.3e} evaluations vs exact "
          f"{rep_e.kernel_evals_performed:.3e}; {gf.num_edges()} vs {ge.num_edges()} edges")


def test_autoselect_follows_reference_rule():
    def backend(n, d, family=F.KernelFamily.gaussian):
        rng = np.random.default_rng(n + d)
        ds = F.Dataset(rng.standard_normal((n, d)).astype(np.float32))
        _, rep, _ = F.build_similarity_graph(
            ds, F.Kernel(family, 1.0),
            F.SparsifierConfig(rounds=4, kde_backend=F.KdeBackend.autoselect), report=True)
        return rep.backend
    assert "fast" in backend(4096, 2)
    assert "exact" in backend(4095, 2)
    assert "exact" in backend(4096, 4)
    assert "exact" in backend(4096, 2, F.KernelFamily.laplacian)  # UnsupportedKernel fallback


def test_fast_rejects_bad_epsilon():
    ds = F.Dataset(np.random.default_rng(0).standard_normal((100, 2)).astype(np.float32))
    k = F.Kernel(F.KernelFamily.gaussian, 1.0)
    with pytest.raises(F.InvalidConfig):
        F.build_similarity_graph(ds, k, F.SparsifierConfig(rounds=4, epsilon=1.5,
                                                           kde_backend=F.KdeBackend.fast))
