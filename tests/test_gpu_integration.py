"""The C++ drop-in: the reference's own objects and libfsgg.so in one binary
(oracle/ref/adapter_check.cpp via include/fsgg/fsg_adapter.hpp), comparing
fsg::build_similarity_graph (CPU, exact) with the adapter (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")

pytestmark = pytest.mark.gpu


def test_cpp_adapter_matches_reference_binary():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "adapter ok" in out.stdout


def test_gpu_graph_file_round_trips_through_reference_reader(ref, tmp_path):
    """End to end through the file the reference's CLI writes (--graph-out):
    the reference's own reader loads the GPU graph's text file to the same
    edges as the reference's graph (weights within the fp32-sum tolerance,
    SURVEY.md §8c(5)), and our writer emits the reference's bytes for the
    reference's graph."""
    import numpy as np
    import paper_2310_13870_b200 as F
    from paper_2310_13870_b200 import datasets
    pts = datasets.make_blobs(2000, np.array([[-2.0, 0.0], [2.0, 0.0]]), 0.5, 1)[0]
    p32 = pts.astype(np.float32)
    g = F.build_similarity_graph(F.Dataset(p32), F.Kernel(F.KernelFamily.gaussian, 0.5),
                                 F.SparsifierConfig(rounds=32, seed=1))
    r = ref.build_graph(p32.astype(np.float64), 0.5, 32, seed=1, want_estimates=False)
    path = tmp_path / "gpu.txt"
    g.write_edge_list(str(path))
    back = ref.load_edge_list(str(path))
    np.testing.assert_array_equal(back["u"], r["u"])
    np.testing.assert_array_equal(back["v"], r["v"])
    assert back["w"].tobytes() == g.w.tobytes()  # %.17g round-trips exactly
    np.testing.assert_allclose(back["w"], r["w"], rtol=1e-5)
    np.testing.assert_allclose(back["degrees"], r["degrees"], rtol=1e-5)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    WG = F.WeightedGraph
    WG(n=2000, u=r["u"], v=r["v"], w=r["w"], row_ptr=None, degrees=r["degrees"],
       total_weight=0.0).write_edge_list(str(ours))
    ref.save_edge_list(str(theirs), 2000, r["u"], r["v"], r["w"])
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.parametrize("chunks", ["0", "1", "4", "16"])
def test_build_into_pinned_buffers_matches_device_build(chunks, monkeypatch):
    """fsgg_build_similarity_graph_into (host buffers filled while the graph
    is finished — in u-range chunks streamed one by one, FSGG_E2E_CHUNKS)
    returns exactly the device build's CSR, weights, degrees and total
    weight."""
    import numpy as np
    import paper_2310_13870_b200 as F
    from paper_2310_13870_b200 import datasets
    monkeypatch.setenv("FSGG_E2E_CHUNKS", chunks)
    p, _ = datasets.make_moons(20000, 0.05, 4)
    ds = F.Dataset(p)
    k = F.Kernel(F.KernelFamily.gaussian, 0.08)
    cfg = F.SparsifierConfig(rounds=16, seed=2)
    full = F.build_similarity_graph(ds, k, cfg)
    g = F.api.HostGraphBuffers().build_into(ds, k, cfg, 16)
    assert np.array_equal(g.v, full.v) and np.array_equal(g.w, full.w)
    assert np.array_equal(g.row_ptr, full.row_ptr) and np.array_equal(g.u, full.u)
    assert np.array_equal(g.degrees, full.degrees)
    assert g.total_weight == full.total_weight
