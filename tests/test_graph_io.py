"""Graph files either side of the path: the text edge
list must be byte-identical to fsg::save_edge_list and read back exactly as
fsg::load_edge_list does (proj/src/graph.cpp:234-276); the binary CSR must
round-trip. Host-only code, so these run without a GPU; the reference's own
reader/writer (oracle/_ref) is the checker."""
import os

import numpy as np
import pytest

import paper_2310_13870_b200 as F
from paper_2310_13870_b200.api import WeightedGraph


def random_graph(n, m, seed):
    rng = np.random.default_rng(seed)
    keys = set()
    while len(keys) < m:
        a, b = rng.integers(0, n, 2)
        if a != b:
            keys.add((min(a, b), max(a, b)))
    uv = np.array(sorted(keys), np.uint32)
    w = np.exp(rng.normal(0, 8, m))
    special = [1.0, 0.1, 1e-300, 5e-324, 1.7976931348623157e308, 123456789.0,
               2.0 ** 53 + 2, 1e21, 1e-5, 0.30000000000000004, 1 / 3, 2.5e-308]
    w[:len(special)] = special
    u, v = uv[:, 0].copy(), uv[:, 1].copy()
    deg = np.zeros(n)
    for a, b, c in zip(u, v, w):
        deg[a] += c
        deg[b] += c
    row_ptr = np.searchsorted(u, np.arange(n + 1), side="left").astype(np.uint64)
    return WeightedGraph(n=n, u=u, v=v, w=w, row_ptr=row_ptr, degrees=deg,
                         total_weight=float(np.sum(w)))


@pytest.fixture(scope="module")
def graph():
    return random_graph(3000, 20000, 11)


@pytest.mark.parametrize("threads", [1, 7, 0])
def test_text_bytes_match_reference(ref, graph, tmp_path, threads):
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    graph.write_edge_list(str(ours), threads=threads)
    ref.save_edge_list(str(theirs), graph.n, graph.u, graph.v, graph.w)
    assert ours.read_bytes() == theirs.read_bytes()


def test_text_read_matches_reference(ref, graph, tmp_path):
    path = tmp_path / "g.txt"
    ref.save_edge_list(str(path), graph.n, graph.u, graph.v, graph.w)
    g = F.read_edge_list(str(path))
    r = ref.load_edge_list(str(path))
    assert g.n == r["n"]
    np.testing.assert_array_equal(g.u, r["u"])
    np.testing.assert_array_equal(g.v, r["v"])
    assert g.w.tobytes() == r["w"].tobytes()
    assert g.degrees.tobytes() == r["degrees"].tobytes()
    assert g.total_weight == r["total_weight"]
    np.testing.assert_array_equal(g.row_ptr, graph.row_ptr)


def test_text_unsorted_swapped_and_whitespace(ref, tmp_path):
    rng = np.random.default_rng(3)
    g0 = random_graph(400, 1500, 5)
    order = rng.permutation(g0.num_edges())
    lines = []
    for e in order:
        a, b = int(g0.u[e]), int(g0.v[e])
        if rng.random() < 0.5:
            a, b = b, a
        sep = ["\t", "  ", " \n ", " "][int(rng.integers(0, 4))]
        lines.append(f"{a}{sep}{b} {float(g0.w[e])!r}")
    path = tmp_path / "messy.txt"
    path.write_text(f"{g0.n}\n{g0.num_edges()}\n" + "\n".join(lines) + "\n\n7 8 9\n")
    g = F.read_edge_list(str(path), threads=3)
    r = ref.load_edge_list(str(path))
    np.testing.assert_array_equal(g.u, r["u"])
    np.testing.assert_array_equal(g.v, r["v"])
    assert g.w.tobytes() == r["w"].tobytes()
    assert g.degrees.tobytes() == r["degrees"].tobytes()


@pytest.mark.parametrize("body", ["", "5", "5 x\n", "5 2\n0 1 0.5\n", "5 1\n0 1 zz\n",
                                  "5 1\n0 1\n"])
def test_text_malformed(ref, tmp_path, body):
    path = tmp_path / "bad.txt"
    path.write_text(body)
    with pytest.raises(F.IoError):
        F.read_edge_list(str(path))
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError) as e:
        ref.load_edge_list(str(path))
    assert e.value.code == 3


def test_missing_files(tmp_path):
    with pytest.raises(F.IoError):
        F.read_edge_list(str(tmp_path / "nope.txt"))
    with pytest.raises(F.IoError):
        F.load_csr(str(tmp_path / "nope.csr"))
    with pytest.raises(F.IoError):
        random_graph(10, 20, 1).write_edge_list(str(tmp_path / "no" / "dir.txt"))


def test_csr_round_trip(graph, tmp_path):
    path = tmp_path / "g.csr"
    graph.save_csr(str(path))
    g = F.load_csr(str(path))
    assert g.n == graph.n and g.total_weight == graph.total_weight
    for k in ("u", "v", "w", "row_ptr", "degrees"):
        assert getattr(g, k).tobytes() == getattr(graph, k).astype(getattr(g, k).dtype).tobytes()
    assert os.path.getsize(path) == 32 + 8 * (graph.n + 1) + 12 * graph.num_edges() + 8 * graph.n
    data = path.read_bytes()
    (tmp_path / "cut.csr").write_bytes(data[:-8])
    with pytest.raises(F.IoError):
        F.load_csr(str(tmp_path / "cut.csr"))
    (tmp_path / "magic.csr").write_bytes(b"X" + data[1:])
    with pytest.raises(F.IoError):
        F.load_csr(str(tmp_path / "magic.csr"))
