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


# ---- point files: fsg::load_csv / save_csv (proj/src/dataset.cpp:54-130) ----

def _points(n, d, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 3, (n, d)) * np.exp(rng.normal(0, 4, (n, d)))
    special = [0.0, -0.0, 1.0, 0.1, 1e-300, 5e-324, -1.7976931348623157e308, 2.0 ** 53 + 2,
               1 / 3, -2.5e-308]
    x.flat[:len(special)] = special
    return x


@pytest.mark.parametrize("labels", [False, True])
def test_csv_save_bytes_match_reference(ref, tmp_path, labels):
    x = _points(5000, 3, 1)
    lab = (np.arange(5000) * 7 % 11).astype(np.uint32) if labels else None
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    F.save_csv(str(ours), x, lab, threads=3)
    ref.save_csv(str(theirs), x, lab)
    assert ours.read_bytes() == theirs.read_bytes()


CSV_CASES = {
    "header_labels": "x0,x1,label\n1,2,0\n3.5,-4e-3,1\n",
    "no_header": "1,2\n3,4\n\n5,6\n",
    "crlf_spaces": "x0,x1\r\n 1 , 2\r\n3,\t4 \r\n",
    "header_no_label": "a,b,c\n1,2,3\n",
    "label_fraction": "x0,label\n1.5,2.9\n2.5,0\n",
    "trailing_no_newline": "x0\n1\n2",
    "blank_lines": "\n\nx0,x1\n\n1,2\n\n",
    "exponents": "1e300,-2.5E-308\n0x1p3,inf\n",
    "bad_count": "x0,x1\n1,2\n3\n",
    "bad_value": "x0,x1\n1,2\n3,abc\n",
    "negative_label": "x0,label\n1,-1\n",
    "empty_field": "x0,x1\n1,\n",
    "no_rows": "x0,x1\n\n",
    "nonfinite": "x0\nnan\n",
    "header_only_label": "label\n1\n",
}


@pytest.mark.parametrize("case", sorted(CSV_CASES))
def test_csv_load_matches_reference(ref, tmp_path, case):
    path = tmp_path / f"{case}.csv"
    path.write_bytes(CSV_CASES[case].encode())
    from oracle.pyoracle import OracleError
    try:
        want = ref.load_csv(str(path))
        want_err = None
    except OracleError as e:  # the reference's exit code decides ours
        want, want_err = None, e.code
    try:
        got = F.load_csv(str(path), threads=2)
        got_err = None
    except F.Error as e:
        got, got_err = None, e
    if want is None:
        assert got is None, f"reference failed ({want_err}) but we parsed {case}"
        assert got_err.exit_code == want_err, (got_err, want_err)
    else:
        assert got_err is None, got_err
        assert np.array_equal(got[0], want[0]) and got[0].shape == want[0].shape
        assert (got[1] is None) == (want[1] is None)
        if want[1] is not None:
            assert np.array_equal(got[1], want[1])


def test_csv_large_parallel_round_trip(ref, tmp_path):
    x = _points(200_000, 5, 2)
    lab = (np.arange(200_000) % 7).astype(np.uint32)
    path = tmp_path / "big.csv"
    F.save_csv(str(path), x, lab)
    for t in (1, 4, 0):
        y, l = F.load_csv(str(path), threads=t)
        assert np.array_equal(y, x) and np.array_equal(l, lab)
    y2, l2 = ref.load_csv(str(path))
    assert np.array_equal(y2, x) and np.array_equal(l2, lab)
