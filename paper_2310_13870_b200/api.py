"""Host-side mirror of the reference's hot-path interface, over the C ABI.

Names, argument meaning and error behaviour follow the reference library
``fsg`` so a caller (and the parity tests) read like the reference's own:

==============================  ============================================
this module                     reference
==============================  ============================================
``Dataset``                     fsg::Dataset (proj/include/fsg/dataset.hpp:12)
``Kernel`` / ``KernelFamily``   fsg::Kernel (proj/include/fsg/kernel.hpp:21)
``SparsifierConfig``            proj/include/fsg/sparsifier.hpp:14-26
``build_similarity_graph``      proj/src/sparsifier.cpp:51-142
``sample_neighbors_counted``    proj/src/sampler.cpp:77-247
``sample_neighbors``            proj/src/sampler.cpp:249-269
``make_estimator(...).eval``    fsg::KdeEstimator::eval (kde.hpp:54-58)
``WeightedGraph``               proj/include/fsg/graph.hpp:20-40
``BuildReport``/``EdgeEstimate`` proj/include/fsg/sparsifier.hpp:29-58
==============================  ============================================

All compute runs in libfsgg.so on an sm_100a device; nothing here loops
over points or edges.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import InvalidConfig, LengthMismatch, TooFewPoints


class KernelFamily(enum.IntEnum):
    gaussian = 0
    exponential = 1
    laplacian = 2


class RngMode(enum.IntEnum):
    reference = 0  # bit-exact keyed splitmix64 streams (proj/include/fsg/rng.hpp)
    philox = 1     # Philox4x32-10, same law, not edge-for-edge


class LogBase(enum.IntEnum):
    two = 0
    natural = 1


@dataclass(frozen=True)
class Kernel:
    """proj/include/fsg/kernel.hpp:21-58. Bandwidth must be positive
    (proj/src/kernel.cpp:23-26)."""

    family: KernelFamily = KernelFamily.gaussian
    sigma: float = 1.0

    def __post_init__(self):
        if not (self.sigma > 0.0):
            raise InvalidConfig("kernel bandwidth must be positive")

    def _c(self):
        return N.fsgg_kernel(int(self.family), float(self.sigma))

    def __call__(self, x, y) -> float:
        """k(x, y) in fp64 (host helper for small checks only)."""
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        if self.family == KernelFamily.gaussian:
            return math.exp(-float(np.sum((x - y) ** 2)) / (self.sigma * self.sigma))
        if self.family == KernelFamily.exponential:
            return math.exp(-math.sqrt(float(np.sum((x - y) ** 2))) / self.sigma)
        return math.exp(-float(np.sum(np.abs(x - y))) / self.sigma)


def default_epsilon(n: int, log_base: LogBase = LogBase.two) -> float:
    """proj/src/kde.cpp:15-18."""
    return N.lib().fsgg_default_epsilon(n, int(log_base))


class KdeBackend(enum.IntEnum):
    """fsg::KdeBackend (proj/include/fsg/kde.hpp:20). ``exact`` is this
    library's default (the reference's is ``autoselect``): see fsgg.h,
    fsgg_config::kde_backend, for the fast backend's certified budget."""

    exact = 0
    fast = 1
    autoselect = 2


@dataclass
class SparsifierConfig:
    """proj/include/fsg/sparsifier.hpp:14-26 (+ rng_mode, query shard)."""

    C: float = 1.0
    lambda_k1_estimate: float = 1.0
    rounds: int = 0
    epsilon: float = 0.0
    log_base: LogBase = LogBase.two
    seed: int = 1
    rng_mode: RngMode = RngMode.reference
    query_begin: int = 0
    query_end: int = 0
    dense_kde: bool = False  # True: evaluate every kernel term (no certified pruning)
    kde_backend: KdeBackend = KdeBackend.exact  # SparsifierConfig::kde.backend

    def _c(self):
        c = N.fsgg_config()
        c.C = self.C
        c.lambda_k1_estimate = self.lambda_k1_estimate
        c.rounds = self.rounds
        c.epsilon = self.epsilon
        c.log_base = int(self.log_base)
        c.seed = self.seed
        c.rng_mode = int(self.rng_mode)
        c.query_begin = self.query_begin
        c.query_end = self.query_end
        c.dense_kde = int(self.dense_kde)
        c.kde_backend = int(self.kde_backend)
        return c

    def rounds_for(self, n: int) -> int:
        """proj/src/sparsifier.cpp:17-23."""
        out = C.c_uint32()
        c = self._c()
        N.check(N.lib().fsgg_rounds_for(C.byref(c), n, C.byref(out)))
        return out.value

    def epsilon_for(self, n: int) -> float:
        """proj/src/sparsifier.cpp:25-28."""
        return self.epsilon if self.epsilon > 0 else default_epsilon(n, self.log_base)


class Dataset:
    """Device-resident fp32 point set (fsg::Dataset, index order = tree order).

    ``points`` may be a numpy array (host, fp32 or fp64 — fp64 is rounded to
    fp32) or a CUDA torch tensor (device pointer, fp32, contiguous)."""

    def __init__(self, points, device: int = 0):
        self._h = None
        lib = N.lib()
        h = C.c_void_p()
        if hasattr(points, "is_cuda") and points.is_cuda:
            import torch
            if points.dtype != torch.float32 or points.dim() != 2:
                raise InvalidConfig("device points must be a 2-D float32 tensor")
            pts = points.contiguous()
            n, d = pts.shape
            # the library copies on its own stream, which does not wait for
            # torch's: finish whatever is still writing the tensor first
            torch.cuda.current_stream(pts.device).synchronize()
            device = pts.device.index if pts.device.index is not None else torch.cuda.current_device()
            N.check(lib.fsgg_dataset_create(C.c_void_p(pts.data_ptr()), n, d, 1,
                                            device, C.byref(h)))
        else:
            arr = np.asarray(points)
            if arr.ndim != 2:
                raise InvalidConfig("points must be a 2-D array (n x d)")
            n, d = arr.shape
            if arr.dtype == np.float64:
                arr = np.ascontiguousarray(arr)
                N.check(lib.fsgg_dataset_create_f64(arr.ctypes.data_as(C.c_void_p), n, d,
                                                    device, C.byref(h)))
            else:
                arr = np.ascontiguousarray(arr, np.float32)
                N.check(lib.fsgg_dataset_create(arr.ctypes.data_as(C.c_void_p), n, d, 0,
                                                device, C.byref(h)))
        self._h = h
        self.n, self.d, self.device = int(n), int(d), device

    def size(self) -> int:
        return self.n

    def dim(self) -> int:
        return self.d

    def upload(self, host_points: np.ndarray):
        """Replace coordinates from pinned/pageable host fp32 memory."""
        arr = np.ascontiguousarray(host_points, np.float32)
        if arr.shape != (self.n, self.d):
            raise LengthMismatch("upload shape does not match the dataset")
        N.check(N.lib().fsgg_dataset_upload(self._h, arr.ctypes.data_as(C.c_void_p)))

    def upload_ptr(self, host_ptr: int):
        N.check(N.lib().fsgg_dataset_upload(self._h, C.c_void_p(host_ptr)))

    def device_ptr(self) -> int:
        return int(N.lib().fsgg_dataset_device_points(self._h) or 0)

    def close(self):
        if self._h is not None and N._lib is not None:
            N.lib().fsgg_dataset_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class WeightedGraph:
    """Sorted (u < v) undirected edge list + CSR (proj/include/fsg/graph.hpp)."""

    n: int
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    row_ptr: np.ndarray
    degrees: np.ndarray
    total_weight: float

    def num_vertices(self) -> int:
        return self.n

    def num_edges(self) -> int:
        return int(self.v.size)

    def __getattr__(self, name):
        # graphs read back as CSR only (HostGraphBuffers.fetch) expand the
        # row index of every edge on first use
        if name == "u":
            u = np.repeat(np.arange(self.n, dtype=np.uint32),
                          np.diff(np.asarray(self.row_ptr, np.int64)))
            object.__setattr__(self, "u", u)
            return u
        raise AttributeError(name)

    def degree(self, v: int) -> float:
        return float(self.degrees[v])

    def edges(self):
        return list(zip(self.u.tolist(), self.v.tolist(), self.w.tolist()))

    def write_edge_list(self, path: str, threads: int = 0):
        """fsg::save_edge_list (proj/src/graph.cpp:234-241, 265-270): "n m"
        then "u v %.17g" per edge, byte-identical to the reference's file."""
        u = np.ascontiguousarray(self.u, np.uint32)
        v = np.ascontiguousarray(self.v, np.uint32)
        w = np.ascontiguousarray(self.w, np.float64)
        N.check(N.lib().fsgg_graph_save_text(os.fsencode(path), self.n, u.size,
                                             u.ctypes.data, v.ctypes.data, w.ctypes.data,
                                             threads))

    def _c(self):
        """fsgg_graph view of this graph's arrays (and the arrays keeping it alive)."""
        g = N.fsgg_graph()
        keep = [np.ascontiguousarray(self.u, np.uint32), np.ascontiguousarray(self.v, np.uint32),
                np.ascontiguousarray(self.w, np.float64),
                np.ascontiguousarray(self.row_ptr, np.uint64),
                np.ascontiguousarray(self.degrees, np.float64)]
        g.n, g.num_edges, g.total_weight = self.n, keep[0].size, self.total_weight
        g.u, g.v, g.w, g.row_ptr, g.degrees = (C.cast(a.ctypes.data, f) for a, f in zip(
            keep, [C.POINTER(C.c_uint32)] * 2 + [C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                                 C.POINTER(C.c_double)]))
        return g, keep

    def save_csr(self, path: str):
        """Binary upper-triangular CSR (include/fsgg.h: fsgg_graph_save_csr)."""
        g, _keep = self._c()
        N.check(N.lib().fsgg_graph_save_csr(os.fsencode(path), C.byref(g)))


def _load_graph(fn, path, *extra) -> WeightedGraph:
    g = N.fsgg_graph()
    lib = N.lib()
    N.check(getattr(lib, fn)(os.fsencode(path), *extra, C.byref(g)))
    try:
        return _graph_from_c(g)
    finally:
        lib.fsgg_graph_free(C.byref(g))


def read_edge_list(path: str, threads: int = 0) -> WeightedGraph:
    """fsg::load_edge_list (proj/src/graph.cpp:243-263, 272-276)."""
    return _load_graph("fsgg_graph_load_text", path, threads)


def load_csr(path: str) -> WeightedGraph:
    """Inverse of WeightedGraph.save_csr."""
    return _load_graph("fsgg_graph_load_csr", path)


def load_csv(path: str, threads: int = 0):
    """fsg::load_csv (proj/src/dataset.cpp:54-102): returns (points as an
    n x d float64 array, labels as uint32 or None)."""
    lib = N.lib()
    pts, lab = C.c_void_p(), C.c_void_p()
    n, d = C.c_uint32(), C.c_uint32()
    N.check(lib.fsgg_csv_load(os.fsencode(path), threads, C.byref(pts), C.byref(n),
                              C.byref(d), C.byref(lab)))
    try:
        x = np.ctypeslib.as_array(C.cast(pts, C.POINTER(C.c_double)),
                                  shape=(n.value * d.value,)).copy().reshape(n.value, d.value)
        labels = None
        if lab.value:
            labels = np.ctypeslib.as_array(C.cast(lab, C.POINTER(C.c_uint32)),
                                           shape=(n.value,)).copy()
        return x, labels
    finally:
        lib.fsgg_free(pts)
        lib.fsgg_free(lab)


def save_csv(path: str, points, labels=None, threads: int = 0):
    """fsg::save_csv (proj/src/dataset.cpp:104-130): "x0,...[,label]" header,
    "%.17g" values."""
    x = np.ascontiguousarray(points, np.float64)
    if x.ndim != 2:
        raise ValueError("points must be n x d")
    n, d = x.shape
    lab = None
    if labels is not None:
        lab = np.ascontiguousarray(labels, np.uint32)
        if lab.size != n:
            from .errors import LengthMismatch
            raise LengthMismatch("label count does not match dataset size")
    N.check(N.lib().fsgg_csv_save(os.fsencode(path), x.ctypes.data, n, d,
                                  lab.ctypes.data if lab is not None else None, threads))


@dataclass
class BuildReport:
    """proj/include/fsg/sparsifier.hpp:40-58 plus device counters."""

    n: int = 0
    rounds: int = 0
    epsilon: float = 0.0
    backend: str = ""
    sampled_pairs: int = 0
    self_pairs_discarded: int = 0
    underflow_edges_discarded: int = 0
    edge_count: int = 0
    degenerate_draws: int = 0
    estimator_build_seconds: float = 0.0
    sampling_seconds: float = 0.0
    degree_kde_seconds: float = 0.0
    weighting_seconds: float = 0.0
    total_seconds: float = 0.0
    estimator_bytes: int = 0
    graph_bytes: int = 0
    kernel_evals: int = 0
    kde_tiled_evals: int = 0
    kde_tiled_seconds: float = 0.0
    kde_tiled_launches: int = 0
    levels: int = 0
    peak_entries: int = 0
    gpu_launches: int = 0
    kernel_evals_performed: int = 0
    kde_tiled_performed_evals: int = 0
    tie_verified_entries: int = 0
    kde_root_performed_evals: int = 0
    kde_root_seconds: float = 0.0

    @classmethod
    def _from_c(cls, r):
        out = cls()
        for name, _ in N.fsgg_report._fields_:
            v = getattr(r, name)
            setattr(out, name, v.decode() if isinstance(v, bytes) else v)
        return out


EDGE_ESTIMATE_DTYPE = np.dtype([("i", "<u4"), ("j", "<u4"), ("k_ij", "<f8"), ("g_i", "<f8"),
                                ("g_j", "<f8"), ("p_hat_i_j", "<f8"), ("p_hat_j_i", "<f8"),
                                ("p_hat", "<f8")])


def _as_numpy(ptr, count, ctype, dtype):
    if count == 0:
        return np.zeros(0, dtype)
    arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,))
    return np.array(arr, dtype=dtype, copy=True)


def _graph_from_c(g) -> WeightedGraph:
    m = int(g.num_edges)
    return WeightedGraph(
        n=int(g.n), u=_as_numpy(g.u, m, C.c_uint32, np.uint32),
        v=_as_numpy(g.v, m, C.c_uint32, np.uint32),
        w=_as_numpy(g.w, m, C.c_double, np.float64),
        row_ptr=_as_numpy(g.row_ptr, int(g.n) + 1, C.c_uint64, np.uint64),
        degrees=_as_numpy(g.degrees, int(g.n), C.c_double, np.float64),
        total_weight=float(g.total_weight))


def device_graph_to_host(ds: Dataset) -> WeightedGraph:
    """Host copy of the graph left on the device by the last device-resident
    or distributed build on ``ds``."""
    g = N.fsgg_graph()
    lib = N.lib()
    N.check(lib.fsgg_device_graph_to_host(ds._h, C.byref(g)))
    try:
        return _graph_from_c(g)
    finally:
        lib.fsgg_graph_free(C.byref(g))


class HostGraphBuffers:
    """Reusable page-locked host buffers for device graph read-back (the
    e2e path): grown on demand, filled by fsgg_device_graph_copy."""

    def __init__(self):
        self._bufs = {}

    def _get(self, name, count, dtype):
        import torch
        tdt = {np.uint32: torch.int32, np.float64: torch.float64, np.uint64: torch.int64}[dtype]
        t = self._bufs.get(name)
        if t is None or t.numel() < count:
            t = torch.empty(max(count, 1) + max(count, 1) // 4, dtype=tdt, pin_memory=True)
            self._bufs[name] = t
        return t.numpy().view(dtype)[:count]

    def fetch(self, ds: "Dataset", graph, with_u: bool = False) -> "WeightedGraph":
        """Copy the device graph into the pinned buffers. By default only the
        CSR (row_ptr, v, w) and degrees cross PCIe — the complete graph; the
        per-edge u (a 4-byte row index per edge) is expanded on the host on
        first access, or copied too with with_u=True."""
        m, n = int(graph.num_edges), int(graph.n)
        u = self._get("u", m, np.uint32) if with_u else None
        v = self._get("v", m, np.uint32)
        w = self._get("w", m, np.float64)
        rp = self._get("row_ptr", n + 1, np.uint64)
        dg = self._get("degrees", n, np.float64)
        N.check(N.lib().fsgg_device_graph_copy(
            ds._h, u.ctypes.data_as(C.c_void_p) if with_u else None,
            v.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p),
            rp.ctypes.data_as(C.c_void_p), dg.ctypes.data_as(C.c_void_p)))
        g = WeightedGraph(n=n, u=u, v=v, w=w, row_ptr=rp, degrees=dg,
                          total_weight=float(graph.total_weight))
        if not with_u:
            del g.u  # expanded lazily from row_ptr (WeightedGraph.__getattr__)
        return g

    def build_into(self, ds: "Dataset", kernel: "Kernel", config: "SparsifierConfig",
                   rounds: int) -> "WeightedGraph":
        """build_similarity_graph straight into the pinned buffers
        (fsgg_build_similarity_graph_into): each CSR array's device-to-host
        copy starts as soon as it is final, overlapping the rest of the
        finish. ``rounds`` sizes the edge buffers (n * L bounds the edges)."""
        n = ds.n
        cap = n * rounds
        v = self._get("v", cap, np.uint32)
        w = self._get("w", cap, np.float64)
        rp = self._get("row_ptr", n + 1, np.uint64)
        dg = self._get("degrees", n, np.float64)
        m = C.c_uint64()
        tw = C.c_double()
        rep = N.fsgg_report()
        N.check(N.lib().fsgg_build_similarity_graph_into(
            ds._h, C.byref(kernel._c()), C.byref(config._c()), cap,
            v.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p),
            rp.ctypes.data_as(C.c_void_p), dg.ctypes.data_as(C.c_void_p), C.byref(m),
            C.byref(tw), C.byref(rep)))
        mm = int(m.value)
        g = WeightedGraph(n=n, u=None, v=v[:mm], w=w[:mm], row_ptr=rp, degrees=dg,
                          total_weight=float(tw.value))
        del g.u  # expanded lazily from row_ptr
        return g


def build_similarity_graph(ds: Dataset, kernel: Kernel, config: SparsifierConfig | None = None,
                           report: bool = False, estimates: bool = False):
    """FastSimilarityGraph (proj/src/sparsifier.cpp:51-142) on the device.

    Returns ``graph`` or ``(graph, report, estimates)`` when either flag is
    set (estimates is a structured array with EdgeEstimate's fields)."""
    cfg = (config or SparsifierConfig())._c()
    k = kernel._c()
    g = N.fsgg_graph()
    rep = N.fsgg_report()
    est = C.POINTER(N.fsgg_edge_estimate)()
    lib = N.lib()
    N.check(lib.fsgg_build_similarity_graph(ds._h, C.byref(k), C.byref(cfg), C.byref(g),
                                            C.byref(rep),
                                            C.byref(est) if estimates else None))
    try:
        graph = _graph_from_c(g)
    finally:
        lib.fsgg_graph_free(C.byref(g))
    est_arr = None
    if estimates:
        m = int(g.num_edges) if g.num_edges else graph.num_edges()
        nbytes = m * C.sizeof(N.fsgg_edge_estimate)
        if m:
            raw = np.ctypeslib.as_array(C.cast(est, C.POINTER(C.c_uint8)), shape=(nbytes,))
            est_arr = raw.view(EDGE_ESTIMATE_DTYPE).copy()
        else:
            est_arr = np.zeros(0, EDGE_ESTIMATE_DTYPE)
        lib.fsgg_free(C.cast(est, C.c_void_p))
    if report or estimates:
        return graph, BuildReport._from_c(rep), est_arr
    return graph


def build_similarity_graph_device(ds: Dataset, kernel: Kernel,
                                  config: SparsifierConfig | None = None):
    """Device-resident build (no graph copy back). Returns (fsgg_device_graph,
    BuildReport); pointers stay valid until the next build on ``ds``."""
    cfg = (config or SparsifierConfig())._c()
    k = kernel._c()
    g = N.fsgg_device_graph()
    rep = N.fsgg_report()
    N.check(N.lib().fsgg_build_similarity_graph_device(ds._h, C.byref(k), C.byref(cfg),
                                                       C.byref(g), C.byref(rep)))
    return g, BuildReport._from_c(rep)


@dataclass
class SampleDiagnostics:
    """proj/include/fsg/sampler.hpp:22-26."""

    entries_per_level: list = field(default_factory=list)
    tickets_per_level: list = field(default_factory=list)
    degenerate_draws: int = 0


def sample_neighbors_counted(ds: Dataset, kernel: Kernel, queries, rounds: int, seed: int,
                             rng_mode: RngMode = RngMode.reference, diagnostics: bool = False,
                             dense_kde: bool = False):
    """proj/src/sampler.cpp:77-247: (query, source, count) rows sorted by
    (query, source), as an (m, 3) uint32 array."""
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.int64))
    if q.size and (q.min() < 0):
        raise InvalidConfig("query index out of range")
    q = q.astype(np.uint32)
    k = kernel._c()
    out = C.c_void_p()
    cnt = C.c_size_t()
    diag = N.fsgg_sample_diag()
    lib = N.lib()
    N.check(lib.fsgg_sample_neighbors_counted(ds._h, C.byref(k), q.ctypes.data_as(C.c_void_p),
                                              q.size, rounds, seed, int(rng_mode),
                                              int(dense_kde), C.byref(out), C.byref(cnt),
                                              C.byref(diag)))
    m = cnt.value
    tri = _as_numpy(out, 3 * m, C.c_uint32, np.uint32).reshape(m, 3)
    lib.fsgg_free(out)
    if diagnostics:
        d = SampleDiagnostics(list(diag.entries_per_level)[: diag.nlevels],
                              list(diag.tickets_per_level)[: diag.nlevels],
                              int(diag.degenerate_draws))
        return tri, d
    return tri


@dataclass
class SampleReport:
    """fsgg_sample_report: diagnostics, evaluation counters and (with
    ``record_sums``) every entry's child sums as the level kernels produced
    them. ``records`` is a numpy structured array with fields level, query,
    first, last, left, right (children [first, mid) and [mid, last),
    mid = first + (last - first) // 2)."""

    diagnostics: SampleDiagnostics
    kernel_evals: int
    kernel_evals_performed: int
    root_evals_performed: int
    tie_verified: int
    records: np.ndarray | None


RECORD_DTYPE = np.dtype([("level", "<u4"), ("query", "<u4"), ("first", "<u4"), ("last", "<u4"),
                         ("left", "<f8"), ("right", "<f8")])


def sample_neighbors_counted_ex(ds: Dataset, kernel: Kernel, queries, rounds: int, seed: int,
                                rng_mode: RngMode = RngMode.reference, dense_kde: bool = False,
                                record_sums: bool = False, walks: bool = True,
                                kde_backend: "KdeBackend" = None, epsilon: float = 0.0):
    """fsgg_sample_neighbors_counted_ex: the descent with options; returns
    (triples, SampleReport)."""
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.int64))
    if q.size and (q.min() < 0):
        raise InvalidConfig("query index out of range")
    q = q.astype(np.uint32)
    k = kernel._c()
    opt = N.fsgg_sample_options()
    lib = N.lib()
    lib.fsgg_sample_options_init(C.byref(opt))
    opt.rng_mode = int(rng_mode)
    opt.dense_kde = int(dense_kde)
    opt.record_sums = int(record_sums)
    opt.walks = int(walks)
    opt.kde_backend = int(KdeBackend.exact if kde_backend is None else kde_backend)
    opt.epsilon = float(epsilon)
    out = C.c_void_p()
    cnt = C.c_size_t()
    rep = N.fsgg_sample_report()
    N.check(lib.fsgg_sample_neighbors_counted_ex(ds._h, C.byref(k), q.ctypes.data_as(C.c_void_p),
                                                 q.size, rounds, seed, C.byref(opt), C.byref(out),
                                                 C.byref(cnt), C.byref(rep)))
    m = cnt.value
    tri = _as_numpy(out, 3 * m, C.c_uint32, np.uint32).reshape(m, 3)
    lib.fsgg_free(out)
    recs = None
    if rep.records:
        nr = rep.num_records
        buf = (C.c_char * (nr * RECORD_DTYPE.itemsize)).from_address(rep.records)
        recs = np.frombuffer(bytes(buf), dtype=RECORD_DTYPE).copy()
        lib.fsgg_free(C.c_void_p(rep.records))
    d = rep.diag
    diag = SampleDiagnostics(list(d.entries_per_level)[: d.nlevels],
                             list(d.tickets_per_level)[: d.nlevels], int(d.degenerate_draws))
    return tri, SampleReport(diag, int(rep.kernel_evals), int(rep.kernel_evals_performed),
                             int(rep.root_evals_performed), int(rep.tie_verified), recs)


def sample_neighbors(ds: Dataset, kernel: Kernel, queries, seed: int,
                     rng_mode: RngMode = RngMode.reference):
    """proj/src/sampler.cpp:249-269: one neighbour per query, sorted by
    query; returns an (len(queries), 2) array of (query, source)."""
    q = np.asarray(queries, dtype=np.int64)
    tri = sample_neighbors_counted(ds, kernel, q, 1, seed, rng_mode)
    choice = {int(a): int(b) for a, b, _ in tri}
    out = np.array([(int(x), choice[int(x)]) for x in q], dtype=np.uint32).reshape(-1, 2)
    order = np.lexsort((out[:, 1], out[:, 0])) if out.size else np.zeros(0, np.int64)
    return out[order]


class KdeEstimator:
    """The plugin seam fsg::KdeEstimator (proj/include/fsg/kde.hpp:49-85),
    exact backend on the device."""

    backend_name = "gpu-exact-sm100a"
    sum_floor = 1e-300

    def __init__(self, ds: Dataset, kernel: Kernel):
        self.ds = ds
        self.kernel = kernel

    def epsilon(self) -> float:
        return 0.0

    def eval(self, first: int, last: int, targets) -> np.ndarray:
        t = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
        if t.size and t.min() < 0:
            raise InvalidConfig("target index out of range")
        t = t.astype(np.uint32)
        if first < 0 or last < 0:
            raise InvalidConfig("invalid source index range")
        out = np.zeros(t.size, np.float64)
        k = self.kernel._c()
        N.check(N.lib().fsgg_kde_eval(self.ds._h, C.byref(k), first, last,
                                      t.ctypes.data_as(C.c_void_p), t.size,
                                      out.ctypes.data_as(C.c_void_p)))
        return out


def make_estimator(ds: Dataset, kernel: Kernel) -> KdeEstimator:
    """proj/src/kde.cpp:104-129; the device path is always exact."""
    return KdeEstimator(ds, kernel)


def exact_kde(ds: Dataset, kernel: Kernel, first: int, last: int, targets) -> np.ndarray:
    """proj/src/kde.cpp:131-138."""
    return make_estimator(ds, kernel).eval(first, last, targets)


def device_available() -> bool:
    return bool(N.lib().fsgg_device_available())


def _ensure_two_points(n):
    if n < 2:
        raise TooFewPoints("similarity graph needs n >= 2")


# ---- spectral clustering (proj/include/fsg/spectral.hpp) on the device ----

@dataclass
class EigenOptions:
    """proj/include/fsg/spectral.hpp:11-16"""
    tol: float = 1e-6
    max_matvecs: int = 0
    max_basis: int = 0
    seed: int = 7

    def _c(self):
        return N.fsgg_eigen_options(self.tol, self.max_matvecs, self.max_basis, self.seed)


@dataclass
class KMeansOptions:
    """proj/include/fsg/spectral.hpp:44-49"""
    restarts: int = 10
    max_iters: int = 300
    rel_tol: float = 1e-8
    seed: int = 7

    def _c(self):
        return N.fsgg_kmeans_options(self.restarts, self.max_iters, self.rel_tol, self.seed)


@dataclass
class SpectralOptions:
    eigen: EigenOptions = field(default_factory=EigenOptions)
    kmeans: KMeansOptions = field(default_factory=KMeansOptions)

    def _c(self):
        return N.fsgg_spectral_options(self.eigen._c(), self.kmeans._c())


@dataclass
class EigenResult:
    """fsg::EigenResult: eigenvalues ascending; eigenvectors[i] is pair i."""
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray | None
    residuals: np.ndarray
    matvecs: int


def smallest_eigenpairs(graph, q: int, options: EigenOptions | None = None,
                        vectors: bool = True, device: int = 0) -> EigenResult:
    """fsg::smallest_eigenpairs (proj/src/spectral.cpp:40-222) of the
    normalised Laplacian, on the device. ``graph`` is a Dataset (its last
    device-built graph) or a WeightedGraph (uploaded for the call)."""
    opts = (options or EigenOptions())._c()
    vals = np.zeros(q)
    res = np.zeros(q)
    mv = C.c_uint64()
    lib = N.lib()
    if isinstance(graph, Dataset):
        n = graph.n
        vecs = np.zeros((q, n)) if vectors else None
        N.check(lib.fsgg_smallest_eigenpairs(graph._h, q, C.byref(opts), vals.ctypes.data,
                                             vecs.ctypes.data if vectors else None,
                                             res.ctypes.data, C.byref(mv)))
    else:
        g, keep = graph._c()
        vecs = np.zeros((q, graph.n)) if vectors else None
        N.check(lib.fsgg_smallest_eigenpairs_graph(C.byref(g), device, q, C.byref(opts),
                                                   vals.ctypes.data,
                                                   vecs.ctypes.data if vectors else None,
                                                   res.ctypes.data, C.byref(mv)))
    return EigenResult(vals, vecs, res, int(mv.value))


def spectral_cluster(graph, k: int, seed: int = 7, options: SpectralOptions | None = None,
                     device: int = 0, report: bool = False):
    """fsg::spectral_cluster (proj/src/spectral.cpp:405-419) on the device:
    labels (uint32, n) in [0, k); with report=True also a dict of counters."""
    opts = (options or SpectralOptions())._c()
    rep = N.fsgg_spectral_report()
    lib = N.lib()
    if isinstance(graph, Dataset):
        labels = np.zeros(graph.n, np.uint32)
        N.check(lib.fsgg_spectral_cluster(graph._h, k, seed, C.byref(opts), labels.ctypes.data,
                                          C.byref(rep)))
    else:
        g, keep = graph._c()
        labels = np.zeros(graph.n, np.uint32)
        N.check(lib.fsgg_spectral_cluster_graph(C.byref(g), device, k, seed, C.byref(opts),
                                                labels.ctypes.data, C.byref(rep)))
    if report:
        return labels, {f: getattr(rep, f) for f, _ in rep._fields_}
    return labels


def kmeans(points, k: int, options: KMeansOptions | None = None, device: int = 0):
    """fsg::kmeans (proj/src/spectral.cpp:257-403) on the device:
    (labels, cost, iterations) of the best restart."""
    pts = np.ascontiguousarray(points, np.float64)
    if pts.ndim != 2:
        raise ValueError("points must be n x dim")
    n, dim = pts.shape
    labels = np.zeros(n, np.uint32)
    cost = C.c_double()
    iters = C.c_uint32()
    opts = (options or KMeansOptions())._c()
    N.check(N.lib().fsgg_kmeans(pts.ctypes.data, n, dim, k, C.byref(opts), device,
                                labels.ctypes.data, C.byref(cost), C.byref(iters)))
    return labels, float(cost.value), int(iters.value)
