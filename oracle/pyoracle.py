"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Ref``    — oracle/_ref/libfsgref.so: the reference's own sources
               (/root/reference/proj/src) compiled in place + ref/ref_driver.cpp.
* ``Oracle`` — oracle/libfsgoracle.so: fsg_oracle.c, our plain-C restatement.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product
(paper_2310_13870_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfsgref.so")
ORACLE_SO = os.path.join(HERE, "libfsgoracle.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _take(lib, ptr, n, dtype):
    """Copy a malloc'd C array into numpy and free it."""
    if not ptr.value:
        return np.zeros(0, dtype)
    ctype = {np.uint32: C.c_uint32, np.float64: C.c_double}[dtype]
    arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(max(n, 1),))
    out = np.array(arr[:n], dtype=dtype, copy=True)
    lib_free = getattr(lib, "fsgref_free", None) or getattr(lib, "oracle_free")
    lib_free(ptr)
    return out


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"rc={code}: {msg}")
        self.code = code


class Ref:
    """The reference implementation (compiled in place)."""

    available = os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        self.lib = lib = C.CDLL(path)
        lib.fsgref_last_error.restype = C.c_char_p
        lib.fsgref_free.argtypes = [C.c_void_p]
        lib.fsgref_default_epsilon.restype = C.c_double
        lib.fsgref_default_epsilon.argtypes = [C.c_uint32, C.c_int]
        lib.fsgref_estimator_create.restype = C.c_void_p
        lib.fsgref_estimator_create.argtypes = [_f64p, C.c_uint32, C.c_uint32, C.c_int,
                                                C.c_double, C.c_int, C.c_double]
        lib.fsgref_estimator_destroy.argtypes = [C.c_void_p]
        lib.fsgref_estimator_backend.restype = C.c_char_p
        lib.fsgref_estimator_backend.argtypes = [C.c_void_p]
        lib.fsgref_estimator_epsilon.restype = C.c_double
        lib.fsgref_estimator_epsilon.argtypes = [C.c_void_p]
        lib.fsgref_kde_eval.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, _u32p,
                                        C.c_size_t, _f64p]
        lib.fsgref_set_threads.argtypes = [C.c_uint]
        lib.fsgref_load_csv.argtypes = [C.c_char_p, C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_void_p)]
        lib.fsgref_save_csv.argtypes = [C.c_char_p, C.c_void_p, C.c_uint32, C.c_uint32,
                                        C.c_void_p]
        lib.fsgref_worker_count.restype = C.c_uint

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.fsgref_last_error().decode())

    def set_threads(self, n: int):
        self.lib.fsgref_set_threads(n)

    def load_csv(self, path: str):
        """fsg::load_csv: (points n x d float64, labels uint32 or None)."""
        pts, lab = C.c_void_p(), C.c_void_p()
        n, d = C.c_uint32(), C.c_uint32()
        self._check(self.lib.fsgref_load_csv(os.fsencode(path), C.byref(pts), C.byref(n),
                                             C.byref(d), C.byref(lab)))
        try:
            x = np.ctypeslib.as_array(C.cast(pts, C.POINTER(C.c_double)),
                                      shape=(n.value * d.value,)).copy()
            labels = None
            if lab.value:
                labels = np.ctypeslib.as_array(C.cast(lab, C.POINTER(C.c_uint32)),
                                               shape=(n.value,)).copy()
            return x.reshape(n.value, d.value), labels
        finally:
            self.lib.fsgref_free(pts)
            self.lib.fsgref_free(lab)

    def save_csv(self, path: str, points, labels=None):
        x = np.ascontiguousarray(points, np.float64)
        lab = None if labels is None else np.ascontiguousarray(labels, np.uint32)
        self._check(self.lib.fsgref_save_csv(os.fsencode(path), x.ctypes.data, x.shape[0],
                                             x.shape[1],
                                             lab.ctypes.data if lab is not None else None))

    def worker_count(self) -> int:
        return int(self.lib.fsgref_worker_count())

    # --- generators (proj/src/datasets.cpp) --------------------------------
    def make_moons(self, n, noise, seed):
        pts = np.zeros(n * 2)
        lab = np.zeros(n, np.uint32)
        self._check(self.lib.fsgref_make_moons(C.c_uint32(n), C.c_double(noise),
                                               C.c_uint64(seed), pts.ctypes.data_as(C.c_void_p),
                                               lab.ctypes.data_as(C.c_void_p)))
        return pts.reshape(n, 2), lab

    def make_blobs(self, n, centers, stddev, seed):
        centers = np.ascontiguousarray(centers, np.float64)
        k, d = centers.shape
        pts = np.zeros(n * d)
        lab = np.zeros(n, np.uint32)
        self._check(self.lib.fsgref_make_blobs(C.c_uint32(n), centers.ctypes.data_as(C.c_void_p),
                                               C.c_uint32(k), C.c_uint32(d), C.c_double(stddev),
                                               C.c_uint64(seed), pts.ctypes.data_as(C.c_void_p),
                                               lab.ctypes.data_as(C.c_void_p)))
        return pts.reshape(n, d), lab

    def default_epsilon(self, n, log_base=0):
        return self.lib.fsgref_default_epsilon(n, log_base)

    def rounds_for(self, n, C_=1.0, lam=1.0, rounds=0, log_base=0):
        out = C.c_uint32()
        self._check(self.lib.fsgref_rounds_for(C.c_uint32(n), C.c_double(C_), C.c_double(lam),
                                               C.c_uint32(rounds), C.c_int(log_base), C.byref(out)))
        return out.value

    def kernel(self, family, sigma, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = C.c_double()
        self._check(self.lib.fsgref_kernel_eval(C.c_int(family), C.c_double(sigma),
                                                x.ctypes.data_as(C.c_void_p),
                                                y.ctypes.data_as(C.c_void_p),
                                                C.c_uint32(x.size), C.byref(out)))
        return out.value

    # --- estimator (proj/include/fsg/kde.hpp:49-89) ------------------------
    def estimator(self, pts, family=0, sigma=1.0, backend=0, epsilon=0.0):
        return RefEstimator(self, pts, family, sigma, backend, epsilon)

    def build_graph(self, pts, sigma, rounds, seed=1, family=0, backend=0, C_=1.0, lam=1.0,
                    epsilon=0.0, log_base=0, want_estimates=True):
        pts = np.ascontiguousarray(pts, np.float64)
        n, d = pts.shape
        m = C.c_size_t()
        u, v, w, deg, est = (C.c_void_p() for _ in range(5))
        rep = (C.c_double * 14)()
        name = C.create_string_buffer(64)
        self._check(self.lib.fsgref_build_graph(
            pts.ctypes.data_as(C.c_void_p), C.c_uint32(n), C.c_uint32(d), C.c_int(family),
            C.c_double(sigma), C.c_uint32(rounds), C.c_uint64(seed), C.c_int(backend),
            C.c_double(C_), C.c_double(lam), C.c_double(epsilon), C.c_int(log_base),
            C.byref(m), C.byref(u), C.byref(v), C.byref(w), C.byref(deg),
            C.byref(est) if want_estimates else None, rep, name, C.c_size_t(64)))
        M = m.value
        out = dict(u=_take(self.lib, u, M, np.uint32), v=_take(self.lib, v, M, np.uint32),
                   w=_take(self.lib, w, M, np.float64), degrees=_take(self.lib, deg, n, np.float64))
        if want_estimates:
            out["estimates"] = _take(self.lib, est, 8 * M, np.float64).reshape(M, 8)
        keys = ["n", "rounds", "epsilon", "sampled_pairs", "self_pairs_discarded",
                "underflow_edges_discarded", "edge_count", "degenerate_draws",
                "estimator_build_seconds", "sampling_seconds", "degree_kde_seconds",
                "weighting_seconds", "total_seconds", "total_weight"]
        out["report"] = dict(zip(keys, list(rep)))
        out["report"]["backend"] = name.value.decode()
        return out

    # --- spectral module (proj/src/spectral.cpp, built on ref/eigen_shim) ----
    @staticmethod
    def _graph_args(u, v, w):
        u = np.ascontiguousarray(u, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        return (u, v, w), (C.c_size_t(u.size), u.ctypes.data_as(C.c_void_p),
                           v.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p))

    def smallest_eigenpairs(self, n, u, v, w, q, tol=1e-6, seed=7, vectors=True):
        keep, args = self._graph_args(u, v, w)
        vals = np.zeros(q)
        res = np.zeros(q)
        vecs = np.zeros((q, n)) if vectors else None
        mv = C.c_uint64()
        self._check(self.lib.fsgref_smallest_eigenpairs(
            C.c_uint32(n), *args, C.c_uint32(q), C.c_double(tol), C.c_uint64(seed),
            vals.ctypes.data_as(C.c_void_p),
            vecs.ctypes.data_as(C.c_void_p) if vectors else None,
            res.ctypes.data_as(C.c_void_p), C.byref(mv)))
        return dict(eigenvalues=vals, eigenvectors=vecs, residuals=res, matvecs=mv.value)

    def spectral_cluster(self, n, u, v, w, k, seed=7):
        keep, args = self._graph_args(u, v, w)
        lab = np.zeros(n, np.uint32)
        self._check(self.lib.fsgref_spectral_cluster(C.c_uint32(n), *args, C.c_uint32(k),
                                                     C.c_uint64(seed),
                                                     lab.ctypes.data_as(C.c_void_p)))
        return lab

    def kmeans(self, pts, k, restarts=10, max_iters=300, rel_tol=1e-8, seed=7):
        pts = np.ascontiguousarray(pts, np.float64)
        n, dim = pts.shape
        lab = np.zeros(n, np.uint32)
        cost = C.c_double()
        iters = C.c_uint32()
        self._check(self.lib.fsgref_kmeans(pts.ctypes.data_as(C.c_void_p), C.c_uint32(n),
                                           C.c_uint32(dim), C.c_uint32(k), C.c_uint32(restarts),
                                           C.c_uint32(max_iters), C.c_double(rel_tol),
                                           C.c_uint64(seed), lab.ctypes.data_as(C.c_void_p),
                                           C.byref(cost), C.byref(iters)))
        return lab, cost.value, iters.value

    # --- edge-list files (proj/src/graph.cpp:234-276) -----------------------
    def save_edge_list(self, path, n, u, v, w):
        u = np.ascontiguousarray(u, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        self._check(self.lib.fsgref_save_edge_list(
            os.fsencode(path), C.c_uint32(n), C.c_size_t(u.size), u.ctypes.data_as(C.c_void_p),
            v.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)))

    def load_edge_list(self, path):
        n = C.c_uint32()
        m = C.c_size_t()
        tot = C.c_double()
        u, v, w, deg = (C.c_void_p() for _ in range(4))
        self._check(self.lib.fsgref_load_edge_list(os.fsencode(path), C.byref(n), C.byref(m),
                                                   C.byref(u), C.byref(v), C.byref(w),
                                                   C.byref(deg), C.byref(tot)))
        M = m.value
        return dict(n=n.value, u=_take(self.lib, u, M, np.uint32),
                    v=_take(self.lib, v, M, np.uint32), w=_take(self.lib, w, M, np.float64),
                    degrees=_take(self.lib, deg, n.value, np.float64), total_weight=tot.value)


class RefEstimator:
    def __init__(self, ref: Ref, pts, family, sigma, backend, epsilon):
        self.ref = ref
        self.pts = np.ascontiguousarray(pts, np.float64)
        n, d = self.pts.shape
        self.n = n
        self.h = ref.lib.fsgref_estimator_create(self.pts.reshape(-1), n, d, family, sigma,
                                                 backend, epsilon)
        if not self.h:
            raise OracleError(2, ref.lib.fsgref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.fsgref_estimator_destroy(self.h)
            self.h = None

    @property
    def backend(self):
        return self.ref.lib.fsgref_estimator_backend(self.h).decode()

    @property
    def epsilon(self):
        return self.ref.lib.fsgref_estimator_epsilon(self.h)

    def eval(self, first, last, targets):
        t = np.ascontiguousarray(targets, np.uint32)
        out = np.zeros(t.size)
        self.ref._check(self.ref.lib.fsgref_kde_eval(self.h, first, last, t, t.size, out))
        return out

    def sample_counted(self, queries, rounds, seed, inline_range=64, record=False):
        q = np.ascontiguousarray(queries, np.uint32)
        lib = self.ref.lib
        tri = C.c_void_p()
        cnt = C.c_size_t()
        epl = (C.c_uint64 * 64)()
        tpl = (C.c_uint64 * 64)()
        nl = C.c_uint32()
        deg = C.c_uint64()
        rf, rl, rq, rs = (C.c_void_p() for _ in range(4))
        rc_ = C.c_size_t()
        self.ref._check(lib.fsgref_sample_counted(
            C.c_void_p(self.h), q.ctypes.data_as(C.c_void_p), C.c_size_t(q.size),
            C.c_uint32(rounds), C.c_uint64(seed), C.c_uint32(inline_range), C.c_int(int(record)),
            C.byref(tri), C.byref(cnt), epl, tpl, C.byref(nl), C.byref(deg),
            C.byref(rf), C.byref(rl), C.byref(rq), C.byref(rs), C.byref(rc_)))
        k = cnt.value
        out = dict(triples=_take(lib, tri, 3 * k, np.uint32).reshape(k, 3),
                   entries_per_level=list(epl)[: nl.value],
                   tickets_per_level=list(tpl)[: nl.value],
                   degenerate_draws=deg.value)
        if record:
            r = rc_.value
            out["rec"] = dict(first=_take(lib, rf, r, np.uint32), last=_take(lib, rl, r, np.uint32),
                              query=_take(lib, rq, r, np.uint32), sum=_take(lib, rs, r, np.float64))
        return out


class Oracle:
    """fsg_oracle.c, the plain-C restatement."""

    available = os.path.exists(ORACLE_SO)

    def __init__(self, path: str = ORACLE_SO):
        self.lib = lib = C.CDLL(path)
        lib.oracle_splitmix64.restype = C.c_uint64
        lib.oracle_splitmix64.argtypes = [C.c_uint64]
        lib.oracle_rng_key.restype = C.c_uint64
        lib.oracle_rng_key.argtypes = [C.c_uint64] * 4
        lib.oracle_rng_double.restype = C.c_double
        lib.oracle_rng_double.argtypes = [C.c_uint64, C.c_uint64]
        lib.oracle_binomial.restype = C.c_uint64
        lib.oracle_binomial.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        lib.oracle_kernel.restype = C.c_double
        lib.oracle_kernel.argtypes = [C.c_int, C.c_double, _f64p, _f64p, C.c_uint32]
        lib.oracle_default_epsilon.restype = C.c_double
        lib.oracle_default_epsilon.argtypes = [C.c_uint32, C.c_int]
        lib.oracle_free.argtypes = [C.c_void_p]
        lib.oracle_kde_exact.argtypes = [_f64p, C.c_uint32, C.c_uint32, C.c_int, C.c_double,
                                         C.c_uint32, C.c_uint32, _u32p, C.c_size_t, C.c_double,
                                         _f64p]

    def splitmix64(self, x):
        return self.lib.oracle_splitmix64(x)

    def rng_key(self, seed, tag, a=0, b=0):
        return self.lib.oracle_rng_key(seed, tag, a, b)

    def rng_double(self, key, counter):
        return self.lib.oracle_rng_double(key, counter)

    def binomial(self, key, m, p):
        return self.lib.oracle_binomial(key, m, p)

    def random_dataset(self, n, d, seed, lo=0.0, hi=1.0):
        out = np.zeros(n * d)
        self.lib.oracle_random_dataset(C.c_uint32(n), C.c_uint32(d), C.c_uint64(seed),
                                       C.c_double(lo), C.c_double(hi),
                                       out.ctypes.data_as(C.c_void_p))
        return out.reshape(n, d)

    def kernel(self, family, sigma, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        return self.lib.oracle_kernel(family, sigma, x, y, x.size)

    def default_epsilon(self, n, log_base=0):
        return self.lib.oracle_default_epsilon(n, log_base)

    def rounds_for(self, n, C_=1.0, lam=1.0, rounds=0, log_base=0):
        out = C.c_uint32()
        rc = self.lib.oracle_rounds_for(C.c_uint32(n), C.c_double(C_), C.c_double(lam),
                                        C.c_uint32(rounds), C.c_int(log_base), C.byref(out))
        if rc:
            raise OracleError(rc)
        return out.value

    def kde_exact(self, pts, first, last, targets, sigma, family=0, floor=1e-300):
        pts = np.ascontiguousarray(pts, np.float64)
        n, d = pts.shape
        t = np.ascontiguousarray(targets, np.uint32)
        out = np.zeros(t.size)
        rc = self.lib.oracle_kde_exact(pts.reshape(-1), n, d, family, sigma, first, last, t,
                                       t.size, floor, out)
        if rc:
            raise OracleError(rc)
        return out

    def sample_counted(self, pts, queries, rounds, seed, sigma, family=0, record=False):
        pts = np.ascontiguousarray(pts, np.float64)
        n, d = pts.shape
        q = np.ascontiguousarray(queries, np.uint32)
        tri = C.c_void_p()
        cnt = C.c_size_t()

        class Diag(C.Structure):
            _fields_ = [("nlevels", C.c_uint32), ("epl", C.c_uint64 * 64),
                        ("tpl", C.c_uint64 * 64), ("degenerate", C.c_uint64)]

        diag = Diag()
        rf, rl, rq, rs = (C.c_void_p() for _ in range(4))
        rc_ = C.c_size_t()
        rec = [C.byref(x) for x in (rf, rl, rq, rs, rc_)] if record else [None] * 5
        rc = self.lib.oracle_sample_counted(
            pts.ctypes.data_as(C.c_void_p), C.c_uint32(n), C.c_uint32(d), C.c_int(family),
            C.c_double(sigma), q.ctypes.data_as(C.c_void_p), C.c_size_t(q.size),
            C.c_uint32(rounds), C.c_uint64(seed), C.byref(tri), C.byref(cnt), C.byref(diag), *rec)
        if rc:
            raise OracleError(rc)
        k = cnt.value
        out = dict(triples=_take(self.lib, tri, 3 * k, np.uint32).reshape(k, 3),
                   entries_per_level=list(diag.epl)[: diag.nlevels],
                   tickets_per_level=list(diag.tpl)[: diag.nlevels],
                   degenerate_draws=diag.degenerate)
        if record:
            r = rc_.value
            out["rec"] = dict(first=_take(self.lib, rf, r, np.uint32),
                              last=_take(self.lib, rl, r, np.uint32),
                              query=_take(self.lib, rq, r, np.uint32),
                              sum=_take(self.lib, rs, r, np.float64))
        return out

    def build_graph(self, pts, sigma, rounds, seed=1, family=0):
        pts = np.ascontiguousarray(pts, np.float64)
        n, d = pts.shape
        m = C.c_size_t()
        u, v, w, deg, est = (C.c_void_p() for _ in range(5))
        g = np.zeros(n)
        rep = (C.c_double * 8)()
        rc = self.lib.oracle_build_graph(
            pts.ctypes.data_as(C.c_void_p), C.c_uint32(n), C.c_uint32(d), C.c_int(family),
            C.c_double(sigma), C.c_uint32(rounds), C.c_uint64(seed), C.byref(m), C.byref(u),
            C.byref(v), C.byref(w), C.byref(deg), C.byref(est), g.ctypes.data_as(C.c_void_p), rep)
        if rc:
            raise OracleError(rc)
        M = m.value
        keys = ["n", "rounds", "sampled_pairs", "self_pairs_discarded",
                "underflow_edges_discarded", "edge_count", "degenerate_draws", "total_weight"]
        return dict(u=_take(self.lib, u, M, np.uint32), v=_take(self.lib, v, M, np.uint32),
                    w=_take(self.lib, w, M, np.float64),
                    degrees=_take(self.lib, deg, n, np.float64),
                    estimates=_take(self.lib, est, 8 * M, np.float64).reshape(M, 8),
                    g_full=g, report=dict(zip(keys, list(rep))))
