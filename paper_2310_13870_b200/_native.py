"""ctypes binding of the C ABI in include/fsgg.h (libfsgg.so, sm_100a).

The shared library is built in-tree by ``__graft_entry__.build()``
(``paper_2310_13870_b200/csrc/Makefile``). There is no CPU fallback: if the
library is missing every call raises :class:`DeviceError`, and without a
usable B200 every compute call returns FSGG_ERR_DEVICE.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# FSGG_LIB_PATH: load an alternative in-tree build (development A/B runs)
LIB_PATH = os.environ.get("FSGG_LIB_PATH") or os.path.join(HERE, "_lib", "libfsgg.so")
INCLUDE_DIR = os.path.join(os.path.dirname(HERE), "include")

FSGG_OK = 0
FSGG_ERR_CONFIG = 2
FSGG_ERR_IO = 3
FSGG_ERR_NUMERIC = 4
FSGG_ERR_DEVICE = 5


class fsgg_kernel(C.Structure):
    _fields_ = [("family", C.c_int), ("sigma", C.c_double)]


class fsgg_config(C.Structure):
    _fields_ = [("C", C.c_double), ("lambda_k1_estimate", C.c_double),
                ("rounds", C.c_uint32), ("epsilon", C.c_double), ("log_base", C.c_int),
                ("seed", C.c_uint64), ("rng_mode", C.c_int),
                ("query_begin", C.c_uint32), ("query_end", C.c_uint32),
                ("dense_kde", C.c_int), ("kde_backend", C.c_int)]


class fsgg_report(C.Structure):
    _fields_ = [("n", C.c_uint32), ("rounds", C.c_uint32), ("epsilon", C.c_double),
                ("backend", C.c_char * 32), ("sampled_pairs", C.c_uint64),
                ("self_pairs_discarded", C.c_uint64),
                ("underflow_edges_discarded", C.c_uint64), ("edge_count", C.c_uint64),
                ("degenerate_draws", C.c_uint64), ("estimator_build_seconds", C.c_double),
                ("sampling_seconds", C.c_double), ("degree_kde_seconds", C.c_double),
                ("weighting_seconds", C.c_double), ("total_seconds", C.c_double),
                ("estimator_bytes", C.c_uint64), ("graph_bytes", C.c_uint64),
                ("kernel_evals", C.c_uint64), ("kde_tiled_evals", C.c_uint64),
                ("kde_tiled_seconds", C.c_double), ("kde_tiled_launches", C.c_uint32),
                ("levels", C.c_uint32), ("peak_entries", C.c_uint64),
                ("gpu_launches", C.c_uint32), ("kernel_evals_performed", C.c_uint64),
                ("kde_tiled_performed_evals", C.c_uint64),
                ("tie_verified_entries", C.c_uint64),
                ("kde_root_performed_evals", C.c_uint64), ("kde_root_seconds", C.c_double)]


class fsgg_edge_estimate(C.Structure):
    _fields_ = [("i", C.c_uint32), ("j", C.c_uint32), ("k_ij", C.c_double),
                ("g_i", C.c_double), ("g_j", C.c_double), ("p_hat_i_j", C.c_double),
                ("p_hat_j_i", C.c_double), ("p_hat", C.c_double)]


class fsgg_graph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("num_edges", C.c_uint64),
                ("u", C.POINTER(C.c_uint32)), ("v", C.POINTER(C.c_uint32)),
                ("w", C.POINTER(C.c_double)), ("row_ptr", C.POINTER(C.c_uint64)),
                ("degrees", C.POINTER(C.c_double)), ("total_weight", C.c_double)]


class fsgg_eigen_options(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_matvecs", C.c_uint64), ("max_basis", C.c_uint32),
                ("seed", C.c_uint64)]


class fsgg_kmeans_options(C.Structure):
    _fields_ = [("restarts", C.c_uint32), ("max_iters", C.c_uint32), ("rel_tol", C.c_double),
                ("seed", C.c_uint64)]


class fsgg_spectral_options(C.Structure):
    _fields_ = [("eigen", fsgg_eigen_options), ("kmeans", fsgg_kmeans_options)]


class fsgg_spectral_report(C.Structure):
    _fields_ = [("matvecs", C.c_uint64), ("components", C.c_uint32),
                ("kmeans_iterations", C.c_uint32), ("kmeans_cost", C.c_double),
                ("eigen_seconds", C.c_double), ("kmeans_seconds", C.c_double),
                ("gpu_launches", C.c_uint64)]


class fsgg_device_graph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("num_edges", C.c_uint64), ("u", C.c_void_p),
                ("v", C.c_void_p), ("w", C.c_void_p), ("row_ptr", C.c_void_p),
                ("degrees", C.c_void_p), ("total_weight", C.c_double)]


class fsgg_sample_diag(C.Structure):
    _fields_ = [("nlevels", C.c_uint32), ("entries_per_level", C.c_uint64 * 64),
                ("tickets_per_level", C.c_uint64 * 64), ("degenerate_draws", C.c_uint64)]


class fsgg_entry_record(C.Structure):
    _fields_ = [("level", C.c_uint32), ("query", C.c_uint32), ("first", C.c_uint32),
                ("last", C.c_uint32), ("left", C.c_double), ("right", C.c_double)]


class fsgg_sample_options(C.Structure):
    _fields_ = [("rng_mode", C.c_int), ("dense_kde", C.c_int), ("record_sums", C.c_int),
                ("walks", C.c_int), ("kde_backend", C.c_int), ("epsilon", C.c_double)]


class fsgg_sample_report(C.Structure):
    _fields_ = [("diag", fsgg_sample_diag), ("kernel_evals", C.c_uint64),
                ("kernel_evals_performed", C.c_uint64), ("root_evals_performed", C.c_uint64),
                ("tie_verified", C.c_uint64), ("records", C.c_void_p),
                ("num_records", C.c_size_t)]


class fsgg_shard(C.Structure):
    _fields_ = [("query_begin", C.c_uint32), ("query_end", C.c_uint32),
                ("rounds", C.c_uint32), ("num_pairs", C.c_uint64), ("pairs", C.c_void_p),
                ("g_full", C.c_void_p), ("sampled_pairs", C.c_uint64),
                ("self_pairs", C.c_uint64), ("degenerate_draws", C.c_uint64)]


_P = C.c_void_p
_SIGS = {
    "fsgg_version": (C.c_char_p, []),
    "fsgg_last_error": (C.c_char_p, []),
    "fsgg_device_available": (C.c_int, []),
    "fsgg_config_init": (None, [C.POINTER(fsgg_config)]),
    "fsgg_rounds_for": (C.c_int, [C.POINTER(fsgg_config), C.c_uint32, C.POINTER(C.c_uint32)]),
    "fsgg_default_epsilon": (C.c_double, [C.c_uint32, C.c_int]),
    "fsgg_dataset_create": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                      C.POINTER(_P)]),
    "fsgg_dataset_create_f64": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_int,
                                          C.POINTER(_P)]),
    "fsgg_dataset_upload": (C.c_int, [_P, _P]),
    "fsgg_dataset_destroy": (None, [_P]),
    "fsgg_dataset_size": (C.c_uint32, [_P]),
    "fsgg_dataset_dim": (C.c_uint32, [_P]),
    "fsgg_dataset_device_points": (_P, [_P]),
    "fsgg_dataset_stream": (_P, [_P]),
    "fsgg_shard_export": (C.c_int, [_P, _P, _P]),
    "fsgg_build_similarity_graph": (C.c_int, [_P, C.POINTER(fsgg_kernel),
                                              C.POINTER(fsgg_config), C.POINTER(fsgg_graph),
                                              C.POINTER(fsgg_report),
                                              C.POINTER(C.POINTER(fsgg_edge_estimate))]),
    "fsgg_build_similarity_graph_device": (C.c_int, [_P, C.POINTER(fsgg_kernel),
                                                     C.POINTER(fsgg_config),
                                                     C.POINTER(fsgg_device_graph),
                                                     C.POINTER(fsgg_report)]),
    "fsgg_build_similarity_graph_into": (C.c_int, [_P, C.POINTER(fsgg_kernel),
                                                   C.POINTER(fsgg_config), C.c_uint64, _P, _P,
                                                   _P, _P, C.POINTER(C.c_uint64),
                                                   C.POINTER(C.c_double),
                                                   C.POINTER(fsgg_report)]),
    "fsgg_build_similarity_graph_host": (C.c_int, [_P, C.c_uint32, C.c_uint32,
                                                   C.POINTER(fsgg_kernel),
                                                   C.POINTER(fsgg_config), C.c_int,
                                                   C.POINTER(fsgg_graph),
                                                   C.POINTER(fsgg_report)]),
    "fsgg_graph_free": (None, [C.POINTER(fsgg_graph)]),
    "fsgg_device_graph_to_host": (C.c_int, [_P, C.POINTER(fsgg_graph)]),
    "fsgg_device_graph_copy": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "fsgg_free": (None, [_P]),
    "fsgg_spectral_options_init": (None, [C.POINTER(fsgg_spectral_options)]),
    "fsgg_smallest_eigenpairs": (C.c_int, [_P, C.c_uint32, C.POINTER(fsgg_eigen_options), _P, _P,
                                           _P, C.POINTER(C.c_uint64)]),
    "fsgg_spectral_cluster": (C.c_int, [_P, C.c_uint32, C.c_uint64,
                                        C.POINTER(fsgg_spectral_options), _P,
                                        C.POINTER(fsgg_spectral_report)]),
    "fsgg_spectral_cluster_graph": (C.c_int, [C.POINTER(fsgg_graph), C.c_int, C.c_uint32,
                                              C.c_uint64, C.POINTER(fsgg_spectral_options), _P,
                                              C.POINTER(fsgg_spectral_report)]),
    "fsgg_smallest_eigenpairs_graph": (C.c_int, [C.POINTER(fsgg_graph), C.c_int, C.c_uint32,
                                                 C.POINTER(fsgg_eigen_options), _P, _P, _P,
                                                 C.POINTER(C.c_uint64)]),
    "fsgg_kmeans": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32,
                              C.POINTER(fsgg_kmeans_options), C.c_int, _P,
                              C.POINTER(C.c_double), C.POINTER(C.c_uint32)]),
    "fsgg_rows_transposed": (C.c_int, [_P, _P, _P]),
    "fsgg_rows_degrees": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32, _P]),
    "fsgg_graph_save_text": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint64, _P, _P, _P,
                                       C.c_uint32]),
    "fsgg_graph_load_text": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(fsgg_graph)]),
    "fsgg_graph_save_csr": (C.c_int, [C.c_char_p, C.POINTER(fsgg_graph)]),
    "fsgg_graph_load_csr": (C.c_int, [C.c_char_p, C.POINTER(fsgg_graph)]),
    "fsgg_csv_load": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(_P), C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32), C.POINTER(_P)]),
    "fsgg_csv_save": (C.c_int, [C.c_char_p, _P, C.c_uint32, C.c_uint32, _P, C.c_uint32]),
    "fsgg_sample_neighbors_counted": (C.c_int, [_P, C.POINTER(fsgg_kernel), _P, C.c_size_t,
                                                C.c_uint32, C.c_uint64, C.c_int, C.c_int,
                                                C.POINTER(_P), C.POINTER(C.c_size_t),
                                                C.POINTER(fsgg_sample_diag)]),
    "fsgg_sample_options_init": (None, [C.POINTER(fsgg_sample_options)]),
    "fsgg_sample_neighbors_counted_ex": (C.c_int, [_P, C.POINTER(fsgg_kernel), _P, C.c_size_t,
                                                   C.c_uint32, C.c_uint64,
                                                   C.POINTER(fsgg_sample_options),
                                                   C.POINTER(_P), C.POINTER(C.c_size_t),
                                                   C.POINTER(fsgg_sample_report)]),
    "fsgg_kde_eval": (C.c_int, [_P, C.POINTER(fsgg_kernel), C.c_uint32, C.c_uint32, _P,
                                C.c_size_t, _P]),
    "fsgg_make_moons": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, _P, _P]),
    "fsgg_make_blobs": (C.c_int, [C.c_uint32, _P, C.c_uint32, C.c_uint32, C.c_double,
                                  C.c_uint64, _P, _P]),
    "fsgg_make_image_features": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                           C.c_uint64, _P, _P]),
    "fsgg_make_gmm": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                _P, _P]),
    "fsgg_make_moons_device": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.c_int, _P, _P,
                                         _P]),
    "fsgg_make_blobs_device": (C.c_int, [C.c_uint32, _P, C.c_uint32, C.c_uint32, C.c_double,
                                         C.c_uint64, C.c_int, _P, _P, _P]),
    "fsgg_make_image_features_device": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32,
                                                  C.c_double, C.c_uint64, C.c_int, _P, _P, _P]),
    "fsgg_make_gmm_device": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                       C.c_uint64, C.c_int, _P, _P, _P]),
    "fsgg_sample_shard_routed": (C.c_int, [_P, C.POINTER(fsgg_kernel), C.POINTER(fsgg_config),
                                           C.c_uint32, C.POINTER(C.c_uint32),
                                           C.POINTER(C.c_uint64), C.POINTER(fsgg_shard),
                                           C.POINTER(fsgg_report)]),
    "fsgg_rows_row_ptr": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint64, _P]),
    "fsgg_sample_shard": (C.c_int, [_P, C.POINTER(fsgg_kernel), C.POINTER(fsgg_config),
                                    C.POINTER(fsgg_shard), C.POINTER(fsgg_report)]),
    "fsgg_probe_ex2_throughput": (C.c_int, [C.c_int, C.POINTER(C.c_double),
                                            C.POINTER(C.c_double)]),
    "fsgg_shard_bounds": (C.c_int, [_P, C.POINTER(fsgg_kernel), C.c_uint32,
                                    C.POINTER(C.c_uint32)]),
    "fsgg_shard_root_prepare": (C.c_int, [_P, C.POINTER(fsgg_kernel), C.POINTER(fsgg_config),
                                          C.POINTER(C.c_uint64)]),
    "fsgg_shard_root_export": (C.c_int, [_P, _P]),
    "fsgg_shard_root_receive": (C.c_int, [_P, _P, C.c_uint64]),
    "fsgg_finish_graph": (C.c_int, [_P, C.POINTER(fsgg_kernel), C.c_uint32, _P, _P,
                                    C.c_uint64, C.POINTER(fsgg_device_graph),
                                    C.POINTER(fsgg_report)]),
}


def header_functions(include_dir: str = INCLUDE_DIR) -> list[str]:
    """Every function name declared in include/*.h."""
    names = set()
    for fn in sorted(os.listdir(include_dir)):
        if fn.endswith(".h"):
            text = open(os.path.join(include_dir, fn)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            names |= set(re.findall(r"\b(fsgg_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


_lib = None


def lib():
    """Load libfsgg.so once; raise loudly if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from .errors import DeviceError
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != FSGG_OK:
        from .errors import error_for
        raise error_for(rc, lib().fsgg_last_error().decode(errors="replace"))
