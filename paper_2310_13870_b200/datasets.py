"""Benchmark configurations (BASELINE.json ``configs``) and their inputs.

Points are generated on the host by libfsgg.so's generators
(``csrc/datasets.cpp``: make_moons/make_blobs restate
proj/src/datasets.cpp:20-124 bit-for-bit; C4/C5 are harness-defined, see
SURVEY.md §8d) and rounded to fp32, the precision the device path consumes.
Public benchmark data (BSDS images) is not available offline: C4/C5 are
seeded synthetic stand-ins with the configs' shapes and distributions.

``*_device`` / ``config_device`` run the same generators on the GPU
(``csrc/datasets_dev.cu``, correctly rounded log/sin/cos in double-double):
fp32 points identical to the host generators' (tests/test_gpu_generators.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


def make_moons(n: int, noise: float, seed: int):
    pts = np.zeros((n, 2), np.float64)
    lab = np.zeros(n, np.uint32)
    N.check(N.lib().fsgg_make_moons(n, noise, seed, pts.ctypes.data_as(C.c_void_p),
                                    lab.ctypes.data_as(C.c_void_p)))
    return pts, lab


def make_blobs(n: int, centers, stddev: float, seed: int):
    c = np.ascontiguousarray(centers, np.float64)
    k, d = c.shape
    pts = np.zeros((n, d), np.float64)
    lab = np.zeros(n, np.uint32)
    N.check(N.lib().fsgg_make_blobs(n, c.ctypes.data_as(C.c_void_p), k, d, stddev, seed,
                                    pts.ctypes.data_as(C.c_void_p),
                                    lab.ctypes.data_as(C.c_void_p)))
    return pts, lab


def make_image_features(height: int, width: int, regions: int, noise: float, seed: int):
    pts = np.zeros((height * width, 5), np.float64)
    lab = np.zeros(height * width, np.uint32)
    N.check(N.lib().fsgg_make_image_features(height, width, regions, noise, seed,
                                             pts.ctypes.data_as(C.c_void_p),
                                             lab.ctypes.data_as(C.c_void_p)))
    return pts, lab


def make_gmm(n: int, d: int, k: int, stddev: float, seed: int):
    pts = np.zeros((n, d), np.float64)
    lab = np.zeros(n, np.uint32)
    N.check(N.lib().fsgg_make_gmm(n, d, k, stddev, seed, pts.ctypes.data_as(C.c_void_p),
                                  lab.ctypes.data_as(C.c_void_p)))
    return pts, lab


# ---- the same generators on the device (csrc/datasets_dev.cu) -----------
def _device_outputs(n, d, device, fp64):
    import torch
    dev = torch.device("cuda", device)
    p32 = torch.empty((n, d), dtype=torch.float32, device=dev)
    p64 = torch.empty((n, d), dtype=torch.float64, device=dev) if fp64 else None
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    return (p32, p64, lab), (ptr(p64), ptr(p32), ptr(lab))


def make_moons_device(n: int, noise: float, seed: int, device: int = 0, fp64: bool = False):
    """make_moons generated on GPU ``device``: (fp32 points, fp64 points or
    None, labels) as torch tensors; fp32 identical to ``make_moons(...)``
    rounded to fp32 (include/fsgg.h)."""
    out, ptrs = _device_outputs(n, 2, device, fp64)
    N.check(N.lib().fsgg_make_moons_device(n, noise, seed, device, *ptrs))
    return out


def make_blobs_device(n: int, centers, stddev: float, seed: int, device: int = 0,
                      fp64: bool = False):
    c = np.ascontiguousarray(centers, np.float64)
    k, d = c.shape
    out, ptrs = _device_outputs(n, d, device, fp64)
    N.check(N.lib().fsgg_make_blobs_device(n, c.ctypes.data_as(C.c_void_p), k, d, stddev, seed,
                                           device, *ptrs))
    return out


def make_image_features_device(height: int, width: int, regions: int, noise: float, seed: int,
                               device: int = 0, fp64: bool = False):
    out, ptrs = _device_outputs(height * width, 5, device, fp64)
    N.check(N.lib().fsgg_make_image_features_device(height, width, regions, noise, seed, device,
                                                    *ptrs))
    return out


def make_gmm_device(n: int, d: int, k: int, stddev: float, seed: int, device: int = 0,
                    fp64: bool = False):
    out, ptrs = _device_outputs(n, d, device, fp64)
    N.check(N.lib().fsgg_make_gmm_device(n, d, k, stddev, seed, device, *ptrs))
    return out


def config_device(name: str, seed: int = 1, n: int | None = None, device: int = 0):
    """Points of ``config(name, seed, n)`` generated on the device (fp32 torch
    tensor, labels); sigma and rounds as ``config``. C5's bandwidth is the
    median pairwise distance of a 1,000-point subsample, computed on the host
    from those rows."""
    if name == "C1":
        p, _, lab = make_blobs_device(n or 2000, [[-2.0, 0.0], [2.0, 0.0]], 0.5, seed, device)
        return p, lab, 0.5, 32
    if name in ("C2", "C3"):
        nn = n or (100_000 if name == "C2" else 1_000_000)
        p, _, lab = make_moons_device(nn, 0.05, seed, device)
        return p, lab, (0.1 if name == "C2" else 0.05), 64
    if name == "C4":
        if n:
            h = max(2, int(round((n * 481 / 321) ** 0.5)))
            w = max(2, n // h)
        else:
            h, w = 481, 321
        p, _, lab = make_image_features_device(h, w, 8, 0.03, seed, device)
        return p, lab, 0.2, 32
    if name == "C5":
        nn = n or 70_000
        p, _, lab = make_gmm_device(nn, 784, 10, 0.1, seed, device)
        rng = np.random.default_rng(seed)
        idx = np.sort(rng.choice(nn, size=min(1000, nn), replace=False))
        sub = p[idx].cpu().numpy().astype(np.float64)
        return p, lab, median_pairwise_distance(sub, sub.shape[0], seed), 32
    raise ValueError(f"unknown config {name}")


def median_pairwise_distance(pts: np.ndarray, sample: int = 1000, seed: int = 1) -> float:
    """C5 bandwidth: median pairwise distance of a seeded subsample."""
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(pts.shape[0], size=min(sample, pts.shape[0]), replace=False))
    x = pts[idx].astype(np.float64)
    sq = (x * x).sum(1)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * x @ x.T, 0.0)
    iu = np.triu_indices(len(idx), 1)
    return float(np.median(np.sqrt(d2[iu])))


@dataclass
class Workload:
    name: str
    points: np.ndarray  # fp32 (n, d)
    labels: np.ndarray
    sigma: float
    rounds: int

    @property
    def n(self):
        return self.points.shape[0]

    @property
    def d(self):
        return self.points.shape[1]


def config(name: str, seed: int = 1, n: int | None = None) -> Workload:
    """C1..C5 of BASELINE.json (``n`` overrides the size for parity runs)."""
    if name == "C1":
        nn = n or 2000
        p, lab = make_blobs(nn, [[-2.0, 0.0], [2.0, 0.0]], 0.5, seed)
        return Workload("C1-blobs", p.astype(np.float32), lab, 0.5, 32)
    if name == "C2":
        nn = n or 100_000
        p, lab = make_moons(nn, 0.05, seed)
        return Workload("C2-moons-100k", p.astype(np.float32), lab, 0.1, 64)
    if name == "C3":
        nn = n or 1_000_000
        p, lab = make_moons(nn, 0.05, seed)
        return Workload("C3-moons-1M", p.astype(np.float32), lab, 0.05, 64)
    if name == "C4":
        if n:
            h = max(2, int(round((n * 481 / 321) ** 0.5)))
            w = max(2, n // h)
        else:
            h, w = 481, 321
        p, lab = make_image_features(h, w, 8, 0.03, seed)
        return Workload("C4-image-154k", p.astype(np.float32), lab, 0.2, 32)
    if name == "C5":
        nn = n or 70_000
        p, lab = make_gmm(nn, 784, 10, 0.1, seed)
        p32 = p.astype(np.float32)
        sigma = median_pairwise_distance(p32.astype(np.float64), 1000, seed)
        return Workload("C5-gmm-784d", p32, lab, sigma, 32)
    raise ValueError(f"unknown config {name}")
