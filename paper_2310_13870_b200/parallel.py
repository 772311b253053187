"""Multi-GPU build: one process per GPU, queries sharded, points replicated.

A query's descent reads only the replicated points and its own keyed RNG
stream (proj/src/sampler.cpp:213-214), and every child sum is reduced over
node-aligned source chunks in a fixed order, so partitioning the queries
changes nothing observable: the sharded graph is bit-identical to the
1-GPU graph. The only data exchange is at the end (north star: "NCCL over
NVLink is used only for the final edge-list all-gather"):

  1. all-gather of the degree KDE slices g_full (n fp64), needed because
     p_j uses the other endpoint's estimate (proj/src/sparsifier.cpp:110-111);
  2. all-gather of the shards' sorted unique pair keys (variable length:
     counts all-gather + padded all-gather);
then every rank runs the same dedupe/weight/CSR/degree kernels
(fsgg_finish_graph) on the concatenation. The exchange helpers below are
device-agnostic so the CPU suite exercises them with ``gloo``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import replace

import torch
import torch.distributed as dist

from . import _native as N
from .api import BuildReport, Dataset, Kernel, SparsifierConfig


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous query block of ``rank`` (index order = spatial locality)."""
    return n * rank // world, n * (rank + 1) // world


def allgather_varlen(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather 1-D tensors of different lengths, concatenated in rank order."""
    world = dist.get_world_size(group)
    cnt = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    sizes = [int(c.item()) for c in counts]
    cap = max(max(sizes), 1)
    padded = torch.zeros(cap, dtype=t.dtype, device=t.device)
    padded[: t.numel()] = t
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)])


class DistributedResult:
    """Device graph of the sharded build (valid until the next build on ds)."""

    def __init__(self, graph, report: BuildReport, shard_report: BuildReport,
                 exchange_bytes: int):
        self.graph = graph
        self.report = report
        self.shard_report = shard_report
        self.exchange_bytes = exchange_bytes


def sample_shard(ds: Dataset, kernel: Kernel, cfg: SparsifierConfig):
    k = kernel._c()
    c = cfg._c()
    sh = N.fsgg_shard()
    rep = N.fsgg_report()
    N.check(N.lib().fsgg_sample_shard(ds._h, C.byref(k), C.byref(c), C.byref(sh),
                                      C.byref(rep)))
    dev = torch.device("cuda", ds.device)
    pairs = torch.empty(int(sh.num_pairs), dtype=torch.int64, device=dev)
    g = torch.empty(int(sh.query_end - sh.query_begin), dtype=torch.float64, device=dev)
    N.check(N.lib().fsgg_shard_export(ds._h, C.c_void_p(pairs.data_ptr() if pairs.numel() else 0),
                                      C.c_void_p(g.data_ptr() if g.numel() else 0)))
    return sh, BuildReport._from_c(rep), pairs, g


def finish_graph(ds: Dataset, kernel: Kernel, rounds: int, g_full: torch.Tensor,
                 pairs: torch.Tensor):
    k = kernel._c()
    out = N.fsgg_device_graph()
    rep = N.fsgg_report()
    torch.cuda.synchronize(ds.device)  # collectives ran on torch's stream
    N.check(N.lib().fsgg_finish_graph(ds._h, C.byref(k), rounds, C.c_void_p(g_full.data_ptr()),
                                      C.c_void_p(pairs.data_ptr() if pairs.numel() else 0),
                                      pairs.numel(), C.byref(out), C.byref(rep)))
    return out, BuildReport._from_c(rep)


def build_similarity_graph_distributed(ds: Dataset, kernel: Kernel,
                                       config: SparsifierConfig | None = None,
                                       group=None) -> DistributedResult:
    """build_similarity_graph over all ranks of ``group`` (one GPU each)."""
    cfg = config or SparsifierConfig()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    qb, qe = shard_range(ds.n, rank, world)
    sh, srep, pairs, g = sample_shard(ds, kernel, replace(cfg, query_begin=qb, query_end=qe))
    g_full = allgather_varlen(g, group)
    all_pairs = allgather_varlen(pairs, group)
    graph, frep = finish_graph(ds, kernel, int(sh.rounds), g_full, all_pairs)
    frep.sampled_pairs = srep.sampled_pairs
    frep.self_pairs_discarded = srep.self_pairs_discarded
    frep.degenerate_draws = srep.degenerate_draws
    frep.kernel_evals = srep.kernel_evals
    frep.kde_tiled_evals = srep.kde_tiled_evals
    frep.kde_tiled_seconds = srep.kde_tiled_seconds
    frep.kde_tiled_launches = srep.kde_tiled_launches
    frep.sampling_seconds = srep.sampling_seconds
    frep.gpu_launches += srep.gpu_launches
    exchange = (g_full.numel() * 8 + all_pairs.numel() * 8)
    return DistributedResult(graph, frep, srep, exchange)
