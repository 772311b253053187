"""Multi-GPU build: one process per GPU, queries sharded, points replicated.

A query's descent reads only the replicated points and its own keyed RNG
stream (proj/src/sampler.cpp:213-214), and every child sum is reduced over
node-aligned source chunks in a fixed order, so partitioning the queries
changes nothing observable: the sharded graph is bit-identical to the
1-GPU graph. There is no collective during the descent; the exchanges are
at the end, all over NCCL:

  1. all-gather of the degree KDE slices g_full (n fp64), needed because
     p_j uses the other endpoint's estimate (proj/src/sparsifier.cpp:110-111);
  2. all-to-all of the pair keys (u << 32 | v, u < v) to the rank owning
     row u (rows are sharded like the queries) — every rank then dedupes and
     weights only its own rows (fsgg_finish_graph);
  3. all-to-all of the rows' (v, w) to the rank owning v, which sums each
     vertex's degree in exactly the 1-GPU order (fsgg_rows_transposed,
     fsgg_rows_degrees);
  4. optionally the final all-gather of the edge lists and degrees (the
     north star's "final edge-list all-gather"), concatenated in rank order
     = the global (u, v) order.
The graph finish is thus split N ways instead of repeated on every rank.

With the symmetric root pass (low d) there is one exchange before the
descent: shard bounds sit on the root's block boundaries
(fsgg_shard_bounds), every block-pair tile is evaluated by exactly one rank,
and the other rank's side (one fp32 value per point of its block) is sent to it as a
record with one all-to-all (exchange_root) — the root's n^2 work is split
N ways instead of each rank also evaluating the tiles it shares with its
neighbours.
The exchange helpers are device-agnostic so the CPU suite exercises them
with ``gloo``.
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


def shard_bounds(n: int, world: int) -> list[int]:
    return [shard_range(n, r, world)[0] for r in range(world)] + [n]


def block_shard_bounds(ds: Dataset, world: int, kernel: Kernel | None = None) -> list[int]:
    """Query bounds on the symmetric root's block boundaries (plain
    shard_bounds when the root pass is not symmetric for this data); with
    ``kernel``, balanced by the library's per-block cost model."""
    b = (C.c_uint32 * (world + 1))()
    k = kernel._c() if kernel is not None else None
    N.check(N.lib().fsgg_shard_bounds(ds._h, C.byref(k) if k is not None else None, world, b))
    return [int(x) for x in b]


RECORD_WORDS = 324  # X, Y, first point of X, |X|, 320 values (include/fsgg.h)


def record_destinations(records: torch.Tensor, bounds: list[int]) -> torch.Tensor:
    """Rank owning each record's block (word 2 = the block's first point)."""
    first = records[:, 2].to(torch.int64)
    b = torch.tensor(bounds[1:-1], dtype=torch.int64, device=records.device)
    return torch.searchsorted(b, first, right=True)


def route_records(records: torch.Tensor, bounds: list[int], group=None) -> torch.Tensor:
    """All-to-all of exchange records (int32 [m, RECORD_WORDS]) to the ranks
    owning their blocks; returns the records this rank received."""
    world = dist.get_world_size(group)
    dest = record_destinations(records, bounds)
    order = torch.argsort(dest, stable=True)
    counts = torch.bincount(dest, minlength=world).tolist()
    flat = records.index_select(0, order).reshape(-1)
    recv = alltoall_varlen(flat, [c * RECORD_WORDS for c in counts], group)
    return recv.reshape(-1, RECORD_WORDS)


def prepare_root(ds: Dataset, kernel: Kernel, cfg: SparsifierConfig) -> torch.Tensor:
    """fsgg_shard_root_prepare: this shard's root tiles; returns the records
    owed to other ranks (a device copy, int32 [m, RECORD_WORDS])."""
    k = kernel._c()
    c = cfg._c()
    n = C.c_uint64(0)
    N.check(N.lib().fsgg_shard_root_prepare(ds._h, C.byref(k), C.byref(c), C.byref(n)))
    dev = torch.device("cuda", ds.device)
    m = int(n.value)
    out = torch.empty((m, RECORD_WORDS), dtype=torch.int32, device=dev)
    if m:
        N.check(N.lib().fsgg_shard_root_export(ds._h, C.c_void_p(out.data_ptr())))
    return out


def receive_root(ds: Dataset, records: torch.Tensor):
    torch.cuda.synchronize(ds.device)  # the all-to-all ran on torch's stream
    N.check(N.lib().fsgg_shard_root_receive(
        ds._h, C.c_void_p(records.data_ptr() if records.numel() else 0), records.shape[0]))


def exchange_root(ds: Dataset, kernel: Kernel, cfg: SparsifierConfig, bounds: list[int],
                  group=None) -> int:
    """Owner-mode symmetric root for this rank's shard (cfg.query_begin/end
    must be its entry of `bounds`): compute, exchange, store. Returns the
    bytes this rank sent."""
    recs = prepare_root(ds, kernel, cfg)
    # every rank joins the collective, also with nothing to send
    recv = route_records(recs, bounds, group)
    receive_root(ds, recv)
    return recs.numel() * 4


def gather_sizes(n: int, device, group=None) -> list[int]:
    world = dist.get_world_size(group)
    cnt = torch.tensor([n], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    return [int(c.item()) for c in counts]


def allgather_varlen(t: torch.Tensor, group=None, sizes: list[int] | None = None) -> torch.Tensor:
    """All-gather 1-D tensors of different lengths, concatenated in rank order.
    NCCL gathers the uneven pieces directly into one buffer; gloo (CPU
    tests) needs equal sizes, so pieces are padded there."""
    world = dist.get_world_size(group)
    if sizes is None:
        sizes = gather_sizes(t.numel(), t.device, group)
    out = torch.empty(sum(sizes), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather(list(torch.split(out, sizes)), t.contiguous(), group=group)
        return out
    cap = max(max(sizes), 1)
    padded = torch.zeros(cap, dtype=t.dtype, device=t.device)
    padded[: t.numel()] = t
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)])


def owner_splits(keys: torch.Tensor, bounds: list[int]) -> list[int]:
    """Per-destination counts of a sorted key array cut at ``bounds``."""
    b = torch.tensor(bounds[1:-1], dtype=keys.dtype, device=keys.device)
    cuts = torch.searchsorted(keys, b).tolist() if b.numel() else []
    edges = [0] + cuts + [keys.numel()]
    return [edges[i + 1] - edges[i] for i in range(len(edges) - 1)]


def alltoall_varlen(t: torch.Tensor, send_counts: list[int], group=None) -> torch.Tensor:
    """Send t[sum(send_counts[:r]) : ...] to rank r; received slices are
    concatenated in source-rank order."""
    world = dist.get_world_size(group)
    sc = torch.tensor(send_counts, dtype=torch.int64, device=t.device)
    rc = torch.empty(world, dtype=torch.int64, device=t.device)
    dist.all_to_all_single(rc, sc, group=group)
    recv = rc.tolist()
    out = torch.empty(sum(recv), dtype=t.dtype, device=t.device)
    dist.all_to_all_single(out, t.contiguous(), output_split_sizes=recv,
                           input_split_sizes=list(send_counts), group=group)
    return out


class DistributedResult:
    """Sharded build: this rank's rows [row_begin, row_end) of the graph
    (u, v, w sorted by (u, v)) and their degrees; with ``gathered`` the
    full graph (edge arrays, row_ptr, degrees) on every rank."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


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


def sample_shard_routed(ds: Dataset, kernel: Kernel, cfg: SparsifierConfig, bounds: list[int]):
    """fsgg_sample_shard_routed: the shard's descent and its pair keys grouped
    by the owner of row u (unsorted, no dedup on the sending side); returns
    (shard, report, pairs, per-destination counts, g_full slice)."""
    k = kernel._c()
    c = cfg._c()
    world = len(bounds) - 1
    b = (C.c_uint32 * (world + 1))(*bounds)
    counts = (C.c_uint64 * world)()
    sh = N.fsgg_shard()
    rep = N.fsgg_report()
    N.check(N.lib().fsgg_sample_shard_routed(ds._h, C.byref(k), C.byref(c), world, b, counts,
                                             C.byref(sh), C.byref(rep)))
    dev = torch.device("cuda", ds.device)
    pairs = torch.empty(int(sh.num_pairs), dtype=torch.int64, device=dev)
    g = torch.empty(int(sh.query_end - sh.query_begin), dtype=torch.float64, device=dev)
    N.check(N.lib().fsgg_shard_export(ds._h, C.c_void_p(pairs.data_ptr() if pairs.numel() else 0),
                                      C.c_void_p(g.data_ptr() if g.numel() else 0)))
    return sh, BuildReport._from_c(rep), pairs, [int(x) for x in counts], g


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


def finish_rows(ds: Dataset, kernel: Kernel, rounds: int, g_full: torch.Tensor,
                pairs: torch.Tensor, row_begin: int, row_end: int, bounds: list[int],
                group=None, counts: list[int] | None = None):
    """Phase 2 of the row-sharded finish on one rank: `pairs` are this
    shard's keys grouped by destination (`counts` per rank, from
    sample_shard_routed) or sorted (then split at the bounds); returns (rows
    graph tensors, degrees of the rank's rows, report)."""
    dev = torch.device("cuda", ds.device)
    splits = counts if counts is not None else owner_splits(pairs >> 32, bounds)
    routed = alltoall_varlen(pairs, splits, group)
    graph, frep = finish_graph(ds, kernel, rounds, g_full, routed)
    m = int(graph.num_edges)
    v = torch.empty(m, dtype=torch.int32, device=dev)
    w = torch.empty(m, dtype=torch.float64, device=dev)
    N.check(N.lib().fsgg_rows_transposed(ds._h, C.c_void_p(v.data_ptr() if m else 0),
                                         C.c_void_p(w.data_ptr() if m else 0)))
    splits = owner_splits(v.to(torch.int64), bounds)
    lower_v = alltoall_varlen(v, splits, group)
    lower_w = alltoall_varlen(w, splits, group)
    torch.cuda.synchronize(dev)
    deg = torch.empty(row_end - row_begin, dtype=torch.float64, device=dev)
    N.check(N.lib().fsgg_rows_degrees(
        ds._h, C.c_void_p(lower_v.data_ptr() if lower_v.numel() else 0),
        C.c_void_p(lower_w.data_ptr() if lower_w.numel() else 0), lower_v.numel(), row_begin,
        row_end, C.c_void_p(deg.data_ptr() if deg.numel() else 0)))
    rows = dict(u=torch.empty(m, dtype=torch.int32, device=dev),
                v=torch.empty(m, dtype=torch.int32, device=dev),
                w=torch.empty(m, dtype=torch.float64, device=dev))
    if m:  # device-to-device copy of the rank's rows out of the library
        N.check(N.lib().fsgg_device_graph_copy(
            ds._h, C.c_void_p(rows["u"].data_ptr()), C.c_void_p(rows["v"].data_ptr()),
            C.c_void_p(rows["w"].data_ptr()), None, None))
    return rows, deg, frep, routed.numel() * 8 + (lower_v.numel() * 12)


def build_similarity_graph_distributed(ds: Dataset, kernel: Kernel,
                                       config: SparsifierConfig | None = None,
                                       group=None, gather: bool = True) -> DistributedResult:
    """build_similarity_graph over all ranks of ``group`` (one GPU each)."""
    cfg = config or SparsifierConfig()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = ds.n
    bounds = block_shard_bounds(ds, world, kernel)
    qb, qe = bounds[rank], bounds[rank + 1]
    shard_cfg = replace(cfg, query_begin=qb, query_end=qe)
    root_bytes = exchange_root(ds, kernel, shard_cfg, bounds, group)
    sh, srep, pairs, counts, g = sample_shard_routed(ds, kernel, shard_cfg, bounds)
    g_full = allgather_varlen(g, group, [bounds[r + 1] - bounds[r] for r in range(world)])
    rows, deg, frep, moved = finish_rows(ds, kernel, int(sh.rounds), g_full, pairs, qb, qe,
                                         bounds, group, counts)
    frep.sampled_pairs = srep.sampled_pairs
    frep.self_pairs_discarded = srep.self_pairs_discarded
    frep.degenerate_draws = srep.degenerate_draws
    frep.kernel_evals = srep.kernel_evals
    frep.kde_tiled_evals = srep.kde_tiled_evals
    frep.kde_tiled_seconds = srep.kde_tiled_seconds
    frep.kde_tiled_launches = srep.kde_tiled_launches
    frep.sampling_seconds = srep.sampling_seconds
    frep.gpu_launches += srep.gpu_launches
    res = DistributedResult(row_begin=qb, row_end=qe, u=rows["u"], v=rows["v"], w=rows["w"],
                            degrees=deg, report=frep, shard_report=srep,
                            exchange_bytes=g_full.numel() * 8 + moved + root_bytes,
                            gathered=False)
    if gather:
        m_all = gather_sizes(rows["u"].numel(), rows["u"].device, group)
        res.u = allgather_varlen(rows["u"], group, m_all)
        res.v = allgather_varlen(rows["v"], group, m_all)
        res.w = allgather_varlen(rows["w"], group, m_all)
        row_sizes = [bounds[r + 1] - bounds[r] for r in range(world)]
        res.degrees = allgather_varlen(deg, group, row_sizes)
        # global upper CSR: each rank's row_ptr slice shifted by the edges of
        # the ranks before it (fsgg_rows_row_ptr), gathered in rank order
        rp = torch.empty(qe - qb, dtype=torch.int64, device=res.u.device)
        N.check(N.lib().fsgg_rows_row_ptr(ds._h, qb, qe, sum(m_all[:rank]),
                                          C.c_void_p(rp.data_ptr() if rp.numel() else 0)))
        total = torch.tensor([sum(m_all)], dtype=torch.int64, device=res.u.device)
        res.row_ptr = torch.cat([allgather_varlen(rp, group, row_sizes), total])
        res.gathered = True
        res.exchange_bytes += res.u.numel() * 16 + n * 16
    res.num_edges = int(res.v.numel())
    return res
