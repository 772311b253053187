"""World-size-2 test of the multi-GPU exchange logic on CPU (gloo).

The product path (paper_2310_13870_b200.parallel) shards queries, then
all-gathers g_full slices and the shards' pair keys with
``allgather_varlen``. Here each rank produces its shard with the C oracle
instead of the GPU and runs the very same exchange helpers over gloo; the
merged result must equal the single-process oracle graph.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Oracle
    from paper_2310_13870_b200.parallel import allgather_varlen, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    pts = orc.random_dataset(301, 2, 7)
    n, sigma, L, seed = 301, 0.2, 6, 5
    qb, qe = shard_range(n, rank, world)
    tri = orc.sample_counted(pts, np.arange(qb, qe), L, seed, sigma)["triples"]
    q, s = tri[:, 0].astype(np.int64), tri[:, 1].astype(np.int64)
    keep = q != s
    lo, hi = np.minimum(q, s)[keep], np.maximum(q, s)[keep]
    keys = np.unique((lo << 32) | hi)
    g = orc.kde_exact(pts, 0, n, np.arange(qb, qe), sigma)
    all_keys = allgather_varlen(torch.from_numpy(keys.astype(np.int64)))
    g_full = allgather_varlen(torch.from_numpy(g))
    merged = np.unique(all_keys.numpy())
    if rank == 0:
        np.save(os.path.join(out_dir, "merged.npy"), merged)
        np.save(os.path.join(out_dir, "gfull.npy"), g_full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_exchange_matches_single_process(tmp_path):
    from oracle.pyoracle import Oracle
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    merged = np.load(tmp_path / "merged.npy")
    g_full = np.load(tmp_path / "gfull.npy")
    orc = Oracle()
    pts = orc.random_dataset(301, 2, 7)
    full = orc.build_graph(pts, 0.2, 6, seed=5)
    expect = (full["u"].astype(np.int64) << 32) | full["v"].astype(np.int64)
    assert np.array_equal(merged, expect)
    assert np.array_equal(g_full, full["g_full"])


def test_shard_ranges_partition():
    from paper_2310_13870_b200.parallel import shard_range
    for n in (1, 2, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _route_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Oracle
    from paper_2310_13870_b200.parallel import (alltoall_varlen, owner_splits, shard_bounds,
                                                shard_range)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    n, sigma, L, seed = 301, 0.2, 6, 5
    pts = orc.random_dataset(n, 2, 7)
    qb, qe = shard_range(n, rank, world)
    tri = orc.sample_counted(pts, np.arange(qb, qe), L, seed, sigma)["triples"]
    q, s = tri[:, 0].astype(np.int64), tri[:, 1].astype(np.int64)
    keep = q != s
    keys = np.unique((np.minimum(q, s)[keep] << 32) | np.maximum(q, s)[keep])
    bounds = shard_bounds(n, world)
    t = torch.from_numpy(keys)
    # step 2 of parallel.py: pair keys to the owner of row u
    routed = alltoall_varlen(t, owner_splits(t >> 32, bounds))
    mine = np.unique(routed.numpy())
    assert np.all((mine >> 32) >= qb) and np.all((mine >> 32) < qe)
    np.save(os.path.join(out_dir, f"rows{rank}.npy"), mine)
    # step 3: (v, w) of the rows to the owner of v, concatenated in rank order
    v = np.sort((mine & 0xffffffff).astype(np.int64), kind="stable")
    tv = torch.from_numpy(v)
    lower = alltoall_varlen(tv, owner_splits(tv, bounds)).numpy()
    assert np.all(lower >= qb) and np.all(lower < qe)
    np.save(os.path.join(out_dir, f"lower{rank}.npy"), lower)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_routing_matches_single_process(tmp_path, world):
    """parallel.py's all-to-all routing over gloo: every rank ends with
    exactly the edges of its rows, and with the degree contributions
    (edges (u, x), u < x) of its vertices."""
    from oracle.pyoracle import Oracle
    from paper_2310_13870_b200.parallel import shard_range
    mp.spawn(_route_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    orc = Oracle()
    full = orc.build_graph(orc.random_dataset(301, 2, 7), 0.2, 6, seed=5)
    u, v = full["u"].astype(np.int64), full["v"].astype(np.int64)
    got = np.concatenate([np.load(tmp_path / f"rows{r}.npy") for r in range(world)])
    assert np.array_equal(got, (u << 32) | v)
    for r in range(world):
        qb, qe = shard_range(301, r, world)
        lower = np.load(tmp_path / f"lower{r}.npy")
        assert np.array_equal(np.sort(lower), np.sort(v[(v >= qb) & (v < qe)]))


def _record_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2310_13870_b200.parallel import RECORD_WORDS, route_records

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds = [0, 1000, 2500, 4000][: world] + [4000]
    rng = np.random.default_rng(rank)
    m = 50 + 10 * rank
    recs = np.zeros((m, RECORD_WORDS), dtype=np.int32)
    recs[:, 0] = rng.integers(0, 64, m)             # block X
    recs[:, 1] = rank                                # sender tag (stands for Y)
    recs[:, 2] = rng.integers(0, bounds[-1], m)      # first point of X
    recs[:, 3] = 7
    recs[:, 4:] = rng.integers(0, 1 << 30, (m, RECORD_WORDS - 4))
    np.save(os.path.join(out_dir, f"sent{rank}.npy"), recs)
    got = route_records(torch.from_numpy(recs), bounds).numpy()
    np.save(os.path.join(out_dir, f"got{rank}.npy"), got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_root_record_routing(tmp_path, world):
    """Owner-mode symmetric root (parallel.route_records): every record
    reaches the rank whose query range holds its block's first point, intact,
    with sender order preserved."""
    mp.spawn(_record_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
             join=True)
    bounds = [0, 1000, 2500, 4000][: world] + [4000]
    sent = [np.load(tmp_path / f"sent{r}.npy") for r in range(world)]
    for d in range(world):
        got = np.load(tmp_path / f"got{d}.npy")
        expect = np.concatenate([s[(s[:, 2] >= bounds[d]) & (s[:, 2] < bounds[d + 1])]
                                 for s in sent])
        assert np.array_equal(got, expect)
