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
