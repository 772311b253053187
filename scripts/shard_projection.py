"""Per-rank cost of the multi-GPU build, measured on ONE GPU.

The descent has no collective (parallel.py), so what rank r of N does is a
function of its query range alone: this script runs each rank's shard
descent (owner-mode root: fsgg_shard_root_prepare + the records the other
ranks owe it + fsgg_sample_shard_routed) and its row-sharded finish (fsgg_finish_graph on
the keys routed to it + fsgg_rows_transposed + fsgg_rows_degrees) one after
another on one GPU, times each with a device sync on both sides (best of
`--reps`), and reports max over ranks per phase. The NCCL exchanges are not
run here (one GPU); their bytes are counted and reported separately.

    python scripts/shard_projection.py [--n 1000000] [--worlds 1,2,4,8]

This is a PROJECTION (the ranks never run concurrently here); bench.py under
torchrun is the measurement.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_13870_b200 as F  # noqa: E402
from paper_2310_13870_b200 import _native as N  # noqa: E402
from paper_2310_13870_b200 import datasets, parallel  # noqa: E402


def timed(fn, reps):
    best, out = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--sigma", type=float, default=0.05)
    ap.add_argument("--rounds", type=int, default=64)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--no-owner", action="store_true",
                    help="plain query shards (each rank evaluates every root tile it touches)")
    a = ap.parse_args()
    p, _ = datasets.make_moons(a.n, 0.05, 1)
    p = p.astype(np.float32)
    ds = F.Dataset(p)
    k = F.Kernel(F.KernelFamily.gaussian, a.sigma)
    L = a.rounds
    # warm the arena with the full problem
    F.build_similarity_graph_device(ds, k, F.SparsifierConfig(rounds=L, seed=1))
    torch.cuda.synchronize()
    full_t, _ = timed(lambda: F.build_similarity_graph_device(
        ds, k, F.SparsifierConfig(rounds=L, seed=1)), a.reps)
    result = {"n": a.n, "sigma": a.sigma, "L": L, "one_gpu_build_s": full_t, "worlds": {}}
    print(f"1-GPU build {full_t * 1e3:.1f} ms", flush=True)
    for world in [int(x) for x in a.worlds.split(",")]:
        # owner mode (default): block-aligned bounds, each root tile on one
        # rank, one handle per rank (their root values must coexist for the
        # emulated record exchange)
        if a.no_owner:
            bounds = parallel.shard_bounds(a.n, world)
            handles = [ds] * world
        else:
            bounds = parallel.block_shard_bounds(ds, world, k)
            handles = [ds] + [F.Dataset(p) for _ in range(world - 1)]
        cfgs = [F.SparsifierConfig(rounds=L, seed=1, query_begin=bounds[r],
                                   query_end=bounds[r + 1]) for r in range(world)]
        sample_s, root_s, pairs, gs, prep_s, recv_s, rec_bytes = [], [], [], [], [], [], []
        key_counts = []
        for rep_i in range(a.reps):
            recs = []
            for r in range(world):
                if a.no_owner:
                    prep_s.append(0.0)
                    recs.append(None)
                    continue
                t, x = timed(lambda: parallel.prepare_root(handles[r], k, cfgs[r]), 1)
                prep_s.append(t)
                recs.append(x)
            for d in range(world):
                if a.no_owner:
                    recv_s.append(0.0)
                    rec_bytes.append(0)
                    continue
                inbox = torch.cat([x[parallel.record_destinations(x, bounds) == d] for x in recs])
                rec_bytes.append(int(inbox.numel()) * 4)
                t, _ = timed(lambda: parallel.receive_root(handles[d], inbox), 1)
                recv_s.append(t)
            for r in range(world):
                t, (sh, rep, pr, cnt, g) = timed(lambda: parallel.sample_shard_routed(
                    handles[r], k, cfgs[r], bounds), 1)
                if rep_i == 0:
                    sample_s.append(t)
                    root_s.append(rep.kde_root_seconds)
                    pairs.append(pr)
                    key_counts.append(cnt)
                    gs.append(g)
                else:
                    sample_s[r] = min(sample_s[r], t)
        prep_s = [min(prep_s[r::world]) for r in range(world)]
        recv_s = [min(recv_s[r::world]) for r in range(world)]
        sample_s = [sample_s[r] + prep_s[r] + recv_s[r] for r in range(world)]
        g_full = torch.cat(gs)
        routed = [[] for _ in range(world)]
        for src, t in enumerate(pairs):
            for d, piece in enumerate(torch.split(t, key_counts[src])):
                routed[d].append(piece)
        routed = [torch.cat(x) for x in routed]
        finish_s, lower_bytes, vs, ws = [], [], [], []
        for d in range(world):
            def fin():
                graph, _ = parallel.finish_graph(ds, k, L, g_full, routed[d])
                m = int(graph.num_edges)
                v = torch.empty(m, dtype=torch.int32, device="cuda")
                w = torch.empty(m, dtype=torch.float64, device="cuda")
                N.check(N.lib().fsgg_rows_transposed(ds._h, C.c_void_p(v.data_ptr()),
                                                     C.c_void_p(w.data_ptr())))
                return v, w
            t, (v, w) = timed(fin, a.reps)
            vs.append(v)
            ws.append(w)
            # degrees: received lower contributions (emulated routing) + own rows
            sp = parallel.owner_splits(v.to(torch.int64), bounds)
            lower_bytes.append(sum(sp[i] for i in range(world) if i != d) * 12)
            finish_s.append(t)
        deg_s = []
        for d in range(world):
            lv = torch.cat([torch.split(vs[s], parallel.owner_splits(vs[s].to(torch.int64),
                                                                     bounds))[d]
                            for s in range(world)])
            lw = torch.cat([torch.split(ws[s], parallel.owner_splits(vs[s].to(torch.int64),
                                                                     bounds))[d]
                            for s in range(world)])
            deg = torch.empty(bounds[d + 1] - bounds[d], dtype=torch.float64, device="cuda")
            t, _ = timed(lambda: N.check(N.lib().fsgg_rows_degrees(
                ds._h, C.c_void_p(lv.data_ptr() if lv.numel() else 0),
                C.c_void_p(lw.data_ptr() if lw.numel() else 0), lv.numel(), bounds[d],
                bounds[d + 1], C.c_void_p(deg.data_ptr()))), a.reps)
            deg_s.append(t)
        ds = handles[0]
        key_bytes = [sum(c for i, c in enumerate(key_counts[s]) if i != s) * 8
                     for s in range(world)]
        per_rank = [sample_s[r] + finish_s[r] + deg_s[r] for r in range(world)]
        w_out = {
            "sample_s": sample_s, "root_kernel_s": root_s, "finish_s": finish_s,
            "degrees_s": deg_s,
            "max_sample_s": max(sample_s), "max_finish_s": max(finish_s),
            "max_degrees_s": max(deg_s),
            "max_rank_compute_s": max(max(sample_s), 0) + max(finish_s) + max(deg_s),
            "root_prepare_s": prep_s, "root_receive_s": recv_s,
            "root_record_bytes_received": rec_bytes[:world],
            "exchange_bytes_per_rank_max": max(key_bytes) + max(lower_bytes) + 8 * a.n
            + max(rec_bytes[:world] or [0]),
            "projected_speedup_compute_only": full_t / (max(sample_s) + max(finish_s)
                                                        + max(deg_s)),
        }
        result["worlds"][world] = w_out
        print(world, json.dumps({k2: (round(v2, 5) if isinstance(v2, float) else v2)
                                 for k2, v2 in w_out.items() if not isinstance(v2, list)}),
              "sample", [round(x * 1e3, 2) for x in sample_s],
              "root", [round(x * 1e3, 2) for x in root_s], flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(result, f, indent=1)


if __name__ == "__main__":
    main()
