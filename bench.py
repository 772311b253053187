#!/usr/bin/env python
"""Benchmark of the KDE-driven similarity-graph sampler (arXiv 2310.13870).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
    python bench.py --impl reference ...       # the reference's CPU path

One step = one full ``build_similarity_graph`` (tree, level-synchronous
descent with the fused KDE, pair collapse, weights, CSR, degrees) over the
workload, here BASELINE.json configs[2]: two-moons, n = 1,000,000 fp32,
sigma = 0.05, 64 samples/point (it fits one GPU). Prints ONE JSON line.

* value      sampled edges/s (n * L tickets per step / step time), whole job;
             inputs resident in HBM; every step timed with CUDA events on the
             library's launch stream, barrier + synchronize on both sides, L2
             flushed (512 MiB write) between steps outside the timed events;
             max over ranks.
* e2e        same metric through the public API with HOST buffers: each step
             uploads the points from pinned memory and receives the whole
             graph (upper CSR v, w, row_ptr + degrees) in pinned host
             buffers (fsgg_build_similarity_graph_into).
* roofline   the dominant kernel: for low d the symmetric root tile kernel
             (MUFU-bound): Gaussian evaluations (one ex2 each) per launch /
             its mean launch time (CUDA events around the launch on its
             stream), against the MUFU.EX2 throughput measured on this GPU in
             this run; for d >= 64 the tensor-core root launch against the
             TF32 peak.
* cpu_baseline  the reference's own code (oracle/_ref, compiled in place from
             /root/reference) on the host cores, default (auto = FGT for this
             config) backend, bounded sample: a contiguous block of queries.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIG_DOC = {
    "C1": "two 2-D blobs n=2000 sigma=0.5 L=32",
    "C2": "two-moons n=100k sigma=0.1 L=64",
    "C3": "two-moons n=1M sigma=0.05 L=64",
    "C4": "synthetic image pixels n=154401 d=5 sigma=0.2 L=32",
    "C5": "GMM n=70000 d=784 sigma=median dist L=32",
}
TC_MIN_DIM = 64  # kTcMinDim (engine.cuh): gaussian d >= 64 runs on tcgen05
NOMINAL_EX2_PER_CLK_PER_SM = 16
SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def metric_name(cfg: str) -> str:
    return f"sampled edges/sec ({cfg}: {CONFIG_DOC[cfg]})"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C3", choices=sorted(CONFIG_DOC))
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target seconds of CPU work for the cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--kde-backend", default="exact", choices=["exact", "fast", "autoselect"],
                   help="SparsifierConfig::kde.backend (exact: the headline; fast: the "
                        "certified eps-budget backend, include/fsgg.h)")
    return p.parse_args()


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi -lms 200 during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={SMI_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax),
                "power_w_max": max(power), "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------- reference ----
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_inputs(cfg: str):
    """(fp32-rounded fp64 points, sigma, rounds, source) for the reference arm.

    C1-C3 come from the REFERENCE's own generators (oracle/_ref make_blobs /
    make_moons, proj/src/datasets.cpp:32-124), bit-identical to the points
    the GPU arm builds from (tests/test_oracle.py pins them), so this arm never
    loads libfsgg.so. C4/C5 are harness-defined (the reference has no
    generator for them): their points come from the package's host generator."""
    from oracle.pyoracle import Ref
    if cfg in ("C1", "C2", "C3") and Ref.available:
        ref = Ref()
        if cfg == "C1":
            p, _ = ref.make_blobs(2000, [[-2.0, 0.0], [2.0, 0.0]], 0.5, 1)
            sigma, L = 0.5, 32
        elif cfg == "C2":
            p, _ = ref.make_moons(100_000, 0.05, 1)
            sigma, L = 0.1, 64
        else:
            p, _ = ref.make_moons(1_000_000, 0.05, 1)
            sigma, L = 0.05, 64
        return p.astype(np.float32).astype(np.float64), sigma, L, "reference make_moons/make_blobs"
    from paper_2310_13870_b200 import datasets
    w = datasets.config(cfg)
    return (w.points.astype(np.float64), w.sigma, w.rounds,
            "harness generator (libfsgg.so host code; no reference generator for this config)")


def bench_config(cfg: str, n: int, d: int, sigma: float, L: int, world: int,
                 kde_backend: str = "exact") -> dict:
    """The ONE config dict both arms print (same keys and values)."""
    extra = {} if kde_backend == "exact" else {"kde_backend": kde_backend}
    return {**extra, "workload": f"{cfg}: {CONFIG_DOC[cfg]}", "n": n, "d": d, "sigma": sigma,
            "samples_per_point": L, "seed": 1, "rng": "reference (splitmix64)",
            "parallelism": f"query shards x{world}",
            "l2": "GPU arm: flushed (512 MiB write) between steps"}


class RefSample:
    """The reference's own CPU path on a bounded sample of the workload.

    Builds the reference's estimator (make_estimator, proj/src/kde.cpp:104-129;
    backend 2 = auto: FGT for d <= 3, n >= 4096, else exact) once, then runs
    sample_neighbors_counted (proj/src/sampler.cpp:77) plus the degree KDE
    (sparsifier.cpp:74-75) for a contiguous block of queries: their descent is
    exactly the one the full job performs for them. The block is calibrated
    to ~target_s of CPU time. Falls back to the C restatement (exact, single
    thread) when oracle/_ref was not built."""

    def __init__(self, points64, sigma, rounds, seed, target_s, threads, backend=2):
        from oracle.pyoracle import Oracle, Ref
        self.n = points64.shape[0]
        self.rounds, self.seed = rounds, seed
        self.threads = threads
        self.points64, self.sigma = points64, sigma
        if Ref.available:
            self.ref = Ref()
            self.ref.set_threads(threads)
            t0 = time.perf_counter()
            self.est = self.ref.estimator(points64, 0, sigma, backend)
            self.t_build = time.perf_counter() - t0
            self.kind, self.backend = "reference", self.est.backend
        else:
            self.ref, self.est = None, None
            self.orc = Oracle()
            self.t_build, self.kind, self.backend, self.threads = 0.0, "port", "exact (oracle restatement)", 1
        self.start = self.n // 4
        s = 64
        while True:  # calibrate: fixed per-call overheads make tiny probes pessimistic
            t = sum(self.run(np.arange(self.start, self.start + s, dtype=np.uint32)))
            t = max(t, 1e-6)
            if t >= target_s / 4 or s >= self.n - self.start:
                break
            s = int(min(self.n - self.start, s * min(8.0, 0.5 * target_s / t)))
        self.block = int(min(self.n - self.start, max(64, s * target_s / t)))
        self.qs = np.arange(self.start, self.start + self.block, dtype=np.uint32)

    def run(self, qs=None):
        """(sampling seconds, degree-KDE seconds) for one pass over the block."""
        qs = self.qs if qs is None else qs
        t0 = time.perf_counter()
        if self.est is not None:
            self.est.sample_counted(qs, self.rounds, self.seed)
            t1 = time.perf_counter()
            self.est.eval(0, self.n, qs)
        else:
            self.orc.sample_counted(self.points64, qs, self.rounds, self.seed, self.sigma)
            t1 = time.perf_counter()
            self.orc.kde_exact(self.points64, 0, self.n, qs, self.sigma)
        return t1 - t0, time.perf_counter() - t1


def reduced_full_build(points64_fn, sigma, rounds, threads):
    """BuildReport phases (proj/src/sparsifier.cpp:123-140) of one complete
    reference build_similarity_graph at a reduced n (default backend)."""
    from oracle.pyoracle import Ref
    if not Ref.available:
        return None
    ref = Ref()
    ref.set_threads(threads)
    p64, label = points64_fn()
    g = ref.build_graph(p64, sigma, rounds, seed=1, backend=2, want_estimates=False)
    rep = g["report"]
    keys = ("estimator_build_seconds", "sampling_seconds", "degree_kde_seconds",
            "weighting_seconds", "total_seconds")
    return {"points": label, "n": int(p64.shape[0]), "backend": rep["backend"],
            "edge_count": int(rep["edge_count"]),
            "phases": {k: rep[k] for k in keys},
            "sampled_edges_per_s": p64.shape[0] * rounds / max(rep["total_seconds"], 1e-9)}


def cpu_baseline(cfg, points64, sigma, rounds, seed, target_s):
    threads = os.cpu_count() or 1
    rs = RefSample(points64, sigma, rounds, seed, target_s, threads)
    ts, tk = rs.run()
    dt = ts + tk
    n = points64.shape[0]
    value = rs.block * rounds / dt
    out = {
        "value": value, "unit": "sampled edges/s", "cores": rs.threads, "kind": rs.kind,
        "cpu_model": cpu_model(),
        "sample": (f"{rs.backend} backend; sample_neighbors_counted + degree KDE for a "
                   f"contiguous block of {rs.block} of {n} queries (L={rounds}) on the full "
                   f"point set; estimator build {rs.t_build:.2f}s excluded"),
        "sample_seconds": dt, "estimator_build_seconds": rs.t_build,
        "phases_on_sample": {"estimator_build_seconds": rs.t_build, "sampling_seconds": ts,
                             "degree_kde_seconds": tk},
        "extrapolated_full_job_seconds": rs.t_build + dt * n / rs.block,
    }
    if rs.kind == "reference":
        # the exact backend (the one the device path reproduces) on a smaller block
        try:
            ex = RefSample(points64, sigma, rounds, seed, target_s / 3, threads, backend=0)
            es, ek = ex.run()
            out["exact_backend"] = {
                "value": ex.block * rounds / (es + ek), "unit": "sampled edges/s",
                "sample": f"exact backend; contiguous block of {ex.block} queries",
                "sample_seconds": es + ek,
                "extrapolated_full_job_seconds": (es + ek) * n / ex.block}
        except Exception as exc:  # reported, never fatal
            out["exact_backend"] = {"error": repr(exc)}
        if cfg in ("C2", "C3"):
            try:
                def pts():
                    from oracle.pyoracle import Ref
                    p, _ = Ref().make_moons(20_000, 0.05, 1)
                    return p.astype(np.float32).astype(np.float64), "reference make_moons(20000)"
                out["build_report_reduced"] = reduced_full_build(pts, sigma, rounds, threads)
            except Exception as exc:
                out["build_report_reduced"] = {"error": repr(exc)}
    return out


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU code (oracle/_ref, compiled
    in place from /root/reference by oracle/Makefile) on the host cores. Never
    loads libfsgg.so for C1-C3."""
    if rank != 0:
        return
    p64, sigma, L, source = reference_inputs(args.config)
    n, d = p64.shape
    threads = os.cpu_count() or 1
    rs = RefSample(p64, sigma, L, 1, 6.0, threads)
    for _ in range(args.warmup):
        rs.run()
    times, ts_sum, tk_sum = [], 0.0, 0.0
    for _ in range(args.steps):
        ts, tk = rs.run()
        times.append(ts + tk)
        ts_sum += ts
        tk_sum += tk
    step = float(np.mean(times))
    value = rs.block * L / step
    sample = (f"{rs.backend} backend; each step = sample_neighbors_counted + degree KDE "
              f"for a contiguous block of {rs.block} of {n} queries (L={L}); "
              f"estimator build {rs.t_build:.2f}s once, untimed; points: {source}")
    print(json.dumps({
        "impl": "reference", "metric": metric_name(args.config),
        "value": value, "unit": "sampled edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, n, d, sigma, L, world),
        "cpu_baseline": {"value": value, "unit": "sampled edges/s", "cores": rs.threads,
                         "kind": rs.kind, "cpu_model": cpu_model(), "sample": sample,
                         "phases_per_step": {"sampling_seconds": ts_sum / args.steps,
                                             "degree_kde_seconds": tk_sum / args.steps},
                         "estimator_build_seconds": rs.t_build,
                         "extrapolated_full_job_seconds": rs.t_build + step * n / rs.block},
        "e2e": {"value": value, "unit": "sampled edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def relaunch_under_torchrun(args):
    """--gpus N without a torchrun environment: re-exec as N ranks (one per
    GPU, rendezvous on 127.0.0.1), as the driver's own launch would."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------ ours ----
def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2310_13870_b200 as F
    from paper_2310_13870_b200 import _native as N
    from paper_2310_13870_b200 import datasets, parallel

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    w = datasets.config(args.config)
    n, L = w.n, w.rounds
    kernel = F.Kernel(F.KernelFamily.gaussian, w.sigma)
    cfg = F.SparsifierConfig(rounds=L, seed=1, kde_backend=F.KdeBackend[args.kde_backend])
    ds = F.Dataset(w.points, device=local)
    stream = torch.cuda.ExternalStream(N.lib().fsgg_dataset_stream(ds._h), device=local)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step():
        if world == 1:
            g, rep = F.build_similarity_graph_device(ds, kernel, cfg)
            return g, rep
        res = parallel.build_similarity_graph_distributed(ds, kernel, cfg)
        return res, res.report

    for _ in range(args.warmup):
        step()
    barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local).start() if rank == 0 else None
    total_ms, reps, edges = 0.0, [], 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g, rep = step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        total_ms += e0.elapsed_time(e1)
        reps.append(rep)
        edges = int(g.num_edges)
    clk = clocks.stop() if clocks else None
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s = float(t.item()) * 1e-3
    K = args.steps
    sampled_edges = n * L * K                     # tickets routed to leaves
    value = sampled_edges / total_s
    evals = sum(r.kernel_evals for r in reps)
    tiled_evals = sum(r.kde_tiled_evals for r in reps)
    tiled_perf = sum(r.kde_tiled_performed_evals for r in reps)
    performed = sum(r.kernel_evals_performed for r in reps)
    tiled_s = sum(r.kde_tiled_seconds for r in reps)
    tiled_launches = sum(r.kde_tiled_launches for r in reps)
    root_perf = sum(getattr(r, "kde_root_performed_evals", 0) for r in reps)
    root_s = sum(getattr(r, "kde_root_seconds", 0.0) for r in reps)
    launches = sum(r.gpu_launches for r in reps)
    if world > 1:
        agg = torch.tensor([evals, tiled_evals], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(agg)
        evals = float(agg[0])

    # ---- end-to-end through the public host API --------------------------
    e2e = None
    if not args.no_e2e:
        pinned = torch.empty(w.points.shape, dtype=torch.float32, pin_memory=True)
        pinned.numpy()[:] = w.points
        host_ptr = pinned.data_ptr()
        hostbufs = F.api.HostGraphBuffers()
        h2d = w.points.nbytes
        e2e_ms, d2h = 0.0, 0
        for i in range(args.warmup + K):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            ds.upload_ptr(host_ptr)  # pinned host -> device
            if world == 1:
                # device -> pinned host: the graph as CSR (row_ptr, v, w) +
                # degrees, each array's copy started as soon as it is final
                # (fsgg_build_similarity_graph_into); the per-edge u is
                # redundant with row_ptr and expanded on demand
                g = hostbufs.build_into(ds, kernel, cfg, L)
                nbytes = g.v.nbytes + g.w.nbytes + g.row_ptr.nbytes + g.degrees.nbytes
            else:
                # each rank reads back the all-gathered graph (CSR + degrees)
                res = parallel.build_similarity_graph_distributed(ds, kernel, cfg)
                nbytes = 0
                for name in ("v", "w", "row_ptr", "degrees"):
                    t_dev = getattr(res, name)
                    pin = hostbufs._bufs.get(name)
                    if pin is None or pin.numel() < t_dev.numel() or pin.dtype != t_dev.dtype:
                        pin = torch.empty(t_dev.numel(), dtype=t_dev.dtype, pin_memory=True)
                        hostbufs._bufs[name] = pin
                    pin[: t_dev.numel()].copy_(t_dev, non_blocking=True)
                    nbytes += t_dev.numel() * t_dev.element_size()
            torch.cuda.synchronize()
            barrier()
            if i >= args.warmup:
                e2e_ms += (time.perf_counter() - t0) * 1e3
                d2h = nbytes
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": sampled_edges / (float(t.item()) * 1e-3), "unit": "sampled edges/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": float(t.item()) / K}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----------------------------------
    import ctypes as C
    ex2 = C.c_double()
    clk_mhz = C.c_double()
    N.lib().fsgg_probe_ex2_throughput(local, C.byref(ex2), C.byref(clk_mhz))
    props = torch.cuda.get_device_properties(local)
    nominal = NOMINAL_EX2_PER_CLK_PER_SM * props.multi_processor_count * 1965e6
    achieved = tiled_perf / max(tiled_s, 1e-12)  # evaluations the kernel executed
    traffic = None
    # the committed ncu capture of this config's dominant kernel (scripts/ncu_summary.py)
    prof = os.path.join(ROOT, "profiles", f"r2_{args.config.lower()}_wtile_ncu.json"
                        if root_s > 0 else "kde_tiled_ncu.json")
    if os.path.exists(prof):
        try:
            cap = json.load(open(prof))
            # only a capture of this workload's launch says anything about it
            if str(cap.get("config", "")).startswith(args.config):
                traffic = cap.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    tensor = w.d >= TC_MIN_DIM
    if tensor:
        # tcgen05 kind::tf32 path (kde_tc.cu): algorithmic work is the fp32
        # dot-product form, 2*d FLOPs per evaluation; the
        # kernel executes it three times (3xTF32 error compensation).
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except (OSError, ValueError):
            pass
        bf16 = float(peaks.get("bf16_tflops", 2250.0))
        tf32_peak = bf16 / 2.0
        # the root launch (n x n, contiguous query tiles) is the dominant one;
        # deeper tensor-core levels (gathered query blocks) are reported beside
        r_perf, r_s = (root_perf, root_s) if root_s > 0 else (tiled_perf, tiled_s)
        alg = r_perf * 2.0 * w.d / max(r_s, 1e-12) / 1e12
        traffic = None
        prof = os.path.join(ROOT, "profiles", "kde_tc_ncu.json")
        if os.path.exists(prof):
            try:
                cap = json.load(open(prof))
                l0 = cap["launches"][0]
                mul = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
                if str(cap.get("config", "")).startswith(args.config):
                    traffic = sum(float(l0[k][0]) * mul.get(l0[k][1], 1.0)
                                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            except (OSError, ValueError, KeyError, IndexError):
                traffic = None
        # symmetric root (kde_tc_sym_kernel): each executed pair evaluation
        # serves two row sums; the reference evaluates n^2 at the root
        r_ms = (r_s / K if root_s > 0 else tiled_s / max(tiled_launches, 1)) * 1e3
        ref_alg = (n * n * 2.0 * w.d) / max(r_ms * 1e-3, 1e-12) / 1e12 if root_s > 0 else alg
        roofline = {
            "bound": "tensor",
            "kernel": ("kde_tc_sym_kernel<gaussian> (root level, each pair once; tcgen05.mma "
                       "kind::tf32, 3xTF32)"),
            "achieved": alg, "peak": tf32_peak, "unit": "TFLOP/s",
            "frac": alg / tf32_peak,
            "executed_tflops": 3.0 * alg, "executed_frac": 3.0 * alg / tf32_peak,
            "reference_equivalent_tflops": ref_alg,
            "reference_equivalent_frac": ref_alg / tf32_peak,
            "reference_equivalent_note": ("2*d FLOPs x n^2 evaluations (the reference's root "
                                          "pass) / the symmetric launch, which executes each "
                                          "pair once for both row sums"),
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops (burst, cuBLAS) / 2: dense TF32 is "
                            "half the bf16 rate on Blackwell"),
            "algorithmic_unit": "2*d FLOPs per Gaussian evaluation (dot-product form, SURVEY.md §8d)",
            "evals_per_launch": r_perf / K if root_s > 0 else tiled_perf / max(tiled_launches, 1),
            "mean_launch_ms": (r_s / K if root_s > 0 else tiled_s / max(tiled_launches, 1)) * 1e3,
            "share_of_step": r_s / max(total_s, 1e-12) if world == 1 else None,
            "traffic": traffic,
            "all_tensor_launches": {"executed_evals_per_step": tiled_perf / K,
                                    "seconds_per_step": tiled_s / K,
                                    "algorithmic_tflops": tiled_perf * 2.0 * w.d / max(tiled_s, 1e-12) / 1e12,
                                    "launches_per_step": tiled_launches / K},
        }
    elif root_s > 0:
        # the dominant kernel is the symmetric root pass (kde_sym.cu): every
        # pair (q, x) of non-pruned block pairs evaluated once, one ex2 each,
        # serving both q's and x's rows; timed around the tile kernel alone
        root_rate = root_perf / root_s
        roofline = {
            "bound": "mufu",
            "kernel": (f"sym_wtile_kernel<{w.d},gaussian> (root level, each pair once; one warp "
                       "per block-pair tile, persistent)" if w.d <= 6 else
                       f"sym_tile_kernel<{w.d},gaussian> (root level, each pair once)"),
            "achieved": root_rate / 1e9, "peak": ex2.value / 1e9, "unit": "Gex2/s",
            "frac": root_rate / ex2.value if ex2.value else None,
            "peak_source": "measured in this run: MUFU.EX2 microbenchmark (fsgg_probe_ex2_throughput)",
            "nominal_peak": nominal / 1e9, "frac_of_nominal": root_rate / nominal,
            "algorithmic_unit": ("one Gaussian kernel evaluation = one ex2 (SURVEY.md §8d); here "
                                 "each executed ex2 is a pair serving two row sums"),
            "evals_per_launch": root_perf / K,
            "reference_equivalent_evals_per_launch": (n * n) ,
            "reference_equivalent_rate": n * n * K / root_s / 1e9,
            "mean_launch_ms": root_s / K * 1e3,
            "share_of_step": root_s / max(total_s, 1e-12) if world == 1 else None,
            "traffic": traffic,
            "all_tile_kernels": {"executed_evals_per_step": tiled_perf / K,
                                 "seconds_per_step": tiled_s / K,
                                 "rate_gex2_s": achieved / 1e9,
                                 "launches_per_step": tiled_launches / K},
        }
    else:
        roofline = {
            "bound": "mufu", "kernel": "kde_lowd_tiled_kernel<2,gaussian>",
            "achieved": achieved / 1e9, "peak": ex2.value / 1e9, "unit": "Gex2/s",
            "frac": achieved / ex2.value if ex2.value else None,
            "peak_source": "measured in this run: MUFU.EX2 microbenchmark (fsgg_probe_ex2_throughput)",
            "nominal_peak": nominal / 1e9, "frac_of_nominal": achieved / nominal,
            "algorithmic_unit": "one Gaussian kernel evaluation = one ex2 (SURVEY.md §8d)",
            "evals_per_launch": tiled_perf / max(tiled_launches, 1),
            "reference_equivalent_evals_per_launch": tiled_evals / max(tiled_launches, 1),
            "reference_equivalent_rate": tiled_evals / max(tiled_s, 1e-12) / 1e9,
            "mean_launch_ms": tiled_s / max(tiled_launches, 1) * 1e3,
            "share_of_step": tiled_s / max(total_s, 1e-12) if world == 1 else None,
            "traffic": traffic,
        }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, w.points.astype(np.float64), w.sigma, L, 1,
                               args.cpu_seconds)
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "error": repr(exc)}
    line = {
        "metric": metric_name(args.config),
        "value": value, "unit": "sampled edges/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": total_s * 1e3 / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.config, n, w.d, w.sigma, L, world, args.kde_backend),
        "kde_backend": {"name": reps[0].backend, "epsilon": reps[0].epsilon},
        "kernel_evals_per_s": evals / total_s, "kernel_evals_per_step": evals / K / max(world, 1),
        "kernel_evals_performed_per_step": performed / K,
        "kernel_evals_note": ("reference-equivalent Gaussian evaluations (2.38 n^2 sampler + n^2 "
                              "degree KDE in the reference; here the degree KDE is fused, levels "
                              "reuse partial rows and certified pruning skips sub-chunks below "
                              "2^-48 of the node mass, so far fewer are executed)"),
        "undirected_edges": edges, "undirected_edges_per_s": edges * K / total_s,
        "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
