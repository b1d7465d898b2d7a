#!/usr/bin/env python
"""Headline benchmark: MM iterations/s of the Welsch-MM registration hot path
(reference solver.hpp:224-289) on BASELINE.json config 2 — a 316x316 =
99,856-vertex height-field source against a warped, jittered, holed,
outlier-polluted target, ~3,000-node deformation graph, FP64.

One step = one accepted MM iteration (one IterationRecord): correspondence,
Welsch weights + energy, normal-equation assembly, block-Jacobi PCG solve,
rotation projection, Anderson combine (m=5) with its energy safeguard, and
the deformation of the next iterate. The timed run is the reference's
fixed-count single-stage idiom (acceptance_main.cpp:207-215): nu fixed at the
derived values, eps = 1e-300, so exactly `steps` iterations are accepted.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun): config 2 does not shard, so every rank runs
an independent replica ("replicas only"); value = iterations of all ranks /
max-over-ranks device time.

Other configs:
  --config 4   1M-vertex pair; with N > 1 the source vertices are sharded over
               the ranks and K, B, energies are allreduced over NCCL every
               pass ("strong": one registration, value = its iterations/s).
  --config 3   256 independent 20K-vertex pairs, 50 iterations each, pairs
               round-robin over the ranks, no communication.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MM iterations/s (100K-vertex source, config 2)"
UNIT = "iterations/s"


# MM iterations of one registration per BASELINE.json config
CONFIG_ITERS = {0: 100, 1: 100, 2: 100, 3: 50, 4: 50}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=5)
    ap.add_argument("--pcg-rtol", type=float, default=None, help="override the library default (1e-13)")
    ap.add_argument("--pairs", type=int, default=256, help="config 3: number of independent pairs")
    ap.add_argument("--pair-streams", type=int, default=12,
                    help="config 3: pairs run side by side per GPU (12: 9.3K it/s; 6: 8.8K, 9: 9.1K, 18: 6.6K, "
                         "profiles/r04_config3_streams_sweep.txt)")
    ap.add_argument("--pair-iters", type=int, default=50, help="config 3: MM iterations per pair")
    ap.add_argument("--pair-ctas", type=int, default=0,
                    help="config 3: PCG grid cap per pair (0 = SMs / pair-streams)")
    return ap.parse_args()


# ----------------------------------------------------------------- distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if self.local >= torch.cuda.device_count():
                raise SystemExit("bench.py: rank %d needs GPU %d but only %d are visible (one process per GPU)"
                                 % (self.rank, self.local, torch.cuda.device_count()))
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.torch, self.dist = torch, dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v):
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v):
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t)
        return float(t.item())

    def bcast_bytes(self, b):
        if self.world == 1:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi style clock / throttle sampling during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- workload
def problem_for(config, rank=0):
    from paper_2206_03410_b200 import registration as R
    if config == 3:  # one pair of the batch
        return R.make_problem(3, seed=4000)
    return R.make_problem(config)


def pcg_bytes_per_iteration(N, P):
    """one PCG iteration reads K once, the preconditioner and
    six 12N vectors: 128 (N+P) + 128 N + 6 * 96 N bytes."""
    return 128 * (N + P) + 128 * N + 6 * 96 * N


def iteration_fixed_bytes(n, m, sumk, N, P, mk=5):
    """SURVEY.md 8(d) fixed part of one MM iteration (without PCG)."""
    kbar = sumk / n
    per_vertex = (104 + 12 * kbar) * n
    target = 16 * m
    node = 128 * (N + P) + 96 * N + 4 * 96 * N + 16 * P
    aa = (2 * mk + 4) * 96 * N
    return per_vertex + target + node + aa


def kernel_bytes(n, m, sumk, N, P, entries, mk=5):
    """Algorithmic bytes per MM pass of each kernel class (
    SURVEY.md 8(d) split by kernel): compulsory HBM reads + writes, gathers of
    L2-resident node data not counted."""
    kbar = sumk / n
    return {
        "deform": (24 + 4 + 12 * kbar + 24 + 24) * n,           # src, influence CSR, old v, new v
        "nn": 24 * n + 16 * m + 4 * n + 8 * n + 24 * n,         # queries, target, prev idx, out idx/d2/q
        "terms": (8 + 8) * n + 16 * P + 8 * P + 4 * 96 * N,     # d2 -> w_a, pairs -> w_r, X/R
        "assemble": 128 * (N + P) + 96 * N + entries * (4 + 64) + n * (8 + 24),  # K, B, contributors, w_a, q
        "aa": (2 * mk + 4) * 96 * N,
    }


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def h2d_d2h_bytes(p):
    g = p.graph
    h2d = (p.source.nbytes + p.target.nbytes + g.node_positions.nbytes + 4 * g.edges.size +
           4 * g.infl_offsets.size + 4 * g.infl_nodes.size + 8 * g.infl_weights.size + 4 * g.reg_pairs.size +
           8 * g.reg_weights.size)
    d2h = 96 * g.node_count + 24 * p.n
    return int(h2d), int(d2h)


def host_cpu():
    """Core count and CPU model of the host this runs on (the GPU box in a
    driver run)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_baseline(p, cfg_kw, warmup, steps):
    from oracle import binding as O
    cfg = O.config(**cfg_kw)
    sec = O.time_iterations(p, cfg, warmup, steps)
    return steps / sec, sec


def reference_pairs(args, threads):
    """Config 3 on the CPU: independent pairs on `threads` host threads (the
    reference's model: one registration per thread, README.md:217-219); a
    bounded sample of 2 pairs per thread, each the full 50-iteration
    fixed-count run. Returns (iterations/s, pairs, seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import binding as O
    npairs = min(args.pairs, 2 * threads)
    probs = [O.make_problem(3, seed=4000 + q) for q in range(npairs)]
    cfgs = []
    for p in probs:
        prm = O.init_parameters(p)
        cfgs.append(O.config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300))

    def one(k):
        return O.time_iterations(probs[k], cfgs[k], 0, args.pair_iters)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(npairs)))
    wall = time.perf_counter() - t0
    return npairs * args.pair_iters / wall, npairs, wall


def run_reference(args, dist):
    """--impl reference: the reference's own CPU implementation of the path.
    The Eigen reference cannot be built here, so its restatement
    (oracle/, single thread per registration as the reference,
    README.md:217-219) is timed on the box's host cores. Its inputs come from
    the oracle alone (oracle.binding.make_problem: the same seeded arrays,
    tests/test_inputs.py), so this process never loads libnrr_b200.so. Same
    config, steps and warm-up as the GPU arm, except config 4, where one
    iteration of the reference (a 70K-unknown direct solve) takes ~45 s and
    the sample is capped at 3 timed iterations after 1 warm-up."""
    if dist.rank != 0:
        dist.barrier()
        dist.close()
        return
    from oracle import binding as O
    host = host_cpu()
    if args.config == 3:
        threads = host["nproc"] or 1
        value, npairs, sec = reference_pairs(args, threads)
        steps, warm = args.pair_iters, 0
        cores = threads
        sample = (f"{npairs} pairs x {args.pair_iters} fixed-count iterations on {threads} threads (one pair per "
                  "thread at a time); value = their iterations / wall time")
        workload = f"config 3: pairs of 20K source points (~600 nodes), {args.pair_iters} fixed-count iterations each"
        ms = 1e3 * sec / (npairs * args.pair_iters)
    else:
        p = O.make_problem(args.config)
        prm = O.init_parameters(p)
        kw = dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300)
        steps, warm = args.steps, max(3, args.warmup)
        if args.config == 4:
            steps, warm = min(steps, 3), 1
        value, sec = cpu_baseline(p, kw, warm, steps)
        cores = 1
        g = p.graph
        sample = (f"{steps} accepted MM iterations after {warm} warm-up, one registration on one thread "
                  "(the reference is single-threaded)")
        workload = (f"config {args.config}: {p.n} source / {len(p.target)} target points, {g.node_count} nodes, "
                    "fixed-count single stage (nu fixed, eps=1e-300), AA m=5")
        ms = 1e3 * sec / steps
    line = {
        "impl": "reference", "metric": metric_for(args.config), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "host": host,
                         "note": "oracle restatement of the reference (the Eigen reference is unbuildable here)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    dist.barrier()
    dist.close()


def metric_for(config):
    if config == 2:
        return METRIC
    if config == 4:
        return "MM iterations/s (1M-vertex source, config 4)"
    if config == 3:
        return "MM iterations/s (256 independent 20K-vertex pairs, config 3)"
    return f"MM iterations/s (config {config})"


def join_shard(R, ctx, dist, n_global):
    """Vertex sharding (config 4, N > 1): one NCCL communicator per context."""
    uid = dist.bcast_bytes(R.comm_unique_id() if dist.rank == 0 else None)
    ctx.set_comm(uid, dist.world, dist.rank)
    ctx.set_shard(n_global)


def run_b200(args, dist):
    from paper_2206_03410_b200 import registration as R

    p_full = problem_for(args.config, dist.rank)
    sharded = args.config == 4 and dist.world > 1
    if sharded:
        p = R.shard_problem(p_full, *R.shard_bounds(p_full.n, dist.world, dist.rank))
    else:
        p = p_full
    g = p.graph
    n, m, N, P, sumk = p.n, len(p.target), g.node_count, g.pair_count, len(g.infl_nodes)
    kk = np.diff(np.asarray(g.infl_offsets, dtype=np.int64))
    entries = int(np.sum(kk * (kk + 1) // 2))  # assembly contributor entries
    ctx = R.Context(device=dist.local, pcg_rtol=args.pcg_rtol)
    if sharded:
        join_shard(R, ctx, dist, p_full.n)
    ctx.set_problem(p)
    prm = ctx.init_parameters()
    cfg_kw = dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300)
    K, W = args.steps, max(3, args.warmup)
    cfg = R.solver_config(i_max=W + 2 * K + 10, **cfg_kw)
    # the timed passes run without per-kernel-class CUDA events (they cost
    # ~30 us per pass); K further passes with them give the kernel breakdown
    ctx.enable_timing(False)
    ctx.begin(cfg)
    ctx.iterate(W, flush_l2=not args.no_flush)  # untimed warm-up
    l0 = ctx.stats()["launches"]
    dist.barrier()
    with ClockSampler(dist.local) as clocks:
        acc, done, dev_ms = ctx.iterate(K, flush_l2=not args.no_flush)
    dist.barrier()
    launches = ctx.stats()["launches"] - l0
    ctx.enable_timing(True)
    s0 = ctx.stats()
    acc2, _, _ = ctx.iterate(K, flush_l2=not args.no_flush)  # breakdown passes (not the value)
    s1 = ctx.stats()
    X, v, rep = ctx.finish()
    if acc != K or acc2 != K:
        raise RuntimeError(f"only {acc} / {acc2} of {K} iterations accepted")
    max_ms = dist.max(dev_ms)
    total_iters = float(acc) if sharded else dist.sum(float(acc))  # sharded: one registration
    value = total_iters / (max_ms / 1e3)
    kms = {k: s1["kernel_ms"][k] - s0["kernel_ms"][k] for k in s1["kernel_ms"]}
    pcg_iters = s1["pcg_iterations"] - s0["pcg_iterations"]
    dominant = max(kms, key=kms.get)
    peak, peak_src = load_peaks()
    # dominant kernel roofline (per launch)
    if dominant == "pcg":
        bytes_per_launch = (pcg_iters / K) * pcg_bytes_per_iteration(N, P)
        avg_ms = kms["pcg"] / K
    else:
        bytes_per_launch = iteration_fixed_bytes(n, m, sumk, N, P) / 6
        avg_ms = kms[dominant] / K
    achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9
    step_bytes = iteration_fixed_bytes(n, m, sumk, N, P) + (pcg_iters / K) * pcg_bytes_per_iteration(N, P)
    step_gbs = step_bytes / ((dev_ms / K) / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "pcg_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None

    ctx.close()  # the one-shot call below creates its own context, as a user would
    # end-to-end through the C ABI with host buffers (uploads, index build,
    # init_parameters, K iterations, downloads), wall clock around the call
    # (three fresh one-shot registrations; the median is reported: a single
    # ~40 ms wall-clock sample carries the host's scheduling noise)
    # one full registration of the config (BASELINE.json: 100 fixed-count
    # iterations for configs 0-2, 50 for 3-4), at least K
    e2e_k = max(K, CONFIG_ITERS.get(args.config, K))
    cfg_e2e = R.solver_config(i_max=e2e_k, **cfg_kw)
    e2e_samples = []
    for _ in range(3):
        e2e_ctx = R.Context(device=dist.local, pcg_rtol=args.pcg_rtol)
        if sharded:
            join_shard(R, e2e_ctx, dist, p_full.n)
        dist.barrier()
        t0 = time.perf_counter()
        e2e_ctx.register(cfg_e2e, one_shot_problem=p)
        e2e_s = dist.max(time.perf_counter() - t0)
        e2e_iters = e2e_ctx.report()["total_iterations"]
        e2e_ctx.close()
        e2e_samples.append((float(e2e_iters) if sharded else dist.sum(float(e2e_iters))) / e2e_s)
    e2e_value = float(np.median(e2e_samples))
    e2e_s = float(e2e_iters) / e2e_value if sharded else e2e_k / (e2e_value / max(1, dist.world))
    h2d, d2h = h2d_d2h_bytes(p)

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cps, sec = cpu_baseline(p, cfg_kw, 1, args.cpu_steps)
        cpu = {"value": cps, "unit": UNIT, "cores": 1, "kind": "port", "host": host_cpu(),
               "sample": f"{args.cpu_steps} MM iterations of config {args.config} (n={n}) after 1 warm-up, "
                         "oracle restatement, one thread (the reference is single-threaded)"}
    if dist.rank == 0:
        line = {
            "metric": metric_for(args.config), "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
            "warmup": W, "ms_per_step": max_ms / K, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {args.config}: {n} source / {m} target points, {N} nodes, "
                                   f"{P} directed pairs, sum k {sumk}, fixed-count single stage (nu fixed, "
                                   "eps=1e-300), AA m=5",
                       "parallelism": (f"vertex-sharded x{dist.world} (NCCL allreduce of K, B, energies per pass)"
                                       if sharded else f"replicas x{dist.world}" if dist.world > 1 else "1 GPU"),
                       "l2": "flushed (2x L2 write) before every timed iteration, outside the timed interval"
                       if not args.no_flush else "not flushed (working set < L2)"},
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms},
            "step_roofline": {"achieved": step_gbs, "frac": step_gbs / peak, "bytes_per_step": step_bytes},
            "kernel_roofline": {k: {"bytes": b, "achieved_gbs": b / (kms[k] / K / 1e3) / 1e9,
                                    "frac": b / (kms[k] / K / 1e3) / 1e9 / peak}
                                for k, b in kernel_bytes(n, m, sumk, N, P, entries).items() if kms.get(k, 0) > 0},
            "kernel_ms_per_step": {k: v / K for k, v in kms.items()},
            "kernel_ms_note": "per-class CUDA events over K further passes (the timed passes run without them)",
            "pcg_iterations_per_step": pcg_iters / K,
            **({"sharded_split_ms_per_step": {
                "per_vertex (deform + nn + terms + assembly)": sum(kms[k] for k in ("deform", "nn", "terms",
                                                                                      "assemble")) / K,
                "allreduce (K, B)": (s1["comm_ms"] - s0["comm_ms"]) / K,
                "replicated solve (pcg)": kms["pcg"] / K, "replicated anderson": kms["aa"] / K},
                "nccl_ranks": dist.world} if sharded else {}),
            "nn_queries_per_s": n / (kms["nn"] / K / 1e3) if kms["nn"] > 0 else None,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "iterations": e2e_iters, "seconds": e2e_s,
                    "samples": e2e_samples,
                    "note": "median of 3 one-shot nrr_register calls (fresh context each): uploads, BVH, plan, "
                            f"init_parameters, {e2e_k} fixed-count iterations (the config's full registration), "
                            "downloads; h2d/d2h bytes are per registration"},
            "gpu_launches": launches,
            "clocks": clocks.result(),
        }
        print(json.dumps(line), flush=True)
    dist.close()


def run_pairs(args, dist):
    """Config 3: independent pairs round-robin over the ranks (no
    communication). On each GPU the rank's pairs run
    --pair-streams at a time: one context (own stream, PCG grid capped at
    SMs / streams CTAs) per pair, driven by that many host threads, so the
    small per-pair solves fill the GPU side by side. Every pair runs the
    fixed-count idiom for --pair-iters iterations. value = all ranks'
    iterations / max-over-ranks device time of the iterate phase (CUDA events
    around it, every context's stream drained on both sides; problem upload,
    plan and init_parameters excluded); e2e = the same through fresh contexts
    with host buffers (uploads, index build, plan, init, iterations,
    downloads), wall clock."""
    import threading

    import torch

    from paper_2206_03410_b200 import registration as R

    mine = [q for q in range(args.pairs) if q % dist.world == dist.rank]
    probs = [R.make_problem(3, seed=4000 + q) for q in mine]
    sms = torch.cuda.get_device_properties(dist.local).multi_processor_count
    S = max(1, min(args.pair_streams, len(mine)))
    cap = args.pair_ctas if args.pair_ctas > 0 else max(8, sms // S)

    def prepare(p):
        ctx = R.Context(device=dist.local, pcg_rtol=args.pcg_rtol, max_ctas=cap)
        ctx.enable_timing(False)
        ctx.set_problem(p)
        prm = ctx.init_parameters()
        cfg = R.solver_config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300,
                              i_max=args.pair_iters)
        return ctx, cfg

    def run_threads(fn):
        th = [threading.Thread(target=fn, args=(t,)) for t in range(S)]
        for x in th:
            x.start()
        for x in th:
            x.join()

    # phase 1 (untimed): every pair resident on the device, registration begun
    ctxs = [prepare(p) for p in probs]
    for ctx, cfg in ctxs:
        ctx.begin(cfg)
    counts = [0] * S
    launches0 = sum(c.stats()["launches"] for c, _ in ctxs)
    errors = []

    def work(t):
        try:
            for ctx, _ in ctxs[t::S]:
                acc, _, _ = ctx.iterate(args.pair_iters)
                counts[t] += acc
        except Exception as e:  # surfaced after the join
            errors.append(e)

    torch.cuda.synchronize(dist.local)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dist.local) as clocks:
        e0.record()
        run_threads(work)
        torch.cuda.synchronize(dist.local)
        e1.record()
        e1.synchronize()
    if errors:
        raise errors[0]
    dev_ms = e0.elapsed_time(e1)
    iters = sum(counts)
    launches = sum(c.stats()["launches"] for c, _ in ctxs) - launches0
    # algorithmic bytes of the timed iterations (SURVEY 8(d) per pair, with
    # each pair's own PCG iteration count)
    step_bytes = 0.0
    for (ctx, _), p in zip(ctxs, probs):
        g = p.graph
        step_bytes += (args.pair_iters * iteration_fixed_bytes(p.n, len(p.target), len(g.infl_nodes), g.node_count,
                                                               g.pair_count)
                       + ctx.stats()["pcg_iterations"] * pcg_bytes_per_iteration(g.node_count, g.pair_count))
    for ctx, _ in ctxs:
        ctx.finish()
        ctx.close()
    # e2e: fresh contexts, host buffers through the C ABI one-shot register
    e2e_counts = [0] * S

    def work_e2e(t):
        # one context per host thread, reused for its pairs (as a caller
        # running many registrations would); per pair: upload + plan, the
        # reference's init_parameters, the fixed-count registration and the
        # downloads (nrr_ctx_register)
        try:
            ctx = R.Context(device=dist.local, pcg_rtol=args.pcg_rtol, max_ctas=cap)
            ctx.enable_timing(False)
            for p in probs[t::S]:
                ctx.set_problem(p)
                prm = ctx.init_parameters()
                cfg = R.solver_config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"],
                                      eps=1e-300, i_max=args.pair_iters)
                _, _, rep = ctx.register(cfg)
                e2e_counts[t] += rep["total_iterations"]
            ctx.close()
        except Exception as e:
            errors.append(e)

    dist.barrier()
    t0 = time.perf_counter()
    run_threads(work_e2e)
    torch.cuda.synchronize(dist.local)
    wall = time.perf_counter() - t0
    if errors:
        raise errors[0]
    max_ms = dist.max(dev_ms)
    total = dist.sum(float(iters))
    e2e = dist.sum(float(sum(e2e_counts))) / dist.max(wall)
    all_bytes = dist.sum(step_bytes)
    peak, peak_src = load_peaks()
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        host = host_cpu()
        threads = host["nproc"] or 1
        cv, cpairs, csec = reference_pairs(args, threads)
        cpu = {"value": cv, "unit": UNIT, "cores": threads, "kind": "port", "host": host,
               "pairs_per_s": cpairs / csec,
               "sample": f"{cpairs} pairs x {args.pair_iters} fixed-count iterations of the oracle restatement on "
                         f"{threads} threads (one registration per thread, the reference's model)"}
    if dist.rank == 0:
        g = probs[0].graph
        line = {
            "metric": metric_for(3), "value": total / (max_ms / 1e3), "unit": UNIT, "n_gpus": dist.world,
            "steps": args.pair_iters, "warmup": 0, "ms_per_step": max_ms / max(1, iters),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config 3: {args.pairs} pairs x {probs[0].n} source points (~{g.node_count} "
                                   f"nodes), {args.pair_iters} fixed-count iterations each",
                       "parallelism": f"pairs round-robin over {dist.world} GPU(s), no communication; "
                                      f"{S} pairs side by side per GPU (PCG grid <= {cap} CTAs each)",
                       "l2": "not flushed: the batch (all pairs resident) exceeds L2, each pair's working set "
                             "stays resident during its own iterations",
                       "pairs_per_s": args.pairs / (max_ms / 1e3)},
            "roofline": {"bound": "hbm", "kernel": "whole step (all kernels of every pair)",
                         "achieved": all_bytes / (max_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": all_bytes / (max_ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                         "bytes_per_step": all_bytes / max(1.0, total)},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": UNIT, "seconds": wall,
                    "note": "wall clock; one context per host thread, per pair: upload + plan, init_parameters, "
                            "registration, downloads"},
            "gpu_launches": launches, "clocks": clocks.result(),
        }
        print(json.dumps(line), flush=True)
    dist.close()


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: launch the N ranks ourselves (one
    process per GPU, rendezvous on 127.0.0.1) and relay rank 0's line."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    if os.environ.get("BENCH_TRACEBACK_AFTER"):  # debugging aid: dump all thread stacks after N seconds
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["BENCH_TRACEBACK_AFTER"]), exit=True)
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
    elif args.config == 3:
        run_pairs(args, dist)
    else:
        run_b200(args, dist)


if __name__ == "__main__":
    main()
