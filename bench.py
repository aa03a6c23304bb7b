#!/usr/bin/env python3
"""Benchmark: permutation cost evaluations/s (U1 = one reference evaluate()).

Workload (BASELINE.json target: ">= 100x the host CPU in permutation
evaluations/sec on one B200 for N=1024 ring cost"): config C4 -- the
1024-host synthetic hierarchical matrix (fixtures.py, fixed-point variant so
every cost is bit-exact vs the reference), ring all-reduce cost model.  A step
scores one batch of random orders that is resident in HBM (2 GiB of uint16
orders per GPU, far larger than the 126 MB L2), with the per-order bijection
check on, exactly as the reference's evaluate() validates every order.

Arms
  (default)          our CUDA path; one process per GPU under torchrun, each
                     GPU scores its own batch (weak scaling, no collective in
                     the data path), time = max over ranks of CUDA-event time.
  --impl reference   the reference's own evaluate() (oracle/_ref, compiled from
                     the unmodified sources) on all host threads, rank 0 only.

Extra keys: roofline (dominant kernel), cpu_baseline, e2e (host buffers through
the C ABI rw_evaluate_batch, H2D/D2H inside the timed region), clocks,
gpu_launches, and `extras` (N=13 exhaustive time, C1 time-to-best-ring).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "permutation cost evals/sec (ring, N=1024, U1 = one reference evaluate())"
UNIT = "evals/s"
WORKLOAD = "C4: N=1024 ring all-reduce cost, synthetic 3-level hierarchical matrix (fixed-point q/16 us, S=2^27)"
N = 1024
BATCH = 1 << 21  # orders per GPU per step: 2M x 1024 x 2 B = 4 GiB of uint16 orders in HBM
E2E_BATCH = 1 << 16
C4_CHAINS = 592  # time-to-best-ring at C4: 4 chains (warps) per SM, the fastest per chain; DESIGN.md 5
CPU_SECONDS = 10.0


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 5.0  # start timing only once sampling is live
            while not self.lines and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "error": (self.lines[0][:200] if self.lines else "nvidia-smi produced no samples")}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------------- reference --
def cpu_reference_rate(m: np.ndarray, seconds: float, threads: int):
    """Reference evaluate() (oracle/_ref) on `threads` host threads; returns evals/s and the sample."""
    from oracle.pyoracle import Port, Reference, make_spec, reference_available
    spec = make_spec(0, N, float(2 ** 27), 2, 1, 0)
    kind = "reference" if reference_available() else "port"
    eng = Reference() if kind == "reference" else Port()
    rng = np.random.default_rng(7)
    pool = rng.permuted(np.tile(np.arange(N, dtype=np.int32), (max(64, min(65536, threads * 512)), 1)), axis=1)

    def run(orders):
        if kind == "reference":
            eng.evaluate_batch(m, orders, spec, threads=threads)
        else:
            eng.evaluate_batch(m, orders, spec)

    run(pool[: max(threads * 4, 16)])  # warm caches / threads
    done = 0
    t = time.perf_counter()
    while True:
        run(pool)
        done += pool.shape[0]
        dt = time.perf_counter() - t
        if dt >= seconds:
            break
    return done / dt, {"kind": kind, "cores": threads if kind == "reference" else 1,
                       "sample": f"{done} evaluations of random C4 orders (pool of {pool.shape[0]}), {dt:.1f} s"}


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import paper_2105_14088_b200 as rw  # fixture generator only (host code)
    m = rw.fixtures.config_matrix("C4", "fixed")
    threads = os.cpu_count() or 1
    per_step = max(1.0, 20.0 / max(1, args.steps))
    for _ in range(args.warmup):
        cpu_reference_rate(m, min(per_step, 1.0), threads)
    rates = []
    t0 = time.perf_counter()
    info = None
    for _ in range(args.steps):
        r, info = cpu_reference_rate(m, per_step, threads)
        rates.append(r)
    elapsed = time.perf_counter() - t0
    value = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * elapsed / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": N, "model": "ring", "threads": threads},
            "cpu_baseline": dict(info, value=value, unit=UNIT),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm ---
def graph_kernel_nodes(graph) -> int:
    """Kernel launches one replay of the captured step performs (the graph's
    kernel nodes: route + score per chunk, the finalize pass)."""
    from cuda.bindings import runtime as cudart
    raw = graph.raw_cuda_graph()
    g = raw if isinstance(raw, cudart.cudaGraph_t) else cudart.cudaGraph_t(init_value=int(raw))
    err, _, num = cudart.cudaGraphGetNodes(g, 0)
    err, nodes, num = cudart.cudaGraphGetNodes(g, num)
    kernels = 0
    for nd in nodes[:num]:
        err, ty = cudart.cudaGraphNodeGetType(nd)
        if ty == cudart.cudaGraphNodeType.cudaGraphNodeTypeKernel:
            kernels += 1
    return kernels


def make_orders_device(torch, count: int, n: int, seed: int):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    out = torch.empty((count, n), dtype=torch.int16, device="cuda")
    step = 1 << 15
    for s in range(0, count, step):
        e = min(count, s + step)
        out[s:e] = torch.rand((e - s, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2105_14088_b200 as rw
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    m = rw.fixtures.config_matrix("C4", "fixed")
    prob = rw.Problem(m, device=local)
    spec = rw.fixtures.ring_spec(N, rw.fixtures.SIZE_FIXED)
    batch = args.batch
    orders = make_orders_device(torch, batch, N, seed=1234 + rank)
    costs = torch.empty(batch, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def step(p=prob):
        p.evaluate_batch_device(spec, orders.data_ptr(), 2, batch, costs.data_ptr(), stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    prob.sync_errors()

    # parity spot check of this very batch against the reference costs (oracle port, 8 rows)
    if rank == 0:
        from oracle.pyoracle import Port, make_spec
        rows = orders[:8].cpu().numpy().view(np.uint16).astype(np.int32)
        want = Port().evaluate_batch(m, rows, make_spec(0, N, rw.fixtures.SIZE_FIXED))
        assert np.array_equal(costs[:8].cpu().numpy(), want), "GPU costs differ from the oracle"

    # One step (the route/score kernel pairs of every chunk) captured as a CUDA
    # graph; the timed loop replays it.
    graph = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(graph):
        cap = torch.cuda.current_stream()
        prob.evaluate_batch_device(spec, orders.data_ptr(), 2, batch, costs.data_ptr(), cap.cuda_stream)
    graph.replay()
    torch.cuda.synchronize()
    prob.sync_errors()
    launches_per_step = graph_kernel_nodes(graph)

    # ---- timed region: device-resident orders (value) ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    with ClockSampler(local) as clocks:
        ev[0].record(stream)
        for k in range(args.steps):
            graph.replay()
            ev[k + 1].record(stream)
        barrier()
    prob.sync_errors()
    per_launch_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * batch * args.steps / (max_ms / 1000.0)

    def time_path(path, reps=10):
        alt = rw.Problem(m, device=local)
        alt.set_path(path)
        step(alt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            step(alt)
        e1.record(stream)
        torch.cuda.synchronize()
        alt.sync_errors()
        return batch * reps / (e0.elapsed_time(e1) / 1000.0)

    # ---- e2e: host int32 orders through rw_evaluate_batch (H2D + D2H inside) ----
    e2e_batch = args.e2e_batch
    host_orders = torch.empty((e2e_batch, N), dtype=torch.int32, pin_memory=True)
    host_orders.copy_(orders[:e2e_batch].to(torch.int32).cpu())
    host_np = host_orders.numpy()
    host_costs_t = torch.empty(e2e_batch, dtype=torch.float64, pin_memory=True)
    host_costs = host_costs_t.numpy()
    import ctypes as C
    from paper_2105_14088_b200 import _lib
    cs = spec._c()

    def e2e_step():
        _lib.check(_lib.lib.rw_evaluate_batch(prob.handle, C.byref(cs), _lib.ptr(host_np, C.c_int32), e2e_batch,
                                              _lib.ptr(host_costs, C.c_double), 0, None))

    for _ in range(2):
        e2e_step()
    e2e_steps = max(3, min(args.steps, 20))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    barrier()
    e2e_dt = time.perf_counter() - t0
    te = torch.tensor([e2e_dt], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_batch * e2e_steps / float(te.item())

    multi = {}
    if not args.no_extras:
        multi = run_multi_extras(rw, torch, dist, rank, world, local, prob, spec, barrier)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    bytes_per_eval = 2 * N + N * 2 + 8  # order read + L*e lookups (u16) + cost write
    launch_ms = statistics.mean(per_launch_ms)
    achieved = bytes_per_eval * batch / (launch_ms / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        bpo = json.load(open(tpath)).get("bytes_per_order")
        traffic = bpo * batch if bpo else None  # per bench step (one graph replay)
    clock = clocks.summary()
    # The lookups run against shared memory: one random 2-byte scatter (route) and
    # one random 2-byte gather (score) per hop, against the measured random-gather
    # peak (profiles/gather_peaks.json, scripts/microbench/gather_peaks.cu).
    smem_access = None
    gpath_peaks = os.path.join(ROOT, "profiles", "gather_peaks.json")
    if os.path.exists(gpath_peaks):
        gp = json.load(open(gpath_peaks))
        acc_per_s = 2 * N * batch / (launch_ms / 1000.0)
        smem_access = {"accesses_per_s": acc_per_s, "peak_per_s": gp["smem_random_u16_lookups_per_s"],
                       "frac": acc_per_s / gp["smem_random_u16_lookups_per_s"],
                       "note": "route scatter + score gather, 2 random u16 shared-memory accesses per hop"}

    cpu_value, cpu_info = (None, {"kind": "skipped", "cores": 0, "sample": "--no-cpu"})
    if not args.no_cpu:
        cpu_value, cpu_info = cpu_reference_rate(m, CPU_SECONDS, os.cpu_count() or 1)

    extras = {}
    if not args.no_extras:
        extras = run_extras(rw, torch)
        # A/B: the same batch through the alternative ring kernels (not the default path)
        extras["ring_kernel_ab"] = {
            "unit": UNIT,
            "transpose_default": value / world,
            "l2_gather": time_path("l2"),
            "cluster_dsmem": time_path("cluster"),
            "note": "l2_gather: one warp per order, random sector gathers (L1TEX-wavefront bound); "
                    "cluster_dsmem: rows split over a 16-CTA cluster, hops routed by DSMEM stores "
                    "(DSMEM-transaction bound) -- DESIGN.md 4"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": N, "model": "ring", "orders_per_gpu_per_step": batch,
                   "order_bytes_in_hbm": batch * N * 2, "l2_policy": "inputs larger than L2 (2 B x N x batch)",
                   "validation": "bijection check on every order", "parallelism": f"dp{world} (independent batches)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "smem_random_access": smem_access,
                     "kernel": "k_ring_route + k_ring_score (transpose ring path, one pair per chunk)",
                     "algorithmic_bytes_per_eval": bytes_per_eval,
                     "lookups_per_s": N * batch / (launch_ms / 1000.0),
                     "note": "achieved = SURVEY 8(d) algorithmic bytes (2N order + N x 2 B lookups + 8) x evals/s "
                             "over the step's CUDA-event time; the path streams the orders from HBM once and "
                             "keeps its predecessor exchange buffer in L2 -- DESIGN.md 4"},
        "cpu_baseline": dict(cpu_info, value=cpu_value, unit=UNIT),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e_batch * N * 4,
                "d2h_bytes_per_step": e2e_batch * 8, "api": "rw_evaluate_batch (C ABI, pinned host int32 orders)"},
        "clocks": clock,
        "gpu_launches": args.steps * launches_per_step,
        "extras": extras,
        "multi_gpu_configs": multi,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_multi_extras(rw, torch, dist, rank, world, local, prob4, spec4, barrier):
    """BASELINE configs C4 and C5 at this run's GPU count (every rank works;
    times are the max over ranks):
      * C5 halving-doubling (xor) scoring, weak scaling: 16K orders per GPU;
      * C4 annealing with 65,536 chains split over the GPUs (strong scaling in
        chains), winner picked by NCCL all-reduce MIN (cost, chain) + broadcast."""
    from paper_2105_14088_b200 import dist as rwd
    out = {}

    def max_over_ranks(t):
        x = torch.tensor([t], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
        return float(x.item())

    A = rw.Algorithm
    m5 = rw.fixtures.config_matrix("C5", "fixed")
    p5 = rw.Problem(m5, device=local)
    spec5 = rw.CollectiveSpec(A.HalvingDoubling, 4096, rw.fixtures.SIZE_FIXED, 2, rw.CostMode.LatencyTimesSize,
                              rw.HdPairing.XorPairing)
    count, reps = 1 << 14, 4
    o5 = make_orders_device(torch, count, 4096, seed=77 + rank)
    c5 = torch.empty(count, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    p5.evaluate_batch_device(spec5, o5.data_ptr(), 2, count, c5.data_ptr(), st.cuda_stream)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        p5.evaluate_batch_device(spec5, o5.data_ptr(), 2, count, c5.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    p5.sync_errors()
    t5 = max_over_ranks(e0.elapsed_time(e1) / 1000.0)
    out["c5_hd_xor"] = {"value": world * count * reps / t5, "unit": "evals/s", "n_gpus": world,
                        "orders_per_gpu": count * reps, "scaling": "weak",
                        "kernel": "k_rounds_route + k_rounds_score + k_rounds_finalize (transpose path)"}
    del o5, c5, p5

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "anneal_c4.json")))
    target = min(r["cost"] for r in g["results"])
    chains_total, steps = 65536, 2048
    barrier()
    t0 = time.perf_counter()
    sol, rep = rwd.anneal_sharded(prob4, spec4, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                  chains_total, schedule="calibrated")
    barrier()
    ta = max_over_ranks(time.perf_counter() - t0)
    out["c4_anneal_65536_chains"] = {"seconds": ta, "cost": sol.cost, "target_reference_min_seeds0_3": target,
                                     "reached": sol.cost <= target, "chains_total": chains_total,
                                     "chains_per_gpu": chains_total // world, "steps_per_level": steps,
                                     "evaluations": sol.evaluations, "winner_chain": rep["winner_chain"],
                                     "n_gpus": world, "scaling": "strong (fixed total chains)",
                                     "argmin": "NCCL all-reduce MIN on (cost, chain id), broadcast of the order"}
    return out


def time_config(rw, torch, cfg, spec, count, reps=5):
    """evals/s of one config + model through rw_evaluate_batch_device (uint16
    orders resident in HBM, CUDA events on the launching stream)."""
    m = rw.fixtures.config_matrix(cfg, "fixed")
    n = m.shape[0]
    prob = rw.Problem(m)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    o = torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
    c = torch.empty(count, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(2):
        prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    prob.sync_errors()
    return count * reps / (e0.elapsed_time(e1) / 1000.0)


def run_config_extras(rw, torch):
    """Per-config evaluation throughput and C3 local search."""
    A, S = rw.Algorithm, rw.fixtures.SIZE_FIXED
    ref_1t = {"C3_ring": 6.15e4, "C3_dbt": 1.35e5, "C5_hd_xor": 1.16e3, "C5_hd_paper": 1.92e3}  # SURVEY 8(d) [measured]
    rows = {
        "C3_ring": ("C3", rw.CollectiveSpec(A.Ring, 256, S), 1 << 21),
        "C3_dbt": ("C3", rw.CollectiveSpec(A.DoubleBinaryTree, 256, S), 1 << 19),
        "C5_hd_xor": ("C5", rw.CollectiveSpec(A.HalvingDoubling, 4096, S, 2, rw.CostMode.LatencyTimesSize,
                                              rw.HdPairing.XorPairing), 1 << 15),
        "C5_hd_paper": ("C5", rw.CollectiveSpec(A.HalvingDoubling, 4096, S), 1 << 15),
    }
    out = {"unit": "evals/s", "orders": "uint16, device resident", "reference_single_thread_container": ref_1t}
    for k, (cfg, spec, count) in rows.items():
        out[k] = time_config(rw, torch, cfg, spec, count)
    # batched local search to a swap/2-opt local optimum, C3, 148 random orders
    import numpy as np
    rng = np.random.default_rng(3)
    m3 = rw.fixtures.config_matrix("C3", "fixed")
    p3 = rw.Problem(m3)
    starts = np.array([rng.permutation(256) for _ in range(148)], dtype=np.int32)
    ls = {}
    for name, spec in (("ring", rw.CollectiveSpec(A.Ring, 256, S)), ("dbt", rw.CollectiveSpec(A.DoubleBinaryTree, 256, S))):
        t = time.perf_counter()
        orders, costs, evals = p3.local_search(spec, starts, max_rounds=1_000_000)
        dt = time.perf_counter() - t
        ls[name] = {"orders": len(starts), "seconds": dt, "move_evaluations": int(evals),
                    "move_evaluations_per_s": evals / dt, "mean_cost": float(costs.mean()),
                    "start_mean_cost": float(p3.evaluate_batch(spec, starts).mean())}
    out["local_search_c3"] = ls
    return out


def run_extras(rw, torch):
    """Secondary north-star numbers (single GPU, small): exhaustive N=13 and C1 time-to-best-ring."""
    out = {}
    out["configs"] = run_config_extras(rw, torch)
    m13 = rw.fixtures.config_matrix("C2")
    M13 = rw.CostMatrix.from_array(m13)
    spec13 = rw.CollectiveSpec(rw.Algorithm.Ring, 13, 1.0)
    rw.brute_force(M13, spec13, threshold=13)  # warm
    t = time.perf_counter()
    sol = rw.brute_force(M13, spec13, threshold=13)
    out["exhaustive_n13"] = {"seconds": time.perf_counter() - t, "cost": sol.cost, "order": sol.order.perm,
                             "evaluations": sol.evaluations, "reference_seconds_container": 180.8,
                             "golden_cost": 338.0}
    gpath = os.path.join(ROOT, "tests", "golden", "anneal.json")
    if os.path.exists(gpath):
        g = json.load(open(gpath))
        ref = [r for r in g["results"] if r["config"] == "C1"]
        target = min(r["cost"] for r in ref)
        m = rw.fixtures.config_matrix("C1", "fixed")
        prob = rw.Problem(m)
        spec = rw.fixtures.ring_spec(64, rw.fixtures.SIZE_FIXED)
        best = None
        t = time.perf_counter()
        for steps in (16, 64, 256, 1024):
            t1 = time.perf_counter()
            order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                               schedule="calibrated")
            best = (cost, steps, ev, time.perf_counter() - t1, rep["chains"])
            if cost <= target:
                break
        out["time_to_best_ring_c1"] = {"seconds_cumulative": time.perf_counter() - t, "seconds_last_run": best[3],
                                       "target_reference_min_seeds0_9": target, "reached": best[0] <= target,
                                       "cost": best[0], "steps_per_level": best[1], "evaluations": best[2],
                                       "chains": best[4],
                                       "reference_seconds_per_run_container": statistics.median(r["seconds"] for r in ref)}
    gpath4 = os.path.join(ROOT, "tests", "golden", "anneal_c4.json")
    if os.path.exists(gpath4):
        g = json.load(open(gpath4))
        ref = g["results"]
        target = min(r["cost"] for r in ref)
        m = rw.fixtures.config_matrix("C4", "fixed")
        prob = rw.Problem(m)
        spec = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
        best = None
        t = time.perf_counter()
        for steps in (1024, 2048, 4096, 8192, 16384):
            t1 = time.perf_counter()
            order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                               chains=C4_CHAINS, schedule="calibrated")
            best = (cost, steps, ev, time.perf_counter() - t1, rep["chains"])
            if cost <= target:
                break
        out["time_to_best_ring_c4"] = {"seconds_cumulative": time.perf_counter() - t, "seconds_last_run": best[3],
                                       "target_reference_min_seeds0_3": target, "reached": best[0] <= target,
                                       "cost": best[0], "identity_cost": ref[0]["identity_cost"],
                                       "steps_per_level": best[1], "evaluations": best[2], "chains": best[4],
                                       "reference_seconds_per_run_container": statistics.median(r["seconds"] for r in ref)}
    dbt = [r for r in json.load(open(gpath))["results"] if r["config"] == "C3" and r["model"] == "dbt"] \
        if os.path.exists(gpath) else []
    if dbt:
        target = dbt[0]["cost"]
        p3 = rw.Problem(rw.fixtures.config_matrix("C3", "fixed"))
        spec3 = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
        best = None
        t = time.perf_counter()
        for steps in (64, 128, 256, 512):
            t1 = time.perf_counter()
            order, cost, ev, rep = p3.anneal(spec3, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                             chains=C4_CHAINS)
            best = (cost, steps, ev, time.perf_counter() - t1, rep["chains"])
            if cost <= target:
                break
        out["time_to_best_dbt_c3"] = {"seconds_cumulative": time.perf_counter() - t, "seconds_last_run": best[3],
                                      "target_reference_seed0": target, "reached": best[0] <= target,
                                      "cost": best[0], "steps_per_level": best[1], "evaluations": best[2],
                                      "chains": best[4], "reference_seconds_per_run_container": dbt[0]["seconds"]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=120)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--e2e-batch", type=int, default=E2E_BATCH)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
