#!/usr/bin/env python3
"""Benchmark: permutation cost evaluations/s (U1 = one reference evaluate()).

Workload (BASELINE.json target: ">= 100x the host CPU in permutation
evaluations/sec on one B200 for N=1024 ring cost"): config C4 -- the
1024-host synthetic hierarchical matrix (fixtures.py, fixed-point variant so
every cost is bit-exact vs the reference), ring all-reduce cost model.  A step
scores one batch of random orders that is resident in HBM (32 GiB of uint16
orders per GPU, far larger than the 126 MB L2), with the per-order bijection
check on, exactly as the reference's evaluate() validates every order.

Arms
  (default)          our CUDA path; one process per GPU under torchrun, each
                     GPU scores its own batch (weak scaling, no collective in
                     the data path), time = max over ranks of CUDA-event time.
  --impl reference   the reference's own evaluate() (oracle/_ref, compiled from
                     the unmodified sources) on all host threads, rank 0 only.

Extra keys: roofline (dominant kernel, against its binding level -- random
shared-memory accesses -- with the HBM algorithmic-bytes view beside it),
cpu_baseline, e2e (host buffers through the C ABI, H2D/D2H inside every step;
packed, uint16 and int32 wire layouts), clocks (NVML, sampled during the
timed region), gpu_launches, and `extras` (N=13 exhaustive time,
time-to-best-ring, FP32/FP64 storage paths, the reference's searches timed in
the same run).
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
BATCH = 1 << 24  # orders per GPU per step: 16 Mi x 1024 x 2 B = 32 GiB of uint16 orders in HBM (~24 ms/step)
E2E_BATCH = 1 << 18  # orders per e2e step (host buffers through the C ABI)
C4_CHAINS = 592  # time-to-best-ring at C4: 4 chains (warps) per SM, the fastest per chain; DESIGN.md 5
CPU_SECONDS = 10.0


def bench_config(world: int) -> dict:
    """The workload both arms report (identical dicts: the driver compares them)."""
    return {"workload": WORKLOAD, "n": N, "model": "ring", "matrix": "C4 fixed point (bit-exact)",
            "orders_per_gpu_per_step": BATCH, "order_bytes_in_hbm": BATCH * N * 2,
            "l2_policy": "inputs larger than L2 (2 B x N x batch per step)",
            "validation": "bijection check on every order", "parallelism": f"dp{world} (independent batches)"}


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clock and clock-event reasons sampled through NVML every `period`
    seconds on a background thread while the timed region runs (nvidia-smi's
    100 ms loop is too coarse for a sub-second region)."""
    REASONS = (("sw_power_cap", 0x4), ("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, cuda_index: int, period: float = 0.004):
        self.cuda_index = cuda_index
        self.period = period
        self.samples = []
        self.error = None
        self._stop = threading.Event()
        self._t = None

    def _handle(self, nv):
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = self._handle(nv)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # no NVML: report it instead of failing the run
            self.error = f"NVML unavailable: {e}"
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception as e:
                self.error = str(e)
                return
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "error": self.error or "no samples"}
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "sm_mhz_min": min(sm), "period_ms": self.period * 1e3, "source": "NVML"}


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


def reference_matrix(name: str, kind: str = "fixed") -> np.ndarray:
    """BASELINE config matrix built by the reference library alone (no product import)."""
    from oracle.pyoracle import Reference, reference_available, reference_config_matrix
    if not reference_available():
        raise RuntimeError("oracle/_ref is missing")
    return reference_config_matrix(Reference(), name, kind)


def reference_search_same_run():
    """The reference's searches timed on this box in this run (single thread,
    as shipped): ring brute force at N=12 on the C2 block (11! orders) and
    the C1 anneal at seed 0 (default schedule, 2,823,272 evaluations)."""
    from oracle.pyoracle import Reference, make_spec
    ref = Reference()
    out = {}
    m13 = reference_matrix("C2")
    t = time.perf_counter()
    perm, cost, ev = ref.brute_force(np.ascontiguousarray(m13[:12, :12]), make_spec(0, 12, 1.0), threshold=12)
    out["brute_force_n12"] = {"seconds": time.perf_counter() - t, "cost": cost, "evaluations": ev,
                              "order": perm.tolist(), "threads": 1}
    m1 = reference_matrix("C1", "fixed")
    t = time.perf_counter()
    perm, cost, ev = ref.anneal(m1, make_spec(0, 64, float(2 ** 27)), budget_s=1e6, seed=0)
    out["anneal_c1_seed0"] = {"seconds": time.perf_counter() - t, "cost": cost, "evaluations": ev, "threads": 1}
    return out


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    m = reference_matrix("C4", "fixed")
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
            "config": bench_config(world),
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

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    m = rw.fixtures.config_matrix("C4", "fixed")
    prob = rw.Problem(m, device=local)
    spec = rw.fixtures.ring_spec(N, rw.fixtures.SIZE_FIXED)
    batch = args.batch
    orders = make_orders_device(torch, batch, N, seed=1234 + rank)
    costs = torch.empty(batch, dtype=torch.float64, device="cuda")
    # One side stream for warm-up, capture and replay: the library's
    # stream-ordered scratch for this stream is then sized before capture.
    stream = torch.cuda.Stream()

    def step(p=prob, st=None):
        p.evaluate_batch_device(spec, orders.data_ptr(), 2, batch, costs.data_ptr(), (st or stream).cuda_stream)

    with torch.cuda.stream(stream):
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
    with torch.cuda.graph(graph, stream=stream):
        step()
    graph.replay()
    torch.cuda.synchronize()
    prob.sync_errors()
    launches_per_step = graph_kernel_nodes(graph)

    # ---- timed region: device-resident orders (value) ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for k in range(args.steps):
                graph.replay()
                ev[k + 1].record(stream)
        barrier()
    prob.sync_errors()
    per_launch_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    max_ms = max_over_ranks(total_ms)
    value = world * batch * args.steps / (max_ms / 1000.0)

    def time_path(path, reps=10, count=1 << 21):
        alt = rw.Problem(m, device=local)
        alt.set_path(path)
        cst = torch.cuda.current_stream()

        def run():
            alt.evaluate_batch_device(spec, orders.data_ptr(), 2, count, costs.data_ptr(), cst.cuda_stream)
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cst)
        for _ in range(reps):
            run()
        e1.record(cst)
        torch.cuda.synchronize()
        alt.sync_errors()
        return count * reps / (e0.elapsed_time(e1) / 1000.0)

    # ---- e2e: host orders through the C ABI (H2D + D2H inside every step) ----
    e2e = run_e2e(rw, torch, args, prob, spec, orders, barrier, max_over_ranks, world, local)

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
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    bytes_per_eval = 2 * N + N * 2 + 8  # order read + L*e lookups (u16) + cost write
    launch_ms = statistics.mean(per_launch_ms)
    hbm_achieved = bytes_per_eval * batch / (launch_ms / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        bpo = json.load(open(tpath)).get("bytes_per_order")
        traffic = bpo * batch if bpo else None  # DRAM bytes per bench step (one graph replay), from ncu
    clock = clocks.summary()
    # The binding level: shared-memory random accesses -- one random 2-byte
    # scatter (route) and one random 2-byte gather (score) per hop -- against
    # the measured random-access peak (profiles/gather_peaks.json,
    # scripts/microbench/gather_peaks.cu).  ncu: both passes at 90-91% L1TEX.
    gp = json.load(open(os.path.join(ROOT, "profiles", "gather_peaks.json")))
    smem_peak = gp["smem_random_u16_lookups_per_s"]
    acc_per_s = 2 * N * batch / (launch_ms / 1000.0)

    cpu_value, cpu_info = (None, {"kind": "skipped", "cores": 0, "sample": "--no-cpu"})
    if not args.no_cpu:
        cpu_value, cpu_info = cpu_reference_rate(m, CPU_SECONDS, os.cpu_count() or 1)

    extras = {}
    if not args.no_extras:
        extras = run_extras(rw, torch)
        extras["storage_kinds"] = run_storage_extras(rw, torch, hbm_peak)
        if not args.no_cpu:
            extras["reference_search_same_run"] = reference_search_same_run()
        # A/B: the same orders through the alternative ring kernels (not the default path)
        extras["ring_kernel_ab"] = {
            "unit": UNIT, "orders": 1 << 21,
            "transpose_default": time_path("auto"),
            "l2_gather": time_path("l2"),
            "cluster_dsmem": time_path("cluster"),
            "note": "l2_gather: one warp per order, random sector gathers (L1TEX-wavefront bound); "
                    "cluster_dsmem: rows split over a 16-CTA cluster, hops routed by DSMEM stores "
                    "(DSMEM-transaction bound) -- DESIGN.md 4"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": bench_config(world),
        "roofline": {"bound": "smem", "achieved": acc_per_s / 1e9, "peak": smem_peak / 1e9,
                     "unit": "G random shared-memory accesses/s", "frac": acc_per_s / smem_peak,
                     "traffic": traffic, "peak_source": "measured (profiles/gather_peaks.json: random 2-byte "
                                                        "shared-memory accesses, all SMs)",
                     "kernel": "k_ring_route + k_ring_score (transpose ring path, one pair per 262,144-order chunk)",
                     "accesses_per_eval": 2 * N,
                     "hbm": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                             "frac": hbm_achieved / hbm_peak, "peak_source": peak_src,
                             "algorithmic_bytes_per_eval": bytes_per_eval,
                             "note": "SURVEY 8(d) algorithmic bytes (2N order + N x 2 B lookups + 8 B cost) per "
                                     "evaluation over the step's CUDA-event time"},
                     "note": "the lookups are served from shared memory (route scatter + score gather: 2 random "
                             "accesses per hop); both passes run at 90-91% of L1TEX throughput (ncu, profiles/). "
                             "The predecessor exchange buffer (2N B per order) is written and re-read through "
                             "HBM; `traffic` is the ncu DRAM bytes per step -- DESIGN.md 4, 7"},
        "cpu_baseline": dict(cpu_info, value=cpu_value, unit=UNIT),
        "e2e": e2e,
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


def run_e2e(rw, torch, args, prob, spec, orders, barrier, max_over_ranks, world, local):
    """The metric through the public C ABI with HOST buffers: every step copies
    that step's orders host -> device (pinned memory) and reads the costs back.
    Three wire layouts of the same orders: packed (10 bits per host at N=1024,
    rw_evaluate_batch_packed -- the headline), uint16 (rw_evaluate_batch_u16)
    and int32 (rw_evaluate_batch, the reference's RankOrder element type)."""
    import ctypes as C
    from paper_2105_14088_b200 import _lib
    eb = args.e2e_batch
    host16 = orders[:eb].cpu().numpy().view(np.uint16)
    bits = rw.api.packed_bits(N)
    variants = {
        "packed": (torch.from_numpy(rw.api.pack_orders(host16.astype(np.int32), bits)).pin_memory(),
                   rw.api.packed_row_bytes(N, bits)),
        "u16": (torch.from_numpy(host16.copy().view(np.int16)).pin_memory(), 2 * N),
        "int32": (torch.from_numpy(host16.astype(np.int32)).pin_memory(), 4 * N),
    }
    costs_t = torch.empty(eb, dtype=torch.float64).pin_memory()
    cptr = C.cast(costs_t.data_ptr(), C.POINTER(C.c_double))
    cs = spec._c()

    def call(kind, buf):
        if kind == "packed":
            return _lib.lib.rw_evaluate_batch_packed(prob.handle, C.byref(cs), C.c_void_p(buf.data_ptr()), bits, eb,
                                                     cptr, 0, None)
        if kind == "u16":
            return _lib.lib.rw_evaluate_batch_u16(prob.handle, C.byref(cs), C.cast(buf.data_ptr(),
                                                  C.POINTER(C.c_uint16)), eb, cptr, 0, None)
        return _lib.lib.rw_evaluate_batch(prob.handle, C.byref(cs), C.cast(buf.data_ptr(), C.POINTER(C.c_int32)),
                                          eb, cptr, 0, None)

    steps = max(3, min(args.steps, 20))
    out = {}
    ref_costs = None
    for kind, (buf, row) in variants.items():
        for _ in range(2):
            _lib.check(call(kind, buf))
        got = costs_t.numpy().copy()
        if ref_costs is None:
            ref_costs = got
        assert np.array_equal(got, ref_costs), f"e2e {kind}: costs differ between wire layouts"
        barrier()
        with ClockSampler(local, period=0.01) as clk:
            t0 = time.perf_counter()
            for _ in range(steps):
                _lib.check(call(kind, buf))
            dt = time.perf_counter() - t0
        barrier()
        dt = max_over_ranks(dt)
        out[kind] = {"value": world * eb * steps / dt, "unit": UNIT, "steps": steps, "orders_per_step": eb,
                     "h2d_bytes_per_step": eb * row, "d2h_bytes_per_step": eb * 8,
                     "h2d_GBps": eb * row * steps / dt / 1e9, "clocks": clk.summary()}
    head = out["packed"]
    return {"value": head["value"], "unit": UNIT, "h2d_bytes_per_step": head["h2d_bytes_per_step"],
            "d2h_bytes_per_step": head["d2h_bytes_per_step"],
            "api": f"rw_evaluate_batch_packed (C ABI; pinned host orders, {bits} bits per host, "
                   f"{rw.api.packed_row_bytes(N, bits)} B per order; H2D + device unpack + score + D2H of the costs "
                   f"inside every step, wall clock, max over ranks)",
            "variants": out}


def run_storage_extras(rw, torch, hbm_peak):
    """A probed CostMatrix is FP64 (types.hpp:42-53): throughput of the FP32
    and FP64 storage paths a real matrix takes, next to the fixed-point one,
    with a parity assert on every case (north star: FP32 within 1e-6)."""
    from oracle.pyoracle import Port, make_spec
    port = Port()
    A, P = rw.Algorithm, rw.HdPairing
    cases = [("C4", "ring", 0, 0, 1 << 21), ("C5", "hd_xor", 1, 1, 1 << 15), ("C5", "hd_paper", 1, 0, 1 << 15)]
    names = {1: "u16", 2: "f32", 3: "f64"}
    out = {"unit": "evals/s", "orders": "uint16, device resident"}
    for cfg, model, alg, pair, count in cases:
        for kind in ("fixed", "f32", "f64"):
            m = rw.fixtures.config_matrix(cfg, kind)
            n = m.shape[0]
            size = rw.fixtures.size_for(kind)
            spec = rw.CollectiveSpec(A(alg), n, size, 2, rw.CostMode.LatencyTimesSize, P(pair))
            prob = rw.Problem(m)
            g = torch.Generator(device="cuda")
            g.manual_seed(5)
            o = torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
            c = torch.empty(count, dtype=torch.float64, device="cuda")
            st = torch.cuda.current_stream()
            for _ in range(2):
                prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            prob.sync_errors()
            rows = o[:8].cpu().numpy().view(np.uint16).astype(np.int32)
            want = port.evaluate_batch(m, rows, make_spec(alg, n, size, 2, 1, pair))
            rel = float(np.max(np.abs(c[:8].cpu().numpy() - want) / np.abs(want)))
            assert rel <= (0.0 if kind == "fixed" else 1e-6), (cfg, model, kind, rel)
            reps = 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            prob.sync_errors()
            rate = count * reps / (e0.elapsed_time(e1) / 1000.0)
            e = prob.info["storage"]
            esz = {1: 2, 2: 4, 3: 8}[e]
            lookups = port.lookups(make_spec(alg, n, size, 2, 1, pair))
            alg_bytes = 2 * n + lookups * esz + 8
            out[f"{cfg}_{model}_{kind}"] = {
                "storage": names[e], "evals_per_s": rate, "max_rel_err_vs_oracle": rel,
                "roofline_hbm": {"algorithmic_bytes_per_eval": alg_bytes, "achieved_GBps": rate * alg_bytes / 1e9,
                                 "frac": rate * alg_bytes / 1e9 / hbm_peak}}
            del prob, o, c
            torch.cuda.empty_cache()
    return out


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
    # time-to-best-ring on this run's GPUs: 592 chains per GPU (4 per SM, the
    # fastest per chain), split over the ranks; escalate the steps per level
    # until the incumbent beats the reference's best run (max over ranks).
    tt = {"target_reference_min_seeds0_3": target, "chains_total": C4_CHAINS * world, "n_gpus": world,
          "reached": False}
    barrier()
    t0 = time.perf_counter()
    for steps in (512, 1024, 2048, 4096, 8192, 16384):
        s2, r2 = rwd.anneal_sharded(prob4, spec4, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                    C4_CHAINS * world, schedule="calibrated")
        tt.update({"cost": s2.cost, "steps_per_level": steps, "evaluations": s2.evaluations})
        if s2.cost <= target:
            tt["reached"] = True
            break
    barrier()
    tt["seconds_cumulative"] = max_over_ranks(time.perf_counter() - t0)
    out["time_to_best_ring_c4"] = tt
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
        "C5_bcube4": ("C5", rw.CollectiveSpec(A.BCube, 4096, S, 4), 1 << 15),
        "C5_bcube8": ("C5", rw.CollectiveSpec(A.BCube, 4096, S, 8), 1 << 15),
        "C5_dbt": ("C5", rw.CollectiveSpec(A.DoubleBinaryTree, 4096, S), 1 << 15),
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
