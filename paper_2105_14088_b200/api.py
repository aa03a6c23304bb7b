"""Python mirror of the rankweave solver API (proj/include/rankweave/*.hpp).

The reference ships no Python binding (proj/python/CMakeLists.txt:1 is a
placeholder), so this module mirrors the C++ names one to one -- CostMatrix,
RankOrder, CollectiveSpec, evaluate, ring_cost, ..., brute_force, anneal,
two_stage_solve, sample_costs, distribution_stats -- with NumPy arrays in and
out, plus batch entry points.  Every cost is computed by librankweave_b200.so
on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import DomainError, IOError_, RankweaveError, check, lib, ptr

domain_error = DomainError
io_error = IOError_


class Algorithm(enum.IntEnum):
    Ring = 0
    HalvingDoubling = 1
    DoubleBinaryTree = 2
    BCube = 3


class CostMode(enum.IntEnum):
    LatencyOnly = 0
    LatencyTimesSize = 1


class HdPairing(enum.IntEnum):
    PaperFormula = 0
    XorPairing = 1


class SolveMethod(enum.IntEnum):
    BruteForce = 0
    Anneal = 1
    External = 2


class ScheduleSemantics(enum.IntEnum):
    SequentialHops = 0
    BulkSynchronousRounds = 1
    CriticalPath = 2


_ALGO_NAMES = {"ring": Algorithm.Ring, "hd": Algorithm.HalvingDoubling, "dbt": Algorithm.DoubleBinaryTree,
               "bcube": Algorithm.BCube}


def to_string(v) -> str:
    if isinstance(v, Algorithm):
        return {v2: k for k, v2 in _ALGO_NAMES.items()}[v]
    if isinstance(v, CostMode):
        return "latency" if v == CostMode.LatencyOnly else "latency-size"
    if isinstance(v, HdPairing):
        return "paper" if v == HdPairing.PaperFormula else "xor"
    if isinstance(v, SolveMethod):
        return v.name
    raise TypeError(f"no string form for {v!r}")


def algorithm_from_string(s: str) -> Algorithm:
    if s not in _ALGO_NAMES:
        raise DomainError(f"unknown algorithm '{s}' (expected ring|hd|dbt|bcube)")
    return _ALGO_NAMES[s]


# --------------------------------------------------------------------------
class Problem:
    """A cost matrix resident on one GPU (the C ABI's rw_problem)."""

    def __init__(self, rtt_us: np.ndarray, storage: int = _lib.RW_STORAGE_AUTO, device: int = -1):
        m = np.ascontiguousarray(rtt_us, dtype=np.float64)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise DomainError("matrix is not square")
        self.n = int(m.shape[0])
        h = C.c_void_p()
        check(lib.rw_problem_create(ptr(m, C.c_double), self.n, storage, device, C.byref(h)))
        self._h = h
        info = _lib.rw_problem_info()
        check(lib.rw_problem_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in info._fields_}

    @property
    def handle(self):
        return self._h

    def set_path(self, path: str) -> None:
        """Ring kernel path for matrices beyond one CTA's shared memory (A/B measurements):
        'auto' (default), 'l2' (random L2 gathers), 'cluster' (DSMEM routing), 'transpose'."""
        check(lib.rw_problem_set_path(self._h, {"auto": 0, "l2": 1, "cluster": 2, "transpose": 3}[path]))

    def set_resident(self, idle_us: int) -> None:
        """Serve single-order evaluate() calls from a resident CTA on the device
        (no kernel launch per call) that leaves after idle_us without a call;
        0 stops it (rw_problem_set_resident)."""
        check(lib.rw_problem_set_resident(self._h, int(idle_us)))

    def close(self):
        if getattr(self, "_h", None):
            lib.rw_problem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def evaluate(self, spec: "CollectiveSpec", perm) -> float:
        """One order through rw_evaluate (the reference's evaluate(); served by
        the resident evaluator when set_resident is on)."""
        p = np.ascontiguousarray(perm, dtype=np.int32)
        out = C.c_double()
        check(lib.rw_evaluate(self._h, C.byref(spec._c()), ptr(p, C.c_int32), C.byref(out)))
        return out.value

    # batch scoring ---------------------------------------------------------
    def evaluate_batch(self, spec: "CollectiveSpec", orders: np.ndarray, exact: bool = False,
                       validate: bool = True, report: Optional[dict] = None) -> np.ndarray:
        """(B, n) host orders -> B costs.  uint16 arrays go through
        rw_evaluate_batch_u16 (half the host-to-device bytes); anything else
        as int32 through rw_evaluate_batch."""
        u16 = isinstance(orders, np.ndarray) and orders.dtype == np.uint16
        o = np.ascontiguousarray(orders, dtype=np.uint16 if u16 else np.int32)
        if o.ndim == 1:
            o = o[None, :]
        if o.shape[1] != spec.n:
            raise DomainError(f"rank order has {o.shape[1]} entries, expected {spec.n}")
        out = np.empty(o.shape[0], dtype=np.float64)
        flags = (_lib.RW_EVAL_EXACT if exact else 0) | (0 if validate else _lib.RW_EVAL_NO_VALIDATE)
        rep = _lib.rw_eval_report()
        if u16:
            check(lib.rw_evaluate_batch_u16(self._h, C.byref(spec._c()), ptr(o, C.c_uint16), o.shape[0],
                                            ptr(out, C.c_double), flags, C.byref(rep)))
        else:
            check(lib.rw_evaluate_batch(self._h, C.byref(spec._c()), ptr(o, C.c_int32), o.shape[0],
                                        ptr(out, C.c_double), flags, C.byref(rep)))
        if report is not None:
            report.update({f: getattr(rep, f) for f, _ in rep._fields_})
        return out

    def evaluate_batch_packed(self, spec: "CollectiveSpec", packed: np.ndarray, bits: int, batch: int,
                              exact: bool = False, validate: bool = True) -> np.ndarray:
        """Packed host orders (pack_orders) -> costs through rw_evaluate_batch_packed."""
        row = packed_row_bytes(spec.n, bits)
        p = np.ascontiguousarray(packed)
        if p.nbytes < row * batch:
            raise DomainError(f"packed buffer holds {p.nbytes} bytes, need {row * batch}")
        out = np.empty(batch, dtype=np.float64)
        flags = (_lib.RW_EVAL_EXACT if exact else 0) | (0 if validate else _lib.RW_EVAL_NO_VALIDATE)
        check(lib.rw_evaluate_batch_packed(self._h, C.byref(spec._c()), C.c_void_p(p.ctypes.data), bits, batch,
                                           ptr(out, C.c_double), flags, None))
        return out

    def evaluate_batch_device(self, spec: "CollectiveSpec", d_orders: int, perm_bytes: int, batch: int,
                              d_costs: int, stream: int = 0, exact: bool = False, validate: bool = True) -> None:
        """Device-pointer variant (e.g. torch tensors' data_ptr()); asynchronous on `stream`."""
        flags = (_lib.RW_EVAL_EXACT if exact else 0) | (0 if validate else _lib.RW_EVAL_NO_VALIDATE)
        check(lib.rw_evaluate_batch_device(self._h, C.byref(spec._c()), C.c_void_p(d_orders), perm_bytes, batch,
                                           C.c_void_p(d_costs), C.c_void_p(stream), flags))

    def sync_errors(self, stream: int = 0) -> None:
        check(lib.rw_sync_errors(self._h, C.c_void_p(stream)))

    def brute_force_range(self, spec: "CollectiveSpec", first: int, count: int):
        c = C.c_double()
        i = C.c_uint64()
        check(lib.rw_brute_force_range(self._h, C.byref(spec._c()), first, count, C.byref(c), C.byref(i)))
        return c.value, i.value

    def local_search(self, spec: "CollectiveSpec", orders: np.ndarray, max_rounds: int = 1000):
        o = np.ascontiguousarray(orders, dtype=np.int32).copy()
        if o.ndim == 1:
            o = o[None, :]
        costs = np.empty(o.shape[0], dtype=np.float64)
        ev = C.c_uint64()
        check(lib.rw_local_search(self._h, C.byref(spec._c()), ptr(o, C.c_int32), o.shape[0], max_rounds,
                                  ptr(costs, C.c_double), C.byref(ev)))
        return o, costs, ev.value

    def anneal(self, spec: "CollectiveSpec", cfg: "SolverConfig", chains: int = 0, chain_begin: int = 0,
               chain_total: int = 0, max_proposals: int = 0, schedule: str = "reference"):
        """schedule: 'reference' (T0 = stddev of random costs, floor T0*1e-6) or
        'calibrated' (ring: temperatures from sampled 2-opt deltas)."""
        order = np.empty(spec.n, dtype=np.int32)
        cost = C.c_double()
        ev = C.c_uint64()
        rep = _lib.rw_search_report()
        g = _lib.rw_gpu_config(chains, chain_begin, chain_total, {"reference": 0, "calibrated": 1}[schedule],
                               max_proposals)
        check(lib.rw_anneal(self._h, C.byref(spec._c()), C.byref(cfg._c()), C.byref(g), ptr(order, C.c_int32),
                            C.byref(cost), C.byref(ev), C.byref(rep)))
        return order, cost.value, ev.value, {f: getattr(rep, f) for f, _ in rep._fields_}


class ProblemSet:
    """A cost matrix replicated on several GPUs of this process with an
    in-process NCCL communicator (the C ABI's rw_problem_set): sharded batch
    scoring, exhaustive search and annealing, reduced with NCCL."""

    def __init__(self, rtt_us: np.ndarray, devices: Optional[Sequence[int]] = None,
                 storage: int = _lib.RW_STORAGE_AUTO):
        m = np.ascontiguousarray(rtt_us, dtype=np.float64)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise DomainError("matrix is not square")
        self.n = int(m.shape[0])
        devs = np.asarray(list(devices) if devices is not None else [], dtype=np.int32)
        h = C.c_void_p()
        check(lib.rw_problem_set_create(ptr(m, C.c_double), self.n, storage,
                                        ptr(devs, C.c_int32) if devs.size else None, int(devs.size), C.byref(h)))
        self._h = h
        k = C.c_int32()
        check(lib.rw_problem_set_devices(self._h, C.byref(k), None))
        out = np.empty(k.value, dtype=np.int32)
        check(lib.rw_problem_set_devices(self._h, C.byref(k), ptr(out, C.c_int32)))
        self.devices = out.tolist()

    def close(self):
        if getattr(self, "_h", None):
            lib.rw_problem_set_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def evaluate_batch(self, spec: "CollectiveSpec", orders: np.ndarray, exact: bool = False,
                       validate: bool = True) -> np.ndarray:
        u16 = isinstance(orders, np.ndarray) and orders.dtype == np.uint16
        o = np.ascontiguousarray(orders, dtype=np.uint16 if u16 else np.int32)
        if o.ndim == 1:
            o = o[None, :]
        if o.shape[1] != spec.n:
            raise DomainError(f"rank order has {o.shape[1]} entries, expected {spec.n}")
        out = np.empty(o.shape[0], dtype=np.float64)
        flags = (_lib.RW_EVAL_EXACT if exact else 0) | (0 if validate else _lib.RW_EVAL_NO_VALIDATE)
        check(lib.rw_evaluate_batch_set(self._h, C.byref(spec._c()), C.c_void_p(o.ctypes.data), 2 if u16 else 4, 0,
                                        o.shape[0], ptr(out, C.c_double), flags))
        return out

    def evaluate_batch_packed(self, spec: "CollectiveSpec", packed: np.ndarray, bits: int, batch: int,
                              exact: bool = False, validate: bool = True) -> np.ndarray:
        """Packed host orders (pack_orders), one slice per device."""
        p = np.ascontiguousarray(packed)
        if p.nbytes < packed_row_bytes(spec.n, bits) * batch:
            raise DomainError("packed buffer too small")
        out = np.empty(batch, dtype=np.float64)
        flags = (_lib.RW_EVAL_EXACT if exact else 0) | (0 if validate else _lib.RW_EVAL_NO_VALIDATE)
        check(lib.rw_evaluate_batch_set(self._h, C.byref(spec._c()), C.c_void_p(p.ctypes.data), 0, bits, batch,
                                        ptr(out, C.c_double), flags))
        return out

    def brute_force(self, spec: "CollectiveSpec", threshold: int = 10) -> "Solution":
        perm = np.empty(spec.n, dtype=np.int32)
        cost = C.c_double()
        ev = C.c_uint64()
        check(lib.rw_brute_force_set(self._h, C.byref(spec._c()), threshold, ptr(perm, C.c_int32), C.byref(cost),
                                     C.byref(ev)))
        return Solution(RankOrder(perm.tolist()), cost.value, SolveMethod.BruteForce, ev.value)

    def anneal(self, spec: "CollectiveSpec", cfg: "SolverConfig", chains: int = 0, max_proposals: int = 0,
               schedule: str = "reference"):
        order = np.empty(spec.n, dtype=np.int32)
        cost = C.c_double()
        ev = C.c_uint64()
        rep = _lib.rw_search_report()
        g = _lib.rw_gpu_config(chains, 0, 0, {"reference": 0, "calibrated": 1}[schedule], max_proposals)
        check(lib.rw_anneal_set(self._h, C.byref(spec._c()), C.byref(cfg._c()), C.byref(g), ptr(order, C.c_int32),
                                C.byref(cost), C.byref(ev), C.byref(rep)))
        return order, cost.value, ev.value, {f: getattr(rep, f) for f, _ in rep._fields_}


class CostMatrix:
    """N x N pairwise costs in microseconds (types.hpp:42-53).

    The matrix array is read-only so the device copy attached to it can be
    reused safely; use copy() / with_entry() to derive modified matrices."""

    def __init__(self, hosts: Sequence[str], rows):
        arr = np.array(rows, dtype=np.float64)
        hosts = list(hosts)
        if arr.ndim != 2 or arr.shape[0] != len(hosts):
            raise DomainError(f"matrix has {arr.shape[0] if arr.ndim else 0} rows for {len(hosts)} hosts")
        if arr.shape[1] != len(hosts):
            raise DomainError("matrix is not square")
        arr.setflags(write=False)
        self.hosts = hosts
        self.rtt_us = arr
        self._problem: Optional[Problem] = None

    @classmethod
    def from_array(cls, arr, hosts: Optional[Sequence[str]] = None) -> "CostMatrix":
        arr = np.asarray(arr, dtype=np.float64)
        return cls(hosts or [f"h{i}" for i in range(arr.shape[0])], arr)

    def n(self) -> int:
        return len(self.hosts)

    def at(self, i: int, j: int) -> float:
        return float(self.rtt_us[i, j])

    def rows(self):
        return self.rtt_us.tolist()

    def copy(self) -> "CostMatrix":
        return CostMatrix(self.hosts, self.rtt_us.copy())

    def with_entry(self, i: int, j: int, value: float) -> "CostMatrix":
        a = self.rtt_us.copy()
        a[i, j] = value
        return CostMatrix(self.hosts, a)

    def problem(self) -> Problem:
        if self._problem is None:
            self._problem = Problem(self.rtt_us)
        return self._problem


@dataclass
class RankOrder:
    perm: List[int]

    @staticmethod
    def identity(n: int) -> "RankOrder":
        return RankOrder(list(range(n)))

    def size(self) -> int:
        return len(self.perm)


@dataclass
class CollectiveSpec:
    algorithm: Algorithm = Algorithm.Ring
    n: int = 0
    size_bytes: float = 0.0
    bcube_b: int = 2
    cost_mode: CostMode = CostMode.LatencyTimesSize
    hd_pairing: HdPairing = HdPairing.PaperFormula

    def _c(self) -> _lib.rw_spec:
        return _lib.rw_spec(int(self.algorithm), int(self.n), float(self.size_bytes), int(self.bcube_b),
                            int(self.cost_mode), int(self.hd_pairing))


@dataclass
class SolverConfig:
    budget: float = 10.0  # seconds
    seed: int = 0
    initial_temperature: float = 0.0
    cooling: float = 0.995
    steps_per_temperature: int = 0
    restarts: int = 4
    brute_force_threshold: int = 10

    def _c(self) -> _lib.rw_solver_config:
        return _lib.rw_solver_config(float(self.budget), int(self.seed), float(self.initial_temperature),
                                     float(self.cooling), int(self.steps_per_temperature), int(self.restarts),
                                     int(self.brute_force_threshold), 0)


@dataclass
class Solution:
    order: RankOrder = field(default_factory=lambda: RankOrder([]))
    cost: float = 0.0
    method: SolveMethod = SolveMethod.BruteForce
    evaluations: int = 0


@dataclass
class DistributionStats:
    min: float = 0.0
    max: float = 0.0
    mean: float = 0.0
    stddev: float = 0.0
    count: int = 0


# ------------------------------------------------------------ validation ---
def validate_spec(spec: CollectiveSpec) -> None:
    check(lib.rw_validate_spec(C.byref(spec._c())))


def _order_array(order: RankOrder, n: int) -> np.ndarray:
    """validate(RankOrder, n) (types.cpp:100-110) on a NumPy copy of the order;
    returns the int32 array the C ABI takes."""
    if order.size() != n:
        raise DomainError(f"rank order has {order.size()} entries, expected {n}")
    try:
        a = np.asarray(order.perm, dtype=np.int64)
    except (OverflowError, ValueError, TypeError):
        raise DomainError(f"rank order is not a permutation of [0, {n})")
    if n and (a.ndim != 1 or a.min() < 0 or a.max() >= n or np.bincount(a, minlength=n).max() != 1):
        raise DomainError(f"rank order is not a permutation of [0, {n})")
    return a.astype(np.int32)


def validate_order(order: RankOrder, n: int) -> None:
    _order_array(order, n)


def validate_matrix(m: CostMatrix) -> None:
    n = m.n()
    if n == 0:
        raise DomainError("cost matrix is empty")
    a = m.rtt_us
    bad = ~np.isfinite(a) | (a < 0)
    if bad.any():
        i, j = map(int, np.argwhere(bad)[0])
        raise DomainError(f"rtt[{i}][{j}] is not a finite nonnegative value")
    d = np.nonzero(np.diag(a) != 0)[0]
    if d.size:
        raise DomainError(f"rtt[{int(d[0])}][{int(d[0])}] must be 0")


def is_symmetric(m: CostMatrix) -> bool:
    return bool(np.array_equal(m.rtt_us, m.rtt_us.T))


def rotated(order: RankOrder, k: int) -> RankOrder:
    n = order.size()
    return RankOrder([order.perm[((i + k) % n + n) % n] for i in range(n)])


def inverse(order: RankOrder) -> RankOrder:
    out = [0] * order.size()
    for i, v in enumerate(order.perm):
        out[v] = i
    return RankOrder(out)


def alias_rank(r: int, n: int) -> int:
    return ((r % n) + n) % n


def round_bytes(size_bytes: float, base: int, rnd: int) -> float:
    divisor = 1.0
    for _ in range(rnd + 1):
        divisor *= float(base)
    return size_bytes / divisor


def transfer_cost(m: CostMatrix, i: int, j: int, nbytes: float, mode: CostMode) -> float:
    n = m.n()
    rtt = float(m.rtt_us[alias_rank(i, n), alias_rank(j, n)])
    return rtt if mode == CostMode.LatencyOnly else rtt * nbytes


# ------------------------------------------------------------- cost model --
def _check_inputs(m: CostMatrix, order: RankOrder, spec: CollectiveSpec) -> np.ndarray:
    validate_spec(spec)
    if m.n() != spec.n:
        raise DomainError(f"matrix is {m.n()}x{m.n()} but spec has N={spec.n}")
    return _order_array(order, spec.n)


def evaluate(m: CostMatrix, order: RankOrder, spec: CollectiveSpec) -> float:
    """evaluate (cost_model.hpp:28): reference-identical FP64 bits."""
    perm = np.ascontiguousarray(_check_inputs(m, order, spec))
    out = C.c_double()
    check(lib.rw_evaluate(m.problem().handle, C.byref(spec._c()), ptr(perm, C.c_int32), C.byref(out)))
    return out.value


def _model(m, order, spec, want: Algorithm, name: str) -> float:
    _check_inputs(m, order, spec)
    if spec.algorithm != want:
        raise DomainError(f"{name}: spec is not {to_string(want)}")
    return evaluate(m, order, spec)


def ring_cost(m, order, spec):
    return _model(m, order, spec, Algorithm.Ring, "ring_cost")


def halving_doubling_cost(m, order, spec):
    return _model(m, order, spec, Algorithm.HalvingDoubling, "halving_doubling_cost")


def double_binary_tree_cost(m, order, spec):
    return _model(m, order, spec, Algorithm.DoubleBinaryTree, "double_binary_tree_cost")


def bcube_cost(m, order, spec):
    return _model(m, order, spec, Algorithm.BCube, "bcube_cost")


def evaluate_batch(m: CostMatrix, orders: np.ndarray, spec: CollectiveSpec, exact: bool = False) -> np.ndarray:
    validate_spec(spec)
    if m.n() != spec.n:
        raise DomainError(f"matrix is {m.n()}x{m.n()} but spec has N={spec.n}")
    return m.problem().evaluate_batch(spec, orders, exact=exact)


# ----------------------------------------------------------------- solver --
def brute_force(m: CostMatrix, spec: CollectiveSpec, threshold: int = 10) -> Solution:
    validate_spec(spec)
    if spec.n > threshold:
        raise DomainError(f"N={spec.n} exceeds the brute-force threshold {threshold}; use anneal")
    if m.n() != spec.n:
        raise DomainError(f"matrix is {m.n()}x{m.n()} but spec has N={spec.n}")
    perm = np.empty(spec.n, dtype=np.int32)
    cost = C.c_double()
    ev = C.c_uint64()
    check(lib.rw_brute_force(m.problem().handle, C.byref(spec._c()), threshold, ptr(perm, C.c_int32),
                             C.byref(cost), C.byref(ev)))
    return Solution(RankOrder(perm.tolist()), cost.value, SolveMethod.BruteForce, ev.value)


def validate_config(cfg: SolverConfig) -> None:
    if not cfg.budget > 0.0:
        raise DomainError("solver budget must be > 0")
    if not (0.0 < cfg.cooling < 1.0):
        raise DomainError("cooling factor must be in (0, 1)")
    if cfg.restarts < 1:
        raise DomainError("restarts must be >= 1")
    if cfg.brute_force_threshold < 2:
        raise DomainError("brute-force threshold must be >= 2")


def anneal(m: CostMatrix, spec: CollectiveSpec, cfg: SolverConfig, chains: int = 0,
           report: Optional[dict] = None) -> Solution:
    validate_spec(spec)
    validate_config(cfg)
    if m.n() != spec.n:
        raise DomainError("matrix dimension does not match spec.n")
    order, cost, ev, rep = m.problem().anneal(spec, cfg, chains=chains)
    if report is not None:
        report.update(rep)
    return Solution(RankOrder(order.tolist()), cost, SolveMethod.Anneal, ev)


def parse_model_file(text: str, n: int) -> RankOrder:
    """parse_model_file (smtlib.hpp:22-25) through the C ABI (the C++ drop-in's code)."""
    perm = np.empty(max(n, 0), dtype=np.int32)
    check(lib.rw_parse_model_file(text.encode("utf-8"), n, ptr(perm, C.c_int32)))
    return RankOrder(perm.tolist())


def balanced_sexpr(text: str) -> bool:
    out = C.c_int32()
    check(lib.rw_balanced_sexpr(text.encode("utf-8"), C.byref(out)))
    return bool(out.value)


def emit_smtlib(m: CostMatrix, spec: CollectiveSpec, upper_bound: Optional[float] = None,
                emission_cap: int = 64) -> str:
    """emit_smtlib (smtlib.cpp:104-158): the reference's SMT-LIB text, byte for byte."""
    a = np.ascontiguousarray(m.rtt_us, dtype=np.float64)
    has = upper_bound is not None
    ub = float(upper_bound) if has else 0.0
    length = C.c_int64()
    check(lib.rw_emit_smtlib(ptr(a, C.c_double), m.n(), C.byref(spec._c()), int(has), ub, emission_cap, None, 0,
                             C.byref(length)))
    buf = C.create_string_buffer(length.value + 1)
    check(lib.rw_emit_smtlib(ptr(a, C.c_double), m.n(), C.byref(spec._c()), int(has), ub, emission_cap, buf,
                             length.value + 1, C.byref(length)))
    return buf.value.decode("utf-8")


def two_stage_solve(m: CostMatrix, spec: CollectiveSpec, cfg: SolverConfig, external_model_path: str = "",
                    log: Optional[Callable[[str], None]] = None, emit_smt_path: str = "") -> Solution:
    """two_stage_solve (solver.cpp:204-261) through the C ABI: the C++ drop-in's
    routing, SMT side file and external-model handling, unchanged."""
    a = np.ascontiguousarray(m.rtt_us, dtype=np.float64)
    perm = np.empty(max(spec.n, 0), dtype=np.int32)
    cost = C.c_double()
    method = C.c_int32()
    ev = C.c_uint64()
    cb = _lib.LOG_FN((lambda msg, _u: log(msg.decode("utf-8", "replace"))) if log else (lambda msg, _u: None))
    check(lib.rw_two_stage_solve(ptr(a, C.c_double), m.n(), C.byref(spec._c()), C.byref(cfg._c()),
                                 emit_smt_path.encode() if emit_smt_path else None,
                                 external_model_path.encode() if external_model_path else None,
                                 C.cast(cb, C.c_void_p), None, ptr(perm, C.c_int32), C.byref(cost),
                                 C.byref(method), C.byref(ev)))
    return Solution(RankOrder(perm.tolist()), cost.value, SolveMethod(method.value), ev.value)


# ------------------------------------------------------------------ stats --
def distribution_stats(values: Sequence[float]) -> DistributionStats:
    """distribution_stats (stats.cpp:64-81) through the C ABI: serial sums, population stddev."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).ravel())
    out = np.empty(4, dtype=np.float64)
    check(lib.rw_distribution_stats(ptr(v, C.c_double), v.size, ptr(out, C.c_double)))
    return DistributionStats(float(out[0]), float(out[1]), float(out[2]), float(out[3]), int(v.size))


def sample_orders(n: int, n_samples: int, seed: int) -> np.ndarray:
    """sample_orders (stats.cpp:83-94): the reference's orders for this seed
    (std::mt19937_64 + std::shuffle), one row per sample."""
    if n_samples < 1:
        raise DomainError("sample_orders: need at least 1 sample")
    out = np.empty((n_samples, max(n, 0)), dtype=np.int32)
    check(lib.rw_sample_orders(n, n_samples, seed, ptr(out, C.c_int32)))
    return out


def sample_costs(m: CostMatrix, spec: CollectiveSpec, n_samples: int, seed: int) -> np.ndarray:
    """sample_costs (stats.cpp:96-103): the reference's orders, scored on the GPU."""
    if n_samples < 1:
        raise DomainError("sample_orders: need at least 1 sample")
    validate_spec(spec)
    if m.n() != spec.n:
        raise DomainError(f"matrix is {m.n()}x{m.n()} but spec has N={spec.n}")
    out = np.empty(n_samples, dtype=np.float64)
    check(lib.rw_sample_costs(m.problem().handle, C.byref(spec._c()), n_samples, seed, ptr(out, C.c_double)))
    return out


def sample_orders_philox(n: int, n_samples: int, seed: int) -> np.ndarray:
    """GPU extension: uniform orders from a device Philox stream (not the reference's sequence)."""
    if n_samples < 1:
        raise DomainError("sample_orders: need at least 1 sample")
    out = np.empty((n_samples, n), dtype=np.int32)
    check(lib.rw_sample_orders_philox(n, n_samples, seed, ptr(out, C.c_int32)))
    return out


def sample_costs_philox(m: CostMatrix, spec: CollectiveSpec, n_samples: int, seed: int) -> np.ndarray:
    validate_spec(spec)
    if m.n() != spec.n:
        raise DomainError(f"matrix is {m.n()}x{m.n()} but spec has N={spec.n}")
    out = np.empty(n_samples, dtype=np.float64)
    check(lib.rw_sample_costs_philox(m.problem().handle, C.byref(spec._c()), n_samples, seed,
                                     ptr(out, C.c_double)))
    return out


def sample_cost_distribution(m: CostMatrix, spec: CollectiveSpec, n_samples: int, seed: int) -> DistributionStats:
    return distribution_stats(sample_costs(m, spec, n_samples, seed))


# --------------------------------------------------------------- fixtures --
def generate_matrix(levels, jitter: float = 0.0, seed: int = 0) -> np.ndarray:
    """generate_matrix (topology.hpp:40): levels = [(fanout, latency_us, bandwidth, oversub), ...]."""
    k = len(levels)
    fan = np.array([int(l[0]) for l in levels], dtype=np.int32)
    lat = np.array([float(l[1]) for l in levels], dtype=np.float64)
    bw = np.array([float(l[2]) if len(l) > 2 else 1000.0 for l in levels], dtype=np.float64)
    ov = np.array([float(l[3]) if len(l) > 3 else 1.0 for l in levels], dtype=np.float64)
    n = C.c_int32()
    check(lib.rw_generate_matrix(k, ptr(fan, C.c_int32), ptr(lat, C.c_double), ptr(bw, C.c_double),
                                 ptr(ov, C.c_double), jitter, seed, None, 0, C.byref(n)))
    out = np.empty((n.value, n.value), dtype=np.float64)
    check(lib.rw_generate_matrix(k, ptr(fan, C.c_int32), ptr(lat, C.c_double), ptr(bw, C.c_double),
                                 ptr(ov, C.c_double), jitter, seed, ptr(out, C.c_double), out.size, C.byref(n)))
    return out


def expand_schedule(spec: CollectiveSpec):
    """expand_schedule (cost_model.hpp:33) -> (semantics, [ [(src, dst, bytes, parent), ...] per round ])."""
    sem, nr, cnt = C.c_int32(), C.c_int32(), C.c_int64()
    z = None
    check(lib.rw_expand_schedule(C.byref(spec._c()), C.byref(sem), C.byref(nr), C.byref(cnt), z, z, z, z, z))
    off = np.empty(nr.value + 1, dtype=np.int32)
    src, dst, par = (np.empty(cnt.value, dtype=np.int32) for _ in range(3))
    by = np.empty(cnt.value, dtype=np.float64)
    check(lib.rw_expand_schedule(C.byref(spec._c()), C.byref(sem), C.byref(nr), C.byref(cnt), ptr(off, C.c_int32),
                                 ptr(src, C.c_int32), ptr(dst, C.c_int32), ptr(par, C.c_int32), ptr(by, C.c_double)))
    rounds = [[(int(src[t]), int(dst[t]), float(by[t]), int(par[t])) for t in range(off[r], off[r + 1])]
              for r in range(nr.value)]
    return ScheduleSemantics(sem.value), rounds


def simulate_batch(m: CostMatrix, levels, spec: CollectiveSpec, orders: np.ndarray) -> np.ndarray:
    """Batched simulate_collective (simulate.hpp:24) on the GPU; `m` must be
    generate_matrix(levels, ...); levels = [(fanout, latency_us, bandwidth, oversub), ...]."""
    o = np.ascontiguousarray(orders, dtype=np.int32)
    if o.ndim == 1:
        o = o[None, :]
    fan = np.array([int(l[0]) for l in levels], dtype=np.int32)
    bw = np.array([float(l[2]) for l in levels], dtype=np.float64)
    ov = np.array([float(l[3]) if len(l) > 3 else 1.0 for l in levels], dtype=np.float64)
    out = np.empty(o.shape[0], dtype=np.float64)
    check(lib.rw_simulate_batch(m.problem().handle, len(levels), ptr(fan, C.c_int32), ptr(bw, C.c_double),
                                ptr(ov, C.c_double), C.byref(spec._c()), ptr(o, C.c_int32), o.shape[0],
                                ptr(out, C.c_double)))
    return out


def spearman(xs, ys) -> float:
    """spearman (stats.hpp:14) through the C ABI: Pearson correlation of average ranks."""
    x = np.ascontiguousarray(np.asarray(xs, dtype=np.float64).ravel())
    y = np.ascontiguousarray(np.asarray(ys, dtype=np.float64).ravel())
    out = C.c_double()
    check(lib.rw_spearman(ptr(x, C.c_double), ptr(y, C.c_double), x.size, y.size, C.byref(out)))
    return out.value


def gpu_options() -> dict:
    """The C++ drop-in's process-wide GpuOptions (rankweave.hpp), which
    two_stage_solve uses: device, chains, exact_batch, immutable_matrices,
    num_devices (> 1 or 0 = all: device sets with in-process NCCL)."""
    o = _lib.rw_gpu_options()
    check(lib.rw_get_gpu_options(C.byref(o)))
    return {f: getattr(o, f) for f, _ in o._fields_}


def set_gpu_options(**kw) -> None:
    cur = gpu_options()
    unknown = set(kw) - set(cur)
    if unknown:
        raise TypeError(f"unknown GPU options {sorted(unknown)}")
    cur.update({k: int(v) for k, v in kw.items()})
    check(lib.rw_set_gpu_options(C.byref(_lib.rw_gpu_options(**cur))))


def packed_row_bytes(n: int, bits: int) -> int:
    r = int(lib.rw_packed_row_bytes(n, bits))
    if r < 0:
        raise DomainError("packed orders need n >= 1 and 1 <= bits <= 16")
    return r


def packed_bits(n: int) -> int:
    """Smallest width that holds every host index of an n-host order."""
    return max(1, (max(n, 2) - 1).bit_length())


def pack_orders(orders: np.ndarray, bits: Optional[int] = None) -> np.ndarray:
    """(B, n) orders -> the packed wire layout of rw_evaluate_batch_packed, as bytes."""
    o = np.ascontiguousarray(orders, dtype=np.int32)
    if o.ndim == 1:
        o = o[None, :]
    b = packed_bits(o.shape[1]) if bits is None else int(bits)
    out = np.empty(packed_row_bytes(o.shape[1], b) * o.shape[0], dtype=np.uint8)
    check(lib.rw_pack_orders(ptr(o, C.c_int32), o.shape[1], o.shape[0], b, C.c_void_p(out.ctypes.data)))
    return out


def device_count() -> int:
    return int(lib.rw_device_count())
