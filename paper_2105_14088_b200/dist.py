"""Multi-GPU driver (one process per GPU, torch.distributed over NCCL).

SURVEY.md 8(e): the path shards without any data-path collective.
  * batch scoring   -- each rank scores its own slice of the orders;
  * exhaustive      -- the lexicographic index space [0, (N-1)!) is cut into
                       contiguous slices; each rank returns (min cost, min
                       index); the global answer is an all-reduce MIN on the
                       cost followed by an all-reduce MIN on the index among
                       ranks at that cost (lower index = lexicographically
                       smaller order, the reference's tie rule) -- every rank
                       then unranks the winner locally, no broadcast needed;
  * annealing       -- global chain ids are split over ranks; Philox streams
                       are keyed by (seed, global chain id), so the result does
                       not depend on the number of GPUs; end-of-search
                       exchange: MIN cost, MIN chain id at that cost, then a
                       broadcast of the winning order (N int32) from its rank.
The only collectives are these O(1)-size reductions (16 B + N*4 B per
search) and the one-time matrix broadcast (C2).  torch.distributed is the
plumbing; the compute is librankweave_b200.so.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Tuple

import numpy as np

from ._lib import check, lib, ptr
from .api import CollectiveSpec, CostMatrix, Problem, RankOrder, Solution, SolveMethod, SolverConfig

INT64_MAX = np.iinfo(np.int64).max


def _dist():
    import torch.distributed as dist
    return dist


def _device():
    import torch
    dist = _dist()
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def rank_world() -> Tuple[int, int]:
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(), dist.get_world_size()


def broadcast_matrix(m: Optional[np.ndarray], n: int, src: int = 0) -> np.ndarray:
    """C2: replicate the cost matrix from `src` to every rank (N*N float64)."""
    import torch
    dist = _dist()
    r, w = rank_world()
    if w == 1:
        return np.ascontiguousarray(m, dtype=np.float64)
    t = torch.empty((n, n), dtype=torch.float64, device=_device())
    if r == src:
        t.copy_(torch.from_numpy(np.ascontiguousarray(m, dtype=np.float64)))
    dist.broadcast(t, src=src)
    return t.cpu().numpy()


def reduce_argmin(cost: float, key: int, payload: Optional[np.ndarray] = None, n: int = 0):
    """Global (cost, key) argmin across ranks; returns (cost, key, payload of the winner).

    Deterministic: the smallest cost wins, ties go to the smallest key.  The
    payload (e.g. the winning order) is broadcast from the rank that owns it."""
    import torch
    dist = _dist()
    r, w = rank_world()
    if w == 1:
        return cost, key, payload
    dev = _device()
    c = torch.tensor([cost], dtype=torch.float64, device=dev)
    dist.all_reduce(c, op=dist.ReduceOp.MIN)
    best = float(c.item())
    k = torch.tensor([key if cost == best else INT64_MAX], dtype=torch.int64, device=dev)
    dist.all_reduce(k, op=dist.ReduceOp.MIN)
    win_key = int(k.item())
    if payload is None:
        return best, win_key, None
    owner = torch.tensor([r if (cost == best and key == win_key) else w], dtype=torch.int64, device=dev)
    dist.all_reduce(owner, op=dist.ReduceOp.MIN)
    buf = torch.empty(n, dtype=torch.int32, device=dev)
    if r == int(owner.item()):
        buf.copy_(torch.from_numpy(np.ascontiguousarray(payload, dtype=np.int32)))
    dist.broadcast(buf, src=int(owner.item()))
    return best, win_key, buf.cpu().numpy()


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def brute_force_sharded(prob: Problem, spec: CollectiveSpec, threshold: int = 10) -> Solution:
    """brute_force over `world` GPUs: identical answer to the single-GPU call."""
    from .api import DomainError, validate_spec
    validate_spec(spec)
    if spec.n > threshold:
        raise DomainError(f"N={spec.n} exceeds the brute-force threshold {threshold}; use anneal")
    cnt = C.c_uint64()
    check(lib.rw_brute_force_space(C.byref(spec._c()), C.byref(cnt)))
    r, w = rank_world()
    first, count = shard(cnt.value, r, w)
    cost, index = prob.brute_force_range(spec, first, count)
    if count == 0:
        cost, index = float("inf"), INT64_MAX
    best, win, _ = reduce_argmin(cost, int(index))
    perm = np.empty(spec.n, dtype=np.int32)
    # Best::offer (solver.cpp:34-46): the first order of the enumeration stays
    # when its cost is NaN or when no order costs less than +inf
    check(lib.rw_unrank(C.byref(spec._c()), 0, ptr(perm, C.c_int32)))
    if win >= cnt.value or math.isnan(float(prob.evaluate_batch(spec, perm[None, :], exact=True)[0])):
        win = 0
    check(lib.rw_unrank(C.byref(spec._c()), win, ptr(perm, C.c_int32)))
    exact = float(prob.evaluate_batch(spec, perm, exact=True)[0])
    return Solution(RankOrder(perm.tolist()), exact, SolveMethod.BruteForce, int(cnt.value))


def anneal_sharded(prob: Problem, spec: CollectiveSpec, cfg: SolverConfig, chains_total: int,
                   max_proposals: int = 0, schedule: str = "reference"):
    """Simulated annealing with `chains_total` chains split over the ranks.
    Returns (Solution, report) where evaluations are summed over ranks."""
    import torch
    dist = _dist()
    r, w = rank_world()
    begin, count = shard(chains_total, r, w)
    per_rank_budget = max_proposals * count // max(1, chains_total) if max_proposals else 0
    order, cost, ev, rep = prob.anneal(spec, cfg, chains=count, chain_begin=begin, chain_total=chains_total,
                                       max_proposals=per_rank_budget, schedule=schedule)
    best, chain, perm = reduce_argmin(cost, int(rep["winner_chain"]), order, spec.n)
    total_ev = ev
    if w > 1:
        t = torch.tensor([ev], dtype=torch.int64, device=_device())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_ev = int(t.item())
    rep = dict(rep, winner_chain=chain, world=w, chains_total=chains_total)
    return Solution(RankOrder(perm.tolist()), best, SolveMethod.Anneal, total_ev), rep


def evaluate_batch_sharded(prob: Problem, spec: CollectiveSpec, orders: np.ndarray) -> np.ndarray:
    """Each rank scores its slice of `orders`; the costs are all-gathered."""
    import torch
    dist = _dist()
    r, w = rank_world()
    lo, cnt = shard(orders.shape[0], r, w)
    mine = prob.evaluate_batch(spec, orders[lo:lo + cnt]) if cnt else np.empty(0)
    if w == 1:
        return mine
    dev = _device()
    sizes = [shard(orders.shape[0], k, w)[1] for k in range(w)]
    out = [torch.empty(s, dtype=torch.float64, device=dev) for s in sizes]
    dist.all_gather(out, torch.from_numpy(mine).to(dev))
    return torch.cat(out).cpu().numpy()
