"""Multi-GPU inside the library (one process, a device set, in-process NCCL):
rw_problem_set_* / rw_*_set through the Python binding and the C++ drop-in.

Sharded exhaustive search and annealing must give the same order, cost and
evaluation count at every device count (Lehmer range split +
NCCL MIN (cost, index); chain ids split + NCCL MIN (cost, chain) + broadcast).
Runs on whatever the box has: 1 device checks the set path itself; 2 or 4
devices check invariance across device counts."""
import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from paper_2105_14088_b200 import fixtures
from oracle.pyoracle import Port, make_spec

pytestmark = pytest.mark.gpu


def device_counts():
    k = rw.device_count()
    return [c for c in (1, 2, 4, 8) if c <= k]


def test_set_brute_force_is_device_count_invariant():
    m = fixtures.config_matrix("C2")[:11, :11].copy()
    spec = rw.CollectiveSpec(rw.Algorithm.Ring, 11, 1.0)
    single = rw.brute_force(rw.CostMatrix.from_array(m), spec, threshold=11)
    for k in device_counts():
        s = rw.api.ProblemSet(m, devices=list(range(k)))
        sol = s.brute_force(spec, threshold=11)
        assert (sol.cost, sol.order.perm, sol.evaluations) == (single.cost, single.order.perm, single.evaluations), k
        s.close()
    # all models at N=8 (every order enumerated)
    m8 = fixtures.config_matrix("C2")[:8, :8].copy()
    for alg in (1, 2, 3):
        spec8 = rw.CollectiveSpec(rw.Algorithm(alg), 8, 1024.0)
        want = rw.brute_force(rw.CostMatrix.from_array(m8), spec8)
        s = rw.api.ProblemSet(m8, devices=list(range(device_counts()[-1])))
        got = s.brute_force(spec8)
        assert (got.cost, got.order.perm, got.evaluations) == (want.cost, want.order.perm, want.evaluations)


def test_set_anneal_is_device_count_invariant():
    m = fixtures.config_matrix("C1", "fixed")
    spec = fixtures.ring_spec(64, fixtures.SIZE_FIXED)
    cfg = rw.SolverConfig(seed=3, budget=1e6, steps_per_temperature=64)
    prob = rw.Problem(m)
    o1, c1, e1, r1 = prob.anneal(spec, cfg, chains=64)
    for k in device_counts():
        s = rw.api.ProblemSet(m, devices=list(range(k)))
        o, c, e, r = s.anneal(spec, cfg, chains=64)
        assert c == c1 and o.tolist() == o1.tolist() and r["winner_chain"] == r1["winner_chain"], k
        assert c == Port().evaluate(m, o, make_spec(0, 64, fixtures.SIZE_FIXED))
        s.close()


def test_set_batch_scoring_splits_one_host_batch():
    m = fixtures.config_matrix("C4", "fixed")
    spec = fixtures.ring_spec(1024, fixtures.SIZE_FIXED)
    rng = np.random.default_rng(4)
    o = np.array([rng.permutation(1024) for _ in range(20000)], dtype=np.int32)
    want = rw.Problem(m).evaluate_batch(spec, o)
    for k in device_counts():
        s = rw.api.ProblemSet(m, devices=list(range(k)))
        assert np.array_equal(s.evaluate_batch(spec, o), want)
        assert np.array_equal(s.evaluate_batch(spec, o.astype(np.uint16)), want)
        assert np.array_equal(s.evaluate_batch_packed(spec, rw.api.pack_orders(o, 10), 10, len(o)), want)
        bad = o[:4000].copy()
        bad[3333, 5] = bad[3333, 6]
        with pytest.raises(rw.DomainError, match="batch entry 3333"):
            s.evaluate_batch(spec, bad)
        s.close()


def test_set_rejects_bad_device_lists():
    m = np.zeros((4, 4))
    with pytest.raises(rw.DomainError):
        rw.api.ProblemSet(m, devices=[0, 0])
    with pytest.raises(rw.DomainError):
        rw.api.ProblemSet(m, devices=[rw.device_count()])


def test_cpp_drop_in_over_device_sets_is_device_count_invariant():
    """The reference C++ API (brute_force, anneal, two_stage_solve,
    evaluate_batch) with GpuOptions::num_devices = 1, 2, 4: identical output
    (oracle/multi_dump.cpp, linked against librankweave_b200.so only)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "multi_on_b200")
    if not os.path.exists(exe):
        pytest.skip("make -C oracle multi not built")
    outs = {}
    for k in device_counts():
        r = subprocess.run([exe, str(k)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        outs[k] = "".join(l for l in r.stdout.splitlines(True) if not l.startswith("NCCL"))
    first = outs[1]
    assert first.count("\n") == 6 and "brute ring cost=" in first
    for k, out in outs.items():
        assert out == first, k


def test_set_lifecycle_releases_its_threads_resources():
    """A device set owns one host thread per member; destroying the set frees
    those threads' streams and scratch (repeated sets do not leak device memory)."""
    import torch
    m = fixtures.config_matrix("C4", "fixed")
    spec = fixtures.ring_spec(1024, fixtures.SIZE_FIXED)
    o = np.array([np.random.default_rng(k).permutation(1024) for k in range(20000)], dtype=np.int32)
    k = device_counts()[-1]

    def one():
        s = rw.api.ProblemSet(m, devices=list(range(k)))
        s.evaluate_batch(spec, o)
        s.close()

    one()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(0)[0]
    for _ in range(4):
        one()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(0)[0]
    assert free0 - free1 < (64 << 20), (free0, free1)
