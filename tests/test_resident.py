"""Resident evaluator (rw_problem_set_resident, csrc/rw_resident.cu): the
single-order evaluate() served by a resident CTA through a mapped mailbox.

Bar: bit-identical to the launched path and to the oracle port (the reference's
evaluate(), cost_model.cpp:140-148) for every model and storage kind, and a
mailbox protocol that neither loses nor duplicates requests across idle exits,
the 5 ms lifetime cap, stops, restarts and concurrent callers.
"""
import threading
import time

import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from oracle.pyoracle import Port, make_spec

pytestmark = pytest.mark.gpu


def matrix(n, kind, sym, seed):
    rng = np.random.default_rng(seed)
    if kind == "fixed":
        a = rng.integers(0, 6000, size=(n, n)).astype(np.float64) / 8.0
    elif kind == "f32":
        a = (rng.random((n, n)) * 300.0).astype(np.float32).astype(np.float64)
    else:
        a = rng.random((n, n)) * 300.0
    m = (np.triu(a, 1) + np.triu(a, 1).T) if sym else a
    np.fill_diagonal(m, 0.0)
    return m


def models(n):
    out = [(0, 2, 0)]
    if n & (n - 1) == 0:
        out += [(2, 2, 0), (1, 2, 0), (1, 2, 1), (3, 2, 0)]
    if n in (16, 64, 256, 1024):
        out.append((3, 4, 0))
    if n in (64, 512):
        out.append((3, 8, 0))
    return out


@pytest.fixture(scope="module")
def port():
    return Port()


@pytest.mark.parametrize("n", [1, 2, 3, 16, 64, 100, 256, 1024, 4096])
@pytest.mark.parametrize("kind", ["fixed", "f32", "f64"])
def test_resident_matches_launched_and_oracle(n, kind, port):
    m = matrix(n, kind, sym=(n % 2 == 0), seed=n)
    prob = rw.Problem(m)
    rng = np.random.default_rng(7 + n)
    perms = [rng.permutation(n).astype(np.int32) for _ in range(6)]
    for alg, b, pair in models(n):
        for mode in (1, 0):
            spec = rw.CollectiveSpec(rw.Algorithm(alg), n, 2.0 ** 17 + 3, b, rw.CostMode(mode), rw.HdPairing(pair))
            prob.set_resident(0)
            launched = [prob.evaluate(spec, p) for p in perms]
            prob.set_resident(1000)
            resident = [prob.evaluate(spec, p) for p in perms]
            assert np.array_equal(np.array(resident), np.array(launched), equal_nan=True), (alg, b, pair, mode)
            if n <= 1024:
                want = port.evaluate_batch(m, np.stack(perms[:2]), make_spec(alg, n, 2.0 ** 17 + 3, b, mode, pair))
                assert np.array_equal(np.array(resident[:2]), want), (alg, b, pair, mode)
    prob.close()


def test_resident_survives_idle_exits_and_lifetime_cap():
    n = 64
    m = matrix(n, "fixed", True, 3)
    prob = rw.Problem(m)
    spec = rw.CollectiveSpec(rw.Algorithm.Ring, n, 1.0)
    rng = np.random.default_rng(1)
    perms = [rng.permutation(n).astype(np.int32) for _ in range(32)]
    want = prob.evaluate_batch(spec, np.stack(perms), exact=True)
    prob.set_resident(20)  # leaves after 20 us idle
    for k in range(200):
        if k % 3 == 0:
            time.sleep(0.0002)  # the server has left: the next call relaunches it
        assert prob.evaluate(spec, perms[k % 32]) == want[k % 32]
    # continuous calls past the 5 ms lifetime cap
    prob.set_resident(100000)
    t0 = time.time()
    k = 0
    while time.time() - t0 < 0.05:
        assert prob.evaluate(spec, perms[k % 32]) == want[k % 32]
        k += 1
    assert k > 100
    # stop, evaluate launched, restart, close with a live server
    prob.set_resident(0)
    assert prob.evaluate(spec, perms[0]) == want[0]
    prob.set_resident(500)
    assert prob.evaluate(spec, perms[1]) == want[1]
    prob.close()


def test_resident_concurrent_callers():
    n = 256
    m = matrix(n, "f64", False, 5)
    prob = rw.Problem(m)
    prob.set_resident(2000)
    spec = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, n, 4096.0)
    rng = np.random.default_rng(2)
    perms = np.stack([rng.permutation(n) for _ in range(64)]).astype(np.int32)
    want = prob.evaluate_batch(spec, perms)
    errors = []

    def worker(t):
        try:
            for k in range(300):
                i = (k * 7 + t) % 64
                if prob.evaluate(spec, perms[i]) != want[i]:
                    errors.append((t, i))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors
    prob.close()


def test_resident_reconfigured_while_callers_run():
    """set_resident toggled from one thread while others evaluate: a call in
    flight keeps the server it took (shared ownership), later calls take the
    launched path or a new server; every result stays exact."""
    n = 128
    m = matrix(n, "fixed", True, 12)
    prob = rw.Problem(m)
    spec = rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, n, 1e5, 2, rw.CostMode.LatencyTimesSize,
                             rw.HdPairing.XorPairing)
    rng = np.random.default_rng(5)
    perms = np.stack([rng.permutation(n) for _ in range(32)]).astype(np.int32)
    want = prob.evaluate_batch(spec, perms)
    errors = []
    stop = threading.Event()

    def caller(t):
        k = 0
        try:
            while not stop.is_set():
                i = (k * 5 + t) % 32
                if prob.evaluate(spec, perms[i]) != want[i]:
                    errors.append((t, i))
                k += 1
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=caller, args=(t,)) for t in range(3)]
    for th in threads:
        th.start()
    for k in range(60):
        prob.set_resident(0 if k % 2 else 100 + k)
        time.sleep(0.002)
    stop.set()
    for th in threads:
        th.join()
    assert not errors
    prob.close()


def test_resident_rejects_large_n_and_keeps_batches_exact():
    n = 5000
    prob = rw.Problem(matrix(n, "fixed", False, 9))
    with pytest.raises(rw.DomainError):
        prob.set_resident(100)
    prob.close()
    # batch calls on a problem with a live server take their normal paths
    n = 512
    m = matrix(n, "fixed", True, 4)
    prob = rw.Problem(m)
    prob.set_resident(100000)
    spec = rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, n, 1e6, 2, rw.CostMode.LatencyTimesSize,
                             rw.HdPairing.XorPairing)
    rng = np.random.default_rng(3)
    perms = np.stack([rng.permutation(n) for _ in range(600)]).astype(np.int32)
    one = prob.evaluate(spec, perms[0])
    batch = prob.evaluate_batch(spec, perms)
    assert one == batch[0]
    assert prob.evaluate(spec, perms[599]) == batch[599]
    prob.close()


def test_cpp_drop_in_resident_option():
    cpp = pytest.importorskip("paper_2105_14088_b200._rankweave_cpp")
    n = 64
    m = matrix(n, "fixed", True, 11)
    cm = cpp.CostMatrix([f"h{i}" for i in range(n)], m.tolist())
    spec = cpp.CollectiveSpec(cpp.Algorithm.Ring, n, 1.0)
    rng = np.random.default_rng(4)
    orders = [rng.permutation(n).tolist() for _ in range(8)]
    o = cpp.gpu_options()
    base = [cpp.evaluate(cm, cpp.RankOrder(p), spec) for p in orders]
    o.resident_idle_us = 500
    cpp.set_gpu_options(o)
    try:
        res = [cpp.evaluate(cm, cpp.RankOrder(p), spec) for p in orders]
    finally:
        o.resident_idle_us = 0
        cpp.set_gpu_options(o)
    assert res == base
