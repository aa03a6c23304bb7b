"""The pybind11 module (paper_2105_14088_b200/_rankweave_cpp, the reference's
RANKWEAVE_BUILD_PYTHON slot, proj/CMakeLists.txt:11,19-21) binds the C++
drop-in names; it must agree with the reference, the oracle and the ctypes
package."""
import os
import subprocess

import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from paper_2105_14088_b200 import fixtures
from oracle.pyoracle import Port, make_spec

rwc = pytest.importorskip("paper_2105_14088_b200._rankweave_cpp")
REF_DUMP = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "neighbor_on_reference")


def test_types_and_errors_mirror_the_reference():
    m = rwc.CostMatrix(np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], dtype=float), ["a", "b", "c"])
    assert m.n() == 3 and m.hosts == ["a", "b", "c"] and m.at(1, 2) == 3.0
    assert rwc.RankOrder.identity(4).perm == [0, 1, 2, 3]
    s = rwc.CollectiveSpec(rwc.Algorithm.Ring, 3, 10.0)
    assert s.cost_mode == rwc.CostMode.LatencyTimesSize and s.bcube_b == 2
    with pytest.raises(rwc.DomainError, match="power of 2"):
        rwc.validate(rwc.CollectiveSpec(rwc.Algorithm.DoubleBinaryTree, 6, 1.0))
    cfg = rwc.SolverConfig()
    assert cfg.cooling == 0.995 and cfg.restarts == 4 and cfg.brute_force_threshold == 10


def test_neighbor_matches_reference_dump():
    """Same walks as oracle/neighbor_dump.cpp run against the reference."""
    if not os.path.exists(REF_DUMP):
        pytest.skip("make -C oracle neighbor not built (needs /root/reference)")
    lines = subprocess.run([REF_DUMP], capture_output=True, text=True, check=True).stdout.splitlines()
    k = 0
    for n in (1, 2, 3, 5, 8, 13, 64, 1000):
        for seed in range(6):
            o = rwc.neighbor(rwc.RankOrder.identity(n), 1000003 * seed + n, 300)
            want = lines[k].split(":", 1)[1].split("|")[0].split()
            assert o.perm == [int(v) for v in want], (n, seed)
            k += 1


@pytest.mark.gpu
def test_gpu_paths_agree_with_ctypes_and_oracle():
    port = Port()
    m = fixtures.config_matrix("C1", "fixed")
    n = m.shape[0]
    cm = rwc.CostMatrix(m)
    rng = np.random.default_rng(4)
    orders = np.array([rng.permutation(n) for _ in range(64)], dtype=np.int32)
    for alg in range(4):
        spec = rwc.CollectiveSpec(rwc.Algorithm(alg), n, fixtures.SIZE_FIXED)
        want = port.evaluate_batch(m, orders, make_spec(alg, n, fixtures.SIZE_FIXED))
        assert np.array_equal(rwc.evaluate_batch(cm, orders, spec), want)
        assert rwc.evaluate(cm, rwc.RankOrder(orders[0].tolist()), spec) == want[0]
    m8 = np.ascontiguousarray(fixtures.config_matrix("C2")[:8, :8])
    sol = rwc.brute_force(rwc.CostMatrix(m8), rwc.CollectiveSpec(rwc.Algorithm.Ring, 8, 1.0), 8)
    ref = rw.brute_force(rw.CostMatrix.from_array(m8), rw.CollectiveSpec(rw.Algorithm.Ring, 8, 1.0), threshold=8)
    assert sol.cost == ref.cost and sol.order.perm == list(ref.order.perm) and sol.evaluations == ref.evaluations
    cfg = rwc.SolverConfig()
    cfg.seed, cfg.steps_per_temperature = 3, 16
    a = rwc.anneal(cm, rwc.CollectiveSpec(rwc.Algorithm.Ring, n, fixtures.SIZE_FIXED), cfg)
    assert a.method == rwc.SolveMethod.Anneal
    assert a.cost == port.evaluate(m, np.array(a.order.perm, dtype=np.int32), make_spec(0, n, fixtures.SIZE_FIXED))
