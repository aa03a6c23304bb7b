"""Host-side logic of the Python mirror that needs no GPU."""
import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from paper_2105_14088_b200 import api
from oracle.pyoracle import Port


def test_distribution_stats_matches_oracle():
    port = Port()
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 100):
        v = rng.uniform(0, 1e11, n)
        st = api.distribution_stats(v)
        assert (st.min, st.max, st.mean, st.stddev) == port.distribution_stats(v)
        assert st.count == n
    with pytest.raises(rw.DomainError):
        api.distribution_stats([])


def test_parse_model_file():  # smtlib.cpp:160-186 behaviour
    o = api.parse_model_file("; comment\n# other\n\nr_0 = 2\nr_1 = 0\n r_2 = 1 \n", 3)
    assert o.perm == [2, 0, 1]
    for bad in ("r_0 = 0\nr_1 = 0\n", "r_0 = 0\n", "r_5 = 0\nr_1 = 1\n", "x = 1\n", "r_0 = 0\nr_0 = 1\n"):
        with pytest.raises(rw.DomainError):
            api.parse_model_file(bad, 2)


def test_order_helpers():  # test_cost_model.cpp:335-343
    o = rw.RankOrder([2, 0, 3, 1])
    api.validate_order(o, 4)
    assert api.rotated(o, 1).perm == [0, 3, 1, 2]
    assert api.rotated(o, -1).perm == [1, 2, 0, 3]
    assert api.inverse(o).perm == [1, 3, 0, 2]
    with pytest.raises(rw.DomainError):
        api.validate_order(rw.RankOrder([0, 0, 1]), 3)
    with pytest.raises(rw.DomainError):
        api.validate_order(rw.RankOrder([0, 1, 3]), 3)


def test_matrix_validation():  # test_cost_model.cpp:345-351
    with pytest.raises(rw.DomainError):
        api.validate_matrix(rw.CostMatrix(["a", "b"], [[0, 1], [1, 0.5]]))
    with pytest.raises(rw.DomainError):
        api.validate_matrix(rw.CostMatrix(["a", "b"], [[0, -1], [1, 0]]))
    ok = rw.CostMatrix(["a", "b", "c"], [[0, 1, 2], [4, 0, 3], [2, 9, 0]])
    api.validate_matrix(ok)
    assert not api.is_symmetric(ok)


def test_transfer_cost_and_round_bytes():  # test_cost_model.cpp:55-63
    m = rw.CostMatrix(["a", "b", "c"], [[0, 50, 7], [50, 0, 1], [7, 1, 0]])
    assert api.transfer_cost(m, 1, 2, 123.0, rw.CostMode.LatencyOnly) == 1.0
    assert api.transfer_cost(m, 0, 1, 4.0, rw.CostMode.LatencyTimesSize) == 200.0
    assert api.transfer_cost(m, 2, 2, 99.0, rw.CostMode.LatencyTimesSize) == 0.0
    assert api.transfer_cost(m, 0, -1, 1.0, rw.CostMode.LatencyOnly) == 7.0
    assert api.transfer_cost(m, 3, 1, 1.0, rw.CostMode.LatencyOnly) == 50.0
    assert api.round_bytes(100.0, 2, 0) == 50.0 and api.round_bytes(100.0, 2, 1) == 25.0


def test_cost_matrix_is_read_only():
    m = rw.CostMatrix(["a", "b"], [[0, 1], [1, 0]])
    with pytest.raises(ValueError):
        m.rtt_us[0, 1] = 3.0
    m2 = m.with_entry(0, 1, 3.0)
    assert m2.at(0, 1) == 3.0 and m.at(0, 1) == 1.0


def test_string_conversions():
    assert api.algorithm_from_string("dbt") == rw.Algorithm.DoubleBinaryTree
    assert api.to_string(rw.Algorithm.BCube) == "bcube"
    with pytest.raises(rw.DomainError):
        api.algorithm_from_string("mesh")


def test_neighbor_matches_reference_bit_for_bit():
    """neighbor() (solver.hpp:44-47) stays host-side with the caller's
    std::mt19937_64; built against the reference sources and against this
    library (oracle/neighbor_dump.cpp), 300-step walks from seeded generators
    give identical orders and leave the generator in the same state."""
    import os
    import subprocess
    ref = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "neighbor_on_reference")
    ours = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "neighbor_on_b200")
    if not (os.path.exists(ref) and os.path.exists(ours)):
        pytest.skip("make -C oracle neighbor not built (needs /root/reference)")
    a = subprocess.run([ref], capture_output=True, text=True, check=True).stdout
    b = subprocess.run([ours], capture_output=True, text=True, check=True).stdout
    assert a.count("\n") == 48 and a == b
