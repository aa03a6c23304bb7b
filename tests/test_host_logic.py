"""Host-side logic of the Python mirror that needs no GPU."""
import json
import os

import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from paper_2105_14088_b200 import api
from oracle.pyoracle import Port

GOLD = os.path.join(os.path.dirname(__file__), "golden")


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


def test_sample_orders_are_the_references_for_the_same_seed():
    """sample_orders (stats.cpp:83-94): one std::mt19937_64(seed) stream,
    identity std::shuffle'd per sample -- host code, so this runs without a
    GPU; bit-equal to the reference's orders (tests/golden/sample.npz)."""
    g = np.load(os.path.join(GOLD, "sample.npz"))
    keys = [k for k in g.files if k.startswith("orders_")]
    assert len(keys) >= 8
    for k in keys:
        _, n, samples, seed = k.split("_")
        got = api.sample_orders(int(n), int(samples), int(seed))
        assert np.array_equal(got, g[k]), k
    with pytest.raises(rw.DomainError, match="at least 1 sample"):
        api.sample_orders(4, 0, 0)


def test_emit_smtlib_is_byte_identical_to_the_reference():
    """emit_smtlib (smtlib.cpp:104-158): the same text byte for byte on every
    model, both cost modes, with and without a bound (tests/golden/smtlib.json,
    from oracle/_ref).  Host code; no GPU needed."""
    g = json.load(open(os.path.join(GOLD, "smtlib.json")))
    assert len(g) >= 9
    for name, case in g.items():
        alg, n, size, b, mode, pair = case["spec"]
        spec = rw.CollectiveSpec(rw.Algorithm(alg), n, size, b, rw.CostMode(mode), rw.HdPairing(pair))
        m = rw.CostMatrix.from_array(np.array(case["matrix"]))
        text = api.emit_smtlib(m, spec, case["bound"])
        assert text == case["text"], name
        assert api.balanced_sexpr(text)
    with pytest.raises(rw.DomainError, match="term blow-up"):
        u = np.ones((8, 8)) - np.eye(8)
        api.emit_smtlib(rw.CostMatrix.from_array(u), rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 8, 1.0), None, 4)


def test_spearman_and_stats_match_the_reference_bits():
    """spearman / distribution_stats run the C++ drop-in's code through the C
    ABI (one implementation for C++, Python and FFI users); bit-equal to the
    reference library on random and tied series."""
    from oracle.pyoracle import reference_available, Reference
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    import ctypes as C
    ref = Reference()
    L = ref.lib
    L.ref_spearman.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double)]
    rng = np.random.default_rng(11)
    for n in (2, 5, 50, 1000):
        x = rng.integers(0, 7, n).astype(float)  # ties
        y = rng.uniform(0, 1, n)
        x[0] = 7.0  # never a constant series
        out = C.c_double()
        assert L.ref_spearman(x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_double)), n,
                              C.byref(out)) == 0
        assert api.spearman(x, y) == out.value
        st = api.distribution_stats(y)
        o4 = np.empty(4)
        assert L.ref_distribution_stats(y.ctypes.data_as(C.POINTER(C.c_double)), n,
                                        o4.ctypes.data_as(C.POINTER(C.c_double))) == 0
        assert (st.min, st.max, st.mean, st.stddev) == tuple(o4)
    # special values: NaN, infinities, signed zeros, overflow of the sum
    nan, inf = float("nan"), float("inf")
    for c in ([nan, 1.0, 2.0], [1.0, nan], [inf, 1.0], [-inf, inf], [5.0], [-0.0, 0.0], [nan, nan],
              [1e308, 1e308, -1e308]):
        y = np.array(c)
        o4 = np.empty(4)
        assert L.ref_distribution_stats(y.ctypes.data_as(C.POINTER(C.c_double)), len(y),
                                        o4.ctypes.data_as(C.POINTER(C.c_double))) == 0
        st = api.distribution_stats(y)
        assert np.array([st.min, st.max, st.mean, st.stddev]).tobytes() == o4.tobytes(), c
    for c in ([nan, 1.0, 2.0, 3.0], [1.0, 2.0, inf, 0.5], [1.0, nan, nan, 2.0]):
        x, y = np.array(c), rng.uniform(0, 1, len(c))
        out = C.c_double()
        assert L.ref_spearman(x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_double)),
                              len(x), C.byref(out)) == 0
        assert np.float64(api.spearman(x, y)).tobytes() == np.float64(out.value).tobytes(), c
    with pytest.raises(rw.DomainError, match="lengths differ"):
        api.spearman([1.0, 2.0], [1.0, 2.0, 3.0])
    with pytest.raises(rw.DomainError, match="constant series"):
        api.spearman([1.0, 1.0, 1.0], [1.0, 2.0, 3.0])


def test_two_stage_solve_routing_without_gpu_work():
    """N <= 2 routes to the identity; an invalid spec raises the reference's domain_error."""
    with pytest.raises(rw.DomainError):
        api.two_stage_solve(rw.CostMatrix.from_array(np.zeros((3, 3))),
                            rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, 3, 1.0), rw.SolverConfig())
