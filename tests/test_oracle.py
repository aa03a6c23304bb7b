"""Pin the CPU oracle (oracle/rw_oracle.c) before trusting it as the checker.

1. Known-answer tests transcribed from the reference's own suites
   (proj/tests/test_cost_model.cpp, test_solver.cpp, test_stats.cpp).
2. Golden vectors produced by the reference itself (tests/golden/, made by
   tests/golden/make_golden.py from oracle/_ref).
3. Live comparison with oracle/_ref when it is present.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle.pyoracle import Port, Reference, make_spec, reference_available

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def port():
    return Port()


def uniform(n, v):
    m = np.full((n, n), float(v))
    np.fill_diagonal(m, 0.0)
    return m


ABS = np.array([[0, 1, 2, 3], [1, 0, 1, 2], [2, 1, 0, 1], [3, 2, 1, 0]], dtype=float)


# --- test_cost_model.cpp KATs ------------------------------------------------
def test_ring_uniform_is_n_times_t(port):  # test_cost_model.cpp:65-72
    assert port.evaluate(uniform(4, 1.0), range(4), make_spec(0, 4, 8.0, cost_mode=0)) == 4.0
    assert port.evaluate(uniform(8, 2.5), range(8), make_spec(0, 8, 1.0, cost_mode=0)) == 20.0


def test_ring_hand_sums(port):  # test_cost_model.cpp:74-91
    assert port.evaluate(ABS, range(4), make_spec(0, 4, 1.0, cost_mode=0)) == 6.0
    m3 = np.array([[0, 2, 5], [2, 0, 1], [5, 1, 0]], dtype=float)
    for p in ([0, 1, 2], [0, 2, 1], [1, 0, 2], [1, 2, 0], [2, 0, 1], [2, 1, 0]):
        assert port.evaluate(m3, p, make_spec(0, 3, 1.0, cost_mode=0)) == 8.0


def test_ring_rotation_reflection_exact(port):  # test_cost_model.cpp:93-105
    rng = np.random.default_rng(7)
    for n in (3, 4, 8, 13):
        m = rng.uniform(1, 1000, (n, n))
        m = np.triu(m, 1)
        m = m + m.T
        s = make_spec(0, n, 64.0, cost_mode=1)
        o = rng.permutation(n)
        base = port.evaluate(m, o, s)
        for k in range(1, n):
            assert port.evaluate(m, np.roll(o, -k), s) == base
        assert port.evaluate(m, o[::-1].copy(), s) == base


def test_hd_hand_values(port):  # test_cost_model.cpp:107-125
    assert port.evaluate(uniform(4, 1.0), range(4), make_spec(1, 4, 8.0, cost_mode=1)) == 6.0
    assert port.evaluate(uniform(4, 1.0), range(4), make_spec(1, 4, 8.0, cost_mode=1, hd_pairing=1)) == 6.0
    m2 = np.array([[0, 37], [41, 0]], dtype=float)
    assert port.evaluate(m2, [0, 1], make_spec(1, 2, 8.0, cost_mode=0)) == 37.0
    assert port.evaluate(m2, [1, 0], make_spec(1, 2, 8.0, cost_mode=0)) == 41.0
    assert port.evaluate(ABS, range(4), make_spec(1, 4, 1.0, cost_mode=0)) == 3.0


def test_hd_uniform_closed_form(port):  # test_cost_model.cpp:127-133
    for n in (2, 4, 8, 16, 32):
        assert port.evaluate(uniform(n, 2.5), range(n), make_spec(1, n, 1.0, cost_mode=0)) == 2.5 * math.log2(n)


def test_dbt_hand_values(port):  # test_cost_model.cpp:135-149
    assert port.evaluate(uniform(2, 1.0), [0, 1], make_spec(2, 2, 8.0, cost_mode=1)) == 4.0
    assert port.evaluate(uniform(8, 0.0), range(8), make_spec(2, 8, 8.0, cost_mode=0)) == 0.0
    assert port.evaluate(uniform(8, 1.0), range(8), make_spec(2, 8, 8.0, cost_mode=0)) == 2.0


def test_bcube_hand_values_and_hd_identity(port):  # test_cost_model.cpp:165-188
    assert port.evaluate(uniform(4, 1.0), range(4), make_spec(3, 4, 16.0, 4, 1)) == 4.0
    assert port.evaluate(uniform(8, 0.0), range(8), make_spec(3, 8, 64.0, 2, 1)) == 0.0
    rng = np.random.default_rng(13)
    for n in (2, 4, 8, 16):
        for rep in range(10):
            m = rng.uniform(1, 1000, (n, n))
            np.fill_diagonal(m, 0)
            o = rng.permutation(n)
            size = rng.uniform(1, 1e7)
            for mode in (0, 1):
                assert port.evaluate(m, o, make_spec(1, n, size, 2, mode)) == \
                    port.evaluate(m, o, make_spec(3, n, size, 2, mode))


def test_degenerate_and_rejections(port):  # test_cost_model.cpp:204-223
    for alg in range(4):
        assert port.evaluate(np.zeros((1, 1)), [0], make_spec(alg, 1, 8.0)) == 0.0
    m6 = uniform(6, 1.0)
    for s in (make_spec(1, 6, 1.0), make_spec(2, 6, 1.0), make_spec(3, 6, 1.0, 2), make_spec(0, 6, 0.0)):
        with pytest.raises(ValueError):
            port.evaluate(m6, range(6), s)
    with pytest.raises(ValueError):
        port.evaluate(m6, range(4), make_spec(0, 4, 1.0))
    with pytest.raises(ValueError):
        port.evaluate(m6, [0, 1, 2, 3, 4, 4], make_spec(0, 6, 1.0))


# --- test_solver.cpp / test_stats.cpp KATs ------------------------------------
def test_brute_small_kats(port):  # test_solver.cpp:49-64
    perm, cost, ev = port.brute_force(uniform(5, 2.0), make_spec(0, 5, 1.0))
    assert perm.tolist() == [0, 1, 2, 3, 4] and cost == 10.0
    m3 = np.array([[0, 2, 5], [2, 0, 1], [5, 1, 0]], dtype=float)
    perm, cost, ev = port.brute_force(m3, make_spec(0, 3, 1.0))
    assert cost == 8.0 and perm.tolist() == [0, 1, 2] and ev == 2


def test_distribution_stats(port):  # test_stats.cpp:47-57
    assert port.distribution_stats([5.0]) == (5.0, 5.0, 5.0, 0.0)
    mn, mx, mean, sd = port.distribution_stats([2.0, 4.0, 4.0, 4.0, 5.0, 5.0, 7.0, 9.0])
    assert mean == 5.0 and sd == 2.0


def test_splitmix_substream_distinct(port):
    L = port.lib
    assert L.rwo_splitmix64(0) == 0xE220A8397B1DCDAF  # splitmix64 reference vector for x = 0
    assert len({L.rwo_substream(0, k) for k in range(100)}) == 100


def test_lookup_counts(port):  # SURVEY 8(d) L(model, N)
    assert port.lookups(make_spec(0, 1024, 1.0)) == 1024
    assert port.lookups(make_spec(1, 4096, 1.0, hd_pairing=0)) == 2048 * 12
    assert port.lookups(make_spec(1, 4096, 1.0, hd_pairing=1)) == 4096 * 12
    assert port.lookups(make_spec(3, 4096, 1.0, 8)) == 512 * 7 * 4


# --- golden vectors from the reference ---------------------------------------
def test_port_matches_golden_random_small(port):
    z = np.load(os.path.join(GOLD, "random_small.npz"))
    for k in range(int(z["count"][0])):
        alg, n, b, mode, pair = (int(x) for x in z[f"s{k}"])
        s = make_spec(alg, n, float(z[f"z{k}"][0]), b, mode, pair)
        got = port.evaluate_batch(z[f"m{k}"], z[f"p{k}"], s)
        assert np.array_equal(got, z[f"c{k}"]), (k, alg, n, mode)


@pytest.mark.parametrize("cfg", ["C1", "C3", "C4"])
@pytest.mark.parametrize("kind", ["fixed", "f32"])
def test_port_matches_golden_configs(port, cfg, kind):
    from paper_2105_14088_b200 import fixtures
    m = fixtures.config_matrix(cfg, kind)
    z = np.load(os.path.join(GOLD, f"batch_{cfg}_{kind}.npz"))
    perms = z["perms"].astype(np.int32)
    for key in z.files:
        if not key.startswith("cost_"):
            continue
        name = key[5:]
        alg, n, b, mode, pair = (int(x) for x in z[f"spec_{name}"])
        s = make_spec(alg, n, float(z[f"size_{name}"][0]), b, mode, pair)
        got = port.evaluate_batch(m, perms[:8], s)
        assert np.array_equal(got, z[key][:8]), (cfg, kind, name)


def test_port_brute_matches_golden(port):
    g = json.load(open(os.path.join(GOLD, "brute.json")))
    m16 = np.array(g["matrix16_int"])
    for r in g["results"]:
        if r["n"] > 10:
            continue  # the port's scalar enumeration is slow beyond 9!
        s = make_spec(**r["spec"])
        perm, cost, ev = port.brute_force(m16[: r["n"], : r["n"]], s)
        assert cost == r["cost"] and perm.tolist() == r["order"] and ev == r["evaluations"], r["name"]


def test_survey_golden_table():
    """ring brute force on integer-us blocks, reference-produced."""
    g = json.load(open(os.path.join(GOLD, "brute.json")))
    table = {8: 184, 9: 247, 10: 257, 11: 267, 12: 276, 13: 338}
    seen = {r["n"]: r for r in g["results"] if r["name"] == "ring_block"}
    for n, cost in table.items():
        if n in seen:
            assert seen[n]["cost"] == cost
    if 13 in seen:
        assert seen[13]["order"] == [0, 1, 4, 5, 7, 6, 12, 8, 9, 10, 11, 3, 2]


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_port_matches_reference_live(port):
    ref = Reference()
    rng = np.random.default_rng(99)
    for n in (2, 4, 8, 16, 32, 64):
        m = rng.uniform(0, 500, (n, n))
        np.fill_diagonal(m, 0)
        perms = np.array([rng.permutation(n) for _ in range(20)], dtype=np.int32)
        for alg, b, pair in ((0, 2, 0), (1, 2, 0), (1, 2, 1), (2, 2, 0), (3, 2, 0)):
            for mode in (0, 1):
                s = make_spec(alg, n, 3.25e5, b, mode, pair)
                assert np.array_equal(port.evaluate_batch(m, perms, s), ref.evaluate_batch(m, perms, s))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_generator_matches_reference():
    from paper_2105_14088_b200 import api
    ref = Reference()
    for levels in ([(4, 5, 1000, 1), (4, 25, 1000, 4)], [(8, 5, 1000, 1), (8, 25, 1000, 4)]):
        assert np.array_equal(ref.generate_matrix(levels, 0.1, 2105), api.generate_matrix(levels, 0.1, 2105))


def test_reference_arm_builds_the_same_config_matrices():
    """bench.py's reference arm builds the BASELINE matrices from oracle/_ref
    alone (no product import); they must equal the product's fixtures."""
    from oracle.pyoracle import Reference, reference_available, reference_config_matrix
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    from paper_2105_14088_b200 import fixtures
    ref = Reference()
    for name in ("C1", "C2", "C3", "C4"):
        for kind in ("fixed", "f32"):
            assert np.array_equal(reference_config_matrix(ref, name, kind), fixtures.config_matrix(name, kind)), name
