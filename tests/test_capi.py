"""CPU-side checks of the C-ABI boundary (no compute calls need a GPU here)."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from paper_2105_14088_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_functions():
    names = set()
    for h in ("rankweave_c.h",):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*(rw_[a-z0-9_]+)\s*\(", text, re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_abi():
    names = declared_functions()
    assert {"rw_evaluate", "rw_evaluate_batch", "rw_brute_force", "rw_anneal", "rw_problem_create"} <= names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared_functions()) if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table binds exactly the declared set
    assert set(_lib.SIGNATURES) == declared_functions()


def test_abi_version_and_device_query():
    assert _lib.lib.rw_abi_version() == 3
    assert rw.device_count() >= 0


@pytest.mark.parametrize("spec,msg", [
    (rw.CollectiveSpec(rw.Algorithm.Ring, 0, 1.0), "node count must be >= 1"),
    (rw.CollectiveSpec(rw.Algorithm.Ring, 4, 0.0), "data size must be > 0"),
    (rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, 6, 1.0), "hd requires N a power of 2, got 6"),
    (rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 12, 1.0), "dbt requires N a power of 2, got 12"),
    (rw.CollectiveSpec(rw.Algorithm.BCube, 8, 1.0, 1), "BCube group size B must be >= 2"),
    (rw.CollectiveSpec(rw.Algorithm.BCube, 8, 1.0, 4), "BCube requires N a power of B=4, got 8"),
])
def test_spec_validation_wording(spec, msg):
    """types.cpp:143-163 messages, raised as domain_error through the C ABI."""
    with pytest.raises(rw.DomainError, match=re.escape(msg)):
        rw.api.validate_spec(spec)


def test_degenerate_spec_is_valid():
    rw.api.validate_spec(rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, 1, 8.0))


def test_brute_force_space_and_unrank_are_lexicographic():
    spec = rw.CollectiveSpec(rw.Algorithm.Ring, 6, 1.0)._c()
    cnt = C.c_uint64()
    _lib.check(_lib.lib.rw_brute_force_space(C.byref(spec), C.byref(cnt)))
    assert cnt.value == 120
    import itertools
    lex = [(0,) + p for p in itertools.permutations(range(1, 6))]
    out = np.empty(6, dtype=np.int32)
    for idx in (0, 1, 57, 119):
        _lib.check(_lib.lib.rw_unrank(C.byref(spec), idx, _lib.ptr(out, C.c_int32)))
        assert tuple(out) == lex[idx]
    spec_hd = rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, 4, 1.0)._c()
    _lib.check(_lib.lib.rw_brute_force_space(C.byref(spec_hd), C.byref(cnt)))
    assert cnt.value == 24
    with pytest.raises(rw.DomainError):
        _lib.check(_lib.lib.rw_unrank(C.byref(spec), 120, _lib.ptr(out, C.c_int32)))


def test_generator_matches_golden_block():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "brute.json")))
    m = rw.fixtures.config_matrix("C2")
    assert np.array_equal(m, np.array(g["matrix16_int"]))
    assert m.shape == (13, 13) and np.array_equal(m, m.T) and not np.diag(m).any()


def test_generator_validation():
    with pytest.raises(rw.DomainError, match="jitter must be in"):
        rw.api.generate_matrix([(4, 5.0, 1000, 1)], jitter=1.5)
    with pytest.raises(rw.DomainError, match="fanout product must be >= 2"):
        rw.api.generate_matrix([(1, 5.0, 1000, 1)])


def test_fixture_variants_are_exact_types():
    m = rw.fixtures.config_matrix("C1", "fixed")
    q = m * 16
    assert np.array_equal(q, np.round(q)) and q.max() < 65536
    f = rw.fixtures.config_matrix("C1", "f32")
    assert np.array_equal(f.astype(np.float32).astype(np.float64), f)


def test_problem_create_without_gpu_fails_loudly():
    if rw.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(rw.RankweaveError):
        rw.Problem(np.zeros((4, 4)))


def test_null_and_shape_arguments_are_domain_errors():
    with pytest.raises(rw.DomainError):
        _lib.check(_lib.lib.rw_evaluate(None, None, None, None))
    with pytest.raises(rw.DomainError):
        rw.Problem(np.zeros((3, 4)))
    with pytest.raises(rw.DomainError, match="null rw_problem"):
        _lib.check(_lib.lib.rw_problem_set_resident(None, 100))


def test_packed_layout_helpers_on_the_host():
    """rw_packed_row_bytes / rw_pack_orders (host side of the packed wire
    layout): 10 bits per host at N=1024 is 1280 bytes per order; the packing
    round-trips; out-of-width values and bad widths are domain errors."""
    from paper_2105_14088_b200 import api
    assert api.packed_row_bytes(1024, 10) == 1280
    assert api.packed_row_bytes(13, 4) == 16 and api.packed_bits(13) == 4 and api.packed_bits(1024) == 10
    assert int(_lib.lib.rw_packed_row_bytes(0, 10)) == -1 and int(_lib.lib.rw_packed_row_bytes(8, 17)) == -1
    rng = np.random.default_rng(1)
    for n, bits in ((13, 4), (64, 6), (1000, 10), (4096, 12), (300, 16)):
        o = np.array([rng.permutation(n) for _ in range(5)], dtype=np.int32)
        buf = api.pack_orders(o, bits)
        assert buf.size == 5 * api.packed_row_bytes(n, bits)
        w = np.concatenate([buf.view(np.uint32), np.zeros(1, np.uint32)]).astype(np.uint64)
        row = api.packed_row_bytes(n, bits) // 4
        for b in range(5):
            i = np.arange(n, dtype=np.uint64) * np.uint64(bits)
            q = (i >> np.uint64(5)) + np.uint64(b * row)
            sh = i & np.uint64(31)
            v = ((w[q] | (w[q + np.uint64(1)] << np.uint64(32))) >> sh) & np.uint64((1 << bits) - 1)
            assert np.array_equal(v.astype(np.int64), o[b])
    with pytest.raises(rw.DomainError):
        api.pack_orders(np.array([[0, 1, 2, 3, 4, 5, 6, 7, 8]]), 3)  # 2^3 < 9
    with pytest.raises(rw.DomainError):
        api.pack_orders(np.array([[0, 1, 99]]), 2)


def test_gpu_options_round_trip_through_the_c_abi():
    from paper_2105_14088_b200 import api
    before = api.gpu_options()
    try:
        api.set_gpu_options(chains=77, immutable_matrices=1, num_devices=0)
        o = api.gpu_options()
        assert (o["chains"], o["immutable_matrices"], o["num_devices"]) == (77, 1, 0)
        with pytest.raises(rw.DomainError):
            api.set_gpu_options(num_devices=-1)
        with pytest.raises(TypeError):
            api.set_gpu_options(bogus=1)
    finally:
        api.set_gpu_options(**before)
    assert api.gpu_options() == before


def test_problem_set_argument_checks_without_gpu_work():
    from paper_2105_14088_b200 import api
    if rw.device_count() == 0:
        with pytest.raises((rw.DomainError, rw.RankweaveError)):
            api.ProblemSet(np.zeros((4, 4)))
    else:
        with pytest.raises(rw.DomainError):
            api.ProblemSet(np.zeros((4, 4)), devices=[0, 0])
