"""simulate_collective (the validation ground truth) and
the SPEC validate workflow."""
import json
import os

import numpy as np
import pytest

import paper_2105_14088_b200 as rw
from paper_2105_14088_b200 import api, cli

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOPOS = {
    "t64": ([(8, 5, 1000, 1), (8, 25, 1000, 4)], 0.1, 2105),
    "t256": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (2, 100, 1000, 4)], 0.1, 2105),
}


def test_spearman_kats():  # test_stats.cpp:16-45
    assert api.spearman([1, 2, 3], [1, 2, 3]) == 1.0
    assert api.spearman([1, 2, 3], [3, 2, 1]) == -1.0
    assert abs(api.spearman([1, 2, 3, 4, 5], [2, 1, 4, 3, 5]) - 0.8) < 1e-12
    assert abs(api.spearman([1, 1, 2], [1, 2, 3]) - np.sqrt(3.0) / 2.0) < 1e-12
    assert abs(api.spearman([3, 1, 4, 1, 5, 9, 2, 6], [2, 7, 1, 8, 2, 8, 1, 8]) - 0.19885368120992467) < 1e-9
    for xs, ys in (([1, 2], [1, 2, 3]), ([1], [1]), ([2, 2, 2], [1, 2, 3])):
        with pytest.raises(rw.DomainError):
            api.spearman(xs, ys)


def test_expand_schedule_structure():  # test_cost_model.cpp:271-311
    sem, rounds = api.expand_schedule(rw.CollectiveSpec(rw.Algorithm.Ring, 4, 100.0))
    assert sem == api.ScheduleSemantics.SequentialHops and len(rounds) == 4
    assert all(len(r) == 1 and r[0][2] == 100.0 and r[0][0] != r[0][1] for r in rounds)
    sem, rounds = api.expand_schedule(rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, 4, 100.0))
    assert sem == api.ScheduleSemantics.BulkSynchronousRounds and [len(r) for r in rounds] == [2, 2]
    assert rounds[0][0][:3] == (0, 1, 50.0) and rounds[0][1][:2] == (1, 2) and rounds[1][0][2] == 25.0
    sem, rounds = api.expand_schedule(rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 8, 100.0))
    assert sem == api.ScheduleSemantics.CriticalPath
    # depth sizes 4, 8, 4 with the listed first edges
    assert [len(r) for r in rounds] == [4, 8, 4]
    assert rounds[0][0][:2] == (3, 2) and rounds[1][2][:2] == (5, 0) and rounds[2][2] == (5, 2, 50.0, 7)


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["t64", "t256"])
def test_simulate_matches_reference_goldens(topo):
    z = np.load(os.path.join(GOLD, "simulate.npz"))
    levels, jitter, seed = TOPOS[topo]
    rtt = api.generate_matrix(levels, jitter, seed)
    m = rw.CostMatrix.from_array(rtt)
    perms = z[f"{topo}_perms"]
    for key in z.files:
        if not key.startswith(topo + "_") or key.endswith(("_spec", "_perms")):
            continue
        alg, n, b, mode, pair = (int(x) for x in z[key + "_spec"])
        spec = rw.CollectiveSpec(rw.Algorithm(alg), n, 1e6, b, rw.CostMode(mode), rw.HdPairing(pair))
        got = api.simulate_batch(m, levels, spec, perms)
        assert np.array_equal(got, z[key]), key


@pytest.mark.gpu
def test_simulate_rejects_mismatched_topology():
    levels, jitter, seed = TOPOS["t64"]
    m = rw.CostMatrix.from_array(api.generate_matrix(levels, jitter, seed))
    with pytest.raises(rw.DomainError, match="topology has 64 hosts but spec.n=32"):
        api.simulate_batch(m, levels, rw.CollectiveSpec(rw.Algorithm.Ring, 32, 1.0), np.arange(32)[None, :])


@pytest.mark.gpu
def test_validate_command(tmp_path):  # SPEC cmd_validate examples
    t = tmp_path / "topo.json"
    t.write_text(json.dumps({"levels": [{"fanout": 8, "latency_us": 5, "bandwidth_Bpus": 1000},
                                        {"fanout": 8, "latency_us": 25, "bandwidth_Bpus": 1000, "oversub": 4}],
                             "jitter": 0.1, "seed": 7}))
    out = tmp_path / "r.json"
    assert cli.main(["validate", "--topology", str(t), "--algo", "ring", "--size", "1e6", "--samples", "50",
                     "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["spearman"] >= 0.7 and rep["model"]["count"] == 50
    flat = tmp_path / "flat.json"
    flat.write_text(json.dumps({"levels": [{"fanout": 16, "latency_us": 5, "bandwidth_Bpus": 1000}], "seed": 1}))
    assert cli.main(["validate", "--topology", str(flat), "--algo", "ring", "--size", "1e6", "--samples", "20",
                     "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["spearman"] == "undefined" and rep["model"]["stddev"] == 0.0
    assert cli.main(["validate", "--topology", str(t), "--algo", "ring", "--size", "1", "--samples", "1",
                     "--out", str(out)]) == 3
