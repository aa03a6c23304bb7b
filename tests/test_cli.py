"""CLI (SPEC.md cli module) on the reference's file formats."""
import json
import os

import numpy as np
import pytest

from paper_2105_14088_b200 import cli


def test_matrix_json_roundtrip_with_nulls(tmp_path):
    p = tmp_path / "m.json"
    p.write_text(json.dumps({"hosts": ["a", "b"], "rtt_us": [[0, None], [3.5, 0]]}))
    m = cli.load_matrix(str(p))
    assert m.hosts == ["a", "b"] and np.isnan(m.rtt_us[0, 1]) and m.rtt_us[1, 0] == 3.5
    q = tmp_path / "m2.json"
    cli.save_matrix(str(q), m)
    assert json.loads(q.read_text())["rtt_us"] == [[0.0, None], [3.5, 0.0]]


def test_bad_files_exit_code_2(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text("{not json")
    assert cli.main(["solve", "--matrix", str(p), "--algo", "ring", "--size", "1"]) == 2
    assert cli.main(["solve", "--matrix", str(tmp_path / "missing.json"), "--algo", "ring", "--size", "1"]) == 2
    p.write_text(json.dumps({"hosts": ["a", "b"], "rtt_us": [[0, 1]]}))
    assert cli.main(["solve", "--matrix", str(p), "--algo", "ring", "--size", "1"]) == 2


def test_usage_errors_exit_code_1():
    assert cli.main(["solve", "--algo", "mesh"]) == 1


def test_reorder_hostfile(tmp_path):  # SPEC cmd_reorder_hostfile examples
    hosts = tmp_path / "hosts.txt"
    hosts.write_text("# cluster\n10.0.0.1\n10.0.0.2:7000\n\n10.0.0.3\n")
    order = tmp_path / "order.json"
    order.write_text(json.dumps({"order": [2, 0, 1], "cost": 1.0, "method": "Anneal", "evaluations": 5}))
    out = tmp_path / "out.txt"
    assert cli.main(["reorder", "--hosts", str(hosts), "--order", str(order), "--out", str(out)]) == 0
    assert out.read_text() == "10.0.0.3\n10.0.0.1\n10.0.0.2:7000\n"
    order.write_text(json.dumps({"order": [1, 0]}))
    assert cli.main(["reorder", "--hosts", str(hosts), "--order", str(order), "--out", str(out)]) == 3
    hosts.write_text("a\na\n")
    assert cli.main(["reorder", "--hosts", str(hosts), "--order", str(order), "--out", str(out)]) == 3


def test_generate(tmp_path):
    t = tmp_path / "topo.json"
    t.write_text(json.dumps({"levels": [{"fanout": 4, "latency_us": 5, "bandwidth_Bpus": 1000},
                                        {"fanout": 4, "latency_us": 25, "bandwidth_Bpus": 1000, "oversub": 4}],
                             "jitter": 0.1, "seed": 2105}))
    out = tmp_path / "m.json"
    assert cli.main(["generate", "--topology", str(t), "--out", str(out)]) == 0
    m = cli.load_matrix(str(out))
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "brute.json")))
    assert np.array_equal(np.floor(m.rtt_us[:13, :13] + 0.5), np.array(g["matrix16_int"]))


@pytest.mark.gpu
def test_solve_end_to_end(tmp_path):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "brute.json")))
    m = np.array(g["matrix16_int"])[:9, :9]
    p = tmp_path / "m.json"
    p.write_text(json.dumps({"hosts": [f"h{i}" for i in range(9)], "rtt_us": m.tolist()}))
    out = tmp_path / "o.json"
    assert cli.main(["solve", "--matrix", str(p), "--algo", "ring", "--size", "1", "--out", str(out)]) == 0
    sol = json.loads(out.read_text())
    assert sol["cost"] == 247.0 and sol["method"] == "BruteForce" and sol["evaluations"] == 40320
    assert cli.main(["solve", "--matrix", str(p), "--algo", "hd", "--size", "1"]) == 3  # N=9 not a power of 2


@pytest.mark.gpu
def test_solve_emits_smt_and_runs_on_a_device_set(tmp_path):
    """cmd_solve with --emit-smt writes the reference's stage-2 file (bound = the
    stage-1 cost) and --devices 0 runs the search over every visible GPU of the
    process (in-process NCCL) with the same result."""
    from paper_2105_14088_b200 import api
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "brute.json")))
    m = np.array(g["matrix16_int"])[:9, :9]
    p = tmp_path / "m.json"
    p.write_text(json.dumps({"hosts": [f"h{i}" for i in range(9)], "rtt_us": m.tolist()}))
    out, smt = tmp_path / "o.json", tmp_path / "s.smt2"
    try:
        assert cli.main(["solve", "--matrix", str(p), "--algo", "ring", "--size", "1", "--out", str(out),
                         "--emit-smt", str(smt), "--devices", "0"]) == 0
    finally:
        api.set_gpu_options(num_devices=1)
    sol = json.loads(out.read_text())
    assert sol["cost"] == 247.0 and sol["method"] == "BruteForce"
    text = smt.read_text()
    assert api.balanced_sexpr(text) and "(assert (< cost 247.0))" in text
