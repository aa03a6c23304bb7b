"""Command line front end (SPEC.md cli module: cmd_solve, cmd_reorder_hostfile,
plus `generate` and `evaluate` helpers), on the reference's file formats
(proj/src/json_io.cpp, proj/src/hostfile.cpp):

  matrix file   {"hosts": [str...], "rtt_us": [[num|null...]...]}
  solution file {"order": [int...], "cost": num, "method": str, "evaluations": int}
  topology file {"levels": [{"fanout", "latency_us", "bandwidth_Bpus", "oversub"}...], "jitter", "seed"}
  hostfile      one endpoint per line; '#' comments; rank = line index

Exit codes: 0 success, 1 usage, 2 I/O or parse, 3 domain violation.

    python -m paper_2105_14088_b200.cli solve --matrix m.json --algo ring --size 1e8 --out order.json
    python -m paper_2105_14088_b200.cli reorder --hosts hosts.txt --order order.json --out ranked.txt
    python -m paper_2105_14088_b200.cli generate --topology topo.json --out m.json
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

from . import api


class IOFailure(Exception):
    pass


def load_matrix(path: str) -> api.CostMatrix:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise IOFailure(f"cannot read '{path}'")
    except json.JSONDecodeError:
        raise IOFailure("malformed JSON in matrix file")
    try:
        hosts = [str(h) for h in j["hosts"]]
        rows = j["rtt_us"]
    except (KeyError, TypeError) as e:
        raise IOFailure(f"matrix file: missing {e}")
    if not isinstance(rows, list) or len(rows) != len(hosts):
        raise IOFailure("matrix file: rtt_us must have one row per host")
    vals = []
    for row in rows:
        if not isinstance(row, list) or len(row) != len(hosts):
            raise IOFailure("matrix file: rtt_us is not square")
        vals.append([math.nan if v is None else float(v) for v in row])
    return api.CostMatrix(hosts, np.array(vals, dtype=np.float64).reshape(len(hosts), len(hosts)))


def save_matrix(path: str, m: api.CostMatrix) -> None:
    rows = [[(float(v) if math.isfinite(v) else None) for v in r] for r in m.rtt_us.tolist()]
    _write(path, json.dumps({"hosts": m.hosts, "rtt_us": rows}, indent=2) + "\n")


def solution_to_json(s: api.Solution) -> str:
    return json.dumps({"order": list(map(int, s.order.perm)), "cost": s.cost,
                       "method": api.to_string(s.method), "evaluations": int(s.evaluations)}, indent=2) + "\n"


def load_solution(path: str) -> api.Solution:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise IOFailure(f"cannot read '{path}'")
    except json.JSONDecodeError:
        raise IOFailure("malformed JSON in solution file")
    try:
        method = {"BruteForce": api.SolveMethod.BruteForce, "Anneal": api.SolveMethod.Anneal,
                  "External": api.SolveMethod.External}[j.get("method", "BruteForce")]
        return api.Solution(api.RankOrder([int(v) for v in j["order"]]), float(j.get("cost", 0.0)), method,
                            int(j.get("evaluations", 0)))
    except (KeyError, TypeError, ValueError) as e:
        raise IOFailure(f"solution file: {e}")


def parse_hostfile(text: str):
    hosts, seen = [], set()
    for no, line in enumerate(text.splitlines(), 1):
        s = line.strip(" \t\r")
        if not s or s.startswith("#"):
            continue
        if s in seen:
            raise api.DomainError(f"duplicate host '{s}' at line {no}")
        seen.add(s)
        hosts.append(s)
    if not hosts:
        raise api.DomainError("hostfile contains no hosts")
    return hosts


def reorder_hosts(hosts, order: api.RankOrder):
    api.validate_order(order, len(hosts))
    return [hosts[i] for i in order.perm]


def _write(path: str, text: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise IOFailure(f"cannot write '{path}'")


def cmd_solve(a) -> int:
    m = load_matrix(a.matrix)
    api.validate_matrix(m)
    spec = api.CollectiveSpec(api.algorithm_from_string(a.algo), m.n(), a.size, a.b,
                              api.CostMode.LatencyOnly if a.latency_only else api.CostMode.LatencyTimesSize)
    cfg = api.SolverConfig(budget=a.budget, seed=a.seed, brute_force_threshold=a.threshold)
    log = (lambda s: print(s, file=sys.stderr))
    if a.devices != 1:
        api.set_gpu_options(num_devices=a.devices)
    sol = api.two_stage_solve(m, spec, cfg, external_model_path=a.external_model or "", log=log,
                              emit_smt_path=a.emit_smt or "")
    ident = api.evaluate(m, api.RankOrder.identity(m.n()), spec)
    ratio = ident / sol.cost if sol.cost > 0 else 1.0
    print(f"identity cost {ident:.6g}  solved cost {sol.cost:.6g}  improvement x{ratio:.4f}  "
          f"({api.to_string(sol.method)}, {sol.evaluations} evaluations)", file=sys.stderr)
    text = solution_to_json(sol)
    if a.out:
        _write(a.out, text)
    else:
        sys.stdout.write(text)
    return 0


def cmd_reorder(a) -> int:
    try:
        text = open(a.hosts).read()
    except OSError:
        raise IOFailure(f"cannot read hostfile '{a.hosts}'")
    hosts = parse_hostfile(text)
    sol = load_solution(a.order)
    out = reorder_hosts(hosts, sol.order)
    _write(a.out, "".join(h + "\n" for h in out))
    return 0


def cmd_generate(a) -> int:
    try:
        t = json.load(open(a.topology))
    except OSError:
        raise IOFailure(f"cannot read '{a.topology}'")
    except json.JSONDecodeError:
        raise IOFailure("malformed JSON in topology file")
    levels = [(int(l["fanout"]), float(l["latency_us"]), float(l["bandwidth_Bpus"]), float(l.get("oversub", 1.0)))
              for l in t["levels"]]
    rtt = api.generate_matrix(levels, float(t.get("jitter", 0.0)), int(t.get("seed", 0)))
    save_matrix(a.out, api.CostMatrix([f"node{i}" for i in range(rtt.shape[0])], rtt))
    return 0


def cmd_validate(a) -> int:
    """SPEC cmd_validate: model cost vs simulated time over K random orders (GPU for both),
    Spearman coefficient and DistributionStats of each series."""
    try:
        t = json.load(open(a.topology))
    except OSError:
        raise IOFailure(f"cannot read '{a.topology}'")
    except json.JSONDecodeError:
        raise IOFailure("malformed JSON in topology file")
    if a.samples < 2:
        raise api.DomainError("validate needs at least 2 samples")
    levels = [(int(l["fanout"]), float(l["latency_us"]), float(l["bandwidth_Bpus"]), float(l.get("oversub", 1.0)))
              for l in t["levels"]]
    rtt = api.generate_matrix(levels, float(t.get("jitter", 0.0)), int(t.get("seed", 0)))
    m = api.CostMatrix([f"node{i}" for i in range(rtt.shape[0])], rtt)
    spec = api.CollectiveSpec(api.algorithm_from_string(a.algo), m.n(), a.size, a.b)
    orders = api.sample_orders(m.n(), a.samples, a.seed)
    model = m.problem().evaluate_batch(spec, orders, exact=True)
    sim = api.simulate_batch(m, levels, spec, orders)

    def stats(v):
        s = api.distribution_stats(v)
        return {"min": s.min, "max": s.max, "mean": s.mean, "stddev": s.stddev, "count": s.count}

    try:
        rho = api.spearman(model, sim)
    except api.DomainError:
        rho = "undefined"
    report = {"algorithm": a.algo, "n": m.n(), "size_bytes": a.size, "samples": a.samples, "spearman": rho,
              "model": stats(model), "simulated": stats(sim)}
    _write(a.out, json.dumps(report, indent=2) + "\n")
    print(f"spearman {rho}", file=sys.stderr)
    return 0


def cmd_evaluate(a) -> int:
    m = load_matrix(a.matrix)
    spec = api.CollectiveSpec(api.algorithm_from_string(a.algo), m.n(), a.size, a.b)
    sol = load_solution(a.order)
    print(json.dumps({"cost": api.evaluate(m, sol.order, spec)}))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="rankweave-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("--matrix", required=True)
    s.add_argument("--algo", required=True, choices=["ring", "hd", "dbt", "bcube"])
    s.add_argument("--size", type=float, required=True)
    s.add_argument("--b", type=int, default=2)
    s.add_argument("--budget", type=float, default=10.0)
    s.add_argument("--seed", type=int, default=int(os.environ.get("RANKWEAVE_SEED", "0")))
    s.add_argument("--threshold", type=int, default=10)
    s.add_argument("--latency-only", action="store_true")
    s.add_argument("--external-model", default="")
    s.add_argument("--emit-smt", default="", help="write the stage-2 SMT-LIB encoding (bound: the stage-1 cost)")
    s.add_argument("--devices", type=int, default=1,
                   help="GPUs of this process for the search (0: all visible; in-process NCCL)")
    s.add_argument("--out", default="")
    r = sub.add_parser("reorder")
    r.add_argument("--hosts", required=True)
    r.add_argument("--order", required=True)
    r.add_argument("--out", required=True)
    g = sub.add_parser("generate")
    g.add_argument("--topology", required=True)
    g.add_argument("--out", required=True)
    v = sub.add_parser("validate")
    v.add_argument("--topology", required=True)
    v.add_argument("--algo", required=True, choices=["ring", "hd", "dbt", "bcube"])
    v.add_argument("--size", type=float, required=True)
    v.add_argument("--b", type=int, default=2)
    v.add_argument("--samples", type=int, required=True)
    v.add_argument("--seed", type=int, default=int(os.environ.get("RANKWEAVE_SEED", "0")))
    v.add_argument("--out", required=True)
    e = sub.add_parser("evaluate")
    e.add_argument("--matrix", required=True)
    e.add_argument("--algo", required=True, choices=["ring", "hd", "dbt", "bcube"])
    e.add_argument("--size", type=float, required=True)
    e.add_argument("--b", type=int, default=2)
    e.add_argument("--order", required=True)
    try:
        a = ap.parse_args(argv)
    except SystemExit as ex:
        return 1 if ex.code else 0
    try:
        return {"solve": cmd_solve, "reorder": cmd_reorder, "generate": cmd_generate, "evaluate": cmd_evaluate,
                "validate": cmd_validate}[a.cmd](a)
    except IOFailure as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 2
    except api.DomainError as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
