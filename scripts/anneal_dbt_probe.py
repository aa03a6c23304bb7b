#!/usr/bin/env python3
"""C3 tree-model anneal at the reference run's evaluation budget (one chain by default):

    python scripts/anneal_dbt_probe.py [chains]
"""
import json, sys, time
sys.path.insert(0, ".")
import paper_2105_14088_b200 as rw
g = json.load(open("tests/golden/anneal.json"))
ref = [r for r in g["results"] if r["config"] == "C3" and r["model"] == "dbt"][0]
m = rw.fixtures.config_matrix("C3", "fixed")
prob = rw.Problem(m)
spec = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
for sched in ("reference", "calibrated"):
    t = time.perf_counter()
    o, c, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6), chains=int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                                max_proposals=ref["evaluations"], schedule=sched)
    print(sched, "gpu %.6e" % c, "ref %.6e" % ref["cost"], "ident %.6e" % ref["identity_cost"], "evals", ev, "%.1fs" % (time.perf_counter() - t), rep.get("levels"), flush=True)
