#!/usr/bin/env python3
"""One C3 tree-model annealing chain with a small budget (ncu target):
    ncu --set full -k regex:k_anneal_full -c 1 python scripts/anneal_dbt_one_chain.py
"""
import sys
sys.path.insert(0, ".")
import paper_2105_14088_b200 as rw  # noqa: E402

m = rw.fixtures.config_matrix("C3", "fixed")
prob = rw.Problem(m)
spec = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
o, c, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=64), chains=1,
                            max_proposals=400000)
print("cost", c, "evals", ev, rep["proposals"])
