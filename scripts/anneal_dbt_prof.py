#!/usr/bin/env python3
"""Short C3 tree-model anneal for ncu captures of k_anneal_full (one GPU)."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import paper_2105_14088_b200 as rw  # noqa: E402

m = rw.fixtures.config_matrix("C3", "fixed")
prob = rw.Problem(m)
spec = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
o, c, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=int(sys.argv[1]) if len(sys.argv) > 1 else 16),
                            chains=int(os.environ.get("CHAINS", "592")))
print(c, ev, rep)
