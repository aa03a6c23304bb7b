#!/usr/bin/env python3
"""Short C4 anneal for ncu captures of k_anneal_ring (one GPU).

    CHAINS=592 python scripts/anneal_prof.py 512      # steps per temperature level
"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import paper_2105_14088_b200 as rw  # noqa: E402

m = rw.fixtures.config_matrix("C4", "fixed")
prob = rw.Problem(m)
spec = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
chains = int(os.environ.get("CHAINS", "592"))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 512
o, c, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                            chains=chains, schedule="calibrated")
print(c, ev, rep)
