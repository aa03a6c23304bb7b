#!/usr/bin/env python3
"""C4 ring time-to-best against the chain count (one GPU): for each chain
count, escalate the steps per level (as bench.py's time-to-best extra does)
until the incumbent is <= the reference's best run, and print the cumulative
and last-run wall time.

    python scripts/time_to_best_chains.py
"""
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main():
    import paper_2105_14088_b200 as rw
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "anneal_c4.json")))
    target = min(r["cost"] for r in g["results"])
    m = rw.fixtures.config_matrix("C4", "fixed")
    prob = rw.Problem(m)
    spec = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
    prob.anneal(spec, rw.SolverConfig(seed=1, budget=1e6, steps_per_temperature=2), chains=592, schedule="calibrated")
    for chains in [int(a) for a in sys.argv[1:]] or [592, 1184, 2368, 4736]:
        t0 = time.perf_counter()
        for steps in (256, 512, 1024, 2048, 4096, 8192):
            t1 = time.perf_counter()
            order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                               chains=chains, schedule="calibrated")
            last = time.perf_counter() - t1
            if cost <= target:
                break
        print(json.dumps({"chains": chains, "steps_per_level": steps, "reached": cost <= target, "cost": cost,
                          "seconds_cumulative": time.perf_counter() - t0, "seconds_last_run": last,
                          "evaluations": ev}), flush=True)


if __name__ == "__main__":
    main()
