#!/usr/bin/env python3
"""Anneal quality/time probe against the reference goldens (one GPU).

    python scripts/anneal_probe.py c4 4096 16384      # steps per level
    python scripts/anneal_probe.py c3dbt 1024
"""
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main():
    import paper_2105_14088_b200 as rw
    which = sys.argv[1]
    steps_list = [int(x) for x in sys.argv[2:]] or [4096]
    chains = int(os.environ.get("CHAINS", "0"))
    if which == "c4":
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "anneal_c4.json")))
        target = min(r["cost"] for r in g["results"])
        m = rw.fixtures.config_matrix("C4", "fixed")
        spec = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
    elif which == "c3dbt":
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "anneal.json")))
        print(json.dumps({k: v for k, v in g.items() if k != "results"})[:400])
        target = None
        m = rw.fixtures.config_matrix("C3", "fixed")
        spec = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
    else:
        raise SystemExit(which)
    prob = rw.Problem(m)
    for steps in steps_list:
        for sched in os.environ.get("SCHED", "calibrated").split(","):
            t = time.perf_counter()
            order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps),
                                               chains=chains, schedule=sched)
            dt = time.perf_counter() - t
            print(f"{which} steps={steps} sched={sched} cost={cost:.9e} target={target} "
                  f"reached={target is not None and cost <= target} evals={ev:.3e} {dt:.1f}s "
                  f"rate={ev / dt:.3e}/s rep={ {k: rep[k] for k in rep if k in ('chains', 'levels', 'levels_run', 'winner_chain')} }",
                  flush=True)


if __name__ == "__main__":
    main()
