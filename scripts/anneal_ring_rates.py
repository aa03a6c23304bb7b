#!/usr/bin/env python3
"""C4 ring annealing throughput: proposals/s for 592 chains (4 per SM) and
65,536 chains, a fixed number of steps per level.

    python scripts/anneal_ring_rates.py
"""
import sys
import time

sys.path.insert(0, ".")


def main():
    import paper_2105_14088_b200 as rw
    m = rw.fixtures.config_matrix("C4", "fixed")
    prob = rw.Problem(m)
    spec = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
    for chains, steps in ((592, 256), (65536, 16)):
        cfg = rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=steps)
        prob.anneal(spec, rw.SolverConfig(seed=1, budget=1e6, steps_per_temperature=2), chains=chains,
                    schedule="calibrated")
        t = time.perf_counter()
        order, cost, ev, rep = prob.anneal(spec, cfg, chains=chains, schedule="calibrated")
        dt = time.perf_counter() - t
        print(f"chains {chains} steps {steps}: {rep['proposals'] / dt:.4e} proposals/s "
              f"({rep['proposals'] / dt / chains:.4e} per chain), cost {cost:.6e}, {dt:.2f} s", flush=True)


if __name__ == "__main__":
    main()
