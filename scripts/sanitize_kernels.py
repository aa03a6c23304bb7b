#!/usr/bin/env python3
"""Small invocation of every kernel family (all scoring paths including the
validation branches, exhaustive, local search, anneal, simulate):

    python scripts/sanitize_kernels.py

Written as the workload for compute-sanitizer (memcheck / racecheck /
synccheck); the tool is closed on the current GPU pool, so the script runs
plain and parity is carried by tests/.
"""
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main():
    import paper_2105_14088_b200 as rw
    A, S = rw.Algorithm, rw.fixtures.SIZE_FIXED
    rng = np.random.default_rng(0)
    # K1: smem paths (C1), all models, host int32 orders, exact and fast
    m1 = rw.fixtures.config_matrix("C1", "fixed")
    p1 = rw.Problem(m1)
    o1 = np.array([rng.permutation(64) for _ in range(37)], dtype=np.int32)
    for alg in range(4):
        spec = rw.CollectiveSpec(A(alg), 64, S)
        p1.evaluate_batch(spec, o1)
        p1.evaluate_batch(spec, o1, exact=True)
    # K1 beyond shared memory: ring (transpose, l2, cluster) and HD transpose at N=1024
    m4 = rw.fixtures.config_matrix("C4", "fixed")
    o4 = np.array([rng.permutation(1024) for _ in range(70)], dtype=np.int32)
    for path in ("transpose", "l2", "cluster"):
        p = rw.Problem(m4)
        p.set_path(path)
        p.evaluate_batch(rw.CollectiveSpec(A.Ring, 1024, S), o4)
    p = rw.Problem(m4)
    for pair in (rw.HdPairing.PaperFormula, rw.HdPairing.XorPairing):
        p.evaluate_batch(rw.CollectiveSpec(A.HalvingDoubling, 1024, S, 2, rw.CostMode.LatencyTimesSize, pair), o4)
    p.evaluate_batch(rw.CollectiveSpec(A.DoubleBinaryTree, 1024, S), o4[:8])
    # invalid orders through the transpose paths (validation branches)
    bad = o4.copy()
    bad[3, 5] = bad[3, 6]
    for alg in (0, 1):
        try:
            p.evaluate_batch(rw.CollectiveSpec(A(alg), 1024, S), bad)
        except rw.DomainError:
            pass
    # K2 exhaustive, K3 local search (ring + full models), K4 anneal (ring + full)
    m2 = rw.fixtures.config_matrix("C2")
    rw.brute_force(rw.CostMatrix.from_array(m2[:9, :9].copy()), rw.CollectiveSpec(A.Ring, 9, 1.0), threshold=9)
    m8 = np.ascontiguousarray(m2[:8, :8])
    for alg in range(4):
        rw.brute_force(rw.CostMatrix.from_array(m8), rw.CollectiveSpec(A(alg), 8, 1024.0), threshold=8)
    o3 = o1[:4]
    for alg in (0, 1, 2):
        p1.local_search(rw.CollectiveSpec(A(alg), 64, S), o3, max_rounds=50)
    for alg in (0, 2):
        p1.anneal(rw.CollectiveSpec(A(alg), 64, S), rw.SolverConfig(seed=1, steps_per_temperature=8), chains=16,
                  schedule="calibrated")
    rw.Problem(m4).anneal(rw.CollectiveSpec(A.Ring, 1024, S), rw.SolverConfig(seed=1, steps_per_temperature=4),
                          chains=8, schedule="calibrated")
    # simulate_collective
    levels = [(8, 5, 1000, 1), (8, 25, 1000, 4)]
    mt = rw.CostMatrix.from_array(rw.generate_matrix(levels, 0.1, 3))
    rw.simulate_batch(mt, levels, rw.CollectiveSpec(A.Ring, 64, 1e6), o1[:5])
    print("sanitize workload done")


if __name__ == "__main__":
    main()
