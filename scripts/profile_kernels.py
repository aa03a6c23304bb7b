#!/usr/bin/env python3
"""Small, fixed workloads for ncu captures (one GPU).

    python scripts/profile_kernels.py ring      # C4 ring scoring, 256K orders x 4 launches
    python scripts/profile_kernels.py all       # ring, hd-xor (C5), dbt (C3), exhaustive N=13, anneal C1

Run it plain first; then under ncu, e.g.
    ncu --set full --clock-control none --import-source on -k regex:k_ring -s 2 -c 1 -o gpurun_out/ring \
        python scripts/profile_kernels.py ring
"""
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def orders(torch, count, n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)


def score(torch, rw, cfg, kind, spec_fn, count, launches=4):
    m = rw.fixtures.config_matrix(cfg, kind)
    n = m.shape[0]
    prob = rw.Problem(m)
    spec = spec_fn(n, rw.fixtures.size_for(kind))
    o = orders(torch, count, n, 1)
    c = torch.empty(count, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(launches):
        prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st)
    torch.cuda.synchronize()
    prob.sync_errors()
    print(cfg, kind, spec.algorithm.name, "ok", float(c[0]))


def main():
    import torch

    import paper_2105_14088_b200 as rw
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    A = rw.Algorithm
    if which in ("ring", "all"):
        score(torch, rw, "C4", "fixed", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 18)
    if which in ("ring_f32", "all"):
        score(torch, rw, "C4", "f32", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 18)
    if which in ("ring_f64", "all"):
        score(torch, rw, "C4", "f64", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 18)
    if which in ("hdxor", "all"):
        score(torch, rw, "C5", "fixed",
              lambda n, s: rw.CollectiveSpec(A.HalvingDoubling, n, s, 2, rw.CostMode.LatencyTimesSize,
                                             rw.HdPairing.XorPairing), 1 << 12)
    if which in ("hdpaper", "all"):
        score(torch, rw, "C5", "fixed",
              lambda n, s: rw.CollectiveSpec(A.HalvingDoubling, n, s, 2, rw.CostMode.LatencyTimesSize,
                                             rw.HdPairing.PaperFormula), 1 << 12)
    if which in ("bcube8_c5", "all"):
        score(torch, rw, "C5", "fixed", lambda n, s: rw.CollectiveSpec(A.BCube, n, s, 8), 1 << 14)
    if which in ("dbt_c5", "all"):
        score(torch, rw, "C5", "fixed", lambda n, s: rw.CollectiveSpec(A.DoubleBinaryTree, n, s), 1 << 14)
    if which in ("dbt", "all"):
        score(torch, rw, "C3", "fixed", lambda n, s: rw.CollectiveSpec(A.DoubleBinaryTree, n, s), 1 << 16)
    if which in ("ring256", "all"):
        score(torch, rw, "C3", "fixed", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 18)
    if which in ("brute", "all"):
        m = rw.CostMatrix.from_array(rw.fixtures.config_matrix("C2"))
        for _ in range(2):
            sol = rw.brute_force(m, rw.CollectiveSpec(A.Ring, 13, 1.0), threshold=13)
        print("brute", sol.cost)
    if which in ("anneal", "all"):
        prob = rw.Problem(rw.fixtures.config_matrix("C1", "fixed"))
        spec = rw.fixtures.ring_spec(64, rw.fixtures.SIZE_FIXED)
        r = prob.anneal(spec, rw.SolverConfig(seed=0, steps_per_temperature=64))
        print("anneal", r[1], r[3])


if __name__ == "__main__":
    main()
