#!/usr/bin/env python3
"""Tree-model (double binary tree) rates: C3 scoring and C3 single-chain
annealing proposals/s (the reference budget), C4/C5 scoring.

    python scripts/dbt_rates.py
"""
import json
import sys
import time

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2105_14088_b200 as rw
    A = rw.Algorithm
    g = json.load(open("tests/golden/anneal.json"))
    ref = [r for r in g["results"] if r["config"] == "C3" and r["model"] == "dbt"][0]
    for cfg, count in (("C3", 1 << 19), ("C4", 1 << 17), ("C5", 1 << 15)):
        m = rw.fixtures.config_matrix(cfg, "fixed")
        n = m.shape[0]
        prob = rw.Problem(m)
        spec = rw.CollectiveSpec(A.DoubleBinaryTree, n, rw.fixtures.SIZE_FIXED)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(3)
        o = torch.rand((count, n), device="cuda", generator=gen).argsort(dim=1).to(torch.int16)
        c = torch.empty(count, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream()
        prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        prob.sync_errors()
        print(f"{cfg} dbt scoring {3 * count / (e0.elapsed_time(e1) / 1e3):.4e} evals/s", flush=True)
    m = rw.fixtures.config_matrix("C3", "fixed")
    prob = rw.Problem(m)
    spec = rw.CollectiveSpec(A.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
    t = time.perf_counter()
    order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6), chains=1,
                                       max_proposals=ref["evaluations"])
    dt = time.perf_counter() - t
    print(f"C3 dbt anneal 1 chain: {rep['proposals'] / dt:.4e} proposals/s, cost {cost:.6e} "
          f"(reference {ref['cost']:.6e} at {ref['evaluations']} evals), {dt:.1f} s", flush=True)


if __name__ == "__main__":
    main()
