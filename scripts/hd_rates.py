#!/usr/bin/env python3
"""Halving-doubling (xor) rates on the non-transpose paths: C1 / C3 scoring
(matrix in shared memory), C5 small batches (L2 gathers), C1 single-chain
annealing proposals/s.

    python scripts/hd_rates.py
"""
import sys
import time

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2105_14088_b200 as rw
    A, P = rw.Algorithm, rw.HdPairing
    for cfg, count in (("C1", 1 << 20), ("C3", 1 << 19), ("C5", 256)):
        m = rw.fixtures.config_matrix(cfg, "fixed")
        n = m.shape[0]
        prob = rw.Problem(m)
        spec = rw.CollectiveSpec(A.HalvingDoubling, n, rw.fixtures.SIZE_FIXED, 2, rw.CostMode.LatencyTimesSize,
                                 P.XorPairing)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(3)
        o = torch.rand((count, n), device="cuda", generator=gen).argsort(dim=1).to(torch.int16)
        c = torch.empty(count, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream()
        prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        prob.sync_errors()
        print(f"{cfg} hd-xor scoring ({count} orders) {5 * count / (e0.elapsed_time(e1) / 1e3):.4e} evals/s", flush=True)
    m = rw.fixtures.config_matrix("C1", "fixed")
    prob = rw.Problem(m)
    spec = rw.CollectiveSpec(A.HalvingDoubling, 64, rw.fixtures.SIZE_FIXED, 2, rw.CostMode.LatencyTimesSize,
                             P.XorPairing)
    t = time.perf_counter()
    order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6), chains=1, max_proposals=2000000)
    dt = time.perf_counter() - t
    print(f"C1 hd-xor anneal 1 chain: {rep['proposals'] / dt:.4e} proposals/s, cost {cost:.6e}", flush=True)


if __name__ == "__main__":
    main()
