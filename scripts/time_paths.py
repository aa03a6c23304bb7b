#!/usr/bin/env python3
"""A/B throughput of the scoring paths (one GPU, device-resident uint16 orders,
CUDA-event timing after warm-up).  Prints one line per (config, model, path):

    python scripts/time_paths.py            # C4/C5 ring and halving-doubling, every path
"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2105_14088_b200 as rw
    A, P = rw.Algorithm, rw.HdPairing
    cases = [
        ("C4", "ring", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 20, ["l2", "transpose"]),
        ("C4", "hd-xor", lambda n, s: rw.CollectiveSpec(A.HalvingDoubling, n, s, 2, rw.CostMode.LatencyTimesSize,
                                                        P.XorPairing), 1 << 17, ["l2", "transpose"]),
        ("C5", "hd-xor", lambda n, s: rw.CollectiveSpec(A.HalvingDoubling, n, s, 2, rw.CostMode.LatencyTimesSize,
                                                        P.XorPairing), 1 << 16, ["l2", "transpose"]),
        ("C5", "hd-paper", lambda n, s: rw.CollectiveSpec(A.HalvingDoubling, n, s), 1 << 16, ["l2", "transpose"]),
        ("C5", "ring", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 16, ["l2", "transpose"]),
        ("C5h", "ring", lambda n, s: rw.CollectiveSpec(A.Ring, n, s), 1 << 17, ["l2", "transpose"]),
        ("C5h", "hd-xor", lambda n, s: rw.CollectiveSpec(A.HalvingDoubling, n, s, 2, rw.CostMode.LatencyTimesSize,
                                                         P.XorPairing), 1 << 15, ["l2", "transpose"]),
    ]
    only = sys.argv[1:]
    for cfg, name, spec_fn, count, paths in cases:
        if only and f"{cfg}-{name}" not in only:
            continue
        if cfg == "C5h":  # C5 truncated to 2048 hosts (crossover probe)
            m = rw.fixtures.config_matrix("C5", "fixed")[:2048, :2048].copy()
        else:
            m = rw.fixtures.config_matrix(cfg, "fixed")
        n = m.shape[0]
        spec = spec_fn(n, rw.fixtures.SIZE_FIXED)
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        o = torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
        st = torch.cuda.current_stream()
        ref = None
        for pth in paths:
            prob = rw.Problem(m)
            prob.set_path(pth)
            c = torch.empty(count, dtype=torch.float64, device="cuda")
            for _ in range(2):
                prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            prob.sync_errors()
            reps = 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            prob.sync_errors()
            ms = e0.elapsed_time(e1) / reps
            same = "" if ref is None else ("same" if torch.equal(c, ref) else "DIFFERENT")
            ref = c.clone() if ref is None else ref
            print(f"{cfg} {name:9s} {pth:10s} {count / (ms * 1e-3):12.4e} evals/s  {ms:9.3f} ms/launch {same}",
                  flush=True)
            del prob


if __name__ == "__main__":
    main()
