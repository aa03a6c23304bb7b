#!/usr/bin/env python3
"""Throughput of the scoring paths per matrix storage kind (one GPU,
device-resident uint16 orders, CUDA-event timing after warm-up).

A probed CostMatrix is FP64 (types.hpp:42-53); rw_problem_create stores it as
u16 fixed point when that is exact, else FP32 when exact, else FP64.  This
prints evals/s for the fixture variants that land on each storage kind and
checks the first rows against the oracle port:

    python scripts/time_storage.py                 # C4 ring, C5 HD xor/paper
    python scripts/time_storage.py C4-ring-f32     # one case
"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2105_14088_b200 as rw
    from oracle.pyoracle import Port, make_spec
    A, P = rw.Algorithm, rw.HdPairing
    port = Port()
    models = {
        "ring": (0, 0),
        "hd-xor": (1, 1),
        "hd-paper": (1, 0),
        "dbt": (2, 0),
        "bcube8": (3, 0),
    }
    cases = []
    for kind in ("fixed", "f32", "f64"):
        cases.append(("C4", "ring", kind, 1 << 20))
        cases.append(("C5", "hd-xor", kind, 1 << 15))
        cases.append(("C5", "hd-paper", kind, 1 << 15))
        cases.append(("C4", "dbt", kind, 1 << 17))
        cases.append(("C5", "dbt", kind, 1 << 15))
        cases.append(("C5", "bcube8", kind, 1 << 15))
    only = sys.argv[1:]
    names = {1: "u16", 2: "f32", 3: "f64"}
    for cfg, model, kind, count in cases:
        tag = f"{cfg}-{model}-{kind}"
        if only and tag not in only:
            continue
        m = rw.fixtures.config_matrix(cfg, kind)
        n = m.shape[0]
        size = rw.fixtures.size_for(kind)
        alg, pair = models[model]
        b = 8 if model == "bcube8" else 2
        spec = rw.CollectiveSpec(A(alg), n, size, b, rw.CostMode.LatencyTimesSize, P(pair))
        prob = rw.Problem(m)
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        o = torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
        c = torch.empty(count, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream()
        for _ in range(2):
            prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        prob.sync_errors()
        rows = o[:4].cpu().numpy().view(np.uint16).astype(np.int32)
        want = port.evaluate_batch(m, rows, make_spec(alg, n, size, b, 1, pair))
        got = c[:4].cpu().numpy()
        rel = float(np.max(np.abs(got - want) / np.abs(want)))
        reps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        prob.sync_errors()
        ms = e0.elapsed_time(e1) / reps
        print(f"{tag:22s} storage={names[prob.info['storage']]} {count / (ms * 1e-3):12.4e} evals/s "
              f"{ms:9.3f} ms/launch  max_rel_err_vs_oracle={rel:.3e}", flush=True)
        del prob, o, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
