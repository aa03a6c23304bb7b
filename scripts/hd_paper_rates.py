#!/usr/bin/env python3
"""HD paper-pairing scoring rates on the transpose path at N = 1024, 2048, 4096
(u16 and FP32 random matrices, device-resident uint16 orders, CUDA events).
A/B the compact layout with RW_HD_COMPACT=0.

    python scripts/hd_paper_rates.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2105_14088_b200 as rw
    from paper_2105_14088_b200 import _lib
    rng = np.random.default_rng(1)
    for n in (1024, 2048, 4096):
        for kind, storage in (("u16", _lib.RW_STORAGE_U16), ("f32", _lib.RW_STORAGE_F32)):
            m = rng.integers(1, 60000, size=(n, n)).astype(np.float64)
            if kind == "f32":
                m = (m * 0.375).astype(np.float32).astype(np.float64)
            m = np.triu(m, 1) + np.triu(m, 1).T
            prob = rw.Problem(m, storage)
            prob.set_path("transpose")
            spec = rw.CollectiveSpec(rw.Algorithm.HalvingDoubling, n, 1 << 20, 2, rw.CostMode.LatencyTimesSize,
                                     rw.HdPairing.PaperFormula)
            count = (1 << 27) // (n * 2) if n < 4096 else 1 << 15
            g = torch.Generator(device="cuda")
            g.manual_seed(3)
            o = torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
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
            print(f"N={n} {kind} hd-paper transpose {3 * count / (e0.elapsed_time(e1) / 1e3):.4e} evals/s", flush=True)
            del prob, o, c
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
