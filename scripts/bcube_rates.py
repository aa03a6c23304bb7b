#!/usr/bin/env python3
"""BCube scoring at C5 size (N=4096, B=4 and 8; u16 / FP32 / FP64 fixture
matrices): the L2-gather kernel against the source-compacted transpose path,
device-resident uint16 orders, CUDA events, parity of the first rows against
the oracle.

    python scripts/bcube_rates.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2105_14088_b200 as rw
    from oracle.pyoracle import Port, make_spec
    port = Port()
    count = 1 << 15
    for kind in ("fixed", "f32", "f64"):
        m = rw.fixtures.config_matrix("C5", kind)
        n = m.shape[0]
        size = rw.fixtures.size_for(kind)
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        o = torch.rand((count, n), device="cuda", generator=g).argsort(dim=1).to(torch.int16)
        c = torch.empty(count, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream()
        rows = o[:6].cpu().numpy().view(np.uint16).astype(np.int32)
        for b in (8, 4):
            spec = rw.CollectiveSpec(rw.Algorithm.BCube, n, size, b, rw.CostMode.LatencyTimesSize)
            want = port.evaluate_batch(m, rows, make_spec(3, n, size, b, 1, 0))
            for path in ("l2", "transpose"):
                prob = rw.Problem(m)
                prob.set_path(path)
                prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
                torch.cuda.synchronize()
                prob.sync_errors()
                ok = np.array_equal(c[:6].cpu().numpy(), want)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(3):
                    prob.evaluate_batch_device(spec, o.data_ptr(), 2, count, c.data_ptr(), st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                prob.sync_errors()
                rate = 3 * count / (e0.elapsed_time(e1) / 1e3)
                print(f"C5 bcube{b} {kind:5s} storage={prob.info['storage']} {path:9s} {rate:.4e} evals/s "
                      f"oracle_bits={'ok' if ok else 'MISMATCH'}", flush=True)
                prob.close()
        del o, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
