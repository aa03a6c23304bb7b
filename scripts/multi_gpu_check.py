#!/usr/bin/env python3
"""Multi-GPU parity check, run under torchrun (one process per GPU, NCCL):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/multi_gpu_check.py

* exhaustive N=13 sharded over the ranks == the single-GPU optimum (golden 338)
* annealing with a fixed global chain count: identical result for any world size
* sharded batch scoring == single-GPU scoring
Prints one JSON line from rank 0 and exits non-zero on a mismatch.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def main():
    import torch
    import torch.distributed as dist

    import paper_2105_14088_b200 as rw
    from paper_2105_14088_b200 import dist as rwdist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", init_method="env://")
    r, w = rwdist.rank_world()
    out = {"world": w}

    # C2: matrix from rank 0 to everyone
    m13 = rwdist.broadcast_matrix(rw.fixtures.config_matrix("C2") if r == 0 else None, 13)
    p13 = rw.Problem(m13, device=local)
    spec13 = rw.CollectiveSpec(rw.Algorithm.Ring, 13, 1.0)
    torch.cuda.synchronize()
    dist.barrier()
    t = time.perf_counter()
    sol = rwdist.brute_force_sharded(p13, spec13, threshold=13)
    dist.barrier()
    out["exhaustive_n13"] = {"cost": sol.cost, "order": sol.order.perm, "seconds": time.perf_counter() - t}
    ok = sol.cost == 338.0 and sol.order.perm == [0, 1, 4, 5, 7, 6, 12, 8, 9, 10, 11, 3, 2]

    # annealing: global chain ids -> same answer at any world size
    m1 = rw.fixtures.config_matrix("C1", "fixed")
    p1 = rw.Problem(m1, device=local)
    spec1 = rw.fixtures.ring_spec(64, rw.fixtures.SIZE_FIXED)
    cfg = rw.SolverConfig(seed=11, steps_per_temperature=32)
    sol_s, rep = rwdist.anneal_sharded(p1, spec1, cfg, chains_total=64)
    single = p1.anneal(spec1, cfg, chains=64) if r == 0 else None
    if r == 0:
        same = (single[1] == sol_s.cost and single[0].tolist() == sol_s.order.perm and
                single[3]["winner_chain"] == rep["winner_chain"])
        out["anneal_sharded_equals_single"] = same
        ok = ok and same

    # batch scoring sharded
    m4 = rw.fixtures.config_matrix("C4", "fixed")
    p4 = rw.Problem(m4, device=local)
    spec4 = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
    rng = np.random.default_rng(3)
    orders = np.array([rng.permutation(1024) for _ in range(1000)], dtype=np.int32)
    shard = rwdist.evaluate_batch_sharded(p4, spec4, orders)
    if r == 0:
        same = bool(np.array_equal(shard, p4.evaluate_batch(spec4, orders)))
        out["batch_sharded_equals_single"] = same
        ok = ok and same
    flag = torch.tensor([1 if ok or r != 0 else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if r == 0:
        out["ok"] = bool(flag.item())
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if flag.item() else 1


if __name__ == "__main__":
    sys.exit(main())
