"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/librankweave_ref.so, built
by `make -C oracle ref` from /root/reference sources).  The GPU box never runs
this; it reads the committed .npz / .json files.

    python tests/golden/make_golden.py            # fast goldens (~1 min)
    python tests/golden/make_golden.py --slow     # + N=13 exhaustive, anneal baselines

Contents
  batch_<cfg>_<variant>.npz : seeded random orders and the reference's cost for
                              every applicable model/spec on the BASELINE
                              config matrices (fixtures.py recipe)
  random_small.npz          : random FP64 matrices N=2..32 (generic, asymmetric
                              too) with orders and reference costs, both modes
  brute.json                : reference brute_force results (N=8 all models,
                              ring N=8..12, and N=13 with --slow)
  anneal.json (--slow)      : reference anneal at equal-budget settings
  sample.npz                : sample_orders for several (n, samples, seed) and
                              sample_costs on the config matrices
  smtlib.json               : emit_smtlib texts (ring / hd / dbt / bcube)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, make_spec  # noqa: E402
from paper_2105_14088_b200 import fixtures  # noqa: E402

ALGOS = {"ring": 0, "hd": 1, "dbt": 2, "bcube": 3}


def specs_for(n: int, size: float):
    out = [("ring", make_spec(0, n, size, 2, 1, 0)), ("ring_lat", make_spec(0, n, size, 2, 0, 0))]
    if n & (n - 1) == 0:
        out += [("hd_paper", make_spec(1, n, size, 2, 1, 0)), ("hd_xor", make_spec(1, n, size, 2, 1, 1)),
                ("dbt", make_spec(2, n, size, 2, 1, 0)), ("bcube2", make_spec(3, n, size, 2, 1, 0))]
        for b in (4, 8):
            k = n
            while k % b == 0:
                k //= b
            if k == 1:
                out.append((f"bcube{b}", make_spec(3, n, size, b, 1, 0)))
    return out


def spec_dict(s):
    return {f: getattr(s, f) for f, _ in s._fields_}


def batch_goldens(ref: Reference):
    counts = {"C1": 64, "C3": 32, "C4": 16, "C5": 6}
    for cfg, k in counts.items():
        for kind in ("fixed", "f32"):
            m = fixtures.config_matrix(cfg, kind)
            n = m.shape[0]
            rng = np.random.default_rng(1000 + n)
            perms = np.stack([np.arange(n)] + [rng.permutation(n) for _ in range(k - 1)]).astype(np.int32)
            payload = {"perms": perms.astype(np.uint16)}
            names = []
            for name, s in specs_for(n, fixtures.size_for(kind)):
                if name.startswith(("hd_xor", "bcube2")) and n >= 4096:
                    pass
                payload[f"cost_{name}"] = ref.evaluate_batch(m, perms, s, threads=8)
                payload[f"spec_{name}"] = np.array([s.algorithm, s.n, s.bcube_b, s.cost_mode, s.hd_pairing],
                                                   dtype=np.int64)
                payload[f"size_{name}"] = np.array([s.size_bytes])
                names.append(name)
            np.savez_compressed(os.path.join(HERE, f"batch_{cfg}_{kind}.npz"), **payload)
            print(f"batch {cfg} {kind}: n={n} orders={k} specs={names}", flush=True)


def random_small(ref: Reference):
    rng = np.random.default_rng(7)
    payload = {}
    idx = 0
    for n in (1, 2, 3, 4, 5, 8, 9, 13, 16, 27, 32):
        for rep in range(3):
            sym = rep != 1
            m = rng.uniform(1.0, 1000.0, (n, n))
            if sym:
                m = np.triu(m, 1)
                m = m + m.T
            np.fill_diagonal(m, 0.0)
            perms = np.stack([np.arange(n)] + [rng.permutation(n) for _ in range(15)]).astype(np.int32)
            size = float(rng.uniform(1.0, 1e7))
            cases = [("ring", 0, 2, 0)]
            if n & (n - 1) == 0:
                cases += [("hd_paper", 1, 2, 0), ("hd_xor", 1, 2, 1), ("dbt", 2, 2, 0), ("bcube2", 3, 2, 0)]
            if n in (4, 16):
                cases.append(("bcube4", 3, 4, 0))
            if n in (9, 27):
                cases.append(("bcube3", 3, 3, 0))
            for name, alg, b, pair in cases:
                for mode in (0, 1):
                    s = make_spec(alg, n, size, b, mode, pair)
                    c = ref.evaluate_batch(m, perms, s)
                    payload[f"m{idx}"] = m
                    payload[f"p{idx}"] = perms
                    payload[f"c{idx}"] = c
                    payload[f"s{idx}"] = np.array([alg, n, b, mode, pair], dtype=np.int64)
                    payload[f"z{idx}"] = np.array([size])
                    idx += 1
    payload["count"] = np.array([idx])
    np.savez_compressed(os.path.join(HERE, "random_small.npz"), **payload)
    print(f"random_small: {idx} cases", flush=True)


def brute_goldens(ref: Reference, slow: bool):
    out = {"matrix16_int": fixtures.config_matrix("C2", "int").tolist()}
    base = np.array(fixtures.variant(fixtures.base_matrix("C2"), "int"))
    m8 = base[:8, :8]
    res = []
    for name, s in [("ring", make_spec(0, 8, 1024.0, 2, 1, 0)), ("hd_paper", make_spec(1, 8, 1024.0, 2, 1, 0)),
                    ("hd_xor", make_spec(1, 8, 1024.0, 2, 1, 1)), ("dbt", make_spec(2, 8, 1024.0, 2, 1, 0)),
                    ("bcube2", make_spec(3, 8, 1024.0, 2, 1, 0)), ("bcube8", make_spec(3, 8, 1024.0, 8, 1, 0))]:
        perm, cost, ev = ref.brute_force(m8, s, 16)
        res.append({"name": name, "n": 8, "spec": spec_dict(s), "order": perm.tolist(), "cost": cost,
                    "evaluations": ev})
        print("brute", name, cost, perm.tolist(), flush=True)
    top = 13 if slow else 12
    for k in range(8, top + 1):
        s = make_spec(0, k, 1.0, 2, 1, 0)
        t = time.time()
        perm, cost, ev = ref.brute_force(base[:k, :k], s, 16)
        res.append({"name": "ring_block", "n": k, "spec": spec_dict(s), "order": perm.tolist(), "cost": cost,
                    "evaluations": ev, "seconds": time.time() - t})
        print("brute ring", k, cost, perm.tolist(), f"{time.time() - t:.1f}s", flush=True)
    out["results"] = res
    path = os.path.join(HERE, "brute.json")
    if os.path.exists(path) and not slow:  # keep slow results from an earlier --slow run
        old = json.load(open(path))
        keep = [r for r in old.get("results", []) if r["name"] == "ring_block" and r["n"] > top]
        out["results"] += keep
    json.dump(out, open(path, "w"), indent=1)


def anneal_goldens(ref: Reference):
    """Reference anneal with a non-binding budget (SURVEY 8(d) fixed-budget plan)."""
    from concurrent.futures import ThreadPoolExecutor
    jobs = []
    m1 = fixtures.config_matrix("C1", "fixed")
    for seed in range(10):
        jobs.append(("C1", "fixed", "ring", seed, m1, make_spec(0, 64, fixtures.SIZE_FIXED, 2, 1, 0), 0))
    m3 = fixtures.config_matrix("C3", "fixed")
    jobs.append(("C3", "fixed", "ring", 0, m3, make_spec(0, 256, fixtures.SIZE_FIXED, 2, 1, 0), 0))
    jobs.append(("C3", "fixed", "dbt", 0, m3, make_spec(2, 256, fixtures.SIZE_FIXED, 2, 1, 0), 0))

    def run(job):
        cfg, kind, model, seed, m, s, steps = job
        t = time.time()
        perm, cost, ev = ref.anneal(m, s, budget_s=1e6, seed=seed, steps=steps)
        return {"config": cfg, "variant": kind, "model": model, "seed": seed, "n": s.n, "cost": cost,
                "evaluations": ev, "order": perm.tolist(), "seconds": time.time() - t,
                "identity_cost": float(ref.evaluate_batch(m, np.arange(s.n, dtype=np.int32)[None, :], s)[0])}

    with ThreadPoolExecutor(8) as ex:
        results = list(ex.map(run, jobs))
    for r in results:
        print("anneal", r["config"], r["model"], r["seed"], r["cost"], r["evaluations"], f"{r['seconds']:.1f}s")
    json.dump({"results": results, "budget_s": 1e6, "note": "reference anneal, default schedule, seeds as listed"},
              open(os.path.join(HERE, "anneal.json"), "w"), indent=1)


def anneal_c4_goldens(ref: Reference, seeds=(0, 1, 2, 3)):
    """C4 (N=1024 ring) reference anneal, full schedule (45,170,792 evaluations, ~1 h per seed)."""
    from concurrent.futures import ThreadPoolExecutor
    m = fixtures.config_matrix("C4", "fixed")
    s = make_spec(0, 1024, fixtures.SIZE_FIXED, 2, 1, 0)

    def run(seed):
        t = time.time()
        perm, cost, ev = ref.anneal(m, s, budget_s=1e6, seed=seed)
        return {"config": "C4", "variant": "fixed", "model": "ring", "seed": seed, "n": 1024, "cost": cost,
                "evaluations": ev, "order": perm.tolist(), "seconds": time.time() - t,
                "identity_cost": float(ref.evaluate_batch(m, np.arange(1024, dtype=np.int32)[None, :], s)[0])}

    with ThreadPoolExecutor(len(seeds)) as ex:
        results = list(ex.map(run, seeds))
    for r in results:
        print("anneal C4", r["seed"], r["cost"], r["evaluations"], f"{r['seconds']:.1f}s", flush=True)
    json.dump({"results": results, "budget_s": 1e6}, open(os.path.join(HERE, "anneal_c4.json"), "w"), indent=1)


SIM_TOPOLOGIES = {
    "t64": ([(8, 5, 1000, 1), (8, 25, 1000, 4)], 0.1, 2105),
    "t256": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (2, 100, 1000, 4)], 0.1, 2105),
}


def simulate_goldens(ref: Reference):
    """simulate_collective from the reference on random orders (simulate.cpp:81-138)."""
    import ctypes as C
    P = C.POINTER
    L = ref.lib
    L.ref_simulate_batch.argtypes = [C.c_int32, P(C.c_int32), P(C.c_double), P(C.c_double), P(C.c_double), C.c_double,
                                     C.c_uint64, P(type(make_spec())), P(C.c_int32), C.c_int64, P(C.c_double)]
    payload = {}
    for name, (levels, jitter, seed) in SIM_TOPOLOGIES.items():
        fan = np.array([l[0] for l in levels], dtype=np.int32)
        lat = np.array([l[1] for l in levels], dtype=np.float64)
        bw = np.array([l[2] for l in levels], dtype=np.float64)
        ov = np.array([l[3] for l in levels], dtype=np.float64)
        n = int(np.prod(fan))
        rng = np.random.default_rng(n)
        perms = np.stack([np.arange(n)] + [rng.permutation(n) for _ in range(7)]).astype(np.int32)
        payload[f"{name}_perms"] = perms
        cases = [("ring", 0, 2, 0), ("hd_paper", 1, 2, 0), ("hd_xor", 1, 2, 1), ("dbt", 2, 2, 0), ("bcube2", 3, 2, 0)]
        if name == "t64":
            cases += [("bcube4", 3, 4, 0), ("bcube8", 3, 8, 0)]
        for cname, alg, b, pair in cases:
            s = make_spec(alg, n, 1e6, b, 1, pair)
            out = np.empty(perms.shape[0], dtype=np.float64)
            rc = L.ref_simulate_batch(len(levels), fan.ctypes.data_as(P(C.c_int32)), lat.ctypes.data_as(P(C.c_double)),
                                      bw.ctypes.data_as(P(C.c_double)), ov.ctypes.data_as(P(C.c_double)), jitter, seed,
                                      C.byref(s), perms.ctypes.data_as(P(C.c_int32)), perms.shape[0],
                                      out.ctypes.data_as(P(C.c_double)))
            assert rc == 0, L.ref_last_error()
            payload[f"{name}_{cname}"] = out
            payload[f"{name}_{cname}_spec"] = np.array([alg, n, b, 1, pair], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "simulate.npz"), **payload)
    print("simulate goldens:", sorted(k for k in payload if not k.endswith(("_spec", "_perms"))), flush=True)


SAMPLE_CASES = [(1, 3, 0), (2, 5, 1), (7, 16, 0), (13, 32, 2105), (64, 16, 1234), (256, 4, 7), (1024, 3, 0),
                (4096, 2, 14088)]


def sample_goldens(ref: Reference):
    """sample_orders / sample_costs (stats.cpp:83-103): seeded orders and their costs."""
    payload = {}
    for n, k, seed in SAMPLE_CASES:
        payload[f"orders_{n}_{k}_{seed}"] = ref.sample_orders(n, k, seed)
    for cfg, kind in (("C1", "fixed"), ("C1", "f32"), ("C3", "fixed"), ("C4", "fixed"), ("C4", "f64")):
        m = fixtures.config_matrix(cfg, kind)
        n = m.shape[0]
        size = fixtures.size_for(kind)
        for name, spec in specs_for(n, size)[:4]:
            payload[f"costs_{cfg}_{kind}_{name}"] = ref.sample_costs(m, spec, 24, 99)
            payload[f"costs_{cfg}_{kind}_{name}_spec"] = np.array(
                [spec.algorithm, spec.n, spec.bcube_b, spec.cost_mode, spec.hd_pairing], dtype=np.int64)
            payload[f"costs_{cfg}_{kind}_{name}_size"] = np.array([spec.size_bytes])
    np.savez_compressed(os.path.join(HERE, "sample.npz"), **payload)
    print("sample goldens:", len(payload), "arrays", flush=True)


SMT_CASES = [  # (name, n, algorithm, size, mode, b, pairing, bound)
    ("ring2", 2, 0, 8.0, 0, 2, 0, None), ("ring2_bound", 2, 0, 8.0, 0, 2, 0, 12.5),
    ("ring5_size", 5, 0, 1e6, 1, 2, 0, 1e9), ("hd8_paper", 8, 1, 1000.0, 1, 2, 0, 3.25),
    ("hd8_xor", 8, 1, 1000.0, 1, 2, 1, None), ("dbt8", 8, 2, 1000.0, 1, 2, 0, 77.0),
    ("dbt4_lat", 4, 2, 1000.0, 0, 2, 0, None), ("bcube16_b4", 16, 3, 64.0, 1, 4, 0, None),
    ("bcube8_b2", 8, 3, 1e8, 1, 2, 0, 1.0 / 3.0)]


def smtlib_goldens(ref: Reference):
    """emit_smtlib (smtlib.cpp:104-158) texts on small random and fixture matrices."""
    rng = np.random.default_rng(2105)
    out = {}
    for name, n, alg, size, mode, b, pair, bound in SMT_CASES:
        m = rng.uniform(0.5, 300.0, size=(n, n))
        m[2 % n, 1 % n] = 0.0001220703125 if n > 1 else 0.0  # exercises the %.12f rounding
        np.fill_diagonal(m, 0.0)
        spec = make_spec(alg, n, size, b, mode, pair)
        out[name] = {"matrix": m.tolist(), "spec": [alg, n, size, b, mode, pair], "bound": bound,
                     "text": ref.emit_smtlib(m, spec, bound)}
    json.dump(out, open(os.path.join(HERE, "smtlib.json"), "w"))
    print("smtlib goldens:", list(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    ref = Reference()
    steps = a.only.split(",") if a.only else ["batch", "small", "brute"] + (["anneal"] if a.slow else [])
    if "batch" in steps:
        batch_goldens(ref)
    if "small" in steps:
        random_small(ref)
    if "brute" in steps:
        brute_goldens(ref, a.slow)
    if "anneal" in steps:
        anneal_goldens(ref)
    if "anneal_c4" in steps:
        anneal_c4_goldens(ref)
    if "simulate" in steps or not a.only:
        simulate_goldens(ref)
    if "sample" in steps or not a.only:
        sample_goldens(ref)
    if "smtlib" in steps or not a.only:
        smtlib_goldens(ref)


if __name__ == "__main__":
    main()
