#!/usr/bin/env python3
"""Randomised parity sweep (GPU): random matrices (fixed point / FP32 / FP64,
symmetric or not, optionally with NaN, negative and -0.0 entries), random
orders, every model and kernel path, against the oracle port.  Bit-exact for
every max-based model and for ring on fixed point; ring on FP32/FP64 within
1e-12 relative (the reference's own summation order is reproduced only by
the exact mode, which is checked too).  Single-order evaluate() calls go
through the resident evaluator (rw_problem_set_resident) and are held to the
reference bits.

    python scripts/fuzz_parity.py [seconds]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")


def main():
    import paper_2105_14088_b200 as rw
    from oracle.pyoracle import Port, make_spec
    port = Port()
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = np.random.default_rng(int(time.time()) % 100000)
    t0 = time.time()
    cases = fails = 0
    while time.time() - t0 < budget:
        n = int(rng.choice([8, 16, 64, 128, 256, 512, 1024, 2048, 4096]))
        kind = rng.choice(["u16", "f32", "f64"])
        sym = bool(rng.integers(0, 2))
        dirty = kind == "f64" and rng.random() < 0.3
        if kind == "u16":
            a = rng.integers(0, 6000, size=(n, n)).astype(np.float64) / 8.0
        elif kind == "f32":
            a = (rng.random((n, n)) * 300.0).astype(np.float32).astype(np.float64)
        else:
            a = rng.random((n, n)) * 300.0
        if dirty:
            a[rng.random((n, n)) < 0.01] = np.nan
            a[rng.random((n, n)) < 0.03] *= -1.0
            a[rng.random((n, n)) < 0.01] = -0.0
        m = (np.triu(a, 1) + np.triu(a, 1).T) if sym else a.copy()
        np.fill_diagonal(m, 0.0)
        if sym and dirty:
            m[np.isnan(m)] = 1.5
        perms = np.array([rng.permutation(n) for _ in range(int(rng.choice([1, 7, 300, 700])))], dtype=np.int32)
        probs = {}
        for path in ("auto", "l2", "transpose"):
            probs[path] = rw.Problem(m)
            probs[path].set_path(path)
        models = [(0, 2, 0)]
        models += [(1, 2, 0), (1, 2, 1), (2, 2, 0), (3, 2, 0)]
        if n in (16, 64, 256, 1024):
            models.append((3, 4, 0))
        if n in (64, 512):
            models.append((3, 8, 0))
        for alg, b, pair in models:
            for mode in (1, 0):
                spec = rw.CollectiveSpec(rw.Algorithm(alg), n, 2.0 ** 17, b, rw.CostMode(mode), rw.HdPairing(pair))
                ospec = make_spec(alg, n, 2.0 ** 17, b, mode, pair)
                k = min(len(perms), 12)
                want = port.evaluate_batch(m, perms[:k], ospec)
                for path, prob in probs.items():
                    got = prob.evaluate_batch(spec, perms)
                    cases += 1
                    exact_needed = alg != 0 or kind == "u16"
                    if exact_needed:
                        ok = np.array_equal(got[:k], want, equal_nan=True)
                    else:
                        ok = np.allclose(got[:k], want, rtol=1e-12, atol=0, equal_nan=True)
                        ex = prob.evaluate_batch(spec, perms[:k], exact=True)
                        ok = ok and np.array_equal(ex, want, equal_nan=True)
                    if not ok:
                        fails += 1
                        bad = np.nonzero(~np.isclose(got[:k], want, rtol=0, atol=0, equal_nan=True))[0]
                        print(f"MISMATCH n={n} kind={kind} sym={sym} dirty={dirty} alg={alg} b={b} pair={pair} "
                              f"mode={mode} path={path} batch={len(perms)} rows={bad[:5].tolist()} "
                              f"got={got[bad[:3]].tolist()} want={want[bad[:3]].tolist()}", flush=True)
        # the other host layouts (uint16, packed) and device-resident orders score the same
        if n <= 4096 and len(perms) >= 7:
            # (the fast ring sum on FP matrices is path-dependent within 1e-12: compare exact sums)
            spec = rw.CollectiveSpec(rw.Algorithm(0), n, 2.0 ** 17)
            ex = kind != "u16"
            base = probs["auto"].evaluate_batch(spec, perms, exact=ex)
            bits = rw.api.packed_bits(n)
            got_u16 = probs["auto"].evaluate_batch(spec, perms.astype(np.uint16), exact=ex)
            got_pk = probs["auto"].evaluate_batch_packed(spec, rw.api.pack_orders(perms, bits), bits, len(perms),
                                                         exact=ex)
            cases += 2
            for name, got in (("u16", got_u16), ("packed", got_pk)):
                if not np.array_equal(got, base, equal_nan=True):
                    fails += 1
                    print(f"LAYOUT MISMATCH {name} n={n} kind={kind} batch={len(perms)}", flush=True)
        # single-order evaluate() through the resident evaluator (exact path)
        res = rw.Problem(m)
        res.set_resident(300)
        for alg, b, pair in models:
            for mode in (1, 0):
                spec = rw.CollectiveSpec(rw.Algorithm(alg), n, 2.0 ** 17, b, rw.CostMode(mode), rw.HdPairing(pair))
                want = port.evaluate_batch(m, perms[:2], make_spec(alg, n, 2.0 ** 17, b, mode, pair))
                got = np.array([res.evaluate(spec, perms[k]) for k in range(min(2, len(perms)))])
                cases += 1
                if not np.array_equal(got, want[:len(got)], equal_nan=True):
                    fails += 1
                    print(f"RESIDENT MISMATCH n={n} kind={kind} sym={sym} dirty={dirty} alg={alg} b={b} "
                          f"pair={pair} mode={mode} got={got.tolist()} want={want.tolist()}", flush=True)
        res.close()
        del probs
    print(f"fuzz: {cases} comparisons, {fails} mismatches, {time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
