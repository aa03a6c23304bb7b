"""TEST INFRASTRUCTURE ONLY: ctypes access to the oracles.

* ``Port``      -- oracle/librw_oracle.so, the plain-C restatement of the
                   reference algorithms (oracle/rw_oracle.c).
* ``Reference`` -- oracle/_ref/librankweave_ref.so, the unmodified reference
                   sources compiled by oracle/Makefile (present when the
                   reference tree was available at build time; it travels to
                   the GPU box as a built artefact).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs use this module, and only as the checker or the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "librw_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "librankweave_ref.so")

P = C.POINTER


class Spec(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("n", C.c_int32), ("size_bytes", C.c_double),
                ("bcube_b", C.c_int32), ("cost_mode", C.c_int32), ("hd_pairing", C.c_int32)]


def make_spec(algorithm=0, n=0, size_bytes=1.0, bcube_b=2, cost_mode=1, hd_pairing=0) -> Spec:
    return Spec(int(algorithm), int(n), float(size_bytes), int(bcube_b), int(cost_mode), int(hd_pairing))


def _d(a):
    return a.ctypes.data_as(P(C.c_double))


def _i(a):
    return a.ctypes.data_as(P(C.c_int32))


class Port:
    """The C restatement (always buildable with gcc)."""

    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run make -C oracle")
        L = self.lib = C.CDLL(path)
        L.rwo_evaluate.argtypes = [P(C.c_double), C.c_int32, P(C.c_int32), P(Spec), P(C.c_double)]
        L.rwo_evaluate_batch.argtypes = [P(C.c_double), C.c_int32, P(C.c_int32), C.c_int64, P(Spec), P(C.c_double)]
        L.rwo_brute_force.argtypes = [P(C.c_double), P(Spec), C.c_int32, P(C.c_int32), P(C.c_double),
                                      P(C.c_uint64)]
        L.rwo_distribution_stats.argtypes = [P(C.c_double), C.c_int32, P(C.c_double)]
        L.rwo_splitmix64.restype = C.c_uint64
        L.rwo_splitmix64.argtypes = [C.c_uint64]
        L.rwo_substream.restype = C.c_uint64
        L.rwo_substream.argtypes = [C.c_uint64, C.c_uint64]
        L.rwo_lookups.restype = C.c_int64
        L.rwo_lookups.argtypes = [P(Spec)]
        L.rwo_round_bytes.restype = C.c_double
        L.rwo_round_bytes.argtypes = [C.c_double, C.c_int32, C.c_int32]

    def evaluate(self, m: np.ndarray, perm, spec: Spec) -> float:
        m = np.ascontiguousarray(m, dtype=np.float64)
        p = np.ascontiguousarray(perm, dtype=np.int32)
        out = C.c_double()
        if self.lib.rwo_evaluate(_d(m), m.shape[0], _i(p), C.byref(spec), C.byref(out)) != 0:
            raise ValueError("oracle: invalid inputs")
        return out.value

    def evaluate_batch(self, m: np.ndarray, perms: np.ndarray, spec: Spec) -> np.ndarray:
        m = np.ascontiguousarray(m, dtype=np.float64)
        p = np.ascontiguousarray(perms, dtype=np.int32)
        out = np.empty(p.shape[0], dtype=np.float64)
        if self.lib.rwo_evaluate_batch(_d(m), m.shape[0], _i(p), p.shape[0], C.byref(spec), _d(out)) != 0:
            raise ValueError("oracle: invalid inputs")
        return out

    def brute_force(self, m: np.ndarray, spec: Spec, threshold: int = 16):
        m = np.ascontiguousarray(m, dtype=np.float64)
        perm = np.empty(spec.n, dtype=np.int32)
        cost = C.c_double()
        ev = C.c_uint64()
        rc = self.lib.rwo_brute_force(_d(m), C.byref(spec), threshold, _i(perm), C.byref(cost), C.byref(ev))
        if rc != 0:
            raise ValueError("oracle: invalid inputs")
        return perm, cost.value, ev.value

    def distribution_stats(self, v) -> tuple:
        a = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(4, dtype=np.float64)
        if self.lib.rwo_distribution_stats(_d(a), a.size, _d(out)) < 0:
            raise ValueError("no samples")
        return tuple(float(x) for x in out)

    def lookups(self, spec: Spec) -> int:
        return int(self.lib.rwo_lookups(C.byref(spec)))


class Reference:
    """The reference library itself (oracle/_ref)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run make -C oracle ref (needs /root/reference)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_evaluate_batch.argtypes = [P(C.c_double), C.c_int32, P(Spec), P(C.c_int32), C.c_int64,
                                         P(C.c_double), C.c_int32]
        L.ref_brute_force.argtypes = [P(C.c_double), P(Spec), C.c_int32, P(C.c_int32), P(C.c_double),
                                      P(C.c_uint64)]
        L.ref_anneal.argtypes = [P(C.c_double), P(Spec), C.c_double, C.c_uint64, C.c_double, C.c_double,
                                 C.c_int32, C.c_int32, P(C.c_int32), P(C.c_double), P(C.c_uint64)]
        L.ref_generate_matrix.argtypes = [C.c_int32, P(C.c_int32), P(C.c_double), P(C.c_double), P(C.c_double),
                                          C.c_double, C.c_uint64, P(C.c_double), C.c_int32]
        L.ref_expand_schedule.argtypes = [P(Spec), P(C.c_int32), P(C.c_int32), P(C.c_double), C.c_int64,
                                          P(C.c_int64)]
        L.ref_sample_costs.argtypes = [P(C.c_double), P(Spec), C.c_int32, C.c_uint64, P(C.c_double)]
        L.ref_distribution_stats.argtypes = [P(C.c_double), C.c_int32, P(C.c_double)]
        L.ref_sample_orders.argtypes = [C.c_int32, C.c_int32, C.c_uint64, P(C.c_int32)]
        L.ref_emit_smtlib.argtypes = [P(C.c_double), P(Spec), C.c_int32, C.c_double, C.c_int32, C.c_char_p,
                                      C.c_int64, P(C.c_int64)]

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            raise ValueError(f"reference: {msg}")

    def evaluate_batch(self, m, perms, spec: Spec, threads: int = 1) -> np.ndarray:
        m = np.ascontiguousarray(m, dtype=np.float64)
        p = np.ascontiguousarray(perms, dtype=np.int32)
        out = np.empty(p.shape[0], dtype=np.float64)
        self._check(self.lib.ref_evaluate_batch(_d(m), m.shape[0], C.byref(spec), _i(p), p.shape[0], _d(out),
                                                threads))
        return out

    def brute_force(self, m, spec: Spec, threshold: int = 16):
        m = np.ascontiguousarray(m, dtype=np.float64)
        perm = np.empty(spec.n, dtype=np.int32)
        cost = C.c_double()
        ev = C.c_uint64()
        self._check(self.lib.ref_brute_force(_d(m), C.byref(spec), threshold, _i(perm), C.byref(cost),
                                             C.byref(ev)))
        return perm, cost.value, ev.value

    def anneal(self, m, spec: Spec, budget_s=10.0, seed=0, t0=0.0, cooling=0.995, steps=0, restarts=4):
        m = np.ascontiguousarray(m, dtype=np.float64)
        perm = np.empty(spec.n, dtype=np.int32)
        cost = C.c_double()
        ev = C.c_uint64()
        self._check(self.lib.ref_anneal(_d(m), C.byref(spec), budget_s, seed, t0, cooling, steps, restarts,
                                        _i(perm), C.byref(cost), C.byref(ev)))
        return perm, cost.value, ev.value

    def generate_matrix(self, levels, jitter=0.0, seed=0) -> np.ndarray:
        fan = np.array([l[0] for l in levels], dtype=np.int32)
        lat = np.array([l[1] for l in levels], dtype=np.float64)
        bw = np.array([l[2] for l in levels], dtype=np.float64)
        ov = np.array([l[3] for l in levels], dtype=np.float64)
        n = int(np.prod(fan))
        out = np.empty((n, n), dtype=np.float64)
        self._check(self.lib.ref_generate_matrix(len(levels), _i(fan), _d(lat), _d(bw), _d(ov), jitter, seed,
                                                 _d(out), n))
        return out

    def expand_schedule(self, spec: Spec):
        sem = C.c_int32()
        count = C.c_int64()
        self._check(self.lib.ref_expand_schedule(C.byref(spec), C.byref(sem), None, None, 0, C.byref(count)))
        quad = np.empty((count.value, 4), dtype=np.int32)
        nbytes = np.empty(count.value, dtype=np.float64)
        self._check(self.lib.ref_expand_schedule(C.byref(spec), C.byref(sem), _i(quad), _d(nbytes), count.value,
                                                 C.byref(count)))
        return sem.value, quad, nbytes

    def sample_costs(self, m, spec: Spec, samples: int, seed: int) -> np.ndarray:
        m = np.ascontiguousarray(m, dtype=np.float64)
        out = np.empty(samples, dtype=np.float64)
        self._check(self.lib.ref_sample_costs(_d(m), C.byref(spec), samples, seed, _d(out)))
        return out


    def sample_orders(self, n: int, samples: int, seed: int) -> np.ndarray:
        out = np.empty((samples, n), dtype=np.int32)
        self._check(self.lib.ref_sample_orders(n, samples, seed, _i(out)))
        return out

    def emit_smtlib(self, m, spec: Spec, upper_bound=None, cap: int = 64) -> str:
        m = np.ascontiguousarray(m, dtype=np.float64)
        has = upper_bound is not None
        length = C.c_int64()
        self._check(self.lib.ref_emit_smtlib(_d(m), C.byref(spec), int(has), float(upper_bound or 0.0), cap, None, 0,
                                             C.byref(length)))
        buf = C.create_string_buffer(length.value + 1)
        self._check(self.lib.ref_emit_smtlib(_d(m), C.byref(spec), int(has), float(upper_bound or 0.0), cap, buf,
                                             length.value + 1, C.byref(length)))
        return buf.value.decode()


# The BASELINE config recipe, built from the reference alone --
# generate_matrix (topology.cpp:40-64) + the relabeling shuffle, which is
# sample_orders(n, 1, 14088) (stats.cpp:83-94: std::shuffle of the identity
# with mt19937_64(seed)) -- so the bench's reference arm never loads the
# product library.  Equal to paper_2105_14088_b200.fixtures.config_matrix
# (tests/test_oracle.py checks it).
CONFIG_LEVELS = {
    "C1": ([(8, 5, 1000, 1), (8, 25, 1000, 4)], True, None),
    "C2": ([(4, 5, 1000, 1), (4, 25, 1000, 4)], False, 13),
    "C3": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (2, 100, 1000, 4)], True, None),
    "C4": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (8, 100, 1000, 4)], True, None),
    "C5": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (32, 100, 1000, 4)], True, None),
}


def reference_config_matrix(ref: "Reference", name: str, kind: str = "fixed") -> np.ndarray:
    levels, relabel, trunc = CONFIG_LEVELS[name]
    m = ref.generate_matrix(levels, jitter=0.1, seed=2105)
    if trunc is not None:
        m = np.ascontiguousarray(m[:trunc, :trunc])
    if relabel:
        rl = ref.sample_orders(m.shape[0], 1, 14088)[0]
        m = np.ascontiguousarray(m[np.ix_(rl, rl)])
    if name == "C2":
        kind = "int"
    if kind == "f32":
        return m.astype(np.float32).astype(np.float64)
    if kind == "fixed":
        return np.clip(np.floor(m * 16.0 + 0.5), 0, 65535) / 16.0
    if kind == "int":
        return np.floor(m + 0.5)
    return m


def reference_available() -> bool:
    return os.path.exists(REF_PATH)
