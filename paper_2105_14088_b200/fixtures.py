"""Synthetic hierarchical-datacenter cost matrices for the BASELINE.json configs.

Recipe: generate_matrix (topology.cpp:40-64) with jitter 0.1
and seed 2105, host-relabeled by std::shuffle(iota(N), mt19937_64(14088)),
then one of two variants so the oracle and the GPU see identical values:

* ``f32``   -- every entry rounded through float; S = 1e8 bytes.
* ``fixed`` -- every entry rounded to q/16 us with q a uint16; S = 2^27, so
               every product and partial sum of the reference is exact and
               bit-exact parity is well defined.

Levels are (fanout, latency_us, bandwidth_B_per_us, oversubscription).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib, ptr
from .api import Algorithm, CollectiveSpec, CostMode, generate_matrix

CONFIGS = {
    # name: (levels, relabel, truncate_to)
    "C1": ([(8, 5, 1000, 1), (8, 25, 1000, 4)], True, None),
    "C2": ([(4, 5, 1000, 1), (4, 25, 1000, 4)], False, 13),
    "C3": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (2, 100, 1000, 4)], True, None),
    "C4": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (8, 100, 1000, 4)], True, None),
    "C5": ([(8, 5, 1000, 1), (16, 25, 1000, 4), (32, 100, 1000, 4)], True, None),
}

SIZE_F32 = 1e8
SIZE_FIXED = float(2 ** 27)


def relabel(m: np.ndarray, seed: int = 14088) -> np.ndarray:
    out = np.ascontiguousarray(m, dtype=np.float64).copy()
    check(lib.rw_relabel_matrix(ptr(out, C.c_double), out.shape[0], seed))
    return out


def base_matrix(name: str) -> np.ndarray:
    levels, do_relabel, trunc = CONFIGS[name]
    m = generate_matrix(levels, jitter=0.1, seed=2105)
    if trunc is not None:
        m = np.ascontiguousarray(m[:trunc, :trunc])
    if do_relabel:
        m = relabel(m)
    return m


def variant(m: np.ndarray, kind: str) -> np.ndarray:
    if kind == "f32":
        return m.astype(np.float32).astype(np.float64)
    if kind == "fixed":  # std::round semantics (half away from zero; entries are >= 0)
        q = np.clip(np.floor(m * 16.0 + 0.5), 0, 65535)
        return q / 16.0
    if kind == "int":
        return np.floor(m + 0.5)
    if kind == "f64":
        return m.copy()
    raise ValueError(kind)


def config_matrix(name: str, kind: str = "fixed") -> np.ndarray:
    """C2 is defined on integer microseconds; others take `kind`."""
    m = base_matrix(name)
    if name == "C2":
        return variant(m, "int")
    return variant(m, kind)


def size_for(kind: str) -> float:
    return SIZE_FIXED if kind == "fixed" else SIZE_F32


def ring_spec(n: int, size: float, mode: CostMode = CostMode.LatencyTimesSize) -> CollectiveSpec:
    return CollectiveSpec(Algorithm.Ring, n, size, 2, mode)
