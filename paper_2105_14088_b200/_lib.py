"""ctypes binding of the C ABI in include/rankweave_c.h (librankweave_b200.so).

The shared library is built in-tree by ``make -C paper_2105_14088_b200`` (or
``__graft_entry__.build()``).  There is deliberately no fallback: if the
library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librankweave_b200.so")

RW_OK = 0
RW_ERR_IO = 2
RW_ERR_DOMAIN = 3
RW_ERR_CUDA = 5
RW_ERR_NCCL = 6
RW_ERR_INTERNAL = 7

RW_STORAGE_AUTO, RW_STORAGE_U16, RW_STORAGE_F32, RW_STORAGE_F64 = 0, 1, 2, 3
RW_EVAL_EXACT = 1
RW_EVAL_NO_VALIDATE = 2


class rw_spec(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("n", C.c_int32), ("size_bytes", C.c_double),
                ("bcube_b", C.c_int32), ("cost_mode", C.c_int32), ("hd_pairing", C.c_int32)]


class rw_solver_config(C.Structure):
    _fields_ = [("budget_s", C.c_double), ("seed", C.c_uint64), ("initial_temperature", C.c_double),
                ("cooling", C.c_double), ("steps_per_temperature", C.c_int32), ("restarts", C.c_int32),
                ("brute_force_threshold", C.c_int32), ("reserved", C.c_int32)]


class rw_gpu_config(C.Structure):
    _fields_ = [("chains", C.c_int32), ("chain_begin", C.c_int32), ("chain_total", C.c_int32),
                ("schedule", C.c_int32), ("max_proposals", C.c_int64)]


class rw_problem_info(C.Structure):
    _fields_ = [("n", C.c_int32), ("device", C.c_int32), ("storage", C.c_int32), ("frac_bits", C.c_int32),
                ("symmetric", C.c_int32), ("zero_diagonal", C.c_int32), ("device_bytes", C.c_int64),
                ("max_value", C.c_double)]


class rw_search_report(C.Structure):
    _fields_ = [("winner_chain", C.c_int64), ("chains", C.c_int64), ("proposals", C.c_int64),
                ("levels", C.c_int32), ("levels_run", C.c_int32), ("initial_temperature", C.c_double),
                ("seconds", C.c_double)]


class rw_gpu_options(C.Structure):
    _fields_ = [("device", C.c_int32), ("chains", C.c_int32), ("exact_batch", C.c_int32),
                ("immutable_matrices", C.c_int32), ("num_devices", C.c_int32),
                ("resident_idle_us", C.c_int32)]


class rw_eval_report(C.Structure):
    _fields_ = [("bit_exact", C.c_int32), ("kernel", C.c_int32), ("kernel_ms", C.c_float),
                ("lookups", C.c_int64)]


P = C.POINTER
_vp = C.c_void_p
_i32p = P(C.c_int32)
_dp = P(C.c_double)
_u64p = P(C.c_uint64)

# name -> (restype, argtypes); every symbol declared in include/rankweave_c.h
SIGNATURES = {
    "rw_last_error": (C.c_char_p, []),
    "rw_abi_version": (C.c_int32, []),
    "rw_device_count": (C.c_int32, []),
    "rw_validate_spec": (C.c_int, [P(rw_spec)]),
    "rw_problem_create": (C.c_int, [_dp, C.c_int32, C.c_int32, C.c_int32, P(_vp)]),
    "rw_problem_destroy": (C.c_int, [_vp]),
    "rw_problem_get_info": (C.c_int, [_vp, P(rw_problem_info)]),
    "rw_problem_set_path": (C.c_int, [_vp, C.c_int32]),
    "rw_evaluate": (C.c_int, [_vp, P(rw_spec), _i32p, _dp]),
    "rw_evaluate_batch": (C.c_int, [_vp, P(rw_spec), _i32p, C.c_int64, _dp, C.c_uint32, P(rw_eval_report)]),
    "rw_evaluate_batch_u16": (C.c_int, [_vp, P(rw_spec), P(C.c_uint16), C.c_int64, _dp, C.c_uint32,
                                        P(rw_eval_report)]),
    "rw_packed_row_bytes": (C.c_int64, [C.c_int32, C.c_int32]),
    "rw_pack_orders": (C.c_int, [_i32p, C.c_int32, C.c_int64, C.c_int32, _vp]),
    "rw_evaluate_batch_packed": (C.c_int, [_vp, P(rw_spec), _vp, C.c_int32, C.c_int64, _dp, C.c_uint32,
                                           P(rw_eval_report)]),
    "rw_evaluate_batch_device": (C.c_int, [_vp, P(rw_spec), _vp, C.c_int32, C.c_int64, _vp, _vp, C.c_uint32]),
    "rw_sync_errors": (C.c_int, [_vp, _vp]),
    "rw_schedule_cost": (C.c_int, [_vp, C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _dp, _i32p, C.c_int32,
                                   _i32p, _dp]),
    "rw_brute_force": (C.c_int, [_vp, P(rw_spec), C.c_int32, _i32p, _dp, _u64p]),
    "rw_brute_force_space": (C.c_int, [P(rw_spec), _u64p]),
    "rw_brute_force_range": (C.c_int, [_vp, P(rw_spec), C.c_uint64, C.c_uint64, _dp, _u64p]),
    "rw_unrank": (C.c_int, [P(rw_spec), C.c_uint64, _i32p]),
    "rw_anneal": (C.c_int, [_vp, P(rw_spec), P(rw_solver_config), P(rw_gpu_config), _i32p, _dp, _u64p,
                            P(rw_search_report)]),
    "rw_local_search": (C.c_int, [_vp, P(rw_spec), _i32p, C.c_int64, C.c_int32, _dp, _u64p]),
    "rw_sample_orders": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, _i32p]),
    "rw_sample_costs": (C.c_int, [_vp, P(rw_spec), C.c_int32, C.c_uint64, _dp]),
    "rw_sample_orders_philox": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, _i32p]),
    "rw_sample_costs_philox": (C.c_int, [_vp, P(rw_spec), C.c_int32, C.c_uint64, _dp]),
    "rw_problem_set_create": (C.c_int, [_dp, C.c_int32, C.c_int32, _i32p, C.c_int32, P(_vp)]),
    "rw_problem_set_destroy": (C.c_int, [_vp]),
    "rw_problem_set_devices": (C.c_int, [_vp, _i32p, _i32p]),
    "rw_problem_set_member": (C.c_int, [_vp, C.c_int32, P(_vp)]),
    "rw_evaluate_batch_set": (C.c_int, [_vp, P(rw_spec), _vp, C.c_int32, C.c_int32, C.c_int64, _dp, C.c_uint32]),
    "rw_brute_force_set": (C.c_int, [_vp, P(rw_spec), C.c_int32, _i32p, _dp, _u64p]),
    "rw_anneal_set": (C.c_int, [_vp, P(rw_spec), P(rw_solver_config), P(rw_gpu_config), _i32p, _dp, _u64p,
                                P(rw_search_report)]),
    "rw_set_gpu_options": (C.c_int, [P(rw_gpu_options)]),
    "rw_problem_set_resident": (C.c_int, [_vp, C.c_int32]),
    "rw_get_gpu_options": (C.c_int, [P(rw_gpu_options)]),
    "rw_distribution_stats": (C.c_int, [_dp, C.c_int64, _dp]),
    "rw_spearman": (C.c_int, [_dp, _dp, C.c_int64, C.c_int64, _dp]),
    "rw_parse_model_file": (C.c_int, [C.c_char_p, C.c_int32, _i32p]),
    "rw_balanced_sexpr": (C.c_int, [C.c_char_p, _i32p]),
    "rw_emit_smtlib": (C.c_int, [_dp, C.c_int32, P(rw_spec), C.c_int32, C.c_double, C.c_int32, C.c_char_p,
                                 C.c_int64, P(C.c_int64)]),
    "rw_two_stage_solve": (C.c_int, [_dp, C.c_int32, P(rw_spec), P(rw_solver_config), C.c_char_p, C.c_char_p,
                                     _vp, _vp, _i32p, _dp, _i32p, _u64p]),
    "rw_generate_matrix": (C.c_int, [C.c_int32, _i32p, _dp, _dp, _dp, C.c_double, C.c_uint64, _dp, C.c_int64,
                                     _i32p]),
    "rw_relabel_matrix": (C.c_int, [_dp, C.c_int32, C.c_uint64]),
    "rw_expand_schedule": (C.c_int, [P(rw_spec), _i32p, _i32p, P(C.c_int64), _i32p, _i32p, _i32p, _i32p, _dp]),
    "rw_simulate_batch": (C.c_int, [_vp, C.c_int32, _i32p, _dp, _dp, P(rw_spec), _i32p, C.c_int64, _dp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2105_14088_b200)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class RankweaveError(RuntimeError):
    """CUDA / internal failure inside librankweave_b200."""


class DomainError(ValueError):
    """rankweave::domain_error (types.hpp:14-17)."""


class IOError_(OSError):
    """rankweave::io_error (types.hpp:21-24)."""


def check(status: int) -> None:
    if status == RW_OK:
        return
    msg = lib.rw_last_error().decode("utf-8", "replace")
    if status == RW_ERR_DOMAIN:
        raise DomainError(msg)
    if status == RW_ERR_IO:
        raise IOError_(msg)
    raise RankweaveError(f"status {status}: {msg}")


# void (*rw_log_fn)(const char* message, void* user)
LOG_FN = C.CFUNCTYPE(None, C.c_char_p, C.c_void_p)


def ptr(arr, ctype):
    return arr.ctypes.data_as(P(ctype))
