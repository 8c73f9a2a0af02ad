"""ctypes rendering of ``include/migplan_b200.h`` — the C-ABI boundary.

The same declarations bind all three libraries that implement the header:
the product (``paper_2109_11067_b200/_native/libmigplan_b200.so``), and — in
tests and bench.py only — the CPU restatement ``oracle/liboracle.so`` and the
reference shim ``oracle/_ref/libmigref.so``.
"""
from __future__ import annotations

import ctypes as C
import os

MIG_OK = 0
MIG_ERR_PLANNING = 1
MIG_ERR_SCHEMA = 2
MIG_ERR_DEVICE = 3
MIG_ERR_ARGUMENT = 4
MAX_INST = 7


class ProfileEntryC(C.Structure):
    _fields_ = [("size", C.c_int32), ("batch", C.c_int32), ("throughput_rps", C.c_double), ("p90_ms", C.c_double)]


class ModelProfileC(C.Structure):
    _fields_ = [("model_name", C.c_char_p), ("entries", C.POINTER(ProfileEntryC)), ("n_entries", C.c_int32)]


class ServiceC(C.Structure):
    _fields_ = [("service_id", C.c_char_p), ("model_name", C.c_char_p), ("required_rps", C.c_double),
                ("max_p90_ms", C.c_double)]


class RulesC(C.Structure):
    _fields_ = [("n_sizes", C.c_int32), ("size", C.c_int32 * 8), ("n_slots", C.c_int32 * 8),
                ("slots", (C.c_int32 * 16) * 8), ("n_weights", C.c_int32), ("weight_size", C.c_int32 * 8),
                ("weight", C.c_int32 * 8), ("n_exclusions", C.c_int32), ("exclusion", (C.c_int32 * 2) * 16),
                ("memory_budget", C.c_int32)]


class InstanceC(C.Structure):
    _fields_ = [("slices", C.c_int32), ("slot", C.c_int32), ("service", C.c_int32), ("batch", C.c_int32)]


class ConfigC(C.Structure):
    _fields_ = [("n_instances", C.c_int32), ("inst", InstanceC * MAX_INST)]


class CandidateC(C.Structure):
    _fields_ = [("config", ConfigC), ("nnz", C.c_int32), ("util_idx", C.c_int32 * MAX_INST),
                ("util_val", C.c_double * MAX_INST), ("util_sum", C.c_double)]


class PartitionC(C.Structure):
    _fields_ = [("n", C.c_int32), ("slices", C.c_int32 * MAX_INST), ("slot", C.c_int32 * MAX_INST)]


class MctsParamsC(C.Structure):
    _fields_ = [("budget_iters", C.c_int32), ("topk", C.c_int32), ("pick_services", C.c_int32),
                ("ucb_c", C.c_double)]


class GaParamsC(C.Structure):
    _fields_ = [("population", C.c_int32), ("erase_fraction", C.c_double), ("mutation_pairs", C.c_int32),
                ("stall_rounds", C.c_int32), ("time_budget_s", C.c_double), ("seed", C.c_uint64),
                ("max_rounds", C.c_int32), ("workers", C.c_int32), ("slow", MctsParamsC)]


class StatsC(C.Structure):
    _fields_ = [("rows_scored", C.c_int64), ("greedy_rows", C.c_int64), ("topk_rows", C.c_int64),
                ("greedy_calls", C.c_int64), ("topk_calls", C.c_int64), ("greedy_steps", C.c_int64),
                ("ext_events", C.c_int64), ("ext_rows", C.c_int64), ("kernel_launches", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("greedy_ms", C.c_double),
                ("topk_ms", C.c_double), ("phase_ms", C.c_double * 5), ("rollout_steps", C.c_int64),
                ("rollout_calls", C.c_int64), ("rollout_ms", C.c_double), ("mcts_ms", C.c_double),
                ("mcts_launches", C.c_int64), ("mcts_rows", C.c_int64), ("mcts_topk_calls", C.c_int64)]


class RolloutParamsC(C.Structure):
    _fields_ = [("n_rollouts", C.c_int64), ("topk", C.c_int32), ("max_depth", C.c_int32), ("seed", C.c_uint64),
                ("id_offset", C.c_int64), ("batch", C.c_int64), ("table_log2", C.c_int32)]


class RolloutResultC(C.Structure):
    _fields_ = [("best_len", C.c_int32), ("max_depth", C.c_int32), ("best_id", C.c_int64),
                ("completed", C.c_int64), ("capped", C.c_int64), ("failed", C.c_int64), ("steps", C.c_int64),
                ("keys", C.c_int64), ("rounds", C.c_int32), ("path_len", C.c_int32), ("device_ms", C.c_double)]


GREEDY_TRACE = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(CandidateC), C.c_double,
                           C.POINTER(C.c_double), C.c_int32)
MCTS_TRACE = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32)
GA_LOG = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_double)

_P = C.c_void_p
_I = C.c_int
_DP = C.POINTER(C.c_double)
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)

# name -> (restype, argtypes)
SIGNATURES = {
    "mig_last_error": (C.c_char_p, []),
    "mig_abi_version": (C.c_int32, []),
    "mig_impl_name": (C.c_char_p, []),
    "mig_rules_defaults": (None, [C.POINTER(RulesC)]),
    "mig_is_legal_partition": (_I, [C.POINTER(RulesC), _I32P, _I32P, C.c_int32, _I32P]),
    "mig_enumerate_maximal_partitions": (_I, [C.POINTER(RulesC), C.POINTER(PartitionC), C.c_int32, _I32P]),
    "mig_validate_services": (_I, [C.POINTER(ModelProfileC), C.c_int32, C.POINTER(ServiceC), C.c_int32, _I32P]),
    "mig_ctx_create": (_I, [C.POINTER(RulesC), C.POINTER(ModelProfileC), C.c_int32, C.POINTER(ServiceC),
                            C.c_int32, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "mig_ctx_destroy": (None, [_P]),
    "mig_ctx_n_services": (C.c_int32, [_P]),
    "mig_pool_size": (_I, [_P, _I64P]),
    "mig_pool_candidate": (_I, [_P, C.c_int64, C.POINTER(CandidateC)]),
    "mig_pool_best_single_util": (_I, [_P, _DP]),
    "mig_score": (_I, [_P, C.c_int64, _DP, C.c_int32, _DP]),
    "mig_topk_candidates": (_I, [_P, _DP, C.c_int32, C.c_int32, _I64P, C.c_int64, _I64P, _I32P]),
    "mig_fast_algo": (_I, [_P, _DP, C.c_int32, C.POINTER(ConfigC), C.c_int32, _I32P, GREEDY_TRACE, _P]),
    "mig_rng_create": (_I, [C.c_uint64, C.POINTER(_P)]),
    "mig_rng_destroy": (None, [_P]),
    "mig_rng_next": (C.c_uint64, [_P]),
    "mig_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "mig_pick_index": (C.c_uint64, [_P, C.c_uint64]),
    "mig_mcts_params_defaults": (None, [C.POINTER(MctsParamsC)]),
    "mig_expand": (_I, [_P, _DP, C.c_int32, C.POINTER(MctsParamsC), _P, _I64P, C.c_int32, _I32P]),
    "mig_rollout_cache_create": (_I, [C.POINTER(_P)]),
    "mig_rollout_cache_destroy": (None, [_P]),
    "mig_rollout_cache_builds": (C.c_int32, [_P]),
    "mig_rollout": (_I, [_P, _DP, C.c_int32, C.POINTER(MctsParamsC), _P, _P, C.c_int32, _I64P, C.c_int32, _I32P]),
    "mig_mcts_solve": (_I, [_P, _DP, C.c_int32, C.POINTER(MctsParamsC), C.c_uint64, C.POINTER(ConfigC),
                            C.c_int32, _I32P, MCTS_TRACE, _P]),
    "mig_rollouts": (_I, [_P, _DP, C.c_int32, C.POINTER(RolloutParamsC), _I32P, _I64P, C.c_int32,
                          C.POINTER(RolloutResultC)]),
    "mig_mcts_solve_parallel": (_I, [_P, _DP, C.c_int32, C.POINTER(RolloutParamsC), C.POINTER(ConfigC), C.c_int32,
                                     _I32P, C.POINTER(RolloutResultC)]),
    "mig_board_bytes": (_I, [C.c_int32, _I64P]),
    "mig_board_alloc": (_I, [C.c_int32, C.c_int32, C.POINTER(_P), C.POINTER(C.c_uint8)]),
    "mig_board_open": (_I, [C.c_int32, C.POINTER(C.c_uint8), C.POINTER(_P)]),
    "mig_board_free": (_I, [_P, C.c_int32]),
    "mig_ctx_set_shard": (_I, [_P, C.c_int32, C.c_int32, C.POINTER(_P), C.c_int32]),
    "mig_fast_algo_group": (_I, [C.POINTER(_P), C.c_int32, _DP, C.c_int32, C.POINTER(ConfigC), C.c_int32, _I32P]),
    "mig_ga_params_defaults": (None, [C.POINTER(GaParamsC)]),
    "mig_completion_of": (_I, [_P, C.POINTER(ConfigC), C.c_int32, _DP]),
    "mig_mutate": (_I, [_P, C.POINTER(ConfigC), C.c_int32, C.POINTER(GaParamsC), _P, C.POINTER(ConfigC)]),
    "mig_crossover": (_I, [_P, C.POINTER(ConfigC), C.c_int32, C.c_int32, C.POINTER(GaParamsC), _P,
                           C.POINTER(ConfigC), C.c_int32, _I32P]),
    "mig_two_phase": (_I, [_P, C.POINTER(GaParamsC), C.POINTER(ConfigC), C.c_int32, _I32P, GA_LOG, _P]),
    "mig_two_phase_parallel": (_I, [_P, C.POINTER(GaParamsC), C.POINTER(ConfigC), C.c_int32, _I32P, GA_LOG, _P]),
    "mig_two_phase_parallel_mcts": (_I, [_P, C.POINTER(GaParamsC), C.POINTER(RolloutParamsC), C.POINTER(ConfigC),
                                         C.c_int32, _I32P, GA_LOG, _P]),
    "mig_lower_bound": (_I, [_P, _I32P]),
    "mig_baseline": (_I, [_P, C.c_int32, _P, C.c_int32, _I32P]),
    "mig_brute_force_optimum": (_I, [_P, C.c_int32, C.c_int64, _P, C.c_int32, _I32P, _I32P]),
    "mig_ctx_stats": (_I, [_P, C.POINTER(StatsC)]),
    "mig_ctx_reset_stats": (None, [_P]),
    "mig_ctx_step_rows": (_I, [_P, _I64P, C.c_int32, _I32P]),
    "mig_device_cache_release": (_I, [C.c_int32]),
    "mig_last_plan": (_I, [C.POINTER(ConfigC), C.c_int32, _I32P]),
    "mig_philox_u64": (_I, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.POINTER(C.c_uint64)]),
}

# Exported by the reference shim only (bench.py reference arm, golden generation).
REF_EXTRAS = {
    "mig_ref_count_rows": (_I, [_P, _DP, C.c_int32, _I64P]),
    "mig_ref_step_rows": (_I, [_P, _DP, C.c_int32, C.c_int64, _I64P, C.c_int32, _I32P, _I64P, C.c_int32, _I32P]),
    "mig_ref_fast_algo_prefix": (_I, [_P, _DP, C.c_int32, C.c_int64, C.c_int64, GREEDY_TRACE, _P, _I32P, _I32P]),
    "mig_ref_plan_transition": (_I, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32,
                                     C.c_char_p, C.c_int32, _I32P]),
    "mig_ref_deployment_json": (_I, [_P, C.POINTER(ConfigC), C.c_int32, C.c_char_p, C.c_int32, _I32P]),
    "mig_ref_gen_workload": (_I, [C.POINTER(ModelProfileC), C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                  C.c_double, C.c_double, C.c_uint64, _I32P, _DP]),
}


class AbiError(RuntimeError):
    pass


def bind(path: str, extras: dict | None = None) -> C.CDLL:
    """dlopen `path` and attach every header signature; a missing symbol is an error."""
    if not os.path.exists(path):
        raise AbiError(f"library not found: {path}")
    lib = C.CDLL(path)
    for name, (res, args) in {**SIGNATURES, **(extras or {})}.items():
        fn = getattr(lib, name)  # AttributeError == the library does not export the header
        fn.restype = res
        fn.argtypes = args
    return lib


def header_symbols() -> list[str]:
    return sorted(SIGNATURES)
