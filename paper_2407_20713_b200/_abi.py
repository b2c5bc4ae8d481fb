"""ctypes mirror of include/sabr_b200.h (the C-ABI boundary).

Only structure layouts and the shared-library loader live here; the
reference-shaped API is in ``paper_2407_20713_b200.api``.
"""
from __future__ import annotations

import ctypes as C
import os

SABR_OK = 0
STATUS_NAMES = {
    0: "SABR_OK",
    1: "SABR_E_DOMAIN",
    2: "SABR_E_OUT_OF_RANGE",
    3: "SABR_E_CONSTRAINT",
    4: "SABR_E_RUNTIME",
    5: "SABR_E_CUDA",
    6: "SABR_E_NCCL",
    7: "SABR_E_INVALID",
    8: "SABR_E_LOGIC",
}

MODEL_STATIC, MODEL_CASE1, MODEL_CASE2 = 0, 1, 2
RNG_XOSHIRO, RNG_PHILOX = 0, 1
FP64, FP32 = 0, 1

OBJ_BOWL3, OBJ_ROSENBROCK4, OBJ_SINQUAD2, OBJ_SQUARE1, OBJ_COSBOWL2, OBJ_CORNER2, OBJ_NANRIGHT1 = range(7)
PRED_NONE, PRED_SUM_LE_1 = 0, 1

MAX_PARAMS = 16
NAME_LEN = 16
MAX_DIM = 12

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


class sabr_surface(C.Structure):
    _fields_ = [
        ("spot", C.c_double),
        ("n_slices", C.c_int64),
        ("maturity", _dp),
        ("rate", _dp),
        ("dividend", _dp),
        ("quote_offset", _ip),
        ("strike", _dp),
        ("vol", _dp),
    ]


class sabr_schedule(C.Structure):
    _fields_ = [
        ("t0", C.c_double),
        ("cooling", C.c_double),
        ("chain_length", C.c_int32),
        ("workers", C.c_int32),
        ("groups", C.c_int32),
        ("omp_threads", C.c_int32),
        ("t_min", C.c_double),
        ("max_evals", C.c_int64),
        ("seed", C.c_uint64),
    ]


class sabr_plan(C.Structure):
    _fields_ = [
        ("num_paths", C.c_uint64),
        ("dt", C.c_double),
        ("seed", C.c_uint64),
        ("workers", C.c_int32),
        ("rng", C.c_int32),
        ("block_size", C.c_uint64),
        ("precision", C.c_int32),
        ("_pad", C.c_int32),
    ]


class sabr_bounds(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("names", C.POINTER(C.c_char_p)),
        ("lo", _dp),
        ("hi", _dp),
    ]


class sabr_fixed(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("names", C.POINTER(C.c_char_p)),
        ("values", _dp),
    ]


class sabr_report_row(C.Structure):
    _fields_ = [
        ("maturity", C.c_double),
        ("strike", C.c_double),
        ("market", C.c_double),
        ("model", C.c_double),
        ("rel_error", C.c_double),
    ]


class sabr_report(C.Structure):
    _fields_ = [
        ("model", C.c_char * NAME_LEN),
        ("technique", C.c_char * NAME_LEN),
        ("quantity", C.c_char * NAME_LEN),
        ("n_params", C.c_int64),
        ("param_names", (C.c_char * NAME_LEN) * MAX_PARAMS),
        ("param_values", C.c_double * MAX_PARAMS),
        ("final_cost", C.c_double),
        ("mean_rel_error", C.c_double),
        ("max_rel_error", C.c_double),
        ("wall_seconds", C.c_double),
        ("evals", C.c_int64),
        ("seed", C.c_uint64),
        ("rows", C.POINTER(sabr_report_row)),
        ("rows_capacity", C.c_int64),
        ("n_rows", C.c_int64),
        ("trace_t", _dp),
        ("trace_f", _dp),
        ("trace_capacity", C.c_int64),
        ("trace_len", C.c_int64),
    ]


class sabr_anneal_result(C.Structure):
    _fields_ = [
        ("best_point", _dp),
        ("best_value", C.c_double),
        ("evals", C.c_int64),
        ("trace_t", _dp),
        ("trace_f", _dp),
        ("trace_capacity", C.c_int64),
        ("trace_len", C.c_int64),
    ]


class sabr_timing(C.Structure):
    _fields_ = [
        ("total_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("kernel_launches", C.c_int64),
        ("total_launches", C.c_int64),
        ("units", C.c_double),
        ("path_steps", C.c_double),
    ]


class sabr_level_record(C.Structure):
    _fields_ = [
        ("end_value", C.c_double),
        ("end_chain", C.c_int64),
        ("best_value", C.c_double),
        ("best_chain", C.c_int64),
        ("evals", C.c_int64),
        ("_pad", C.c_int64),
        ("end_point", C.c_double * MAX_DIM),
        ("best_point", C.c_double * MAX_DIM),
    ]


class sabr_sa_state(C.Structure):
    _fields_ = [
        ("incumbent", C.c_double * MAX_DIM),
        ("incumbent_value", C.c_double),
        ("best", C.c_double * MAX_DIM),
        ("best_value", C.c_double),
        ("evals", C.c_int64),
        ("eval_cap", C.c_int64),
        ("done", C.c_int64),
        ("levels_run", C.c_int64),
    ]


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "libsabr_b200.so")

# exported symbols of include/sabr_b200.h (checked by tests/test_abi.py)
EXPORTS = [
    "sabr_last_error", "sabr_version", "sabr_ctx_create", "sabr_ctx_destroy",
    "sabr_ctx_set_profiling", "sabr_ctx_last_timing", "sabr_comm_unique_id",
    "sabr_ctx_init_comm", "sabr_calibrate_static_T1", "sabr_calibrate_static_T1_slices",
    "sabr_calibrate_dynamic_case1_T1",
    "sabr_calibrate_case2_T2", "sabr_calibrate_case2_formula", "sabr_evaluate_case1",
    "sabr_evaluate_case2_prices", "sabr_cost_batch", "sabr_implied_vol_batch",
    "sabr_case2_feasible_batch", "sabr_mc_simulate_terminals",
    "sabr_mc_price_european_batch", "sabr_mc_price_cliquet", "sabr_minimize_builtin",
    "sabr_merge_level_records", "sabr_surface_csv_dims", "sabr_surface_csv_read",
    "sabr_black_scholes_call", "sabr_bench_fp64_peak", "sabr_black_scholes_call_batch",
    "sabr_implied_vol_from_price_batch", "sabr_ctx_init_host_exchange", "sabr_ctx_enable_peer_exchange",
    "sabr_ctx_disable_peer_exchange", "sabr_bench_mufu_peak",
]

# sabr_allgather_fn
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)

_lib = None


def load_library(path: str | None = None) -> C.CDLL:
    """Load the in-tree CUDA engine (built by __graft_entry__.build()).

    There is no fallback: if the shared library is missing the engine cannot
    run, and this raises.
    """
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} not found: build the sm_100a engine first (python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = C.CDLL(p)
    lib.sabr_last_error.restype = C.c_char_p
    lib.sabr_version.restype = C.c_char_p
    if path is None:
        _lib = lib
    return lib
