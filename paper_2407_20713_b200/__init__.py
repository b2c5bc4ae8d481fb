"""B200-native SABR calibration engine (drop-in for the hot path of
arxiv/paper_2407_20713): parallel simulated annealing, Hagan/Obloj (Eq. 7) and
Osajima (Eq. 8) implied-vol cost functions and the log-Euler Monte Carlo
pricer, as hand-written sm_100a CUDA behind the C-ABI in include/sabr_b200.h.
"""
from ._abi import (LIB_PATH, MODEL_CASE1, MODEL_CASE2, MODEL_STATIC, RNG_PHILOX, RNG_XOSHIRO,
                   load_library)
from .api import (AnnealingSchedule, AnnealResult, CalibrationReport, CaseIIParams, CaseIParams,
                  ConstraintError, DomainError, Engine, NumericalError, OutOfRangeError, ParseError,
                  PriceEstimate, ReportRow, SabrError, SimulationPlan, StaticSabrParams,
                  VolQuote, VolSlice, VolSurface, black_scholes_call, calibrate_case2_formula,
                  calibrate_case2_T2, calibrate_dynamic_case1_T1, calibrate_static_T1,
                  calibrate_static_T1_slices, default_engine, evaluate_case1, evaluate_case2_prices, n_levels, parse_surface)

__all__ = [name for name in dir() if not name.startswith("_")]
