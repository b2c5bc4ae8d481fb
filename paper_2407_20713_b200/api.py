"""Reference-shaped Python API over the C-ABI (include/sabr_b200.h).

Mirrors the calibration API of the reference C++ engine
(proj/include/sabr/calibration.hpp, mc.hpp, annealer.hpp): the same names,
argument meaning and error behaviour, so that the parity tests read like the
reference's own doctest suites.  Exceptions map onto the reference's C++
exception types:

=====================  ==========================================
reference              here
=====================  ==========================================
std::domain_error      DomainError (ValueError)
std::out_of_range      OutOfRangeError (IndexError)
sabr::constraint_error ConstraintError (RuntimeError)
std::runtime_error     NumericalError (RuntimeError)
=====================  ==========================================

All compute goes through the CUDA engine; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Mapping, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A


# --------------------------------------------------------------- errors ---
class SabrError(Exception):
    status = -1


class DomainError(SabrError, ValueError):
    status = 1


class OutOfRangeError(SabrError, IndexError):
    status = 2


class ConstraintError(SabrError, RuntimeError):
    status = 3


class NumericalError(SabrError, RuntimeError):
    status = 4


class ParseError(NumericalError):
    """io::parse_error (io.hpp:14-24), a std::runtime_error: malformed surface
    CSV or parameter file; the message carries "(line N)" when known."""


class CudaError(SabrError, RuntimeError):
    status = 5


class NcclError(SabrError, RuntimeError):
    status = 6


class AbiError(SabrError, ValueError):
    status = 7


class LogicError(SabrError, RuntimeError):
    status = 8


_ERRORS = {c.status: c for c in (DomainError, OutOfRangeError, ConstraintError, NumericalError,
                                 CudaError, NcclError, AbiError, LogicError)}


def raise_for_status(status: int, message: str) -> None:
    if status == A.SABR_OK:
        return
    raise _ERRORS.get(status, SabrError)(message)


# ---------------------------------------------------------- value types ---
@dataclass
class VolQuote:
    strike: float
    vol: float


@dataclass
class VolSlice:
    maturity: float
    rate: float
    dividend: float
    quotes: List[VolQuote] = field(default_factory=list)


@dataclass
class VolSurface:
    """VolSurface, calibration.hpp:16-37."""

    spot: float
    slices: List[VolSlice] = field(default_factory=list)

    def forward(self, slice: int) -> float:
        s = self.slices[slice]
        if not self.spot > 0:
            raise DomainError("forward_price: spot must be positive")
        if not s.maturity > 0:
            raise DomainError("forward_price: maturity must be positive")
        return self.spot * math.exp((s.rate - s.dividend) * s.maturity)

    def total_quotes(self) -> int:
        return sum(len(s.quotes) for s in self.slices)

    def validate(self) -> None:
        """VolSurface::validate, calibration.cpp:233-251."""
        if self.spot <= 0:
            raise DomainError("VolSurface: spot must be positive")
        if not self.slices:
            raise DomainError("VolSurface: no slices")
        for i, s in enumerate(self.slices):
            if s.maturity <= 0:
                raise DomainError("VolSurface: maturity must be positive")
            if i > 0 and s.maturity <= self.slices[i - 1].maturity:
                raise DomainError("VolSurface: maturities must be strictly increasing")
            if not s.quotes:
                raise DomainError(f"VolSurface: empty quote block in slice {i}")
            for j, q in enumerate(s.quotes):
                if q.strike <= 0 or q.vol <= 0:
                    raise DomainError("VolSurface: strikes and vols must be positive")
                if j > 0 and q.strike <= s.quotes[j - 1].strike:
                    raise DomainError("VolSurface: strikes must be strictly increasing")

    # SoA view for the ABI
    def to_abi(self):
        n = len(self.slices)
        T = np.array([s.maturity for s in self.slices], dtype=np.float64)
        r = np.array([s.rate for s in self.slices], dtype=np.float64)
        y = np.array([s.dividend for s in self.slices], dtype=np.float64)
        off = np.zeros(n + 1, dtype=np.int64)
        for i, s in enumerate(self.slices):
            off[i + 1] = off[i] + len(s.quotes)
        K = np.array([q.strike for s in self.slices for q in s.quotes], dtype=np.float64)
        v = np.array([q.vol for s in self.slices for q in s.quotes], dtype=np.float64)
        keep = (T, r, y, off, K, v)
        st = A.sabr_surface(
            spot=float(self.spot), n_slices=n,
            maturity=_dptr(T), rate=_dptr(r), dividend=_dptr(y),
            quote_offset=off.ctypes.data_as(C.POINTER(C.c_int64)),
            strike=_dptr(K), vol=_dptr(v),
        )
        return st, keep

    @staticmethod
    def from_arrays(spot, maturity, rate, dividend, quote_offset, strike, vol) -> "VolSurface":
        slices = []
        for i in range(len(maturity)):
            qs = [VolQuote(float(strike[j]), float(vol[j]))
                  for j in range(int(quote_offset[i]), int(quote_offset[i + 1]))]
            slices.append(VolSlice(float(maturity[i]), float(rate[i]), float(dividend[i]), qs))
        return VolSurface(float(spot), slices)


@dataclass
class AnnealingSchedule:
    """AnnealingSchedule, annealer.hpp:17-29 (same defaults)."""

    t0: float = 10.0
    cooling: float = 0.95
    chain_length: int = 100
    workers: int = 8
    groups: int = 1
    t_min: float = 1e-5
    max_evals: int = 1_000_000
    seed: int = 0
    omp_threads: int = 1

    def to_abi(self) -> A.sabr_schedule:
        return A.sabr_schedule(self.t0, self.cooling, self.chain_length, self.workers, self.groups,
                               self.omp_threads, self.t_min, self.max_evals, self.seed)

    def validate(self) -> None:
        """AnnealingSchedule::validate, annealer.cpp:28-39."""
        if not self.t0 > 0:
            raise DomainError("AnnealingSchedule: t0 must be positive")
        if not (0 < self.cooling < 1):
            raise DomainError("AnnealingSchedule: cooling must be in (0,1)")
        if self.chain_length < 1:
            raise DomainError("AnnealingSchedule: chain_length must be >= 1")
        if self.workers < 1 or self.groups < 1:
            raise DomainError("AnnealingSchedule: workers and groups must be >= 1")
        if not (0 < self.t_min < self.t0):
            raise DomainError("AnnealingSchedule: need 0 < t_min < t0")
        if self.max_evals < 1:
            raise DomainError("AnnealingSchedule: max_evals must be >= 1")


@dataclass
class SimulationPlan:
    """SimulationPlan, mc.hpp:12-20, plus the random stream (``"xoshiro"``
    reproduces the reference streams; ``"philox"`` is counter-based) and the
    path-loop arithmetic (``"fp64"``, the reference's; ``"fp32"``, the MUFU
    fast path)."""

    num_paths: int = 1 << 20
    dt: float = 1.0 / 250.0
    seed: int = 0
    workers: int = 1
    block_size: int = 4096
    rng: str = "xoshiro"
    precision: str = "fp64"

    def to_abi(self) -> A.sabr_plan:
        rng = {"xoshiro": A.RNG_XOSHIRO, "philox": A.RNG_PHILOX}[self.rng]
        prec = {"fp64": A.FP64, "fp32": A.FP32}[self.precision]
        return A.sabr_plan(self.num_paths, self.dt, self.seed, self.workers, rng, self.block_size, prec, 0)

    def validate(self) -> None:
        """SimulationPlan::validate, mc.cpp:161-166."""
        if self.num_paths < 1:
            raise DomainError("SimulationPlan: num_paths must be >= 1")
        if not self.dt > 0:
            raise DomainError("SimulationPlan: dt must be positive")
        if self.workers < 1:
            raise DomainError("SimulationPlan: workers must be >= 1")
        if self.block_size < 1:
            raise DomainError("SimulationPlan: block_size must be >= 1")


@dataclass
class ReportRow:
    maturity: float
    strike: float
    market: float
    model: float
    rel_error: float


@dataclass
class CalibrationReport:
    """CalibrationReport, calibration.hpp:47-59 (+ the annealer trace)."""

    model: str = ""
    technique: str = ""
    quantity: str = ""
    params: Dict[str, float] = field(default_factory=dict)
    final_cost: float = 0.0
    rows: List[ReportRow] = field(default_factory=list)
    mean_rel_error: float = 0.0
    max_rel_error: float = 0.0
    wall_seconds: float = 0.0
    evals: int = 0
    seed: int = 0
    temperature_trace: List[Tuple[float, float]] = field(default_factory=list)


@dataclass
class AnnealResult:
    best_point: List[float]
    best_value: float
    evals: int
    temperature_trace: List[Tuple[float, float]]


@dataclass
class PriceEstimate:
    value: float
    std_error: float
    num_paths: int


@dataclass
class StaticSabrParams:
    alpha: float
    beta: float
    nu: float
    rho: float

    def vector(self):
        return [self.alpha, self.beta, self.nu, self.rho]


@dataclass
class CaseIParams:
    alpha: float
    beta: float
    rho0: float
    nu0: float
    a: float
    b: float

    def vector(self):
        return [self.alpha, self.beta, self.rho0, self.nu0, self.a, self.b]


@dataclass
class CaseIIParams:
    alpha: float
    beta: float
    rho0: float
    q_rho: float
    d_rho: float
    nu0: float
    q_nu: float
    d_nu: float
    a: float
    b: float
    horizon: float

    def vector(self):
        return [self.alpha, self.beta, self.rho0, self.q_rho, self.d_rho, self.nu0, self.q_nu,
                self.d_nu, self.a, self.b, self.horizon]


def model_of(params) -> Tuple[int, List[float]]:
    if isinstance(params, StaticSabrParams):
        return A.MODEL_STATIC, params.vector()
    if isinstance(params, CaseIParams):
        return A.MODEL_CASE1, params.vector()
    if isinstance(params, CaseIIParams):
        return A.MODEL_CASE2, params.vector()
    raise TypeError("params must be StaticSabrParams, CaseIParams or CaseIIParams")


# ------------------------------------------------------------ helpers ---
def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _bounds_abi(bounds: Optional[Mapping[str, Tuple[float, float]]]):
    bounds = dict(bounds or {})
    names = (C.c_char_p * max(1, len(bounds)))(*[k.encode() for k in bounds])
    lo = np.array([v[0] for v in bounds.values()] or [0.0], dtype=np.float64)
    hi = np.array([v[1] for v in bounds.values()] or [0.0], dtype=np.float64)
    return A.sabr_bounds(len(bounds), names, _dptr(lo), _dptr(hi)), (names, lo, hi)


def _fixed_abi(fixed: Optional[Mapping[str, float]]):
    fixed = dict(fixed or {})
    names = (C.c_char_p * max(1, len(fixed)))(*[k.encode() for k in fixed])
    vals = np.array(list(fixed.values()) or [0.0], dtype=np.float64)
    return A.sabr_fixed(len(fixed), names, _dptr(vals)), (names, vals)


class _ReportBuf:
    def __init__(self, n_rows: int, trace_cap: int = 0):
        self.rows = (A.sabr_report_row * max(1, n_rows))()
        self.tt = np.zeros(max(1, trace_cap))
        self.tf = np.zeros(max(1, trace_cap))
        self.rep = A.sabr_report()
        self.rep.rows = C.cast(self.rows, C.POINTER(A.sabr_report_row))
        self.rep.rows_capacity = n_rows
        if trace_cap:
            self.rep.trace_t = _dptr(self.tt)
            self.rep.trace_f = _dptr(self.tf)
            self.rep.trace_capacity = trace_cap

    def report(self) -> CalibrationReport:
        r = self.rep
        params = {r.param_names[i].value.decode(): r.param_values[i] for i in range(r.n_params)}
        rows = [ReportRow(self.rows[i].maturity, self.rows[i].strike, self.rows[i].market,
                          self.rows[i].model, self.rows[i].rel_error) for i in range(r.n_rows)]
        trace = []
        if r.trace_capacity:
            trace = list(zip(self.tt[: r.trace_len].tolist(), self.tf[: r.trace_len].tolist()))
        return CalibrationReport(r.model.decode(), r.technique.decode(), r.quantity.decode(), params,
                                 r.final_cost, rows, r.mean_rel_error, r.max_rel_error,
                                 r.wall_seconds, r.evals, r.seed, trace)


def n_levels(schedule: AnnealingSchedule, all_evals: bool = True) -> int:
    """Number of temperature levels, annealer.cpp:99-100 (repeated product).
    all_evals: every step is an evaluation (no feasibility predicate), so the
    run stops after at most ceil((max_evals - 1) / n_chains) + 1 levels
    (host_common.hpp: level_cap_all_evals)."""
    chains = schedule.workers * schedule.groups
    cap = None
    if all_evals and chains > 0 and schedule.max_evals >= 1:
        cap = (schedule.max_evals - 1 + chains - 1) // chains + 1
    n, t = 0, schedule.t0
    while t >= schedule.t_min and (cap is None or n < cap):
        n += 1
        t *= schedule.cooling
    return n


# -------------------------------------------------------------- engine ---
class Engine:
    """One CUDA context (one GPU, one stream) of the sm_100a engine."""

    def __init__(self, device: int = 0, stream: int = 0, lib: Optional[C.CDLL] = None):
        self.lib = lib or A.load_library()
        self._ctx = C.c_void_p()
        self._check(self.lib.sabr_ctx_create(C.c_int32(device), C.c_void_p(stream),
                                             C.byref(self._ctx)))
        self.device = device
        self.rank, self.nranks = 0, 1

    # -- plumbing --
    def _check(self, status: int) -> None:
        if status != A.SABR_OK:
            raise_for_status(status, self.lib.sabr_last_error().decode(errors="replace"))

    def close(self) -> None:
        if self._ctx:
            self.lib.sabr_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._ctx

    def set_profiling(self, on: bool = True) -> None:
        self._check(self.lib.sabr_ctx_set_profiling(self._ctx, C.c_int32(int(on))))

    def last_timing(self) -> A.sabr_timing:
        t = A.sabr_timing()
        self._check(self.lib.sabr_ctx_last_timing(self._ctx, C.byref(t)))
        return t

    @staticmethod
    def comm_unique_id(lib: Optional[C.CDLL] = None) -> bytes:
        lib = lib or A.load_library()
        buf = (C.c_uint8 * 128)()
        st = lib.sabr_comm_unique_id(buf)
        if st != A.SABR_OK:
            raise_for_status(st, lib.sabr_last_error().decode())
        return bytes(buf)

    def init_comm(self, uid: bytes, rank: int, nranks: int) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.lib.sabr_ctx_init_comm(self._ctx, buf, C.c_int32(rank), C.c_int32(nranks)))
        self.rank, self.nranks = rank, nranks

    # -- calibration (calibration.hpp:82-124) --
    def init_host_exchange(self, rank: int, nranks: int, allgather) -> None:
        """Split the chains over `nranks` ranks with the per-level record
        exchange done on the host: allgather(send: bytes) -> bytes (nranks
        records in rank order), e.g. over a torch.distributed gloo group."""
        def cb(user, send, recv, nbytes):
            try:
                out = allgather(C.string_at(send, nbytes))
                if len(out) != nbytes * nranks:
                    return 1
                C.memmove(recv, out, len(out))
                return 0
            except Exception:  # noqa: BLE001 - reported to the engine as a failed exchange
                return 1

        self._exchange_cb = A.ALLGATHER_FN(cb)  # keep the trampoline alive
        self._check(self.lib.sabr_ctx_init_host_exchange(self._ctx, C.c_int32(rank), C.c_int32(nranks),
                                                         self._exchange_cb, None))

    def enable_peer_exchange(self) -> None:
        """Fused peer-memory exchange of the T_I level records (after
        init_comm / init_host_exchange); see include/sabr_b200.h."""
        self._check(self.lib.sabr_ctx_enable_peer_exchange(self._ctx))

    def disable_peer_exchange(self) -> None:
        self._check(self.lib.sabr_ctx_disable_peer_exchange(self._ctx))

    def calibrate_static_T1(self, surface: VolSurface, slice: int, bounds=None,
                            schedule: Optional[AnnealingSchedule] = None, fixed=None,
                            trace: bool = False) -> CalibrationReport:
        schedule = schedule or AnnealingSchedule()
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        rb = _ReportBuf(surface.total_quotes(), n_levels(schedule) if trace else 0)
        sch = schedule.to_abi()
        self._check(self.lib.sabr_calibrate_static_T1(self._ctx, C.byref(s), C.c_int64(slice),
                                                      C.byref(b), C.byref(sch), C.byref(f),
                                                      C.byref(rb.rep)))
        return rb.report()

    def calibrate_static_T1_slices(self, surface: VolSurface, slices=None, bounds=None,
                                   schedule: Optional[AnnealingSchedule] = None, fixed=None,
                                   trace: bool = False) -> List[CalibrationReport]:
        """calibrate_static_T1 for each of `slices` (default: every slice) in
        one call; on a single-rank engine the slices' annealers run side by side
        on their own streams (sabr_calibrate_static_T1_slices).  Reports equal
        the one-slice calls'."""
        schedule = schedule or AnnealingSchedule()
        idx = list(range(len(surface.slices))) if slices is None else [int(i) for i in slices]
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        bufs = [_ReportBuf(surface.total_quotes(), n_levels(schedule) if trace else 0) for _ in idx]
        reps = (A.sabr_report * max(1, len(idx)))()
        for i, rb in enumerate(bufs):
            reps[i] = rb.rep
        sl = (C.c_int64 * max(1, len(idx)))(*idx)
        sch = schedule.to_abi()
        self._check(self.lib.sabr_calibrate_static_T1_slices(self._ctx, C.byref(s), sl, C.c_int64(len(idx)),
                                                             C.byref(b), C.byref(sch), C.byref(f), reps))
        for i, rb in enumerate(bufs):
            rb.rep = reps[i]
        return [rb.report() for rb in bufs]

    def calibrate_dynamic_case1_T1(self, surface: VolSurface, bounds=None,
                                   schedule: Optional[AnnealingSchedule] = None, fixed=None,
                                   trace: bool = False) -> CalibrationReport:
        schedule = schedule or AnnealingSchedule()
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        rb = _ReportBuf(surface.total_quotes(), n_levels(schedule) if trace else 0)
        sch = schedule.to_abi()
        self._check(self.lib.sabr_calibrate_dynamic_case1_T1(self._ctx, C.byref(s), C.byref(b),
                                                             C.byref(sch), C.byref(f),
                                                             C.byref(rb.rep)))
        return rb.report()

    def calibrate_case2_T2(self, surface: VolSurface, bounds=None,
                           schedule: Optional[AnnealingSchedule] = None,
                           plan: Optional[SimulationPlan] = None, fixed=None,
                           report_plan: Optional[SimulationPlan] = None,
                           start_override: Optional[Sequence[float]] = None,
                           trace: bool = False) -> CalibrationReport:
        schedule = schedule or AnnealingSchedule()
        plan = plan or SimulationPlan()
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        rb = _ReportBuf(surface.total_quotes(), n_levels(schedule, all_evals=False) if trace else 0)
        sch, pl = schedule.to_abi(), plan.to_abi()
        rp = C.byref(report_plan.to_abi()) if report_plan is not None else None
        if start_override is not None:
            st = np.asarray(start_override, dtype=np.float64)
            stp, stn = _dptr(st), len(st)
        else:
            st, stp, stn = None, None, 0
        self._check(self.lib.sabr_calibrate_case2_T2(self._ctx, C.byref(s), C.byref(b),
                                                     C.byref(sch), C.byref(pl), C.byref(f), rp,
                                                     stp, C.c_int64(stn), C.byref(rb.rep)))
        return rb.report()

    def calibrate_case2_formula(self, surface: VolSurface, bounds=None,
                                schedule: Optional[AnnealingSchedule] = None, fixed=None,
                                trace: bool = False) -> CalibrationReport:
        schedule = schedule or AnnealingSchedule()
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        rb = _ReportBuf(surface.total_quotes(), n_levels(schedule, all_evals=False) if trace else 0)
        sch = schedule.to_abi()
        self._check(self.lib.sabr_calibrate_case2_formula(self._ctx, C.byref(s), C.byref(b),
                                                          C.byref(sch), C.byref(f),
                                                          C.byref(rb.rep)))
        return rb.report()

    def evaluate_case1(self, surface: VolSurface, p: CaseIParams) -> CalibrationReport:
        s, keep = surface.to_abi()
        v = np.asarray(p.vector(), dtype=np.float64)
        rb = _ReportBuf(surface.total_quotes())
        self._check(self.lib.sabr_evaluate_case1(self._ctx, C.byref(s), _dptr(v), C.byref(rb.rep)))
        return rb.report()

    def evaluate_case2_prices(self, surface: VolSurface, p: CaseIIParams,
                              plan: SimulationPlan) -> CalibrationReport:
        s, keep = surface.to_abi()
        v = np.asarray(p.vector(), dtype=np.float64)
        rb = _ReportBuf(surface.total_quotes())
        pl = plan.to_abi()
        self._check(self.lib.sabr_evaluate_case2_prices(self._ctx, C.byref(s), _dptr(v),
                                                        C.byref(pl), C.byref(rb.rep)))
        return rb.report()

    # -- batched objective --
    def cost_batch(self, model: int, surface: VolSurface, params: np.ndarray, slice: int = -1,
                   plan: Optional[SimulationPlan] = None) -> np.ndarray:
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64)
        n = P.shape[0] if P.ndim == 2 else 1
        out = np.empty(n, dtype=np.float64)
        pl = plan.to_abi() if plan is not None else None
        self._check(self.lib.sabr_cost_batch(self._ctx, C.c_int32(model), C.byref(s),
                                             C.c_int64(slice), _dptr(P), C.c_int64(n),
                                             C.byref(pl) if pl is not None else None, _dptr(out)))
        return out

    def implied_vol_batch(self, model: int, surface: VolSurface, params: np.ndarray,
                          slice: int = -1) -> np.ndarray:
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64)
        n = P.shape[0] if P.ndim == 2 else 1
        nq = (len(surface.slices[slice].quotes) if model == A.MODEL_STATIC
              else surface.total_quotes())
        if P.ndim == 2 and model == A.MODEL_CASE2 and P.shape[1] != 11:
            raise ValueError("case2 parameter rows are 11 wide (horizon last)")
        out = np.empty((n, nq), dtype=np.float64)
        self._check(self.lib.sabr_implied_vol_batch(self._ctx, C.c_int32(model), C.byref(s),
                                                    C.c_int64(slice), _dptr(P), C.c_int64(n),
                                                    _dptr(out)))
        return out

    def case2_feasible_batch(self, params: np.ndarray) -> np.ndarray:
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
        out = np.zeros(P.shape[0], dtype=np.uint8)
        self._check(self.lib.sabr_case2_feasible_batch(
            self._ctx, _dptr(P), C.c_int64(P.shape[0]), out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out.astype(bool)

    # -- Black-Scholes (black_scholes.hpp), batched on the device --
    def _bs_batch(self, fn, cols):
        arrs = np.broadcast_arrays(*(np.asarray(c, dtype=np.float64) for c in cols))
        arrs = [np.ascontiguousarray(a.ravel()) for a in arrs]
        out = np.zeros(arrs[0].size)
        self._check(fn(self._ctx, C.c_int64(out.size), *(_dptr(a) for a in arrs), _dptr(out)))
        return out.reshape(np.broadcast(*cols).shape)

    def black_scholes_call_batch(self, spot, strike, rate, dividend, maturity, vol) -> np.ndarray:
        """black_scholes_call (black_scholes.cpp:20-35) element-wise; arguments broadcast."""
        return self._bs_batch(self.lib.sabr_black_scholes_call_batch, (spot, strike, rate, dividend, maturity, vol))

    def implied_vol_from_price_batch(self, price, spot, strike, rate, dividend, maturity) -> np.ndarray:
        """implied_vol_from_price (black_scholes.cpp:37-69) element-wise; arguments broadcast."""
        return self._bs_batch(self.lib.sabr_implied_vol_from_price_batch,
                              (price, spot, strike, rate, dividend, maturity))

    # -- Monte Carlo (mc.hpp) --
    def simulate_terminals(self, params, forward0: float, alpha0: float, maturity: float,
                           plan: SimulationPlan) -> np.ndarray:
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        out = np.empty(int(plan.num_paths), dtype=np.float64)
        pl = plan.to_abi()
        self._check(self.lib.sabr_mc_simulate_terminals(
            self._ctx, C.c_int32(model), _dptr(v), C.c_double(forward0), C.c_double(alpha0),
            C.c_double(maturity), C.byref(pl), _dptr(out)))
        return out

    def price_european_batch(self, params, spot: float, strikes: Sequence[float], rate: float,
                             dividend: float, maturity: float,
                             plan: SimulationPlan) -> List[PriceEstimate]:
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        K = np.asarray(strikes, dtype=np.float64)
        val = np.empty(len(K))
        se = np.empty(len(K))
        pl = plan.to_abi()
        self._check(self.lib.sabr_mc_price_european_batch(
            self._ctx, C.c_int32(model), _dptr(v), C.c_double(spot), _dptr(K), C.c_int64(len(K)),
            C.c_double(rate), C.c_double(dividend), C.c_double(maturity), C.byref(pl),
            _dptr(val), _dptr(se)))
        return [PriceEstimate(float(val[j]), float(se[j]), int(plan.num_paths)) for j in range(len(K))]

    def price_european_call(self, params, spot, strike, rate, dividend, maturity,
                            plan: SimulationPlan) -> PriceEstimate:
        return self.price_european_batch(params, spot, [strike], rate, dividend, maturity, plan)[0]

    def price_cliquet(self, params, spot, rate, dividend, local_floor, local_cap, global_floor,
                      global_cap, reset_dates, plan: SimulationPlan) -> PriceEstimate:
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        R = np.asarray(reset_dates, dtype=np.float64)
        val, se = C.c_double(), C.c_double()
        pl = plan.to_abi()
        self._check(self.lib.sabr_mc_price_cliquet(
            self._ctx, C.c_int32(model), _dptr(v), C.c_double(spot), C.c_double(rate),
            C.c_double(dividend), C.c_double(local_floor), C.c_double(local_cap),
            C.c_double(global_floor), C.c_double(global_cap), _dptr(R), C.c_int64(len(R)),
            C.byref(pl), C.byref(val), C.byref(se)))
        return PriceEstimate(val.value, se.value, int(plan.num_paths))

    # -- annealer on device objectives --
    def minimize_builtin(self, objective: int, lower, upper, schedule: AnnealingSchedule, start,
                         predicate: int = A.PRED_NONE) -> AnnealResult:
        lo = np.asarray(lower, dtype=np.float64)
        hi = np.asarray(upper, dtype=np.float64)
        st = np.asarray(start, dtype=np.float64)
        dim = len(lo)
        best = np.zeros(max(1, dim))
        cap = n_levels(schedule, predicate == A.PRED_NONE) if schedule.t0 > 0 and 0 < schedule.cooling < 1 and schedule.t_min > 0 else 1
        tt = np.zeros(max(1, cap))
        tf = np.zeros(max(1, cap))
        res = A.sabr_anneal_result(_dptr(best), 0.0, 0, _dptr(tt), _dptr(tf), cap, 0)
        sch = schedule.to_abi()
        self._check(self.lib.sabr_minimize_builtin(self._ctx, C.c_int32(objective),
                                                   C.c_int32(predicate), _dptr(lo), _dptr(hi),
                                                   C.c_int64(dim), C.byref(sch), _dptr(st),
                                                   C.byref(res)))
        n = res.trace_len
        return AnnealResult(best[:dim].tolist(), res.best_value, res.evals,
                            list(zip(tt[:n].tolist(), tf[:n].tolist())))


# ------------------------------------------------- module-level functions ---
_default: Optional[Engine] = None
_default_lock = threading.Lock()


def default_engine() -> Engine:
    global _default
    with _default_lock:
        if _default is None:
            _default = Engine(0)
        return _default


def _raise_parse(st: int, lib) -> None:
    """io::parse_error is a std::runtime_error: SABR_E_RUNTIME from the surface
    loader is a ParseError (a NumericalError subclass)."""
    msg = lib.sabr_last_error().decode()
    if st == 4:  # SABR_E_RUNTIME
        raise ParseError(msg)
    raise_for_status(st, msg)


def parse_surface(path: str) -> VolSurface:
    """io::parse_surface (proj/src/io.cpp:151-161), implemented by the C++ host."""
    lib = A.load_library()
    ns, nq = C.c_int64(), C.c_int64()
    st = lib.sabr_surface_csv_dims(path.encode(), C.byref(ns), C.byref(nq))
    if st != A.SABR_OK:
        _raise_parse(st, lib)
    T, r, y = (np.zeros(ns.value) for _ in range(3))
    off = np.zeros(ns.value + 1, dtype=np.int64)
    K, v = np.zeros(nq.value), np.zeros(nq.value)
    spot = C.c_double()
    st = lib.sabr_surface_csv_read(path.encode(), C.byref(spot), _dptr(T), _dptr(r), _dptr(y),
                                   off.ctypes.data_as(C.POINTER(C.c_int64)), _dptr(K), _dptr(v))
    if st != A.SABR_OK:
        _raise_parse(st, lib)
    return VolSurface.from_arrays(spot.value, T, r, y, off, K, v)


def black_scholes_call(spot, strike, rate, dividend, maturity, vol) -> float:
    lib = A.load_library()
    out = C.c_double()
    st = lib.sabr_black_scholes_call(C.c_double(spot), C.c_double(strike), C.c_double(rate),
                                     C.c_double(dividend), C.c_double(maturity), C.c_double(vol),
                                     C.byref(out))
    if st != A.SABR_OK:
        raise_for_status(st, lib.sabr_last_error().decode())
    return out.value


def calibrate_static_T1(surface, slice, bounds=None, schedule=None, fixed=None):
    return default_engine().calibrate_static_T1(surface, slice, bounds, schedule, fixed)


def calibrate_static_T1_slices(surface, slices=None, bounds=None, schedule=None, fixed=None):
    return default_engine().calibrate_static_T1_slices(surface, slices, bounds, schedule, fixed)


def calibrate_dynamic_case1_T1(surface, bounds=None, schedule=None, fixed=None):
    return default_engine().calibrate_dynamic_case1_T1(surface, bounds, schedule, fixed)


def calibrate_case2_T2(surface, bounds=None, schedule=None, plan=None, fixed=None,
                       report_plan=None, start_override=None):
    return default_engine().calibrate_case2_T2(surface, bounds, schedule, plan, fixed,
                                               report_plan, start_override)


def calibrate_case2_formula(surface, bounds=None, schedule=None, fixed=None):
    return default_engine().calibrate_case2_formula(surface, bounds, schedule, fixed)


def evaluate_case1(surface, p):
    return default_engine().evaluate_case1(surface, p)


def evaluate_case2_prices(surface, p, plan):
    return default_engine().evaluate_case2_prices(surface, p, plan)
