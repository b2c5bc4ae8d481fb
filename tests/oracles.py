"""Test-side bindings of the two CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Ref``     — oracle/_ref/libsabr_ref.so: the unmodified reference library
                 compiled from /root/reference/proj/src + oracle/ref_capi.cpp.
* ``Restate`` — oracle/_build/libsabr_oracle.so: the plain-C restatement
                 (oracle/sabr_oracle.c), incl. the Philox stream twin.

Both take the same ctypes structures as the product ABI (include/sabr_b200.h).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2407_20713_b200 import _abi as A
from paper_2407_20713_b200.api import (AnnealResult, CalibrationReport, PriceEstimate,
                                       _bounds_abi, _dptr, _fixed_abi, _ReportBuf, model_of,
                                       n_levels, raise_for_status)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libsabr_ref.so")
RESTATE_LIB = os.path.join(ROOT, "oracle", "_build", "libsabr_oracle.so")
DATA_DIR = os.path.join(ROOT, "tests", "data")


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def have_restate() -> bool:
    return os.path.exists(RESTATE_LIB)


class Ref:
    """The compiled reference (OpenMP, libm) behind its own public API."""

    def __init__(self):
        self.lib = C.CDLL(REF_LIB)
        self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, st):
        if st != 0:
            raise_for_status(st, self.lib.ref_last_error().decode())

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    def cost_static(self, surface, slice, params):
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 4)
        out = np.empty(P.shape[0])
        self._check(self.lib.ref_cost_static(C.byref(s), C.c_int64(slice), _dptr(P),
                                             C.c_int64(P.shape[0]), _dptr(out)))
        return out

    def cost_case1(self, surface, params):
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 6)
        out = np.empty(P.shape[0])
        self._check(self.lib.ref_cost_case1(C.byref(s), _dptr(P), C.c_int64(P.shape[0]),
                                            _dptr(out)))
        return out

    def cost_case2_mc(self, surface, params, plan):
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
        out = np.empty(P.shape[0])
        pl = plan.to_abi()
        self._check(self.lib.ref_cost_case2_mc(C.byref(s), _dptr(P), C.c_int64(P.shape[0]),
                                               C.byref(pl), _dptr(out)))
        return out

    def case2_feasible(self, params):
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
        out = np.zeros(P.shape[0], dtype=np.uint8)
        self._check(self.lib.ref_case2_feasible(_dptr(P), C.c_int64(P.shape[0]),
                                                out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out.astype(bool)

    def static_vol(self, p, K, f, T):
        out = C.c_double()
        v = np.asarray(p, dtype=np.float64)
        self._check(self.lib.ref_static_vol(_dptr(v), C.c_double(K), C.c_double(f), C.c_double(T),
                                            C.byref(out)))
        return out.value

    def dyn_coeffs_case1(self, p, T):
        v = np.asarray(p, dtype=np.float64)
        out = np.zeros(4)
        self._check(self.lib.ref_dyn_coeffs_case1(_dptr(v), C.c_double(T), _dptr(out)))
        return out

    def dyn_coeffs_case2(self, p, T, nodes=64):
        v = np.asarray(p, dtype=np.float64)
        out = np.zeros(4)
        self._check(self.lib.ref_dyn_coeffs_case2(_dptr(v), C.c_double(T), C.c_int64(nodes),
                                                  _dptr(out)))
        return out

    def dynamic_vol(self, c, alpha, beta, K, f, T):
        cc = np.asarray(c, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.ref_dynamic_vol(_dptr(cc), C.c_double(alpha), C.c_double(beta),
                                             C.c_double(K), C.c_double(f), C.c_double(T),
                                             C.byref(out)))
        return out.value

    def market_prices(self, surface):
        s, keep = surface.to_abi()
        out = np.zeros(surface.total_quotes())
        self._check(self.lib.ref_market_prices(C.byref(s), _dptr(out)))
        return out

    def black_scholes_call(self, spot, K, r, y, T, vol):
        out = C.c_double()
        self._check(self.lib.ref_black_scholes_call(*(C.c_double(x) for x in (spot, K, r, y, T, vol)),
                                                    C.byref(out)))
        return out.value

    def implied_vol_from_price(self, price, spot, K, r, y, T):
        out = C.c_double()
        self._check(self.lib.ref_implied_vol_from_price(
            *(C.c_double(x) for x in (price, spot, K, r, y, T)), C.byref(out)))
        return out.value

    def _report(self, fn, surface, *args, trace_cap=0):
        rb = _ReportBuf(surface.total_quotes(), trace_cap)
        self._check(fn(*args, C.byref(rb.rep)))
        return rb.report()

    def calibrate_static_T1(self, surface, slice, bounds, schedule, fixed=None):
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        sch = schedule.to_abi()
        return self._report(self.lib.ref_calibrate_static_T1, surface, C.byref(s),
                            C.c_int64(slice), C.byref(b), C.byref(sch), C.byref(f))

    def calibrate_dynamic_case1_T1(self, surface, bounds, schedule, fixed=None):
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        sch = schedule.to_abi()
        return self._report(self.lib.ref_calibrate_dynamic_case1_T1, surface, C.byref(s),
                            C.byref(b), C.byref(sch), C.byref(f))

    def calibrate_case2_T2(self, surface, bounds, schedule, plan, fixed=None, report_plan=None,
                           start_override=None):
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        sch, pl = schedule.to_abi(), plan.to_abi()
        rp = C.byref(report_plan.to_abi()) if report_plan is not None else None
        if start_override is not None:
            st = np.asarray(start_override, dtype=np.float64)
            stp, stn = _dptr(st), len(st)
        else:
            st, stp, stn = None, None, 0
        return self._report(self.lib.ref_calibrate_case2_T2, surface, C.byref(s), C.byref(b),
                            C.byref(sch), C.byref(pl), C.byref(f), rp, stp, C.c_int64(stn))

    def calibrate_case2_formula(self, surface, bounds, schedule, fixed=None):
        s, keep = surface.to_abi()
        b, kb = _bounds_abi(bounds)
        f, kf = _fixed_abi(fixed)
        sch = schedule.to_abi()
        return self._report(self.lib.ref_calibrate_case2_formula, surface, C.byref(s),
                            C.byref(b), C.byref(sch), C.byref(f))

    def evaluate_case1(self, surface, p):
        s, keep = surface.to_abi()
        v = np.asarray(p.vector(), dtype=np.float64)
        return self._report(self.lib.ref_evaluate_case1, surface, C.byref(s), _dptr(v))

    def evaluate_case2_prices(self, surface, p, plan):
        s, keep = surface.to_abi()
        v = np.asarray(p.vector(), dtype=np.float64)
        pl = plan.to_abi()
        return self._report(self.lib.ref_evaluate_case2_prices, surface, C.byref(s), _dptr(v),
                            C.byref(pl))

    def _anneal(self, fn, dim, schedule, *args):
        best = np.zeros(max(1, dim))
        cap = n_levels(schedule, all_evals=False)
        tt, tf = np.zeros(max(1, cap)), np.zeros(max(1, cap))
        res = A.sabr_anneal_result(_dptr(best), 0.0, 0, _dptr(tt), _dptr(tf), cap, 0)
        self._check(fn(*args, C.byref(res)))
        n = res.trace_len
        return AnnealResult(best[:dim].tolist(), res.best_value, res.evals,
                            list(zip(tt[:n].tolist(), tf[:n].tolist())))

    def minimize_builtin(self, objective, lower, upper, schedule, start, predicate=0):
        lo, hi, st = (np.asarray(v, dtype=np.float64) for v in (lower, upper, start))
        sch = schedule.to_abi()
        return self._anneal(self.lib.ref_minimize_builtin, len(lo), schedule, C.c_int(objective),
                            C.c_int(predicate), _dptr(lo), _dptr(hi), C.c_int64(len(lo)),
                            C.byref(sch), _dptr(st))

    def minimize_cost(self, model, surface, slice, lower, upper, schedule, start):
        s, keep = surface.to_abi()
        lo, hi, st = (np.asarray(v, dtype=np.float64) for v in (lower, upper, start))
        sch = schedule.to_abi()
        return self._anneal(self.lib.ref_minimize_cost, len(lo), schedule, C.c_int(model),
                            C.byref(s), C.c_int64(slice), _dptr(lo), _dptr(hi),
                            C.c_int64(len(lo)), C.byref(sch), _dptr(st))

    def propose(self, current, temperature, lower, upper, t0, seed, stream, n):
        cur, lo, hi = (np.asarray(v, dtype=np.float64) for v in (current, lower, upper))
        out = np.zeros((n, len(cur)))
        self._check(self.lib.ref_propose(_dptr(cur), C.c_int64(len(cur)), C.c_double(temperature),
                                         _dptr(lo), _dptr(hi), C.c_double(t0), C.c_uint64(seed),
                                         C.c_uint64(stream), C.c_int64(n), _dptr(out)))
        return out

    def xoshiro_uniforms(self, seed, stream, n):
        out = np.zeros(n)
        self.lib.ref_xoshiro_uniforms(C.c_uint64(seed), C.c_uint64(stream), C.c_int64(n), _dptr(out))
        return out

    def simulate_terminals(self, params, f0, alpha0, T, plan, serial=False):
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        out = np.zeros(int(plan.num_paths))
        pl = plan.to_abi()
        self._check(self.lib.ref_simulate_terminals(C.c_int(model), _dptr(v), C.c_double(f0),
                                                    C.c_double(alpha0), C.c_double(T),
                                                    C.byref(pl), C.c_int(int(serial)), _dptr(out)))
        return out

    def price_european_batch(self, params, spot, strikes, r, y, T, plan):
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        K = np.asarray(strikes, dtype=np.float64)
        val, se = np.zeros(len(K)), np.zeros(len(K))
        pl = plan.to_abi()
        self._check(self.lib.ref_price_european_batch(
            C.c_int(model), _dptr(v), C.c_double(spot), _dptr(K), C.c_int64(len(K)), C.c_double(r),
            C.c_double(y), C.c_double(T), C.byref(pl), _dptr(val), _dptr(se)))
        return [PriceEstimate(float(val[j]), float(se[j]), int(plan.num_paths)) for j in range(len(K))]

    def price_cliquet(self, params, spot, r, y, lf, lc, gf, gc, resets, plan):
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        R = np.asarray(resets, dtype=np.float64)
        val, se = C.c_double(), C.c_double()
        pl = plan.to_abi()
        self._check(self.lib.ref_price_cliquet(
            C.c_int(model), _dptr(v), *(C.c_double(x) for x in (spot, r, y, lf, lc, gf, gc)),
            _dptr(R), C.c_int64(len(R)), C.byref(pl), C.byref(val), C.byref(se)))
        return PriceEstimate(val.value, se.value, int(plan.num_paths))


class Restate:
    """The plain-C restatement (oracle/sabr_oracle.c)."""

    def __init__(self):
        self.lib = C.CDLL(RESTATE_LIB)
        self.lib.orc_static_implied_vol.restype = C.c_double
        self.lib.orc_dynamic_implied_vol.restype = C.c_double
        self.lib.orc_cost_static.restype = C.c_double
        self.lib.orc_cost_case1.restype = C.c_double
        self.lib.orc_forward.restype = C.c_double
        self.lib.orc_black_scholes_call.restype = C.c_double
        self.lib.orc_xoshiro_uniform.restype = C.c_double

    def _check(self, st):
        if st != 0:
            raise_for_status(st, "oracle restatement: status %d" % st)

    def cost_static(self, surface, slice, params):
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 4)
        return np.array([self.lib.orc_cost_static(C.byref(s), C.c_int64(slice), _dptr(P[i]))
                         for i in range(P.shape[0])])

    def cost_case1(self, surface, params):
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 6)
        return np.array([self.lib.orc_cost_case1(C.byref(s), _dptr(np.ascontiguousarray(P[i])))
                         for i in range(P.shape[0])])

    def case2_feasible(self, params):
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
        return np.array([bool(self.lib.orc_case2_feasible(_dptr(np.ascontiguousarray(P[i]))))
                         for i in range(P.shape[0])])

    def cost_case2_mc(self, surface, params, plan):
        s, keep = surface.to_abi()
        P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
        pl = plan.to_abi()
        out = np.zeros(P.shape[0])
        for i in range(P.shape[0]):
            c = C.c_double()
            self._check(self.lib.orc_cost_case2_mc(C.byref(s), _dptr(np.ascontiguousarray(P[i])),
                                                   C.byref(pl), C.byref(c)))
            out[i] = c.value
        return out

    def static_vol(self, p, K, f, T):
        v = np.asarray(p, dtype=np.float64)
        return self.lib.orc_static_implied_vol(_dptr(v), C.c_double(K), C.c_double(f), C.c_double(T))

    def dyn_coeffs_case1(self, p, T):
        v = np.asarray(p, dtype=np.float64)
        out = np.zeros(4)
        self.lib.orc_dyn_coeffs_case1(_dptr(v), C.c_double(T), _dptr(out))
        return out

    def _anneal(self, fn, dim, schedule, *args):
        best = np.zeros(max(1, dim))
        cap = n_levels(schedule, all_evals=False)
        tt, tf = np.zeros(max(1, cap)), np.zeros(max(1, cap))
        res = A.sabr_anneal_result(_dptr(best), 0.0, 0, _dptr(tt), _dptr(tf), cap, 0)
        self._check(fn(*args, C.byref(res)))
        n = res.trace_len
        return AnnealResult(best[:dim].tolist(), res.best_value, res.evals,
                            list(zip(tt[:n].tolist(), tf[:n].tolist())))

    def minimize_cost(self, model, surface, slice, lower, upper, schedule, start):
        s, keep = surface.to_abi()
        lo, hi, st = (np.asarray(v, dtype=np.float64) for v in (lower, upper, start))
        sch = schedule.to_abi()
        return self._anneal(self.lib.orc_minimize_cost, len(lo), schedule, C.c_int(model),
                            C.byref(s), C.c_int64(slice), _dptr(lo), _dptr(hi), C.c_int(len(lo)),
                            C.byref(sch), _dptr(st))

    def minimize_builtin(self, objective, lower, upper, schedule, start, predicate=0):
        lo, hi, st = (np.asarray(v, dtype=np.float64) for v in (lower, upper, start))
        sch = schedule.to_abi()
        return self._anneal(self.lib.orc_minimize_builtin, len(lo), schedule, C.c_int(objective),
                            C.c_int(predicate), _dptr(lo), _dptr(hi), C.c_int(len(lo)),
                            C.byref(sch), _dptr(st))

    def simulate_terminals(self, params, f0, alpha0, T, plan):
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        out = np.zeros(int(plan.num_paths))
        pl = plan.to_abi()
        self._check(self.lib.orc_simulate_terminals(C.c_int(model), _dptr(v), C.c_double(f0),
                                                    C.c_double(alpha0), C.c_double(T),
                                                    C.byref(pl), _dptr(out)))
        return out

    def price_european_batch(self, params, spot, strikes, r, y, T, plan):
        model, v = model_of(params)
        v = np.asarray(v, dtype=np.float64)
        K = np.asarray(strikes, dtype=np.float64)
        val, se = np.zeros(len(K)), np.zeros(len(K))
        pl = plan.to_abi()
        self._check(self.lib.orc_price_european_batch(
            C.c_int(model), _dptr(v), C.c_double(spot), _dptr(K), C.c_int64(len(K)), C.c_double(r),
            C.c_double(y), C.c_double(T), C.byref(pl), _dptr(val), _dptr(se)))
        return [PriceEstimate(float(val[j]), float(se[j]), int(plan.num_paths)) for j in range(len(K))]

    def philox_uniform_pair(self, seed, path, step):
        a, b = C.c_double(), C.c_double()
        self.lib.orc_philox_uniform_pair(C.c_uint64(seed), C.c_uint64(path), C.c_uint32(step),
                                         C.byref(a), C.byref(b))
        return a.value, b.value

    def black_scholes_call(self, spot, K, r, y, T, vol):
        return self.lib.orc_black_scholes_call(*(C.c_double(x) for x in (spot, K, r, y, T, vol)))

    def implied_vol_from_price(self, price, spot, K, r, y, T):
        out = C.c_double()
        self._check(self.lib.orc_implied_vol_from_price(*(C.c_double(x) for x in (price, spot, K, r, y, T)),
                                                        C.byref(out)))
        return out.value


def ref_parse_surface(path):
    """io::parse_surface through the compiled reference."""
    from paper_2407_20713_b200.api import VolSurface
    r = Ref()
    ns, nq = C.c_int64(), C.c_int64()
    r._check(r.lib.ref_surface_csv_dims(path.encode(), C.byref(ns), C.byref(nq)))
    T, rr, y = (np.zeros(ns.value) for _ in range(3))
    off = np.zeros(ns.value + 1, dtype=np.int64)
    K, v = np.zeros(nq.value), np.zeros(nq.value)
    spot = C.c_double()
    r._check(r.lib.ref_surface_csv_read(path.encode(), C.byref(spot), _dptr(T), _dptr(rr), _dptr(y),
                                        off.ctypes.data_as(C.POINTER(C.c_int64)), _dptr(K), _dptr(v)))
    return VolSurface.from_arrays(spot.value, T, rr, y, off, K, v)


def atm_vol_guess(surface, slice):
    """atm_vol_guess, calibration.cpp:143-153 (alpha start of the calibrators)."""
    fwd = surface.forward(slice)
    qs = surface.slices[slice].quotes
    best, dist = qs[0].vol, abs(qs[0].strike - fwd)
    for q in qs:
        if abs(q.strike - fwd) < dist:
            dist, best = abs(q.strike - fwd), q.vol
    return best


def cost_sensitivity(orc, model, surface, slice, params):
    """|cost(libm +-1 ulp) - cost| per vector (oracle/sabr_oracle.c)."""
    orc.lib.orc_cost_sensitivity.restype = C.c_double
    s, keep = surface.to_abi()
    dim = 4 if model == A.MODEL_STATIC else 6
    P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, dim)
    return np.array([orc.lib.orc_cost_sensitivity(C.c_int(model), C.byref(s), C.c_int64(slice),
                                                  _dptr(np.ascontiguousarray(P[i])))
                     for i in range(P.shape[0])])


def ref_cost_case2_formula(ref, surface, params):
    s, keep = surface.to_abi()
    P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
    out = np.empty(P.shape[0])
    ref._check(ref.lib.ref_cost_case2_formula(C.byref(s), _dptr(P), C.c_int64(P.shape[0]), _dptr(out)))
    return out


def orc_cost_case2_formula(orc, surface, params):
    orc.lib.orc_cost_case2_formula.restype = C.c_double
    s, keep = surface.to_abi()
    P = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 11)
    return np.array([orc.lib.orc_cost_case2_formula(C.byref(s), _dptr(np.ascontiguousarray(P[i])))
                     for i in range(P.shape[0])])


def orc_dyn_coeffs_case2(orc, p, T, nodes=8):
    v = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(4)
    orc.lib.orc_dyn_coeffs_case2(_dptr(v), C.c_double(T), C.c_int(nodes), _dptr(out))
    return out


def orc_price_cliquet(orc, params, spot, r, y, lf, lc, gf, gc, resets, plan):
    model, v = model_of(params)
    v = np.asarray(v, dtype=np.float64)
    R = np.asarray(resets, dtype=np.float64)
    val, se = C.c_double(), C.c_double()
    pl = plan.to_abi()
    st = orc.lib.orc_price_cliquet(C.c_int(model), _dptr(v), *(C.c_double(x) for x in (spot, r, y, lf, lc, gf, gc)),
                                   _dptr(R), C.c_int(len(R)), C.byref(pl), C.byref(val), C.byref(se))
    if st != 0:
        raise_for_status(st, "oracle restatement: status %d" % st)
    return PriceEstimate(val.value, se.value, int(plan.num_paths))
