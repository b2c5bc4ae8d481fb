// host_common.hpp — host-side mirror of the reference calibration API
// (validation, ParamSpace, surfaces, schedules) shared by the drivers.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sabr_b200.h"

namespace sabr_gpu {

// An error crossing the ABI: status + message (maps to the reference's
// exception type, see sabr_status).
struct Error : std::runtime_error {
    sabr_status status;
    Error(sabr_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(sabr_status s, const std::string& m) { throw Error(s, m); }
inline void require(bool ok, const char* msg) {
    if (!ok) fail(SABR_E_DOMAIN, msg);
}

// ---------------------------------------------------------------- surface ---
// VolSurface, proj/include/sabr/calibration.hpp:16-37 (SoA).
struct HostSurface {
    double spot = 0.0;
    std::vector<double> T, r, y;
    std::vector<int64_t> off;  // n+1
    std::vector<double> K, vol;

    size_t n() const { return T.size(); }
    size_t total_quotes() const { return K.size(); }
    size_t quotes(size_t i) const { return static_cast<size_t>(off[i + 1] - off[i]); }
    // slices.at(i): std::out_of_range with the libstdc++ message
    void at(size_t i) const {
        if (i >= n())
            fail(SABR_E_OUT_OF_RANGE, "vector::_M_range_check: __n (which is " + std::to_string(i) +
                                          ") >= this->size() (which is " + std::to_string(n()) + ")");
    }
    // VolSurface::forward -> forward_price, calibration.cpp:222-225, analytics.cpp:177-181
    double forward(size_t i) const {
        at(i);
        require(spot > 0, "forward_price: spot must be positive");
        require(T[i] > 0, "forward_price: maturity must be positive");
        return spot * std::exp((r[i] - y[i]) * T[i]);
    }
    // VolSurface::validate, calibration.cpp:233-251
    void validate() const {
        if (spot <= 0) fail(SABR_E_DOMAIN, "VolSurface: spot must be positive");
        if (n() == 0) fail(SABR_E_DOMAIN, "VolSurface: no slices");
        for (size_t i = 0; i < n(); ++i) {
            if (T[i] <= 0) fail(SABR_E_DOMAIN, "VolSurface: maturity must be positive");
            if (i > 0 && T[i] <= T[i - 1])
                fail(SABR_E_DOMAIN, "VolSurface: maturities must be strictly increasing");
            if (quotes(i) == 0)
                fail(SABR_E_DOMAIN, "VolSurface: empty quote block in slice " + std::to_string(i));
            for (int64_t j = off[i]; j < off[i + 1]; ++j) {
                if (K[j] <= 0 || vol[j] <= 0)
                    fail(SABR_E_DOMAIN, "VolSurface: strikes and vols must be positive");
                if (j > off[i] && K[j] <= K[j - 1])
                    fail(SABR_E_DOMAIN, "VolSurface: strikes must be strictly increasing");
            }
        }
    }
    static HostSurface from_abi(const sabr_surface* s) {
        if (!s) fail(SABR_E_INVALID, "surface is null");
        if (s->n_slices < 0) fail(SABR_E_INVALID, "surface: negative slice count");
        HostSurface h;
        h.spot = s->spot;
        const size_t n = static_cast<size_t>(s->n_slices);
        if (n && (!s->maturity || !s->rate || !s->dividend || !s->quote_offset))
            fail(SABR_E_INVALID, "surface: null slice arrays");
        h.T.assign(s->maturity, s->maturity + n);
        h.r.assign(s->rate, s->rate + n);
        h.y.assign(s->dividend, s->dividend + n);
        h.off.assign(s->quote_offset, s->quote_offset + n + 1);
        if (n == 0) h.off = {0};
        for (size_t i = 0; i < n; ++i)
            if (h.off[i + 1] < h.off[i]) fail(SABR_E_INVALID, "surface: quote offsets decrease");
        const int64_t nq = h.off.back() - h.off.front();
        if (h.off.front() != 0) fail(SABR_E_INVALID, "surface: quote offsets must start at 0");
        if (nq && (!s->strike || !s->vol)) fail(SABR_E_INVALID, "surface: null quote arrays");
        h.K.assign(s->strike, s->strike + nq);
        h.vol.assign(s->vol, s->vol + nq);
        return h;
    }
    HostSurface slice_only(size_t i) const {  // VolSurface one{spot, {slices[i]}}
        HostSurface o;
        o.spot = spot;
        o.T = {T[i]};
        o.r = {r[i]};
        o.y = {y[i]};
        o.off = {0, off[i + 1] - off[i]};
        o.K.assign(K.begin() + off[i], K.begin() + off[i + 1]);
        o.vol.assign(vol.begin() + off[i], vol.begin() + off[i + 1]);
        return o;
    }
};

// -------------------------------------------------------------- schedule ---
// AnnealingSchedule::validate, proj/src/annealer.cpp:28-39
inline void validate_schedule(const sabr_schedule& s) {
    if (!(s.t0 > 0)) fail(SABR_E_DOMAIN, "AnnealingSchedule: t0 must be positive");
    if (!(s.cooling > 0 && s.cooling < 1))
        fail(SABR_E_DOMAIN, "AnnealingSchedule: cooling must be in (0,1)");
    if (s.chain_length < 1) fail(SABR_E_DOMAIN, "AnnealingSchedule: chain_length must be >= 1");
    if (s.workers < 1 || s.groups < 1)
        fail(SABR_E_DOMAIN, "AnnealingSchedule: workers and groups must be >= 1");
    if (!(s.t_min > 0 && s.t_min < s.t0))
        fail(SABR_E_DOMAIN, "AnnealingSchedule: need 0 < t_min < t0");
    if (s.max_evals < 1) fail(SABR_E_DOMAIN, "AnnealingSchedule: max_evals must be >= 1");
}

// SimulationPlan::validate, proj/src/mc.cpp:161-166
inline void validate_plan(const sabr_plan& p) {
    if (p.num_paths < 1) fail(SABR_E_DOMAIN, "SimulationPlan: num_paths must be >= 1");
    if (!(p.dt > 0)) fail(SABR_E_DOMAIN, "SimulationPlan: dt must be positive");
    if (p.workers < 1) fail(SABR_E_DOMAIN, "SimulationPlan: workers must be >= 1");
    if (p.block_size < 1) fail(SABR_E_DOMAIN, "SimulationPlan: block_size must be >= 1");
    if (p.rng != SABR_RNG_XOSHIRO && p.rng != SABR_RNG_PHILOX)
        fail(SABR_E_DOMAIN, "SimulationPlan: unknown rng");
    if (p.precision != SABR_FP64 && p.precision != SABR_FP32)
        fail(SABR_E_DOMAIN, "SimulationPlan: unknown precision");
    if (p.num_paths > (1ull << 40)) fail(SABR_E_DOMAIN, "SimulationPlan: num_paths too large");
}

// The temperatures of annealer.cpp:99-100 (repeated product, not t0*c^k).
// The reference's level loop also stops once evals >= max_evals; when every
// step is an evaluation (no feasibility predicate) a level adds at least
// min(n_chains, remaining) evals, so at most ceil((max_evals - 1) / n_chains)
// + 1 levels can run and the list is cut there (a valid but extreme cooling
// such as 1 - 1e-10 would otherwise build ~1e11 temperatures).  max_levels < 0:
// no cut (with a predicate, infeasible steps do not count).
inline std::vector<double> temperatures(const sabr_schedule& s, int64_t max_levels = -1) {
    std::vector<double> t;
    for (double temp = s.t0; temp >= s.t_min; temp *= s.cooling) {
        if (max_levels >= 0 && static_cast<int64_t>(t.size()) >= max_levels) break;
        t.push_back(temp);
    }
    return t;
}

inline int64_t level_cap_all_evals(const sabr_schedule& s) {
    const int64_t n = static_cast<int64_t>(s.workers) * s.groups;
    return (s.max_evals - 1 + n - 1) / n + 1;
}

// ------------------------------------------------------------ ParamSpace ---
struct ParamDef {
    const char* name;
    double lo, hi, start;
};

// Default search boxes, proj/src/calibration.cpp:24-60
inline const std::vector<ParamDef>& static_defs() {
    static const std::vector<ParamDef> d = {
        {"alpha", 1e-4, 2.0, 0.3}, {"beta", 0.0, 1.0, 1.0}, {"nu", 1e-4, 10.0, 0.5}, {"rho", -1.0, 1.0, -0.3}};
    return d;
}
inline const std::vector<ParamDef>& case1_defs() {
    static const std::vector<ParamDef> d = {{"alpha", 1e-4, 2.0, 0.3}, {"beta", 0.0, 1.0, 1.0},
                                            {"rho0", -1.0, 1.0, -0.3}, {"nu0", 1e-4, 10.0, 0.5},
                                            {"a", 0.0, 150.0, 0.1},    {"b", 0.0, 150.0, 0.1}};
    return d;
}
inline const std::vector<ParamDef>& case2_defs() {
    static const std::vector<ParamDef> d = {
        {"alpha", 1e-4, 2.0, 0.3},  {"beta", 0.0, 1.0, 1.0},   {"rho0", -1.0, 1.0, -0.3},
        {"q_rho", -15.0, 15.0, 0.0}, {"d_rho", -1.0, 1.0, 0.0}, {"nu0", 1e-4, 10.0, 0.5},
        {"q_nu", -15.0, 15.0, 0.0},  {"d_nu", -1.0, 1.0, 0.0},  {"a", 0.0, 150.0, 0.1},
        {"b", 0.0, 150.0, 0.1}};
    return d;
}

using Bounds = std::map<std::string, std::pair<double, double>>;
using Fixed = std::map<std::string, double>;

inline Bounds bounds_from_abi(const sabr_bounds* b) {
    Bounds out;
    if (b && b->n > 0) {
        if (!b->names || !b->lo || !b->hi) fail(SABR_E_INVALID, "bounds: null arrays");
        for (int64_t i = 0; i < b->n; ++i) {
            if (!b->names[i]) fail(SABR_E_INVALID, "bounds: null name");
            out[b->names[i]] = {b->lo[i], b->hi[i]};
        }
    }
    return out;
}

inline Fixed fixed_from_abi(const sabr_fixed* f) {
    Fixed out;
    if (f && f->n > 0) {
        if (!f->names || !f->values) fail(SABR_E_INVALID, "fixed: null arrays");
        for (int64_t i = 0; i < f->n; ++i) {
            if (!f->names[i]) fail(SABR_E_INVALID, "fixed: null name");
            out[f->names[i]] = f->values[i];
        }
    }
    return out;
}

// ParamSpace, proj/src/calibration.cpp:64-141 (same checks, same messages).
struct ParamSpace {
    std::vector<ParamDef> defs;
    std::vector<size_t> free_ix;
    std::vector<double> fixed_values;
    std::vector<bool> is_free;

    ParamSpace(const std::vector<ParamDef>& base, const Bounds& bounds, const Fixed& fixed,
               double alpha_start) {
        defs = base;
        for (auto& d : defs) {
            if (auto it = bounds.find(d.name); it != bounds.end()) {
                if (!(it->second.first < it->second.second))
                    fail(SABR_E_DOMAIN, std::string("bounds for ") + d.name + ": lower must be below upper");
                d.lo = it->second.first;
                d.hi = it->second.second;
            }
            if (std::string(d.name) == "alpha" && alpha_start > 0)
                d.start = alpha_start < d.lo ? d.lo : (d.hi < alpha_start ? d.hi : alpha_start);
        }
        for (const auto& kv : bounds) {
            bool found = false;
            for (const auto& d : defs) found = found || kv.first == d.name;
            if (!found) fail(SABR_E_DOMAIN, "unknown bounds parameter: " + kv.first);
        }
        for (const auto& kv : fixed) {
            bool found = false;
            for (const auto& d : defs) found = found || kv.first == d.name;
            if (!found) fail(SABR_E_DOMAIN, "unknown fixed parameter: " + kv.first);
        }
        fixed_values.assign(defs.size(), 0.0);
        is_free.assign(defs.size(), true);
        for (size_t i = 0; i < defs.size(); ++i) {
            if (auto it = fixed.find(defs[i].name); it != fixed.end()) {
                is_free[i] = false;
                fixed_values[i] = it->second;
            } else {
                free_ix.push_back(i);
            }
        }
    }
    std::vector<double> full(const std::vector<double>& x) const {
        std::vector<double> out(defs.size());
        size_t j = 0;
        for (size_t i = 0; i < defs.size(); ++i) out[i] = is_free[i] ? x[j++] : fixed_values[i];
        return out;
    }
    std::vector<double> start_point() const {
        std::vector<double> x;
        for (size_t i : free_ix) {
            const auto& d = defs[i];
            x.push_back(d.start < d.lo ? d.lo : (d.hi < d.start ? d.hi : d.start));
        }
        return x;
    }
    uint32_t free_mask() const {
        uint32_t m = 0;
        for (size_t i : free_ix) m |= 1u << i;
        return m;
    }
    std::map<std::string, double> named(const std::vector<double>& full_params) const {
        std::map<std::string, double> m;
        for (size_t i = 0; i < defs.size(); ++i) m[defs[i].name] = full_params[i];
        return m;
    }
};

// atm_vol_guess, calibration.cpp:143-153
inline double atm_vol_guess(const HostSurface& s, size_t slice) {
    const double fwd = s.forward(slice);
    double best = s.vol[s.off[slice]], dist = std::abs(s.K[s.off[slice]] - fwd);
    for (int64_t j = s.off[slice]; j < s.off[slice + 1]; ++j)
        if (std::abs(s.K[j] - fwd) < dist) {
            dist = std::abs(s.K[j] - fwd);
            best = s.vol[j];
        }
    return best;
}

// ------------------------------------------------- model domain checks ---
// StaticSabrParams::validate, analytics.cpp:120-125
inline void validate_static(const double* p) {
    require(p[0] > 0, "StaticSabrParams: alpha must be positive");
    require(p[1] >= 0 && p[1] <= 1, "StaticSabrParams: beta must be in [0,1]");
    require(p[2] >= 0, "StaticSabrParams: nu must be nonnegative");
    require(p[3] >= -1 && p[3] <= 1, "StaticSabrParams: rho must be in [-1,1]");
}
// CaseIParams::validate, analytics.cpp:130-136
inline void validate_case1(const double* p) {
    require(p[0] > 0, "CaseIParams: alpha must be positive");
    require(p[1] >= 0 && p[1] <= 1, "CaseIParams: beta must be in [0,1]");
    require(p[2] >= -1 && p[2] <= 1, "CaseIParams: rho0 must be in [-1,1]");
    require(p[3] > 0, "CaseIParams: nu0 must be positive");
    require(p[4] >= 0 && p[5] >= 0, "CaseIParams: decay rates must be nonnegative");
}
// CaseIIParams::validate domain part, analytics.cpp:145-149 (the grid part
// raises SABR_E_CONSTRAINT, see engine.cu)
inline void validate_case2_domain(const double* p) {
    require(p[0] > 0, "CaseIIParams: alpha must be positive");
    require(p[1] >= 0 && p[1] <= 1, "CaseIIParams: beta must be in [0,1]");
    require(p[8] >= 0 && p[9] >= 0, "CaseIIParams: decay rates must be nonnegative");
    require(p[10] > 0, "CaseIIParams: horizon must be positive");
}

// black_scholes_call, proj/src/black_scholes.cpp:20-35 (market side of T_II;
// computed once per calibration on the host, like the reference).
inline double black_scholes_call(double spot, double strike, double rate, double dividend,
                                 double maturity, double vol) {
    if (spot <= 0 || strike <= 0 || maturity <= 0)
        fail(SABR_E_DOMAIN, "black_scholes_call: spot, strike, maturity must be positive");
    if (vol < 0) fail(SABR_E_DOMAIN, "black_scholes_call: vol must be nonnegative");
    const double df_div = spot * std::exp(-dividend * maturity);
    const double df_k = strike * std::exp(-rate * maturity);
    if (vol == 0.0) return (df_div - df_k < 0.0) ? 0.0 : df_div - df_k;
    const double sd = vol * std::sqrt(maturity);
    const double d1 = (std::log(spot / strike) + (rate - dividend + 0.5 * vol * vol) * maturity) / sd;
    const double d2 = d1 - sd;
    constexpr double kSqrt2 = 1.41421356237309504880;
    return df_div * (0.5 * std::erfc(-d1 / kSqrt2)) - df_k * (0.5 * std::erfc(-d2 / kSqrt2));
}

}  // namespace sabr_gpu
