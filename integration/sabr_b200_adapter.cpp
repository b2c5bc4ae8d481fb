// integration/sabr_b200_adapter.cpp — see sabr_b200_adapter.hpp.  Converts
// the reference's value types into the C-ABI's SoA views, calls the engine,
// rethrows the matching reference exception type and assembles the
// CalibrationReport the reference returns (calibration.hpp:47-59).
#include "sabr_b200_adapter.hpp"

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "sabr/types.hpp"
#include "sabr_b200.h"

namespace sabr::b200 {
namespace {

struct SurfaceSoA {  // VolSurface -> sabr_surface
    std::vector<double> T, r, y, K, v;
    std::vector<int64_t> off{0};
    sabr_surface view{};
    explicit SurfaceSoA(const VolSurface& s) {
        for (const auto& sl : s.slices) {
            T.push_back(sl.maturity);
            r.push_back(sl.rate);
            y.push_back(sl.dividend);
            for (const auto& q : sl.quotes) {
                K.push_back(q.strike);
                v.push_back(q.vol);
            }
            off.push_back(static_cast<int64_t>(K.size()));
        }
        view = {s.spot, static_cast<int64_t>(T.size()), T.data(), r.data(), y.data(), off.data(), K.data(), v.data()};
    }
};

struct Named {  // BoundsOverrides / FixedParams -> sabr_bounds / sabr_fixed
    std::vector<const char*> names;
    std::vector<double> a, b;
};

[[noreturn]] void rethrow(sabr_status st) {
    const std::string m = sabr_last_error();
    switch (st) {
        case SABR_E_DOMAIN: throw std::domain_error(m);
        case SABR_E_OUT_OF_RANGE: throw std::out_of_range(m);
        case SABR_E_CONSTRAINT: throw constraint_error(m, 0.0);
        default: throw std::runtime_error(m);
    }
}

sabr_ctx* context() {  // one context per process, device from SABR_DEVICE
    static std::once_flag once;
    static sabr_ctx* ctx = nullptr;
    std::call_once(once, [] {
        const char* d = std::getenv("SABR_DEVICE");
        if (sabr_status st = sabr_ctx_create(d ? std::atoi(d) : 0, nullptr, &ctx)) rethrow(st);
    });
    return ctx;
}

sabr_schedule to_abi(const AnnealingSchedule& a) {
    return sabr_schedule{a.t0, a.cooling, a.chain_length, a.workers, a.groups, a.omp_threads,
                         a.t_min, static_cast<int64_t>(a.max_evals), a.seed};
}

sabr_plan to_abi(const mc::SimulationPlan& p) {
    sabr_plan out{};
    out.num_paths = p.num_paths;
    out.dt = p.dt;
    out.seed = p.seed;
    out.workers = p.workers;
    out.rng = SABR_RNG_XOSHIRO;  // the reference's streams
    out.block_size = p.block_size;
    out.precision = SABR_FP64;
    return out;
}

// Run one ABI calibrator with caller-owned report storage, then build the
// reference's CalibrationReport from it.
template <class Call>
CalibrationReport run(const VolSurface& s, const BoundsOverrides& bounds, const FixedParams& fixed, Call&& call) {
    Named nb, nf;
    for (const auto& [k, v] : bounds) {
        nb.names.push_back(k.c_str());
        nb.a.push_back(v.first);
        nb.b.push_back(v.second);
    }
    for (const auto& [k, v] : fixed) {
        nf.names.push_back(k.c_str());
        nf.a.push_back(v);
    }
    const sabr_bounds bb{static_cast<int64_t>(nb.names.size()), nb.names.data(), nb.a.data(), nb.b.data()};
    const sabr_fixed ff{static_cast<int64_t>(nf.names.size()), nf.names.data(), nf.a.data()};
    SurfaceSoA soa(s);
    std::vector<sabr_report_row> rows(soa.K.size());
    sabr_report rep{};
    rep.rows = rows.data();
    rep.rows_capacity = static_cast<int64_t>(rows.size());
    if (sabr_status st = call(context(), &soa.view, &bb, &ff, &rep)) rethrow(st);
    CalibrationReport out{};
    out.model = rep.model;
    out.technique = rep.technique;
    out.quantity = rep.quantity;
    for (int64_t i = 0; i < rep.n_params; ++i) out.params[rep.param_names[i]] = rep.param_values[i];
    for (int64_t i = 0; i < rep.n_rows; ++i)
        out.rows.push_back({rows[i].maturity, rows[i].strike, rows[i].market, rows[i].model, rows[i].rel_error});
    out.final_cost = rep.final_cost;
    out.mean_rel_error = rep.mean_rel_error;
    out.max_rel_error = rep.max_rel_error;
    out.wall_seconds = rep.wall_seconds;
    out.evals = static_cast<long>(rep.evals);
    out.seed = rep.seed;
    return out;
}

// Parameter structs -> (sabr_model, flat vector in the ABI's order).
struct ModelArgs {
    int32_t model;
    std::vector<double> v;
};
ModelArgs model_args(const StaticSabrParams& p) { return {SABR_MODEL_STATIC, {p.alpha, p.beta, p.nu, p.rho}}; }
ModelArgs model_args(const CaseIParams& p) {
    return {SABR_MODEL_CASE1, {p.alpha, p.beta, p.rho0, p.nu0, p.a, p.b}};
}
ModelArgs model_args(const CaseIIParams& p) {
    return {SABR_MODEL_CASE2,
            {p.alpha, p.beta, p.rho0, p.q_rho, p.d_rho, p.nu0, p.q_nu, p.d_nu, p.a, p.b, p.horizon}};
}

}  // namespace

template <class Params>
std::vector<double> simulate_terminals(const Params& p, double forward0, double alpha0, double maturity,
                                       const mc::SimulationPlan& plan) {
    const ModelArgs m = model_args(p);
    const sabr_plan pl = to_abi(plan);
    std::vector<double> out(plan.num_paths);
    if (sabr_status st = sabr_mc_simulate_terminals(context(), m.model, m.v.data(), forward0, alpha0, maturity,
                                                    &pl, out.data()))
        rethrow(st);
    return out;
}

template <class Params>
std::vector<mc::PriceEstimate> price_european_batch(const Params& p, double spot, const std::vector<double>& strikes,
                                                    double rate, double dividend, double maturity,
                                                    const mc::SimulationPlan& plan) {
    const ModelArgs m = model_args(p);
    const sabr_plan pl = to_abi(plan);
    std::vector<double> value(strikes.size()), se(strikes.size());
    if (sabr_status st = sabr_mc_price_european_batch(context(), m.model, m.v.data(), spot, strikes.data(),
                                                      static_cast<int64_t>(strikes.size()), rate, dividend,
                                                      maturity, &pl, value.data(), se.data()))
        rethrow(st);
    std::vector<mc::PriceEstimate> out;
    for (size_t j = 0; j < strikes.size(); ++j) out.push_back({value[j], se[j], plan.num_paths});
    return out;
}

template <class Params>
mc::PriceEstimate price_european_call(const Params& p, double spot, double strike, double rate, double dividend,
                                      double maturity, const mc::SimulationPlan& plan) {
    return price_european_batch(p, spot, std::vector<double>{strike}, rate, dividend, maturity, plan)[0];
}

template <class Params>
mc::PriceEstimate price_cliquet(const Params& p, double spot, double rate, double dividend,
                                const mc::CliquetSpec& spec, const mc::SimulationPlan& plan) {
    const ModelArgs m = model_args(p);
    const sabr_plan pl = to_abi(plan);
    double value = 0.0, se = 0.0;
    if (sabr_status st = sabr_mc_price_cliquet(context(), m.model, m.v.data(), spot, rate, dividend,
                                               spec.local_floor, spec.local_cap, spec.global_floor, spec.global_cap,
                                               spec.reset_dates.data(), static_cast<int64_t>(spec.reset_dates.size()),
                                               &pl, &value, &se))
        rethrow(st);
    return {value, se, plan.num_paths};
}

#define SABR_B200_MC(P)                                                                                        \
    template std::vector<double> simulate_terminals<P>(const P&, double, double, double,                     \
                                                       const mc::SimulationPlan&);                            \
    template std::vector<mc::PriceEstimate> price_european_batch<P>(const P&, double, const std::vector<double>&, \
                                                                    double, double, double,                    \
                                                                    const mc::SimulationPlan&);                \
    template mc::PriceEstimate price_european_call<P>(const P&, double, double, double, double, double,       \
                                                      const mc::SimulationPlan&);                              \
    template mc::PriceEstimate price_cliquet<P>(const P&, double, double, double, const mc::CliquetSpec&,      \
                                                const mc::SimulationPlan&);
SABR_B200_MC(StaticSabrParams)
SABR_B200_MC(CaseIParams)
SABR_B200_MC(CaseIIParams)
#undef SABR_B200_MC

CalibrationReport calibrate_static_T1(const VolSurface& surface, std::size_t slice, const BoundsOverrides& bounds,
                                      const AnnealingSchedule& schedule, const FixedParams& fixed) {
    const sabr_schedule sch = to_abi(schedule);
    return run(surface, bounds, fixed, [&](sabr_ctx* c, const sabr_surface* s, const sabr_bounds* b,
                                           const sabr_fixed* f, sabr_report* r) {
        return sabr_calibrate_static_T1(c, s, static_cast<int64_t>(slice), b, &sch, f, r);
    });
}

CalibrationReport calibrate_dynamic_case1_T1(const VolSurface& surface, const BoundsOverrides& bounds,
                                             const AnnealingSchedule& schedule, const FixedParams& fixed) {
    const sabr_schedule sch = to_abi(schedule);
    return run(surface, bounds, fixed, [&](sabr_ctx* c, const sabr_surface* s, const sabr_bounds* b,
                                           const sabr_fixed* f, sabr_report* r) {
        return sabr_calibrate_dynamic_case1_T1(c, s, b, &sch, f, r);
    });
}

CalibrationReport calibrate_case2_T2(const VolSurface& surface, const BoundsOverrides& bounds,
                                     const AnnealingSchedule& schedule, const mc::SimulationPlan& plan,
                                     const FixedParams& fixed, const std::optional<mc::SimulationPlan>& report_plan,
                                     const std::vector<double>* start_override) {
    const sabr_schedule sch = to_abi(schedule);
    const sabr_plan pl = to_abi(plan);
    const sabr_plan rp = report_plan ? to_abi(*report_plan) : sabr_plan{};
    return run(surface, bounds, fixed, [&](sabr_ctx* c, const sabr_surface* s, const sabr_bounds* b,
                                           const sabr_fixed* f, sabr_report* r) {
        return sabr_calibrate_case2_T2(c, s, b, &sch, &pl, f, report_plan ? &rp : nullptr,
                                       start_override ? start_override->data() : nullptr,
                                       start_override ? static_cast<int64_t>(start_override->size()) : 0, r);
    });
}

CalibrationReport calibrate_case2_formula(const VolSurface& surface, const BoundsOverrides& bounds,
                                          const AnnealingSchedule& schedule, const FixedParams& fixed) {
    const sabr_schedule sch = to_abi(schedule);
    return run(surface, bounds, fixed, [&](sabr_ctx* c, const sabr_surface* s, const sabr_bounds* b,
                                           const sabr_fixed* f, sabr_report* r) {
        return sabr_calibrate_case2_formula(c, s, b, &sch, f, r);
    });
}

CalibrationReport evaluate_case1(const VolSurface& surface, const CaseIParams& p) {
    const ModelArgs m = model_args(p);
    return run(surface, {}, {}, [&](sabr_ctx* c, const sabr_surface* s, const sabr_bounds*, const sabr_fixed*,
                                    sabr_report* r) { return sabr_evaluate_case1(c, s, m.v.data(), r); });
}

CalibrationReport evaluate_case2_prices(const VolSurface& surface, const CaseIIParams& p,
                                        const mc::SimulationPlan& plan) {
    const ModelArgs m = model_args(p);
    const sabr_plan pl = to_abi(plan);
    return run(surface, {}, {}, [&](sabr_ctx* c, const sabr_surface* s, const sabr_bounds*, const sabr_fixed*,
                                    sabr_report* r) { return sabr_evaluate_case2_prices(c, s, m.v.data(), &pl, r); });
}

}  // namespace sabr::b200
