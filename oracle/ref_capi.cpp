// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI wrapper around the UNMODIFIED reference library of
// arxiv/paper_2407_20713 (/root/reference/proj/src/*.cpp), compiled together
// with those sources into oracle/_ref/libsabr_ref.so by oracle/Makefile.  It
// is the checker the parity tests and the golden-vector script use, and the
// `--impl reference` / cpu_baseline leg of bench.py.  Nothing in the product
// (paper_2407_20713_b200/) links or loads it.
//
// The structs are the ones of include/sabr_b200.h, so a test can hand the very
// same ctypes objects to the product ABI and to this oracle.
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "sabr/analytics.hpp"
#include "sabr/annealer.hpp"
#include "sabr/black_scholes.hpp"
#include "sabr/calibration.hpp"
#include "sabr/io.hpp"
#include "sabr/mc.hpp"
#include "sabr_b200.h"

using namespace sabr;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SABR_OK;
    } catch (const constraint_error& e) {
        g_err = e.what();
        return SABR_E_CONSTRAINT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SABR_E_DOMAIN;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return SABR_E_OUT_OF_RANGE;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return SABR_E_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SABR_E_LOGIC;
    }
}

VolSurface to_surface(const sabr_surface* s) {
    VolSurface out;
    out.spot = s->spot;
    for (int64_t i = 0; i < s->n_slices; ++i) {
        VolSlice sl;
        sl.maturity = s->maturity[i];
        sl.rate = s->rate[i];
        sl.dividend = s->dividend[i];
        for (int64_t j = s->quote_offset[i]; j < s->quote_offset[i + 1]; ++j)
            sl.quotes.push_back({s->strike[j], s->vol[j]});
        out.slices.push_back(std::move(sl));
    }
    return out;
}

AnnealingSchedule to_schedule(const sabr_schedule* s) {
    AnnealingSchedule a;
    a.t0 = s->t0;
    a.cooling = s->cooling;
    a.chain_length = s->chain_length;
    a.workers = s->workers;
    a.groups = s->groups;
    a.t_min = s->t_min;
    a.max_evals = s->max_evals;
    a.seed = s->seed;
    a.omp_threads = s->omp_threads;
    return a;
}

mc::SimulationPlan to_plan(const sabr_plan* p) {
    mc::SimulationPlan q;
    q.num_paths = p->num_paths;
    q.dt = p->dt;
    q.seed = p->seed;
    q.workers = p->workers;
    q.block_size = p->block_size;
    return q;
}

BoundsOverrides to_bounds(const sabr_bounds* b) {
    BoundsOverrides out;
    if (b)
        for (int64_t i = 0; i < b->n; ++i) out[b->names[i]] = {b->lo[i], b->hi[i]};
    return out;
}

FixedParams to_fixed(const sabr_fixed* f) {
    FixedParams out;
    if (f)
        for (int64_t i = 0; i < f->n; ++i) out[f->names[i]] = f->values[i];
    return out;
}

void copy_name(char* dst, const std::string& s) {
    std::memset(dst, 0, SABR_NAME_LEN);
    std::strncpy(dst, s.c_str(), SABR_NAME_LEN - 1);
}

void fill_report(const CalibrationReport& r, sabr_report* out) {
    copy_name(out->model, r.model);
    copy_name(out->technique, r.technique);
    copy_name(out->quantity, r.quantity);
    out->n_params = 0;
    for (const auto& [k, v] : r.params) {
        if (out->n_params >= SABR_MAX_PARAMS) break;
        copy_name(out->param_names[out->n_params], k);
        out->param_values[out->n_params] = v;
        ++out->n_params;
    }
    out->final_cost = r.final_cost;
    out->mean_rel_error = r.mean_rel_error;
    out->max_rel_error = r.max_rel_error;
    out->wall_seconds = r.wall_seconds;
    out->evals = r.evals;
    out->seed = r.seed;
    out->n_rows = static_cast<int64_t>(r.rows.size());
    if (out->rows) {
        if (out->rows_capacity < out->n_rows) throw std::logic_error("rows capacity too small");
        for (std::size_t i = 0; i < r.rows.size(); ++i)
            out->rows[i] = {r.rows[i].maturity, r.rows[i].strike, r.rows[i].market,
                            r.rows[i].model, r.rows[i].rel_error};
    }
    out->trace_len = 0;
}

mc::ModelDynamics to_model(int model, const double* p) {
    switch (model) {
        case SABR_MODEL_STATIC:
            return mc::ModelDynamics::from_static(StaticSabrParams{p[0], p[1], p[2], p[3]});
        case SABR_MODEL_CASE1:
            return mc::ModelDynamics::from_case1(CaseIParams{p[0], p[1], p[2], p[3], p[4], p[5]});
        case SABR_MODEL_CASE2:
            return mc::ModelDynamics::from_case2(CaseIIParams{p[0], p[1], p[2], p[3], p[4], p[5],
                                                              p[6], p[7], p[8], p[9], p[10]});
    }
    throw std::domain_error("unknown model");
}

CaseIIParams case2_params(const double* p) {
    return CaseIIParams{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8], p[9], p[10]};
}

// Restatement of the anonymous case2_mc_cost (calibration.cpp:399-416) with
// the reference's own public functions.
double case2_mc_cost(const VolSurface& surface, const CaseIIParams& p,
                     const mc::SimulationPlan& plan,
                     const std::vector<std::vector<double>>& market) {
    const auto model = mc::ModelDynamics::from_case2(p);
    double sum = 0.0;
    for (std::size_t i = 0; i < surface.slices.size(); ++i) {
        const auto& s = surface.slices[i];
        std::vector<double> strikes;
        for (const auto& q : s.quotes) strikes.push_back(q.strike);
        const auto estimates = mc::price_european_batch(model, surface.spot, strikes, s.rate,
                                                        s.dividend, s.maturity, plan);
        for (std::size_t j = 0; j < estimates.size(); ++j) {
            const double rel = (market[i][j] - estimates[j].value) / market[i][j];
            sum += rel * rel;
        }
    }
    return sum;
}

// The closed-form objectives of proj/tests/test_annealer.cpp.
double sq(double x) { return x * x; }
Objective builtin(int id) {
    switch (id) {
        case SABR_OBJ_BOWL3:
            return [](std::span<const double> x) {
                return sq(x[0] - 1.2) + sq(x[1] + 0.7) + sq(x[2] - 3.4);
            };
        case SABR_OBJ_ROSENBROCK4:
            return [](std::span<const double> x) {
                double v = 0.0;
                for (int i = 0; i < 3; ++i) v += 100.0 * sq(x[i + 1] - sq(x[i])) + sq(1.0 - x[i]);
                return v;
            };
        case SABR_OBJ_SINQUAD2:
            return [](std::span<const double> x) {
                return sq(x[0] - 0.3) + 3.0 * sq(x[1] + 2.1) + 0.1 * std::sin(7.0 * x[0]);
            };
        case SABR_OBJ_SQUARE1:
            return [](std::span<const double> x) { return sq(x[0]); };
        case SABR_OBJ_COSBOWL2:
            return [](std::span<const double> x) {
                return sq(x[0]) + sq(x[1]) + std::cos(3.0 * x[0]);
            };
        case SABR_OBJ_CORNER2:
            return [](std::span<const double> x) { return sq(x[0] - 2.0) + sq(x[1] - 2.0); };
        case SABR_OBJ_NANRIGHT1:
            return [](std::span<const double> x) {
                if (x[0] > 0.5) return std::numeric_limits<double>::quiet_NaN();
                return sq(x[0] + 1.0);
            };
    }
    throw std::domain_error("unknown builtin objective");
}

}  // namespace

extern "C" {

SABR_API const char* ref_last_error(void) { return g_err.c_str(); }

SABR_API int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

SABR_API int ref_surface_csv_dims(const char* path, int64_t* n_slices, int64_t* n_quotes) {
    return guarded([&] {
        const auto s = io::parse_surface(path);
        *n_slices = static_cast<int64_t>(s.slices.size());
        *n_quotes = static_cast<int64_t>(s.total_quotes());
    });
}

SABR_API int ref_surface_csv_read(const char* path, double* spot, double* T, double* r,
                                  double* y, int64_t* off, double* K, double* vol) {
    return guarded([&] {
        const auto s = io::parse_surface(path);
        *spot = s.spot;
        int64_t q = 0;
        for (std::size_t i = 0; i < s.slices.size(); ++i) {
            T[i] = s.slices[i].maturity;
            r[i] = s.slices[i].rate;
            y[i] = s.slices[i].dividend;
            off[i] = q;
            for (const auto& quote : s.slices[i].quotes) {
                K[q] = quote.strike;
                vol[q] = quote.vol;
                ++q;
            }
        }
        off[s.slices.size()] = q;
    });
}

SABR_API int ref_forward(const sabr_surface* s, int64_t slice, double* out) {
    return guarded([&] { *out = to_surface(s).forward(static_cast<std::size_t>(slice)); });
}

SABR_API int ref_static_vol(const double* p, double strike, double forward, double T,
                            double* out) {
    return guarded(
        [&] { *out = static_implied_vol(StaticSabrParams{p[0], p[1], p[2], p[3]}, strike, forward, T); });
}

SABR_API int ref_dyn_coeffs_case1(const double* p, double T, double* out4) {
    return guarded([&] {
        const auto c = dyn_coeffs_case1(CaseIParams{p[0], p[1], p[2], p[3], p[4], p[5]}, T);
        out4[0] = c.nu1_sq;
        out4[1] = c.nu2_sq;
        out4[2] = c.eta1;
        out4[3] = c.eta2_sq;
    });
}

SABR_API int ref_dyn_coeffs_case2(const double* p, double T, int64_t nodes, double* out4) {
    return guarded([&] {
        const auto c = dyn_coeffs_case2(case2_params(p), T, static_cast<std::size_t>(nodes));
        out4[0] = c.nu1_sq;
        out4[1] = c.nu2_sq;
        out4[2] = c.eta1;
        out4[3] = c.eta2_sq;
    });
}

SABR_API int ref_dynamic_vol(const double* c4, double alpha, double beta, double strike,
                             double forward, double T, double* out) {
    return guarded([&] {
        *out = dynamic_implied_vol(DynCoefficients{c4[0], c4[1], c4[2], c4[3]}, alpha, beta, strike,
                                   forward, T);
    });
}

// Objective of calibrate_static_T1 (calibration.cpp:300-306) for full params.
SABR_API int ref_cost_static(const sabr_surface* s, int64_t slice, const double* params,
                             int64_t n, double* cost) {
    return guarded([&] {
        const auto surface = to_surface(s);
        const double fwd = surface.forward(static_cast<std::size_t>(slice));
        for (int64_t i = 0; i < n; ++i) {
            const double* v = params + 4 * i;
            const StaticSabrParams p{v[0], v[1], v[2], v[3]};
            cost[i] = cost_individual(surface, static_cast<std::size_t>(slice),
                                      [&](double strike, double T) {
                                          return static_implied_vol(p, strike, fwd, T);
                                      });
        }
    });
}

// Objective of calibrate_dynamic_case1_T1 (calibration.cpp:339-353).
SABR_API int ref_cost_case1(const sabr_surface* s, const double* params, int64_t n,
                            double* cost) {
    return guarded([&] {
        const auto surface = to_surface(s);
        std::vector<double> forwards;
        for (std::size_t i = 0; i < surface.slices.size(); ++i) forwards.push_back(surface.forward(i));
        for (int64_t k = 0; k < n; ++k) {
            const double* v = params + 6 * k;
            const CaseIParams p{v[0], v[1], v[2], v[3], v[4], v[5]};
            double sum = 0.0;
            for (std::size_t i = 0; i < surface.slices.size(); ++i) {
                const auto coeffs = dyn_coeffs_case1(p, surface.slices[i].maturity);
                sum += cost_individual(surface, i, [&](double strike, double T) {
                    return dynamic_implied_vol(coeffs, p.alpha, p.beta, strike, forwards[i], T);
                });
            }
            cost[k] = sum;
        }
    });
}

// Objective of calibrate_case2_T2 (calibration.cpp:464-466); params n x 11.
SABR_API int ref_cost_case2_mc(const sabr_surface* s, const double* params, int64_t n,
                               const sabr_plan* plan, double* cost) {
    return guarded([&] {
        const auto surface = to_surface(s);
        const auto market = market_prices(surface);
        const auto pl = to_plan(plan);
        for (int64_t k = 0; k < n; ++k)
            cost[k] = case2_mc_cost(surface, case2_params(params + 11 * k), pl, market);
    });
}

// The calibrate_case2_formula objective (calibration.cpp:497-520), restated
// with the reference's own public functions; params n x 11 (horizon last).
SABR_API int ref_cost_case2_formula(const sabr_surface* s, const double* params, int64_t n,
                                    double* cost) {
    return guarded([&] {
        const auto surface = to_surface(s);
        const auto market = market_prices(surface);
        std::vector<double> forwards;
        for (std::size_t i = 0; i < surface.slices.size(); ++i) forwards.push_back(surface.forward(i));
        for (int64_t k = 0; k < n; ++k) {
            const auto p = case2_params(params + 11 * k);
            double sum = 0.0;
            bool bad = false;
            for (std::size_t i = 0; i < surface.slices.size() && !bad; ++i) {
                const auto& sl = surface.slices[i];
                const auto coeffs = dyn_coeffs_case2(p, sl.maturity, 8);
                for (std::size_t j = 0; j < sl.quotes.size(); ++j) {
                    const double vol = dynamic_implied_vol(coeffs, p.alpha, p.beta, sl.quotes[j].strike,
                                                           forwards[i], sl.maturity);
                    if (!(vol > 0)) {
                        bad = true;
                        break;
                    }
                    const double price = black_scholes_call(surface.spot, sl.quotes[j].strike, sl.rate,
                                                            sl.dividend, sl.maturity, vol);
                    const double rel = (market[i][j] - price) / market[i][j];
                    sum += rel * rel;
                }
            }
            cost[k] = bad ? 1e10 : sum;
        }
    });
}

SABR_API int ref_case2_feasible(const double* params, int64_t n, uint8_t* out) {
    return guarded([&] {
        for (int64_t k = 0; k < n; ++k) {
            try {
                case2_params(params + 11 * k).validate();
                out[k] = 1;
            } catch (const std::exception&) {
                out[k] = 0;
            }
        }
    });
}

SABR_API int ref_market_prices(const sabr_surface* s, double* out) {
    return guarded([&] {
        const auto p = market_prices(to_surface(s));
        int64_t q = 0;
        for (const auto& row : p)
            for (double v : row) out[q++] = v;
    });
}

SABR_API int ref_black_scholes_call(double spot, double strike, double r, double y, double T,
                                    double vol, double* out) {
    return guarded([&] { *out = black_scholes_call(spot, strike, r, y, T, vol); });
}

SABR_API int ref_implied_vol_from_price(double price, double spot, double strike, double r,
                                        double y, double T, double* out) {
    return guarded([&] { *out = implied_vol_from_price(price, spot, strike, r, y, T); });
}

SABR_API int ref_calibrate_static_T1(const sabr_surface* s, int64_t slice, const sabr_bounds* b,
                                     const sabr_schedule* sch, const sabr_fixed* f,
                                     sabr_report* out) {
    return guarded([&] {
        const auto r = calibrate_static_T1(to_surface(s), static_cast<std::size_t>(slice),
                                           to_bounds(b), to_schedule(sch), to_fixed(f));
        fill_report(r, out);
    });
}

SABR_API int ref_calibrate_dynamic_case1_T1(const sabr_surface* s, const sabr_bounds* b,
                                            const sabr_schedule* sch, const sabr_fixed* f,
                                            sabr_report* out) {
    return guarded([&] {
        const auto r = calibrate_dynamic_case1_T1(to_surface(s), to_bounds(b), to_schedule(sch),
                                                  to_fixed(f));
        fill_report(r, out);
    });
}

SABR_API int ref_calibrate_case2_T2(const sabr_surface* s, const sabr_bounds* b,
                                    const sabr_schedule* sch, const sabr_plan* plan,
                                    const sabr_fixed* f, const sabr_plan* report_plan,
                                    const double* start, int64_t start_len, sabr_report* out) {
    return guarded([&] {
        std::optional<mc::SimulationPlan> rp;
        if (report_plan) rp = to_plan(report_plan);
        std::vector<double> st;
        if (start) st.assign(start, start + start_len);
        const auto r = calibrate_case2_T2(to_surface(s), to_bounds(b), to_schedule(sch),
                                          to_plan(plan), to_fixed(f), rp, start ? &st : nullptr);
        fill_report(r, out);
    });
}

SABR_API int ref_calibrate_case2_formula(const sabr_surface* s, const sabr_bounds* b,
                                         const sabr_schedule* sch, const sabr_fixed* f,
                                         sabr_report* out) {
    return guarded([&] {
        const auto r = calibrate_case2_formula(to_surface(s), to_bounds(b), to_schedule(sch),
                                               to_fixed(f));
        fill_report(r, out);
    });
}

SABR_API int ref_evaluate_case1(const sabr_surface* s, const double* p, sabr_report* out) {
    return guarded([&] {
        fill_report(evaluate_case1(to_surface(s), CaseIParams{p[0], p[1], p[2], p[3], p[4], p[5]}),
                    out);
    });
}

SABR_API int ref_evaluate_case2_prices(const sabr_surface* s, const double* p,
                                       const sabr_plan* plan, sabr_report* out) {
    return guarded(
        [&] { fill_report(evaluate_case2_prices(to_surface(s), case2_params(p), to_plan(plan)), out); });
}

SABR_API int ref_minimize_builtin(int objective, int predicate, const double* lo, const double* hi,
                                  int64_t dim, const sabr_schedule* sch, const double* start,
                                  sabr_anneal_result* res) {
    return guarded([&] {
        SearchSpace space{std::vector<double>(lo, lo + dim), std::vector<double>(hi, hi + dim),
                          nullptr};
        if (predicate == SABR_PRED_SUM_LE_1)
            space.feasible = [](std::span<const double> x) { return x[0] + x[1] <= 1.0; };
        const auto r = minimize(builtin(objective), space, to_schedule(sch),
                                std::vector<double>(start, start + dim));
        for (int64_t i = 0; i < dim; ++i) res->best_point[i] = r.best_point[i];
        res->best_value = r.best_value;
        res->evals = r.evals;
        res->trace_len = static_cast<int64_t>(r.temperature_trace.size());
        if (res->trace_t) {
            if (res->trace_capacity < res->trace_len) throw std::logic_error("trace capacity");
            for (std::size_t i = 0; i < r.temperature_trace.size(); ++i) {
                res->trace_t[i] = r.temperature_trace[i].first;
                res->trace_f[i] = r.temperature_trace[i].second;
            }
        }
    });
}

// Full annealer run of the static / case1 T_I objectives with the trace
// (calibrate_* do not expose it): same ParamSpace-free full-vector search the
// calibrators run when nothing is fixed.
SABR_API int ref_minimize_cost(int model, const sabr_surface* s, int64_t slice, const double* lo,
                               const double* hi, int64_t dim, const sabr_schedule* sch,
                               const double* start, sabr_anneal_result* res) {
    return guarded([&] {
        const auto surface = to_surface(s);
        std::vector<double> forwards;
        for (std::size_t i = 0; i < surface.slices.size(); ++i) forwards.push_back(surface.forward(i));
        Objective obj;
        if (model == SABR_MODEL_STATIC) {
            obj = [&](std::span<const double> v) {
                const StaticSabrParams p{v[0], v[1], v[2], v[3]};
                return cost_individual(surface, static_cast<std::size_t>(slice),
                                       [&](double strike, double T) {
                                           return static_implied_vol(p, strike, forwards[slice], T);
                                       });
            };
        } else {
            obj = [&](std::span<const double> v) {
                const CaseIParams p{v[0], v[1], v[2], v[3], v[4], v[5]};
                double sum = 0.0;
                for (std::size_t i = 0; i < surface.slices.size(); ++i) {
                    const auto coeffs = dyn_coeffs_case1(p, surface.slices[i].maturity);
                    sum += cost_individual(surface, i, [&](double strike, double T) {
                        return dynamic_implied_vol(coeffs, p.alpha, p.beta, strike, forwards[i], T);
                    });
                }
                return sum;
            };
        }
        SearchSpace space{std::vector<double>(lo, lo + dim), std::vector<double>(hi, hi + dim),
                          nullptr};
        const auto r = minimize(obj, space, to_schedule(sch), std::vector<double>(start, start + dim));
        for (int64_t i = 0; i < dim; ++i) res->best_point[i] = r.best_point[i];
        res->best_value = r.best_value;
        res->evals = r.evals;
        res->trace_len = static_cast<int64_t>(r.temperature_trace.size());
        if (res->trace_t) {
            if (res->trace_capacity < res->trace_len) throw std::logic_error("trace capacity");
            for (std::size_t i = 0; i < r.temperature_trace.size(); ++i) {
                res->trace_t[i] = r.temperature_trace[i].first;
                res->trace_f[i] = r.temperature_trace[i].second;
            }
        }
    });
}

SABR_API int ref_propose(const double* current, int64_t dim, double temperature,
                         const double* lo, const double* hi, double t0, uint64_t seed,
                         uint64_t stream, int64_t n, double* out) {
    return guarded([&] {
        SearchSpace space{std::vector<double>(lo, lo + dim), std::vector<double>(hi, hi + dim),
                          nullptr};
        Xoshiro256pp rng(seed, stream);
        std::vector<double> x(current, current + dim);
        for (int64_t k = 0; k < n; ++k) {
            x = propose(x, temperature, space, t0, rng);
            for (int64_t i = 0; i < dim; ++i) out[k * dim + i] = x[i];
        }
    });
}

SABR_API int ref_xoshiro_uniforms(uint64_t seed, uint64_t stream, int64_t n, double* out) {
    Xoshiro256pp rng(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.uniform();
    return SABR_OK;
}

SABR_API int ref_simulate_terminals(int model, const double* params, double f0, double alpha0,
                                    double T, const sabr_plan* plan, int serial, double* out) {
    return guarded([&] {
        const auto m = to_model(model, params);
        const auto v = serial ? mc::reference::simulate_terminals(m, f0, alpha0, T, to_plan(plan))
                              : mc::simulate_terminals(m, f0, alpha0, T, to_plan(plan));
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

SABR_API int ref_price_european_batch(int model, const double* params, double spot,
                                      const double* strikes, int64_t m, double r, double y,
                                      double T, const sabr_plan* plan, double* value,
                                      double* se) {
    return guarded([&] {
        const auto est = mc::price_european_batch(to_model(model, params), spot,
                                                  std::vector<double>(strikes, strikes + m), r, y, T,
                                                  to_plan(plan));
        for (int64_t j = 0; j < m; ++j) {
            value[j] = est[j].value;
            se[j] = est[j].std_error;
        }
    });
}

SABR_API int ref_price_cliquet(int model, const double* params, double spot, double r, double y,
                               double lf, double lc, double gf, double gc, const double* resets,
                               int64_t n_resets, const sabr_plan* plan, double* value,
                               double* se) {
    return guarded([&] {
        mc::CliquetSpec spec{lf, lc, gf, gc, std::vector<double>(resets, resets + n_resets)};
        const auto est = mc::price_cliquet(to_model(model, params), spot, r, y, spec, to_plan(plan));
        *value = est.value;
        *se = est.std_error;
    });
}

}  // extern "C"
