// integration/adapter_check.cpp — runs the reference's calibrate_* (CPU) and
// the adapter's sabr::b200::calibrate_* (B200 engine) on the same inputs and
// prints one JSON line per case (doubles as hex) for tests/test_gpu_adapter.py.
//   adapter_check <data dir>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "sabr/io.hpp"
#include "sabr_b200_adapter.hpp"

using namespace sabr;

static std::string hx(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "\"%a\"", v);
    return b;
}

static void emit(const char* name, const CalibrationReport& r, const CalibrationReport& g) {
    std::string p = "{", q = "{";
    for (const auto& [k, v] : r.params) p += "\"" + k + "\": " + hx(v) + ", ";
    for (const auto& [k, v] : g.params) q += "\"" + k + "\": " + hx(v) + ", ";
    p = p.substr(0, p.size() - 2) + "}";
    q = q.substr(0, q.size() - 2) + "}";
    std::string rm = "[", gm = "[";
    for (const auto& row : r.rows) rm += hx(row.model) + ", ";
    for (const auto& row : g.rows) gm += hx(row.model) + ", ";
    rm = (r.rows.empty() ? "[" : rm.substr(0, rm.size() - 2)) + "]";
    gm = (g.rows.empty() ? "[" : gm.substr(0, gm.size() - 2)) + "]";
    std::printf("{\"case\": \"%s\", \"ref\": {\"cost\": %s, \"evals\": %ld, \"model\": \"%s\", \"params\": %s, "
                "\"rows\": %s}, \"b200\": {\"cost\": %s, \"evals\": %ld, \"model\": \"%s\", \"params\": %s, "
                "\"rows\": %s}}\n",
                name, hx(r.final_cost).c_str(), r.evals, r.model.c_str(), p.c_str(), rm.c_str(),
                hx(g.final_cost).c_str(), g.evals, g.model.c_str(), q.c_str(), gm.c_str());
}

template <class F>
static std::string kind(F&& f) {
    try {
        f();
    } catch (const std::out_of_range&) {
        return "out_of_range";
    } catch (const std::domain_error&) {
        return "domain_error";
    } catch (const constraint_error&) {
        return "constraint_error";
    } catch (const std::runtime_error&) {
        return "runtime_error";
    }
    return "none";
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "tests/data";
    const VolSurface eq = io::parse_surface(dir + "/eurostoxx50.csv");
    const VolSurface fx = io::parse_surface(dir + "/eurusd.csv");

    AnnealingSchedule s1;  // acceptance.cpp:318-323 (C1)
    s1.t0 = 2.0;
    s1.cooling = 0.96;
    s1.chain_length = 100;
    s1.workers = 32;
    s1.t_min = 1e-7;
    s1.seed = 2;
    emit("static_T1", calibrate_static_T1(eq, 1, {}, s1), b200::calibrate_static_T1(eq, 1, {}, s1));

    AnnealingSchedule s3 = s1;
    s3.cooling = 0.8;
    s3.t_min = 1e-4;
    s3.seed = 3;
    emit("case1_T1", calibrate_dynamic_case1_T1(fx, {}, s3, {{"beta", 1.0}}),
         b200::calibrate_dynamic_case1_T1(fx, {}, s3, {{"beta", 1.0}}));

    VolSurface one{eq.spot, {eq.slices[2]}};
    const FixedParams fixed{{"a", 0.0}, {"b", 0.0}, {"q_rho", 0.0}, {"q_nu", 0.0}, {"d_rho", 0.0}, {"d_nu", 0.0},
                            {"beta", 1.0}};
    AnnealingSchedule s4;
    s4.t0 = 2.0;
    s4.cooling = 0.5;
    s4.chain_length = 4;
    s4.workers = 6;
    s4.t_min = 0.2;
    s4.seed = 3;
    mc::SimulationPlan plan;
    plan.num_paths = 4096;
    plan.seed = 1;
    emit("case2_T2", calibrate_case2_T2(one, {}, s4, plan, fixed), b200::calibrate_case2_T2(one, {}, s4, plan, fixed));

    AnnealingSchedule s5 = s1;  // Case II formula objective (calibration.hpp:108-111), short schedule
    s5.chain_length = 20;
    s5.cooling = 0.7;
    s5.t_min = 1e-3;
    s5.seed = 4;
    emit("case2_formula", calibrate_case2_formula(fx, {}, s5, {{"beta", 1.0}}),
         b200::calibrate_case2_formula(fx, {}, s5, {{"beta", 1.0}}));
    const CaseIParams e1{0.13, 1.0, -0.25, 0.9, 0.7, 1.1};
    emit("evaluate_case1", evaluate_case1(fx, e1), b200::evaluate_case1(fx, e1));
    const CaseIIParams e2{0.13, 1.0, -0.25, 0.05, 0.02, 0.9, -0.1, 0.05, 0.7, 1.1, fx.slices.back().maturity};
    mc::SimulationPlan ep;
    ep.num_paths = 1u << 14;
    ep.seed = 5;
    emit("evaluate_case2_prices", evaluate_case2_prices(fx, e2, ep), b200::evaluate_case2_prices(fx, e2, ep));

    // the Monte Carlo operator (mc.hpp:66-84): same streams, prices to rounding
    mc::SimulationPlan mp;
    mp.num_paths = 1u << 16;
    mp.seed = 3;
    const std::vector<double> strikes{1900.0, 2100.0, 2257.37, 2400.0, 2700.0};
    auto emit_prices = [&](const char* name, const std::vector<mc::PriceEstimate>& r,
                           const std::vector<mc::PriceEstimate>& g) {
        std::string a = "[", b = "[";
        for (size_t j = 0; j < r.size(); ++j) {
            a += "[" + hx(r[j].value) + ", " + hx(r[j].std_error) + "]" + (j + 1 < r.size() ? ", " : "");
            b += "[" + hx(g[j].value) + ", " + hx(g[j].std_error) + "]" + (j + 1 < g.size() ? ", " : "");
        }
        std::printf("{\"case\": \"%s\", \"ref\": %s], \"b200\": %s]}\n", name, a.c_str(), b.c_str());
    };
    const StaticSabrParams sp{0.375162, 0.7, 0.331441, -0.6};
    emit_prices("mc_static", mc::price_european_batch(mc::ModelDynamics::from_static(sp), 2257.37, strikes, 0.018196,
                                                      0.034516, 0.495890, mp),
                b200::price_european_batch(sp, 2257.37, strikes, 0.018196, 0.034516, 0.495890, mp));
    const CaseIParams c1{0.3, 1.0, -0.4, 0.6, 1.5, 0.8};
    emit_prices("mc_case1", mc::price_european_batch(mc::ModelDynamics::from_case1(c1), 2257.37, strikes, 0.018196,
                                                     0.034516, 0.99, mp),
                b200::price_european_batch(c1, 2257.37, strikes, 0.018196, 0.034516, 0.99, mp));
    const CaseIIParams c2{0.3, 1.0, -0.4, 0.1, 0.05, 0.6, -0.1, 0.1, 1.0, 0.5, 1.0};
    emit_prices("mc_case2", mc::price_european_batch(mc::ModelDynamics::from_case2(c2), 2257.37, strikes, 0.018196,
                                                     0.034516, 1.0, mp),
                b200::price_european_batch(c2, 2257.37, strikes, 0.018196, 0.034516, 1.0, mp));
    {
        mc::SimulationPlan tp = mp;
        tp.num_paths = 10000;
        tp.block_size = 1000;
        const auto r = mc::simulate_terminals(mc::ModelDynamics::from_static(sp), 2300.0, sp.alpha, 0.75, tp);
        const auto g = b200::simulate_terminals(sp, 2300.0, sp.alpha, 0.75, tp);
        double worst = r.size() == g.size() ? 0.0 : 1.0;
        for (size_t i = 0; i < std::min(r.size(), g.size()); ++i)
            worst = std::max(worst, std::fabs(g[i] - r[i]) / std::fabs(r[i]));
        std::printf("{\"case\": \"mc_terminals\", \"n\": %zu, \"max_rel\": %.3e}\n", g.size(), worst);
    }
    {
        mc::CliquetSpec cs{-0.05, 0.05, 0.0, 0.2, {0.25, 0.5, 0.75, 1.0}};
        const auto r = mc::price_cliquet(mc::ModelDynamics::from_static(sp), 2257.37, 0.018196, 0.034516, cs, mp);
        const auto g = b200::price_cliquet(sp, 2257.37, 0.018196, 0.034516, cs, mp);
        emit_prices("mc_cliquet", {r}, {g});
    }

    // the reference's exception types come back through the adapter (test_calibration.cpp:212-225)
    const std::string r1 = kind([&] { calibrate_static_T1(eq, 9, {}, s1); });
    const std::string g1 = kind([&] { b200::calibrate_static_T1(eq, 9, {}, s1); });
    const std::string r2 = kind([&] { calibrate_static_T1(eq, 0, {{"nu", {5.0, 0.01}}}, s1); });
    const std::string g2 = kind([&] { b200::calibrate_static_T1(eq, 0, {{"nu", {5.0, 0.01}}}, s1); });
    const std::string r3 = kind([&] { calibrate_static_T1(eq, 0, {}, s1, {{"gamma", 1.0}}); });
    const std::string g3 = kind([&] { b200::calibrate_static_T1(eq, 0, {}, s1, {{"gamma", 1.0}}); });
    mc::SimulationPlan bad = mp;
    bad.num_paths = 0;
    const std::string r4 = kind([&] { mc::price_european_batch(mc::ModelDynamics::from_static(sp), 2257.37, strikes, 0.0, 0.0, 1.0, bad); });
    const std::string g4 = kind([&] { b200::price_european_batch(sp, 2257.37, strikes, 0.0, 0.0, 1.0, bad); });
    std::printf("{\"case\": \"errors\", \"ref\": [\"%s\", \"%s\", \"%s\", \"%s\"], "
                "\"b200\": [\"%s\", \"%s\", \"%s\", \"%s\"]}\n",
                r1.c_str(), r2.c_str(), r3.c_str(), r4.c_str(), g1.c_str(), g2.c_str(), g3.c_str(), g4.c_str());
    return 0;
}
