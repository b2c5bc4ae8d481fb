// integration/adapter_check.cpp — runs the reference's calibrate_* (CPU) and
// the adapter's sabr::b200::calibrate_* (B200 engine) on the same inputs and
// prints one JSON line per case (doubles as hex) for tests/test_gpu_adapter.py.
//   adapter_check <data dir>
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

    // the reference's exception types come back through the adapter (test_calibration.cpp:212-225)
    const std::string r1 = kind([&] { calibrate_static_T1(eq, 9, {}, s1); });
    const std::string g1 = kind([&] { b200::calibrate_static_T1(eq, 9, {}, s1); });
    const std::string r2 = kind([&] { calibrate_static_T1(eq, 0, {{"nu", {5.0, 0.01}}}, s1); });
    const std::string g2 = kind([&] { b200::calibrate_static_T1(eq, 0, {{"nu", {5.0, 0.01}}}, s1); });
    const std::string r3 = kind([&] { calibrate_static_T1(eq, 0, {}, s1, {{"gamma", 1.0}}); });
    const std::string g3 = kind([&] { b200::calibrate_static_T1(eq, 0, {}, s1, {{"gamma", 1.0}}); });
    std::printf("{\"case\": \"errors\", \"ref\": [\"%s\", \"%s\", \"%s\"], \"b200\": [\"%s\", \"%s\", \"%s\"]}\n",
                r1.c_str(), r2.c_str(), r3.c_str(), g1.c_str(), g2.c_str(), g3.c_str());
    return 0;
}
