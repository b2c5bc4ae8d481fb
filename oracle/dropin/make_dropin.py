#!/usr/bin/env python3
"""oracle/dropin/make_dropin.py — TEST INFRASTRUCTURE ONLY.

Builds, under oracle/_ref/dropin/ (git-ignored, never committed), the patched
copy of the reference a maintainer would have after applying INTEGRATION.md:

* src/calibration.cpp: the one-line SABR_BACKEND=b200 dispatch at the top of
  calibrate_static_T1 (calibration.cpp:289), calibrate_dynamic_case1_T1
  (:325), evaluate_case1 (:367), evaluate_case2_prices (:420),
  calibrate_case2_T2 (:450) and calibrate_case2_formula (:483), each to the
  same-signature sabr::b200:: function of integration/sabr_b200_adapter.cpp;
* include/sabr/mc.hpp: the one-line accessor INTEGRATION.md names for
  mc::ModelDynamics (its parameter structs are private);
* src/mc.cpp: the same dispatch at the top of simulate_terminals (mc.cpp:231),
  price_european_batch (:249) and price_cliquet (:275); the serial oracle
  mc::reference::simulate_terminals stays on the CPU.

Every insertion is anchored on the exact reference text and asserted, so a
changed reference fails loudly instead of being patched wrongly.  Nothing else
changes: the other sources, the tests (proj/tests/*.cpp) and the CLI
(proj/tools/sabr_cli.cpp) are compiled from /root/reference as they are.
"""
import os
import sys

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/proj"
OUT = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "_ref",
                                                          "dropin")

GATE = 'const char* b = std::getenv("SABR_BACKEND"); b && std::string(b) == "b200"'


def read(rel):
    with open(os.path.join(REF, rel)) as f:
        return f.read()


def write(rel, text):
    path = os.path.join(OUT, rel)
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        f.write(text)


def insert_after(text, anchor, addition):
    assert text.count(anchor) == 1, f"anchor not unique or missing: {anchor[:70]!r}"
    return text.replace(anchor, anchor + addition)


def dispatch(call):
    return f"\n    if ({GATE})\n        return {call};"


def patch_calibration():
    t = read("src/calibration.cpp")
    t = insert_after(t, '#include "sabr/calibration.hpp"',
                     '\n#include <cstdlib>\n#include "sabr_b200_adapter.hpp"  // SABR_BACKEND=b200 (INTEGRATION.md)')
    t = insert_after(t, """CalibrationReport calibrate_static_T1(const VolSurface& surface, std::size_t slice,
                                      const BoundsOverrides& bounds,
                                      const AnnealingSchedule& schedule,
                                      const FixedParams& fixed) {""",
                     dispatch("b200::calibrate_static_T1(surface, slice, bounds, schedule, fixed)"))
    t = insert_after(t, """CalibrationReport calibrate_dynamic_case1_T1(const VolSurface& surface,
                                             const BoundsOverrides& bounds,
                                             const AnnealingSchedule& schedule,
                                             const FixedParams& fixed) {""",
                     dispatch("b200::calibrate_dynamic_case1_T1(surface, bounds, schedule, fixed)"))
    t = insert_after(t, "CalibrationReport evaluate_case1(const VolSurface& surface, const CaseIParams& p) {",
                     dispatch("b200::evaluate_case1(surface, p)"))
    t = insert_after(t, """CalibrationReport evaluate_case2_prices(const VolSurface& surface,
                                        const CaseIIParams& p,
                                        const mc::SimulationPlan& plan) {""",
                     dispatch("b200::evaluate_case2_prices(surface, p, plan)"))
    t = insert_after(t, """                                     const std::optional<mc::SimulationPlan>& report_plan,
                                     const std::vector<double>* start_override) {""",
                     dispatch("b200::calibrate_case2_T2(surface, bounds, schedule, plan, fixed, report_plan, "
                              "start_override)"))
    t = insert_after(t, """CalibrationReport calibrate_case2_formula(const VolSurface& surface,
                                          const BoundsOverrides& bounds,
                                          const AnnealingSchedule& schedule,
                                          const FixedParams& fixed) {""",
                     dispatch("b200::calibrate_case2_formula(surface, bounds, schedule, fixed)"))
    write("src/calibration.cpp", t)


def patch_mc():
    h = read("include/sabr/mc.hpp")
    h = insert_after(h, "    double rho_at(double t) const;\n",
                     "    // b200 dispatch (INTEGRATION.md): the parameters the dynamics were built from\n"
                     "    const StaticSabrParams& static_params() const { return static_; }\n"
                     "    const CaseIParams& case1_params() const { return case1_; }\n"
                     "    const CaseIIParams& case2_params() const { return case2_; }\n")
    write("include/sabr/mc.hpp", h)

    def by_variant(fn, args):
        return (f"\n    if ({GATE}) {{\n"
                f"        switch (model.variant()) {{\n"
                f"            case ModelVariant::Static: return b200::{fn}(model.static_params(), {args});\n"
                f"            case ModelVariant::CaseI: return b200::{fn}(model.case1_params(), {args});\n"
                f"            case ModelVariant::CaseII: return b200::{fn}(model.case2_params(), {args});\n"
                f"        }}\n    }}")

    t = read("src/mc.cpp")
    t = insert_after(t, '#include "sabr/mc.hpp"',
                     '\n#include <cstdlib>\n#include "sabr_b200_adapter.hpp"  // SABR_BACKEND=b200 (INTEGRATION.md)')
    anchor_sim = """std::vector<double> simulate_terminals(const ModelDynamics& model, double forward0,
                                       double alpha0, double maturity,
                                       const SimulationPlan& plan) {
    plan.validate();
    const Grid grid"""
    # the same text opens mc::reference::simulate_terminals (the serial oracle,
    # mc.cpp:324), which must stay on the CPU: patch the first one only
    ref_ns = t.index("namespace reference {")
    at = t.index(anchor_sim)
    assert at < ref_ns and t.count(anchor_sim) == 2
    head = anchor_sim[: anchor_sim.index("\n    plan.validate();")]
    t = (t[:at] + head + by_variant("simulate_terminals", "forward0, alpha0, maturity, plan") +
         "\n    plan.validate();\n    const Grid grid" + t[at + len(anchor_sim):])
    t = insert_after(t, """std::vector<PriceEstimate> price_european_batch(const ModelDynamics& model,
                                                double spot,
                                                const std::vector<double>& strikes,
                                                double rate, double dividend,
                                                double maturity,
                                                const SimulationPlan& plan) {""",
                     by_variant("price_european_batch", "spot, strikes, rate, dividend, maturity, plan"))
    t = insert_after(t, """PriceEstimate price_cliquet(const ModelDynamics& model, double spot, double rate,
                            double dividend, const CliquetSpec& spec,
                            const SimulationPlan& plan) {""",
                     by_variant("price_cliquet", "spot, rate, dividend, spec, plan"))
    write("src/mc.cpp", t)


if __name__ == "__main__":
    patch_calibration()
    patch_mc()
    # the remaining headers unchanged, so include/sabr resolves entirely to the patched tree
    for name in os.listdir(os.path.join(REF, "include", "sabr")):
        if name != "mc.hpp":
            write(os.path.join("include", "sabr", name), read(os.path.join("include", "sabr", name)))
    print("patched reference written to", os.path.abspath(OUT))
