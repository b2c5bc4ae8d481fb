// integration/sabr_b200_adapter.hpp — the reference-side adapter of INTEGRATION.md
// as a compiled, tested file: the reference's calibrate_* signatures
// (proj/include/sabr/calibration.hpp:82-104) implemented on the B200 engine's
// C-ABI (include/sabr_b200.h).  A maintainer adds this file to proj/src and
// dispatches to it from sabr::calibrate_* when SABR_BACKEND=b200; here it is
// linked against the reference's own objects by oracle/Makefile (target
// `adapter`) and checked by tests/test_gpu_adapter.py.
#pragma once

#include <optional>
#include <vector>

#include "sabr/calibration.hpp"
#include "sabr/mc.hpp"

namespace sabr::b200 {

CalibrationReport calibrate_static_T1(const VolSurface& surface, std::size_t slice,
                                      const BoundsOverrides& bounds, const AnnealingSchedule& schedule,
                                      const FixedParams& fixed = {});

CalibrationReport calibrate_dynamic_case1_T1(const VolSurface& surface, const BoundsOverrides& bounds,
                                             const AnnealingSchedule& schedule, const FixedParams& fixed = {});

CalibrationReport calibrate_case2_T2(const VolSurface& surface, const BoundsOverrides& bounds,
                                     const AnnealingSchedule& schedule, const mc::SimulationPlan& plan,
                                     const FixedParams& fixed = {},
                                     const std::optional<mc::SimulationPlan>& report_plan = std::nullopt,
                                     const std::vector<double>* start_override = nullptr);

CalibrationReport calibrate_case2_formula(const VolSurface& surface, const BoundsOverrides& bounds,
                                          const AnnealingSchedule& schedule, const FixedParams& fixed = {});

CalibrationReport evaluate_case1(const VolSurface& surface, const CaseIParams& p);

CalibrationReport evaluate_case2_prices(const VolSurface& surface, const CaseIIParams& p,
                                        const mc::SimulationPlan& plan);

// The Monte Carlo operator (mc.hpp:66-84).  mc::ModelDynamics keeps its
// parameters private, so the device versions take the parameter structs the
// dynamics are built from (ModelDynamics::from_static / from_case1 /
// from_case2): a maintainer dispatches where the parameters are in hand
// (case2_mc_cost, calibration.cpp:399-416; the CLI's price command), or adds
// an accessor to ModelDynamics.  Same streams (xoshiro, block_size paths per
// substream), same results to rounding.
template <class Params>
std::vector<double> simulate_terminals(const Params& p, double forward0, double alpha0, double maturity,
                                       const mc::SimulationPlan& plan);

template <class Params>
std::vector<mc::PriceEstimate> price_european_batch(const Params& p, double spot, const std::vector<double>& strikes,
                                                    double rate, double dividend, double maturity,
                                                    const mc::SimulationPlan& plan);

template <class Params>
mc::PriceEstimate price_european_call(const Params& p, double spot, double strike, double rate, double dividend,
                                      double maturity, const mc::SimulationPlan& plan);

template <class Params>
mc::PriceEstimate price_cliquet(const Params& p, double spot, double rate, double dividend,
                                const mc::CliquetSpec& spec, const mc::SimulationPlan& plan);

}  // namespace sabr::b200
