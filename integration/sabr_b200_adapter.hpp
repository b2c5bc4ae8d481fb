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

}  // namespace sabr::b200
