// slice_qr.hpp — one slice's cost as a 4x4 quadratic form.
//
// The per-quote relative error of both Eq. 7 and Eq. 8 is linear in three
// strike-independent terms x = (C0, A1, A2) = (1 + B T, A1, A2) / omega:
//     r_j = 1 - (C0 + A1 l_j + A2 l_j^2) / m_j,   l_j = ln(K_j / f), m_j = market
// (analytics.cpp:203-204, calibration.cpp:262), so the slice cost
// sum_j r_j^2 (calibration.cpp:253-267) is ||W v||^2 with the n x 4 matrix
// W = [1/m, l/m, l^2/m, 1] and v = (C0, A1, A2, -1).  With the thin QR
// factorisation W = Q R, ||W v||^2 = ||R v||^2:
//     u0 = R00 C0 + R01 A1 + R02 A2 - R03
//     u1 =          R11 A1 + R12 A2 - R13
//     u2 =                   R22 A2 - R23
//     cost = u0^2 + u1^2 + u2^2 + R33^2
// nine FMAs per slice instead of four per quote.  R is computed once per
// surface on the host in binary128 (Householder), then rounded to double.
// Near the optimum the u_i are small and the cost is R33^2 plus their
// squares, so the rounding of R perturbs the cost by O(ulp * |u| * |R||v|),
// not by the O(ulp * |r| * |W||v|) of the per-quote sum: the factored cost
// agrees with the reference's per-quote sum to ~1e-14 relative on the fixture
// surfaces (tests/test_gpu_costs.py) and leaves the SA decisions unchanged.
// Layout (kQrStride doubles per slice): R00 R01 R02 R03 R11 R12 R13 R22 R23
// R33^2 0 0.
#pragma once

#include <cstdint>

namespace sabr_gpu {

constexpr int kQrStride = 12;

// lm[j] = ln(K_j / f) as the reference evaluates it, market[j] != 0.
void slice_qr_factor(const double* lm, const double* market, int64_t n, double out[kQrStride]);

}  // namespace sabr_gpu
