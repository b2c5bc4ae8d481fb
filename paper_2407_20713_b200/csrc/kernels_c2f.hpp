// kernels_c2f.hpp — the Case II formula objective (calibrate_case2_formula).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace sabr_gpu {

constexpr int kC2fThreads = 128;
constexpr int kMaxC2fSlices = 64;
constexpr int kMaxGlNodes = 64;

struct C2fSlice {
    double T, sqrtT;  // maturity and sqrt(maturity) (black_scholes.cpp:28)
    double f;         // forward, VolSurface::forward
    double rmy;       // rate - dividend
};

// Per quote: ln(K/f) and its square for Eq. 8, and the Black-Scholes
// constants of black_scholes.cpp:24-33 (S e^{-yT}, K e^{-rT}, log(S/K)), all
// evaluated on the host with the reference's expressions.
struct C2fQuote {
    double lm, lm2;
    double log_sk;
    double df_div, df_k;
    double market, inv_market;  // market = BS price of the quoted vol (calibration.cpp:277-287)
    int32_t slice;
    int32_t pad;
};

struct C2fView {
    int32_t ns, nq;
    const C2fSlice* sl;
    const C2fQuote* q;
    double horizon;
    int32_t gl_n;      // Gauss-Legendre nodes per panel (8, calibration.cpp:506; 64 = the
                       // dyn_coeffs_case2 default, analytics.hpp:25-26, for model vols)
    double gl_x[kMaxGlNodes];  // gauss_legendre(gl_n) (quadrature.cpp:9-41), host computed
    double gl_w[kMaxGlNodes];
    const double2* exptab;
};

// One temperature level of the calibrate_case2_formula annealer, one CTA per chain.
cudaError_t launch_c2f_level(const C2fView& v, const SaLevelArgs& a, int64_t level, double temp,
                             cudaStream_t s);
// Case II model vols dynamic_implied_vol(dyn_coeffs_case2(p, T_s, gl_n), ...) of
// every quote, vols[i*nq + j], for full vectors params[i*11 ..]; one CTA per vector.
cudaError_t launch_c2f_vols(const C2fView& v, const double* params, int64_t n, double* vols,
                            cudaStream_t s);
// cost[i] of full vectors params[i*11 ..] (horizon last), one CTA per vector.
cudaError_t launch_c2f_cost(const C2fView& v, const double* params, int64_t n, double* cost,
                            cudaStream_t s);

}  // namespace sabr_gpu
