// kernels_bs.cu — batched Black-Scholes pricing and implied-vol inversion
// (proj/src/black_scholes.cpp:20-69) on sm_100a: one thread per contract.
//
// black_scholes_call is evaluated in the reference's operation order with
// round-to-nearest primitives the compiler may not contract into FMAs (the
// reference is built without FMA), so prices agree with the CPU to the libm
// differences of exp/log/erfc (a few ulp).  implied_vol_from_price keeps the
// reference's control flow exactly: the doubling bracket, then up to 200
// Newton steps on vega with the bisection fallback and the |diff| < 1e-10 exit.
#include <cmath>

#include "device_common.cuh"
#include "kernels.hpp"

namespace sabr_gpu {

using namespace sabr_dev;

namespace {

constexpr double kSqrt2 = 1.4142135623730950488;     // std::numbers::sqrt2
constexpr double kTwoPi = 6.283185307179586476925;   // 2.0 * std::numbers::pi (exact product)

__device__ __forceinline__ double norm_cdf(double x) {  // black_scholes.cpp:12
    return SABR_MUL(0.5, erfc(SABR_DIV(-x, kSqrt2)));
}

__device__ __forceinline__ double norm_pdf(double x) {  // black_scholes.cpp:14-16
    return SABR_DIV(exp(SABR_MUL(SABR_MUL(-0.5, x), x)), sqrt(kTwoPi));
}

// black_scholes_call, black_scholes.cpp:20-35, inputs already validated.
__device__ double bs_call(double spot, double strike, double r, double y, double T, double vol) {
    const double df_div = SABR_MUL(spot, exp(SABR_MUL(-y, T)));
    const double df_k = SABR_MUL(strike, exp(SABR_MUL(-r, T)));
    if (vol == 0.0) {
        const double d = SABR_SUB(df_div, df_k);
        return d > 0.0 ? d : 0.0;
    }
    const double sd = SABR_MUL(vol, sqrt(T));
    const double d1 = SABR_DIV(
        SABR_ADD(log(SABR_DIV(spot, strike)), SABR_MUL(SABR_ADD(SABR_SUB(r, y), SABR_MUL(SABR_MUL(0.5, vol), vol)), T)),
        sd);
    const double d2 = SABR_SUB(d1, sd);
    return SABR_SUB(SABR_MUL(df_div, norm_cdf(d1)), SABR_MUL(df_k, norm_cdf(d2)));
}

__device__ __forceinline__ bool bs_inputs_ok(double spot, double strike, double T) {
    return !(spot <= 0 || strike <= 0 || T <= 0);
}

__global__ void bs_call_kernel(int64_t n, const double* __restrict__ spot, const double* __restrict__ strike,
                               const double* __restrict__ r, const double* __restrict__ y,
                               const double* __restrict__ T, const double* __restrict__ vol,
                               double* __restrict__ out, int32_t* __restrict__ status) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t st = BS_OK;
    double v = 0.0;
    if (!bs_inputs_ok(spot[i], strike[i], T[i])) st = BS_E_INPUTS;
    else if (vol[i] < 0) st = BS_E_VOL;
    else v = bs_call(spot[i], strike[i], r[i], y[i], T[i], vol[i]);
    out[i] = v;
    status[i] = st;
}

// implied_vol_from_price, black_scholes.cpp:37-69.
__global__ void implied_vol_kernel(int64_t n, const double* __restrict__ price, const double* __restrict__ spot,
                                   const double* __restrict__ strike, const double* __restrict__ r,
                                   const double* __restrict__ y, const double* __restrict__ T,
                                   double* __restrict__ out, int32_t* __restrict__ status) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p = price[i], S = spot[i], K = strike[i], rr = r[i], yy = y[i], t = T[i];
    out[i] = 0.0;
    if (!bs_inputs_ok(S, K, t)) {  // black_scholes_call(..., 0.0) throws first
        status[i] = BS_E_INPUTS;
        return;
    }
    const double lower = bs_call(S, K, rr, yy, t, 0.0);
    const double upper = SABR_MUL(S, exp(SABR_MUL(-yy, t)));
    if (p <= lower || p >= upper) {
        status[i] = BS_E_BOUNDS;
        return;
    }
    double lo = 0.0, hi = 1.0;
    while (bs_call(S, K, rr, yy, t, hi) < p) hi = SABR_MUL(hi, 2.0);
    constexpr double kTol = 1e-10;
    double vol = SABR_MUL(0.5, SABR_ADD(lo, hi));
    const double sqt = sqrt(t);
    for (int it = 0; it < 200; ++it) {
        const double v = bs_call(S, K, rr, yy, t, vol);
        const double diff = SABR_SUB(v, p);
        if (fabs(diff) < kTol) break;
        if (diff > 0) hi = vol;
        else lo = vol;
        // Newton step on vega, bisection fallback when it leaves the bracket
        const double sd = SABR_MUL(vol, sqt);
        const double d1 = SABR_DIV(
            SABR_ADD(log(SABR_DIV(S, K)), SABR_MUL(SABR_ADD(SABR_SUB(rr, yy), SABR_MUL(SABR_MUL(0.5, vol), vol)), t)),
            sd);
        const double vega = SABR_MUL(SABR_MUL(SABR_MUL(S, exp(SABR_MUL(-yy, t))), norm_pdf(d1)), sqt);
        double next = SABR_SUB(vol, SABR_DIV(diff, vega));
        if (!(next > lo && next < hi)) next = SABR_MUL(0.5, SABR_ADD(lo, hi));
        vol = next;
    }
    out[i] = vol;
    status[i] = BS_OK;
}

}  // namespace

cudaError_t launch_bs_call(int64_t n, const double* spot, const double* strike, const double* r, const double* y,
                           const double* T, const double* vol, double* out, int32_t* status, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    bs_call_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(n, spot, strike, r, y, T, vol, out,
                                                                          status);
    return cudaGetLastError();
}

cudaError_t launch_implied_vol(int64_t n, const double* price, const double* spot, const double* strike,
                               const double* r, const double* y, const double* T, double* out, int32_t* status,
                               cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    implied_vol_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(n, price, spot, strike, r, y, T,
                                                                              out, status);
    return cudaGetLastError();
}

}  // namespace sabr_gpu
