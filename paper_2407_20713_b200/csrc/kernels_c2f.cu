// kernels_c2f.cu — the Case II asymptotic-formula objective of
// calibrate_case2_formula (proj/src/calibration.cpp:483-534) and its
// annealer, CTA-cooperative on sm_100a.
//
// One objective evaluation is ~1e3 evaluations of the inner integral
//   G(s) = int_0^s nu(u) rho(u) du           (analytics.cpp:246-251)
// for the nested 8-node Gauss-Legendre eta2^2 of every slice
// (analytics.cpp:270-287), plus a Black-Scholes price per quote
// (calibration.cpp:507-517).  A single thread per chain would serialise all
// of it, so one CTA runs one chain: every thread carries the same chain state
// and xoshiro stream (identical proposals and Metropolis draws), while the
// (outer node, inner node) pairs, the grid feasibility checks and the quotes
// are split over the 128 threads and combined by fixed-order tree reductions.
#include <algorithm>
#include <climits>
#include <math_constants.h>

#include "device_common.cuh"
#include "kernels_c2f.hpp"

namespace sabr_gpu {

using namespace sabr_dev;

namespace {

constexpr int kT = kC2fThreads;

// Per-candidate polynomial-times-exponential pieces of nu^2(t) and
// (nu rho)(t), analytics.cpp:94-108 (poly_mul accumulation order kept).
struct Pieces {
    double a, b;
    double nn[3];   // k = 2b : (nu0 + q_nu t)^2
    double nb[2];   // k = b  : 2 d_nu (nu0 + q_nu t)
    double n0;      // k = 0  : d_nu^2
    double rab[3];  // k = a+b: (nu0 + q_nu t)(rho0 + q_rho t)
    double rb[2];   // k = b  : d_rho (nu0 + q_nu t)
    double ra[2];   // k = a  : d_nu (rho0 + q_rho t)
    double r0;      // k = 0  : d_nu d_rho
};

// p = {alpha,beta,rho0,q_rho,d_rho,nu0,q_nu,d_nu,a,b,horizon}
__device__ Pieces make_pieces(const double* p) {
    const double rho0 = p[2], q_rho = p[3], d_rho = p[4], nu0 = p[5], q_nu = p[6], d_nu = p[7];
    Pieces c;
    c.a = p[8];
    c.b = p[9];
    c.nn[0] = nu0 * nu0;
    c.nn[1] = SABR_ADD(nu0 * q_nu, q_nu * nu0);
    c.nn[2] = q_nu * q_nu;
    c.nb[0] = SABR_MUL(SABR_MUL(2.0, d_nu), nu0);
    c.nb[1] = SABR_MUL(SABR_MUL(2.0, d_nu), q_nu);
    c.n0 = d_nu * d_nu;
    c.rab[0] = nu0 * rho0;
    c.rab[1] = SABR_ADD(nu0 * q_rho, q_nu * rho0);
    c.rab[2] = q_nu * q_rho;
    c.rb[0] = d_rho * nu0;
    c.rb[1] = d_rho * q_nu;
    c.ra[0] = d_nu * rho0;
    c.ra[1] = d_nu * q_rho;
    c.r0 = d_nu * d_rho;
    return c;
}

// 1/m for the series of exp_moments (m = 1..29) and 1/(n+m+1) (<= 34)
__constant__ double kInvInt[40] = {
    0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8, 1.0 / 9,
    1.0 / 10, 1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19,
    1.0 / 20, 1.0 / 21, 1.0 / 22, 1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28, 1.0 / 29,
    1.0 / 30, 1.0 / 31, 1.0 / 32, 1.0 / 33, 1.0 / 34, 1.0 / 35, 1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39};

// Sum_n poly[n] I_n with I_n = int_0^T t^n e^{-kt} dt: exp_moments
// (analytics.cpp:219-244) and integrate_poly_exp (:80-86).
template <int N>
__device__ double poly_exp_integral(const double* poly, double k, double T, const double2* tab) {
    double mom[N];
    const double x = k * T;
    if (x < 0.5) {
        double tp = T;
#pragma unroll
        for (int n = 0; n < N; ++n) {
            double term = 1.0, sum = kInvInt[n + 1];
            for (int m = 1; m < 30; ++m) {
                term *= -x * kInvInt[m];
                const double contrib = term * kInvInt[n + m + 1];
                sum += contrib;
                if (fabs(contrib) < 1e-18 * fabs(sum)) break;
            }
            mom[n] = tp * sum;
            tp *= T;
        }
    } else {
        const double e = exp_tab(-x, tab);
        const double rk = fast_rcp(k);
        mom[0] = (1.0 - e) * rk;
        double tp = 1.0;
#pragma unroll
        for (int n = 1; n < N; ++n) {
            tp *= T;
            mom[n] = (n * mom[n - 1] - tp * e) * rk;
        }
    }
    double sum = 0.0;
#pragma unroll
    for (int n = 0; n < N; ++n) sum += poly[n] * mom[n];
    return sum;
}

// G(s) = case2_inner_integral (analytics.cpp:246-251): the four nu*rho pieces
__device__ double inner_integral(const Pieces& c, double s, const double2* tab) {
    double g = poly_exp_integral<3>(c.rab, c.a + c.b, s, tab);
    g += poly_exp_integral<2>(c.rb, c.b, s, tab);
    g += poly_exp_integral<2>(c.ra, c.a, s, tab);
    g += poly_exp_integral<1>(&c.r0, 0.0, s, tab);
    return g;
}

// poly_mul(weight, piece) (analytics.cpp:72-77) for a weight of degree W-1
template <int W, int P>
__device__ void poly_mul(const double* w, const double* p, double* r) {
#pragma unroll
    for (int i = 0; i < W + P - 1; ++i) r[i] = 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) r[i + j] += w[i] * p[j];
}

// nu1^2, nu2^2, eta1 of dyn_coeffs_case2 (analytics.cpp:262-268): exact
// integrals via integrate_pieces (:110-116).
__device__ void exact_coeffs(const Pieces& c, double T, double& nu1, double& nu2, double& eta1,
                             const double2* tab) {
    const double T2 = T * T, T3 = T2 * T;
    double r[5];
    {  // weight {T^2, -2T, 1}
        const double w[3] = {T * T, -2.0 * T, 1.0};
        double s = 0.0;
        poly_mul<3, 3>(w, c.nn, r);
        s += poly_exp_integral<5>(r, 2 * c.b, T, tab);
        poly_mul<3, 2>(w, c.nb, r);
        s += poly_exp_integral<4>(r, c.b, T, tab);
        poly_mul<3, 1>(w, &c.n0, r);
        s += poly_exp_integral<3>(r, 0.0, T, tab);
        nu1 = 3.0 / T3 * s;
    }
    {  // weight {0, T, -1}
        const double w[3] = {0.0, T, -1.0};
        double s = 0.0;
        poly_mul<3, 3>(w, c.nn, r);
        s += poly_exp_integral<5>(r, 2 * c.b, T, tab);
        poly_mul<3, 2>(w, c.nb, r);
        s += poly_exp_integral<4>(r, c.b, T, tab);
        poly_mul<3, 1>(w, &c.n0, r);
        s += poly_exp_integral<3>(r, 0.0, T, tab);
        nu2 = 6.0 / T3 * s;
    }
    {  // weight {T, -1}
        const double w[2] = {T, -1.0};
        double s = 0.0;
        poly_mul<2, 3>(w, c.rab, r);
        s += poly_exp_integral<4>(r, c.a + c.b, T, tab);
        poly_mul<2, 2>(w, c.rb, r);
        s += poly_exp_integral<3>(r, c.b, T, tab);
        poly_mul<2, 2>(w, c.ra, r);
        s += poly_exp_integral<3>(r, c.a, T, tab);
        poly_mul<2, 1>(w, &c.r0, r);
        s += poly_exp_integral<2>(r, 0.0, T, tab);
        eta1 = 2.0 / T2 * s;
    }
}

// black_scholes_call (black_scholes.cpp:20-35) with the quote constants
// df_div = S e^{-yT}, df_k = K e^{-rT}, log(S/K) precomputed on the host.
__device__ double bs_call(const C2fQuote& q, const C2fSlice& s, double vol) {
    const double sd = vol * s.sqrtT;
    const double d1 = (q.log_sk + (s.rmy + 0.5 * vol * vol) * s.T) / sd;
    const double d2 = d1 - sd;
    constexpr double kInvSqrt2 = 0.70710678118654752440;
    return q.df_div * (0.5 * erfc(-d1 * kInvSqrt2)) - q.df_k * (0.5 * erfc(-d2 * kInvSqrt2));
}

struct Shared {
    double red[kT / 32];
    double eta2[kMaxC2fSlices];
    SmileTerms terms[kMaxC2fSlices];
    double coef[kMaxC2fSlices][3];
    int flag[kT / 32];
    double2 tab[kExpTableSize];
};

// fixed-order CTA sum (warp shuffles, then warps in order); valid in all threads
__device__ double cta_sum(double v, Shared& sh) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s += sh.red[w];
    return s;
}

__device__ bool cta_all(bool v, Shared& sh) {
    const int b = __all_sync(0xffffffffu, v) ? 1 : 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh.flag[threadIdx.x >> 5] = b;
    __syncthreads();
    int all = 1;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) all &= sh.flag[w];
    return all != 0;
}

// case2_feasible (calibration.cpp:161-168 -> analytics.cpp:145-175) split
// over the CTA: thread t checks grid nodes t+1, t+1+kT, ...; thread 0 the
// stationary points.  Identical predicate, identical result in all threads.
__device__ bool cta_feasible(const double* p, Shared& sh) {
    const double alpha = p[0], beta = p[1], a = p[8], b = p[9], horizon = p[10];
    if (!(alpha > 0) || !(beta >= 0 && beta <= 1) || !(a >= 0 && b >= 0) || !(horizon > 0))
        return false;
    constexpr double kLo = -1 - 1e-9, kHi = 1 + 1e-9;
    bool ok = true;
    for (int i = threadIdx.x + 1; i <= 256; i += kT) {
        const double t = horizon * i / 256;
        const double r = case2_rho_at(p, t);
        ok = ok && !(r < kLo || r > kHi) && !(case2_nu_at(p, t) <= 0);
    }
    if (threadIdx.x == 0) {
        if (a > 0 && p[3] != 0) {
            const double t = 1.0 / a - p[2] / p[3];
            if (t > 0 && t <= horizon) {
                const double r = case2_rho_at(p, t);
                ok = ok && !(r < kLo || r > kHi) && !(case2_nu_at(p, t) <= 0);
            }
        }
        if (b > 0 && p[6] != 0) {
            const double t = 1.0 / b - p[5] / p[6];
            if (t > 0 && t <= horizon) {
                const double r = case2_rho_at(p, t);
                ok = ok && !(r < kLo || r > kHi) && !(case2_nu_at(p, t) <= 0);
            }
        }
    }
    return cta_all(ok, sh);
}

// dyn_coeffs_case2 (analytics.cpp:219-289) for every slice and the
// strike-independent Eq. 8 terms of dynamic_implied_vol (analytics.cpp:291-312)
// into sh.terms[s], for the full vector p (horizon last).
__device__ void c2f_slice_terms(const double* p, const C2fView& v, Shared& sh) {
    const Pieces c = make_pieces(p);
    const double2* tab = sh.tab;
    // exact nu1^2, nu2^2, eta1 per slice: one thread per slice
    for (int s = threadIdx.x; s < v.ns; s += kT)
        exact_coeffs(c, v.sl[s].T, sh.coef[s][0], sh.coef[s][1], sh.coef[s][2], tab);
    // eta2^2: nested GL (analytics.cpp:270-287), 2 panels per axis split at
    // the boundary layer 10/max(a, b); pair (P, o, p, i) -> thread idx % kT
    const double rate = c.a > c.b ? c.a : c.b;
    const int gn = v.gl_n;
    const int pairs = 4 * gn * gn;
    for (int s = 0; s < v.ns; ++s) {
        const double T = v.sl[s].T;
        const double layer = rate > 0 ? 10.0 / rate : T;
        const double split_o = layer < T ? layer : T;
        double part = 0.0;
        for (int idx = threadIdx.x; idx < pairs; idx += kT) {
            const int P = idx / (2 * gn * gn);
            const int o = (idx / (2 * gn)) % gn;
            const int pp = (idx / gn) % 2;
            const int i = idx % gn;
            if (P == 1 && !(split_o < T)) continue;
            const double lo_o = P == 0 ? 0.0 : split_o, hi_o = P == 0 ? split_o : T;
            const double mid_o = 0.5 * (lo_o + hi_o), half_o = 0.5 * (hi_o - lo_o);
            const double t = mid_o + half_o * v.gl_x[o];
            const double split_i = layer < t ? layer : t;
            if (pp == 1 && !(split_i < t)) continue;
            const double lo_i = pp == 0 ? 0.0 : split_i, hi_i = pp == 0 ? split_i : t;
            const double mid_i = 0.5 * (lo_i + hi_i), half_i = 0.5 * (hi_i - lo_i);
            const double g = inner_integral(c, mid_i + half_i * v.gl_x[i], tab);
            part += (half_o * v.gl_w[o]) * (half_i * v.gl_w[i]) * (g * g);
        }
        const double tot = cta_sum(part, sh);
        if (threadIdx.x == 0) {
            const double T2 = T * T, T4 = T2 * T2;
            sh.eta2[s] = 12.0 / T4 * tot;
        }
    }
    __syncthreads();
    // strike-independent Eq. 8 terms per slice (dynamic_implied_vol, analytics.cpp:291-312)
    for (int s = threadIdx.x; s < v.ns; s += kT) {
        const double pw = pow(v.sl[s].f, 1.0 - p[1]);
        sh.terms[s] = dynamic_terms(sh.coef[s][0], sh.coef[s][1], sh.coef[s][2], sh.eta2[s], p[0], p[1],
                                    pw, v.sl[s].T);
    }
    __syncthreads();
}

// The calibrate_case2_formula objective (calibration.cpp:497-520) for the
// full vector p (horizon last); every thread returns the same value.
__device__ double c2f_objective(const double* p, const C2fView& v, Shared& sh) {
    c2f_slice_terms(p, v, sh);
    // quotes: vol -> BS price -> squared relative price error (calibration.cpp:507-517)
    bool ok = true;
    double sum = 0.0;
    for (int j = threadIdx.x; j < v.nq; j += kT) {
        const C2fQuote q = v.q[j];
        const C2fSlice& sl = v.sl[q.slice];
        const double vol = smile_vol(sh.terms[q.slice], q.lm, q.lm2);
        if (!(vol > 0)) ok = false;  // "formula left its validity range"
        const double price = bs_call(q, sl, vol);
        const double rel = (q.market - price) * q.inv_market;
        sum = fma(rel, rel, sum);
    }
    const bool all_ok = cta_all(ok, sh);
    const double tot = cta_sum(sum, sh);
    return all_ok ? tot : 1e10;
}

__device__ void stage_tab(const C2fView& v, Shared& sh) {
    for (int i = threadIdx.x; i < kExpTableSize; i += kT) sh.tab[i] = v.exptab[i];
    __syncthreads();
}

// ---- the annealer level, one CTA per chain (annealer.cpp:107-139) ----
__global__ void __launch_bounds__(kT) c2f_level_kernel(const __grid_constant__ C2fView v,
                                                       const __grid_constant__ SaLevelArgs a,
                                                       const int64_t level, const double temp) {
    __shared__ Shared sh;
    __shared__ int is_last;
    sabr_sa_state* st = a.state;
    if (st->done) return;
    stage_tab(v, sh);
    const int64_t chain = a.chain_begin + blockIdx.x;
    double x[11], y[11], bp[10];
    for (int i = 0; i < 10; ++i) x[i] = bp[i] = st->incumbent[i];
    x[10] = y[10] = v.horizon;
    double fx = st->incumbent_value, bv = fx;
    long long ev = 0;
    const long long cap = st->eval_cap;
    Xoshiro rng;
    rng.init(a.seed, (static_cast<uint64_t>(level) << 20) ^ static_cast<uint64_t>(chain));
    const double ratio = temp / a.t0;
    const double scale = (ratio < 1.0) ? ratio : 1.0;
    for (int step = 0; step < a.chain_length; ++step) {
        if (ev >= cap) break;
        for (int i = 0; i < 10; ++i) {
            if ((a.free_mask >> i) & 1u) {
                const double u = rng.uniform();
                const double stp = __dmul_rn(__dmul_rn(a.range[i], scale), __dsub_rn(__dmul_rn(2.0, u), 1.0));
                double w = __dadd_rn(x[i], stp);
                if (w > a.hi[i]) w = __dsub_rn(__dmul_rn(2.0, a.hi[i]), w);
                if (w < a.lo[i]) w = __dsub_rn(__dmul_rn(2.0, a.lo[i]), w);
                y[i] = (w < a.lo[i]) ? a.lo[i] : (a.hi[i] < w) ? a.hi[i] : w;
            } else {
                y[i] = x[i];
            }
        }
        if (!cta_feasible(y, sh)) continue;  // annealer.cpp:122
        double fy = c2f_objective(y, v, sh);
        if (isnan(fy)) fy = CUDART_INF;
        ++ev;
        bool accept = fy <= fx;
        if (!accept) accept = rng.uniform() < exp(-(fy - fx) / temp);
        if (accept) {
            for (int i = 0; i < 10; ++i) x[i] = y[i];
            fx = fy;
            if (fx < bv) {
                bv = fx;
                for (int i = 0; i < 10; ++i) bp[i] = x[i];
            }
        }
    }
    // one record per CTA (= chain), then the last CTA reduces them
    if (threadIdx.x == 0) {
        sabr_level_record rec{};
        rec.end_value = fx;
        rec.end_chain = chain;
        rec.best_value = bv;
        rec.best_chain = chain;
        rec.evals = ev;
        for (int i = 0; i < 10; ++i) {
            rec.end_point[i] = x[i];
            rec.best_point[i] = bp[i];
        }
        a.block_recs[blockIdx.x] = rec;
        __threadfence();
        is_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last || threadIdx.x != 0) return;
    __threadfence();
    int e = -1, b = -1;
    long long n = 0;
    for (int k = 0; k < static_cast<int>(gridDim.x); ++k) {
        const sabr_level_record* r = a.block_recs + k;
        const double rev = __ldcg(&r->end_value), rbv = __ldcg(&r->best_value);
        const long long rei = __ldcg(reinterpret_cast<const long long*>(&r->end_chain));
        const long long rbi = __ldcg(reinterpret_cast<const long long*>(&r->best_chain));
        if (e < 0 || lex_less(rev, rei, __ldcg(&a.block_recs[e].end_value),
                              __ldcg(reinterpret_cast<const long long*>(&a.block_recs[e].end_chain))))
            e = k;
        if (b < 0 || lex_less(rbv, rbi, __ldcg(&a.block_recs[b].best_value),
                              __ldcg(reinterpret_cast<const long long*>(&a.block_recs[b].best_chain))))
            b = k;
        n += __ldcg(reinterpret_cast<const long long*>(&r->evals));
    }
    sabr_level_record out{};
    out.end_value = __ldcg(&a.block_recs[e].end_value);
    out.end_chain = __ldcg(reinterpret_cast<const long long*>(&a.block_recs[e].end_chain));
    out.best_value = __ldcg(&a.block_recs[b].best_value);
    out.best_chain = __ldcg(reinterpret_cast<const long long*>(&a.block_recs[b].best_chain));
    out.evals = n;
    for (int i = 0; i < SABR_MAX_DIM; ++i) {
        out.end_point[i] = __ldcg(&a.block_recs[e].end_point[i]);
        out.best_point[i] = __ldcg(&a.block_recs[b].best_point[i]);
    }
    *a.rank_rec = out;
    *a.ticket = 0u;
    if (a.nranks == 1)
        merge_level(st, &out, 1, a.n_chains, a.max_evals, a.levels_total, 10, a.trace_f + level);
}

// objective of full vectors (horizon last), one CTA per vector; infeasible
// vectors are the caller's responsibility (validated on the host)
__global__ void __launch_bounds__(kT) c2f_cost_kernel(const __grid_constant__ C2fView v,
                                                      const double* __restrict__ params,
                                                      double* __restrict__ cost) {
    __shared__ Shared sh;
    stage_tab(v, sh);
    double p[11];
    for (int i = 0; i < 11; ++i) p[i] = params[blockIdx.x * 11 + i];
    const double f = c2f_objective(p, v, sh);
    if (threadIdx.x == 0) cost[blockIdx.x] = f;
}

// Case II model vols of every quote, one CTA per vector (validated on the host)
__global__ void __launch_bounds__(kT) c2f_vol_kernel(const __grid_constant__ C2fView v,
                                                     const double* __restrict__ params,
                                                     double* __restrict__ vols) {
    __shared__ Shared sh;
    stage_tab(v, sh);
    double p[11];
    for (int i = 0; i < 11; ++i) p[i] = params[blockIdx.x * 11 + i];
    c2f_slice_terms(p, v, sh);
    for (int j = threadIdx.x; j < v.nq; j += kT) {
        const C2fQuote q = v.q[j];
        vols[static_cast<int64_t>(blockIdx.x) * v.nq + j] = smile_vol(sh.terms[q.slice], q.lm, q.lm2);
    }
}

}  // namespace

cudaError_t launch_c2f_vols(const C2fView& v, const double* params, int64_t n, double* vols,
                            cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    c2f_vol_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(v, params, vols);
    return cudaGetLastError();
}

cudaError_t launch_c2f_level(const C2fView& v, const SaLevelArgs& a, int64_t level, double temp,
                             cudaStream_t s) {
    if (a.n_local <= 0) return cudaSuccess;
    c2f_level_kernel<<<static_cast<unsigned>(a.n_local), kT, 0, s>>>(v, a, level, temp);
    return cudaGetLastError();
}

cudaError_t launch_c2f_cost(const C2fView& v, const double* params, int64_t n, double* cost,
                            cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    c2f_cost_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(v, params, cost);
    return cudaGetLastError();
}

}  // namespace sabr_gpu
