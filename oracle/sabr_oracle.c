/*
 * oracle/sabr_oracle.c — TEST INFRASTRUCTURE ONLY (see sabr_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Compiled with
 * -ffp-contract=off so that, like the reference built for baseline x86-64
 * (no FMA), every expression rounds exactly as written; the operation order
 * of each expression follows the cited reference line.  Pinned against the
 * compiled reference by tests/test_oracle.py (bit-identical results on the
 * same libm) and against tests/golden/.
 */
#include "sabr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846
#define ORC_SQRT2 1.41421356237309504880

/* ---------------------------------------------------------------- RNG --- */

/* splitmix64, proj/include/sabr/rng.hpp:7-12 */
static uint64_t splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Xoshiro256pp(seed, stream), rng.hpp:19-23 */
void orc_xoshiro_init(orc_xoshiro* g, uint64_t seed, uint64_t stream) {
    uint64_t sm = seed ^ (stream * 0xD2B74407B1CE6E93ull + 0x9E3779B97F4A7C15ull);
    for (int i = 0; i < 4; ++i) g->s[i] = splitmix64(&sm);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* xoshiro256++ next(), rng.hpp:29-39 */
uint64_t orc_xoshiro_next(orc_xoshiro* g) {
    uint64_t* s = g->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* uniform() = (next() >> 11) * 2^-53, rng.hpp:42 */
double orc_xoshiro_uniform(orc_xoshiro* g) {
    return (double)(orc_xoshiro_next(g) >> 11) * 0x1.0p-53;
}

/* Philox4x32-10 (Salmon et al. 2011, the Random123 constants).  The GPU
 * engine's SABR_RNG_PHILOX stream: key = seed (lo, hi), counter =
 * (path lo, path hi, step, 0).  Not part of the reference — restated here so
 * the GPU's Philox stream has an identical CPU twin. */
void orc_philox4x32(const uint32_t ctr[4], uint64_t key, uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* Two uniforms in [0,1) with the reference's 53-bit recipe (rng.hpp:42):
 * u_a from words (0,1), u_b from words (2,3). */
void orc_philox_uniform_pair(uint64_t seed, uint64_t path, uint32_t step, double* u_a,
                             double* u_b) {
    const uint32_t ctr[4] = {(uint32_t)path, (uint32_t)(path >> 32), step, 0u};
    uint32_t x[4];
    orc_philox4x32(ctr, seed, x);
    const uint64_t a = ((uint64_t)x[0] << 32) | x[1];
    const uint64_t b = ((uint64_t)x[2] << 32) | x[3];
    *u_a = (double)(a >> 11) * 0x1.0p-53;
    *u_b = (double)(b >> 11) * 0x1.0p-53;
}

/* ----------------------------------------------------------- analytics --- */

/* Last-bit sensitivity probes (test-only): exp and pow inside the analytics
 * can be moved by +-k ulps to measure how much a 1-ulp libm difference moves
 * a cost (the reference's own rounding sensitivity, used as the parity bound
 * where its closed forms cancel). 0 = the plain libm result. */
static int g_exp_ulps = 0, g_pow_ulps = 0;

static double nudge(double v, int k) {
    for (; k > 0; --k) v = nextafter(v, INFINITY);
    for (; k < 0; ++k) v = nextafter(v, -INFINITY);
    return v;
}
static double pexp(double x) { return nudge(exp(x), g_exp_ulps); }
static double ppow(double x, double y) { return nudge(pow(x, y), g_pow_ulps); }

/* std::min / std::max / std::clamp exactly as libstdc++ defines them. */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double sclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : (hi < v) ? hi : v;
}

/* StaticSabrParams::validate, analytics.cpp:120-125 */
static int static_valid(const double p[4]) {
    return p[0] > 0 && p[1] >= 0 && p[1] <= 1 && p[2] >= 0 && p[3] >= -1 && p[3] <= 1;
}

/* CaseIParams::validate, analytics.cpp:130-136 */
static int case1_valid(const double p[6]) {
    return p[0] > 0 && p[1] >= 0 && p[1] <= 1 && p[2] >= -1 && p[2] <= 1 && p[3] > 0 &&
           p[4] >= 0 && p[5] >= 0;
}

/* static_implied_vol (Obloj-corrected Eq. 7), analytics.cpp:183-205.
 * Returns NaN where the reference throws std::domain_error. */
double orc_static_implied_vol(const double p[4], double strike, double forward, double T) {
    if (!static_valid(p) || !(strike > 0) || !(forward > 0) || !(T > 0)) return NAN;
    const double alpha = p[0], beta = p[1], nu = p[2], rho = p[3];
    const double one_m_beta = 1.0 - beta;
    const double omega = ppow(forward, one_m_beta) / alpha;
    const double rnw = rho * nu * omega;
    const double nw = nu * omega;
    const double a1 = -0.5 * (one_m_beta - rnw);
    const double a2 = (one_m_beta * one_m_beta + 3.0 * (one_m_beta - rnw) +
                       (2.0 - 3.0 * rho * rho) * nw * nw) /
                      12.0;
    const double b = one_m_beta * one_m_beta / (24.0 * omega * omega) +
                     beta * rho * nu / (4.0 * omega) + (2.0 - 3.0 * rho * rho) * nu * nu / 24.0;
    const double log_m = log(strike / forward);
    return (1.0 + a1 * log_m + a2 * log_m * log_m + b * T) / omega;
}

/* Taylor coefficients of the scaled Case I functions, analytics.cpp:23-39. */
static const double kSeriesNu1[14] = {
    1.0, -1.0 / 4, 1.0 / 20, -1.0 / 120, 1.0 / 840, -1.0 / 6720, 1.0 / 60480,
    -1.0 / 604800, 1.0 / 6652800, -1.0 / 79833600, 1.0 / 1037836800,
    -1.0 / 14529715200.0, 1.0 / 217945728000.0, -1.0 / 3487131648000.0};
static const double kSeriesNu2[14] = {
    1.0, -1.0 / 2, 3.0 / 20, -1.0 / 30, 1.0 / 168, -1.0 / 1120, 1.0 / 8640,
    -1.0 / 75600, 1.0 / 739200, -1.0 / 7983360, 1.0 / 94348800,
    -1.0 / 1210809600, 1.0 / 16765056000.0, -1.0 / 249080832000.0};
static const double kSeriesEta1[14] = {
    1.0, -1.0 / 3, 1.0 / 12, -1.0 / 60, 1.0 / 360, -1.0 / 2520, 1.0 / 20160,
    -1.0 / 181440, 1.0 / 1814400, -1.0 / 19958400, 1.0 / 239500800,
    -1.0 / 3113510400.0, 1.0 / 43589145600.0, -1.0 / 653837184000.0};
static const double kSeriesEta2[14] = {
    1.0, -3.0 / 5, 7.0 / 30, -1.0 / 14, 31.0 / 1680, -1.0 / 240,
    127.0 / 151200, -17.0 / 110880, 73.0 / 2851200, -31.0 / 7862400,
    2047.0 / 3632428800.0, -1.0 / 13305600, 8191.0 / 871782912000.0,
    -5461.0 / 4940103168000.0};

/* horner, analytics.cpp:41-45 */
static double horner(const double c[14], double x) {
    double acc = 0.0;
    for (int i = 13; i >= 0; --i) acc = acc * x + c[i];
    return acc;
}

#define KX_SWITCH 0.25 /* analytics.cpp:21 */

/* f_nu1 .. f_eta2, analytics.cpp:47-67 */
static double f_nu1(double x) {
    if (x < KX_SWITCH) return horner(kSeriesNu1, x);
    return 6.0 / (x * x * x) * (x * x / 2 - x + 1 - pexp(-x));
}
static double f_nu2(double x) {
    if (x < KX_SWITCH) return horner(kSeriesNu2, x);
    const double e = pexp(-x);
    return 6.0 / (x * x * x) * (2 * (e - 1) + x * (e + 1));
}
static double f_eta1(double x) {
    if (x < KX_SWITCH) return horner(kSeriesEta1, x);
    return 2.0 / (x * x) * (pexp(-x) - (1 - x));
}
static double f_eta2(double x) {
    if (x < KX_SWITCH) return horner(kSeriesEta2, x);
    const double e = pexp(-x);
    return 3.0 / (x * x * x * x) * (e * e - 8 * e + 7 + 2 * x * (x - 3));
}

/* dyn_coeffs_case1, analytics.cpp:207-215 */
void orc_dyn_coeffs_case1(const double p[6], double T, double out[4]) {
    if (!case1_valid(p) || !(T > 0)) {
        out[0] = out[1] = out[2] = out[3] = NAN;
        return;
    }
    const double xb = 2.0 * p[5] * T;
    const double xab = (p[4] + p[5]) * T;
    const double nn = p[3] * p[3];
    const double nr = p[3] * p[2];
    out[0] = nn * f_nu1(xb);
    out[1] = nn * f_nu2(xb);
    out[2] = nr * f_eta1(xab);
    out[3] = nr * nr * f_eta2(xab);
}

/* dynamic_implied_vol (Osajima Eq. 8), analytics.cpp:291-312 */
double orc_dynamic_implied_vol(const double c[4], double alpha, double beta, double strike,
                               double forward, double T) {
    if (!(alpha > 0) || !(strike > 0) || !(forward > 0) || !(T > 0)) return NAN;
    const double nu1_sq = c[0], nu2_sq = c[1], eta1 = c[2], eta2_sq = c[3];
    const double one_m_beta = 1.0 - beta;
    const double omega = ppow(forward, one_m_beta) / alpha;
    const double e1w = eta1 * omega;
    const double a1 = 0.5 * (beta - 1.0) + 0.5 * e1w;
    const double a2 = one_m_beta * one_m_beta / 12.0 + (one_m_beta - e1w) / 4.0 +
                      (4.0 * nu1_sq + 3.0 * (eta2_sq - 3.0 * eta1 * eta1)) * omega * omega / 24.0;
    const double b = one_m_beta * one_m_beta / (24.0 * omega * omega) +
                     beta * eta1 / (4.0 * omega) + (2.0 * nu2_sq - 3.0 * eta2_sq) / 24.0;
    const double log_m = log(strike / forward);
    return (1.0 + a1 * log_m + a2 * log_m * log_m + b * T) / omega;
}

/* VolSurface::forward -> forward_price, calibration.cpp:222-225, analytics.cpp:177-181 */
double orc_forward(const sabr_surface* s, int64_t slice) {
    return s->spot * exp((s->rate[slice] - s->dividend[slice]) * s->maturity[slice]);
}

/* CaseIIParams::rho_at / nu_at, analytics.cpp:138-143 (p: 11-vector) */
static double c2_rho_at(const double* p, double t) { return (p[2] + p[3] * t) * exp(-p[8] * t) + p[4]; }
static double c2_nu_at(const double* p, double t) { return (p[5] + p[6] * t) * exp(-p[9] * t) + p[7]; }

/* CaseIIParams::validate as a predicate (case2_feasible), analytics.cpp:145-175,
 * calibration.cpp:161-168.  p = {alpha,beta,rho0,q_rho,d_rho,nu0,q_nu,d_nu,a,b,horizon}. */
int orc_case2_feasible(const double p[11]) {
    const double alpha = p[0], beta = p[1], a = p[8], b = p[9], horizon = p[10];
    if (!(alpha > 0) || !(beta >= 0 && beta <= 1) || !(a >= 0 && b >= 0) || !(horizon > 0))
        return 0;
    double ts[258];
    int n = 0;
    for (int i = 1; i <= 256; ++i) ts[n++] = horizon * i / 256;
    if (a > 0 && p[3] != 0) {
        const double t_star = 1.0 / a - p[2] / p[3];
        if (t_star > 0 && t_star <= horizon) ts[n++] = t_star;
    }
    if (b > 0 && p[6] != 0) {
        const double t_star = 1.0 / b - p[5] / p[6];
        if (t_star > 0 && t_star <= horizon) ts[n++] = t_star;
    }
    const double kTol = 1e-9;
    for (int k = 0; k < n; ++k) {
        const double r = c2_rho_at(p, ts[k]);
        if (r < -1 - kTol || r > 1 + kTol) return 0;
        if (c2_nu_at(p, ts[k]) <= 0) return 0;
    }
    return 1;
}

/* cost_individual with static_implied_vol, calibration.cpp:253-267, :300-306.
 * NaN signals the reference's domain_error. */
double orc_cost_static(const sabr_surface* s, int64_t slice, const double p[4]) {
    const double fwd = orc_forward(s, slice);
    const double T = s->maturity[slice];
    double sum = 0.0;
    for (int64_t j = s->quote_offset[slice]; j < s->quote_offset[slice + 1]; ++j) {
        const double market = s->vol[j];
        if (market == 0) return NAN;
        const double model = orc_static_implied_vol(p, s->strike[j], fwd, T);
        const double rel = (market - model) / market;
        sum += rel * rel;
    }
    return sum;
}

/* The Case I objective (model_cost), calibration.cpp:339-349 */
double orc_cost_case1(const sabr_surface* s, const double p[6]) {
    double sum = 0.0;
    for (int64_t i = 0; i < s->n_slices; ++i) {
        const double T = s->maturity[i];
        const double fwd = orc_forward(s, i);
        double c[4];
        orc_dyn_coeffs_case1(p, T, c);
        double part = 0.0;
        for (int64_t j = s->quote_offset[i]; j < s->quote_offset[i + 1]; ++j) {
            const double market = s->vol[j];
            if (market == 0) return NAN;
            const double model = orc_dynamic_implied_vol(c, p[0], p[1], s->strike[j], fwd, T);
            const double rel = (market - model) / market;
            part += rel * rel;
        }
        sum += part;
    }
    return sum;
}

/* max |cost(libm +-1 ulp) - cost| over the four (exp, pow) nudges. */
double orc_cost_sensitivity(int model, const sabr_surface* s, int64_t slice, const double* p) {
    const double base = model == SABR_MODEL_STATIC ? orc_cost_static(s, slice, p) : orc_cost_case1(s, p);
    double worst = 0.0;
    for (int e = -1; e <= 1; e += 2)
        for (int w = -1; w <= 1; w += 2) {
            g_exp_ulps = e;
            g_pow_ulps = w;
            const double c = model == SABR_MODEL_STATIC ? orc_cost_static(s, slice, p) : orc_cost_case1(s, p);
            const double d = fabs(c - base);
            if (d > worst) worst = d;
        }
    g_exp_ulps = g_pow_ulps = 0;
    return worst;
}

/* --------------------------------------------- Case II coefficients --- */

/* GaussLegendreRule(n), quadrature.cpp:13-33 */
static void gauss_legendre(int n, double* nodes, double* weights) {
    const int m = (n + 1) / 2;
    for (int i = 0; i < m; ++i) {
        double x = cos(ORC_PI * (i + 0.75) / (n + 0.5));
        double pp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int j = 2; j <= n; ++j) {
                const double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            pp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / pp;
            x -= dx;
            if (fabs(dx) < 1e-15) break;
        }
        nodes[i] = -x;
        nodes[n - 1 - i] = x;
        weights[i] = weights[n - 1 - i] = 2.0 / ((1.0 - x * x) * pp * pp);
    }
}

/* detail::exp_moments, analytics.cpp:219-244 */
static void exp_moments(double k, double T, double* out, int size) {
    const double x = k * T;
    if (x < 0.5) {
        double tp = T;
        for (int n = 0; n < size; ++n) {
            double term = 1.0, sum = 1.0 / (n + 1);
            for (int m = 1; m < 30; ++m) {
                term *= -x / m;
                const double contrib = term / (n + m + 1);
                sum += contrib;
                if (fabs(contrib) < 1e-18 * fabs(sum)) break;
            }
            out[n] = tp * sum;
            tp *= T;
        }
        return;
    }
    const double e = exp(-x);
    out[0] = (1.0 - e) / k;
    double tp = 1.0;
    for (int n = 1; n < size; ++n) {
        tp *= T;
        out[n] = (n * out[n - 1] - tp * e) / k;
    }
}

/* integrate_poly_exp, analytics.cpp:80-86 */
static double integrate_poly_exp(const double* p, int size, double k, double T) {
    double mom[8] = {0};
    exp_moments(k, T, mom, size);
    double sum = 0.0;
    for (int n = 0; n < size; ++n) sum += p[n] * mom[n];
    return sum;
}

/* poly_mul, analytics.cpp:72-77; returns the product size */
static int poly_mul(const double* p, int np, const double* q, int nq, double* r) {
    for (int i = 0; i < np + nq - 1; ++i) r[i] = 0.0;
    for (int i = 0; i < np; ++i)
        for (int j = 0; j < nq; ++j) r[i + j] += p[i] * q[j];
    return np + nq - 1;
}

typedef struct {
    double k;
    double poly[3];
    int n;
} piece_t;

/* case2_nu_sq_pieces / case2_nurho_pieces, analytics.cpp:94-108 */
static int nu_sq_pieces(const double* p, piece_t* out) {
    const double nu_lin[2] = {p[5], p[6]};
    out[0].k = 2 * p[9];
    out[0].n = poly_mul(nu_lin, 2, nu_lin, 2, out[0].poly);
    out[1].k = p[9];
    out[1].poly[0] = 2 * p[7] * p[5];
    out[1].poly[1] = 2 * p[7] * p[6];
    out[1].n = 2;
    out[2].k = 0.0;
    out[2].poly[0] = p[7] * p[7];
    out[2].n = 1;
    return 3;
}

static int nurho_pieces(const double* p, piece_t* out) {
    const double nu_lin[2] = {p[5], p[6]};
    const double rho_lin[2] = {p[2], p[3]};
    out[0].k = p[8] + p[9];
    out[0].n = poly_mul(nu_lin, 2, rho_lin, 2, out[0].poly);
    out[1].k = p[9];
    out[1].poly[0] = p[4] * p[5];
    out[1].poly[1] = p[4] * p[6];
    out[1].n = 2;
    out[2].k = p[8];
    out[2].poly[0] = p[7] * p[2];
    out[2].poly[1] = p[7] * p[3];
    out[2].n = 2;
    out[3].k = 0.0;
    out[3].poly[0] = p[7] * p[4];
    out[3].n = 1;
    return 4;
}

/* integrate_pieces, analytics.cpp:110-116 */
static double integrate_pieces(const piece_t* pieces, int np, const double* w, int nw, double T) {
    double sum = 0.0;
    for (int i = 0; i < np; ++i) {
        double r[8];
        const int n = poly_mul(w, nw, pieces[i].poly, pieces[i].n, r);
        sum += integrate_poly_exp(r, n, pieces[i].k, T);
    }
    return sum;
}

/* detail::case2_inner_integral, analytics.cpp:246-251 */
static double case2_inner_integral(const double* p, double s) {
    piece_t pc[4];
    const int np = nurho_pieces(p, pc);
    double sum = 0.0;
    for (int i = 0; i < np; ++i) sum += integrate_poly_exp(pc[i].poly, pc[i].n, pc[i].k, s);
    return sum;
}

/* GaussLegendreRule::integrate, quadrature.hpp:18-25, for the two nested
 * integrands of dyn_coeffs_case2 */
typedef struct {
    const double* p;
    const double* x;
    const double* w;
    int n;
    double layer;
} gl_ctx;

static double gl_inner(const gl_ctx* c, double lo, double hi) {
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    double sum = 0.0;
    for (int i = 0; i < c->n; ++i) {
        const double g = case2_inner_integral(c->p, mid + half * c->x[i]);
        sum += c->w[i] * (g * g);
    }
    return half * sum;
}

static double integrate_inner(const gl_ctx* c, double hi) {
    const double split = smin(c->layer, hi);
    double sum = gl_inner(c, 0.0, split);
    if (split < hi) sum += gl_inner(c, split, hi);
    return sum;
}

static double gl_outer(const gl_ctx* c, double lo, double hi) {
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    double sum = 0.0;
    for (int i = 0; i < c->n; ++i) sum += c->w[i] * integrate_inner(c, mid + half * c->x[i]);
    return half * sum;
}

/* dyn_coeffs_case2, analytics.cpp:255-289 (p must be feasible: the caller
 * validates, as the reference does on entry). */
void orc_dyn_coeffs_case2(const double p[11], double T, int nodes, double out[4]) {
    const double T2 = T * T, T3 = T2 * T, T4 = T3 * T;
    piece_t nu_sq[3], nurho[4];
    nu_sq_pieces(p, nu_sq);
    nurho_pieces(p, nurho);
    const double w1[3] = {T * T, -2.0 * T, 1.0};
    const double w2[3] = {0.0, T, -1.0};
    const double w3[2] = {T, -1.0};
    out[0] = 3.0 / T3 * integrate_pieces(nu_sq, 3, w1, 3, T);
    out[1] = 6.0 / T3 * integrate_pieces(nu_sq, 3, w2, 3, T);
    out[2] = 2.0 / T2 * integrate_pieces(nurho, 4, w3, 2, T);
    double x[64], w[64];
    gauss_legendre(nodes, x, w);
    const double rate = smax(p[8], p[9]);
    gl_ctx c = {p, x, w, nodes, rate > 0 ? 10.0 / rate : T};
    const double split = smin(c.layer, T);
    double sum = gl_outer(&c, 0.0, split);
    if (split < T) sum += gl_outer(&c, split, T);
    out[3] = 12.0 / T4 * sum;
}

/* The calibrate_case2_formula objective, calibration.cpp:497-520 */
double orc_cost_case2_formula(const sabr_surface* s, const double p[11]) {
    double sum = 0.0;
    for (int64_t i = 0; i < s->n_slices; ++i) {
        const double T = s->maturity[i];
        const double fwd = orc_forward(s, i);
        double c[4];
        orc_dyn_coeffs_case2(p, T, 8, c);
        for (int64_t j = s->quote_offset[i]; j < s->quote_offset[i + 1]; ++j) {
            const double vol = orc_dynamic_implied_vol(c, p[0], p[1], s->strike[j], fwd, T);
            if (!(vol > 0)) return 1e10;
            const double price = orc_black_scholes_call(s->spot, s->strike[j], s->rate[i],
                                                        s->dividend[i], T, vol);
            const double market = orc_black_scholes_call(s->spot, s->strike[j], s->rate[i],
                                                         s->dividend[i], T, s->vol[j]);
            const double rel = (market - price) / market;
            sum += rel * rel;
        }
    }
    return sum;
}

/* ------------------------------------------------------------ annealer --- */

/* propose, annealer.cpp:60-74 (in place into `next`) */
static void propose(const double* cur, double* next, int dim, double temperature,
                    const double* lo, const double* hi, double t0, orc_xoshiro* rng) {
    const double scale = smin(1.0, temperature / t0);
    for (int i = 0; i < dim; ++i) {
        const double range = hi[i] - lo[i];
        const double step = range * scale * (2.0 * orc_xoshiro_uniform(rng) - 1.0);
        double x = cur[i] + step;
        if (x > hi[i]) x = 2.0 * hi[i] - x;
        if (x < lo[i]) x = 2.0 * lo[i] - x;
        next[i] = sclamp(x, lo[i], hi[i]);
    }
}

/* AnnealingSchedule::validate, annealer.cpp:28-39 */
static int schedule_valid(const sabr_schedule* s) {
    return s->t0 > 0 && s->cooling > 0 && s->cooling < 1 && s->chain_length >= 1 &&
           s->workers >= 1 && s->groups >= 1 && s->t_min > 0 && s->t_min < s->t0 &&
           s->max_evals >= 1;
}

typedef struct {
    double* endpoint;
    double endpoint_value;
    double* best_point;
    double best_value;
    long evals;
} chain_result;

/* minimize, annealer.cpp:76-167 (serial over chains: the reference result is
 * independent of the thread count). */
int orc_minimize(orc_objective f, void* user, orc_predicate feasible, void* puser,
                 const double* lo, const double* hi, int dim, const sabr_schedule* sch,
                 const double* start, sabr_anneal_result* res) {
    if (!schedule_valid(sch)) return SABR_E_DOMAIN;
    for (int i = 0; i < dim; ++i)
        if (!(lo[i] < hi[i])) return SABR_E_DOMAIN;
    for (int i = 0; i < dim; ++i)
        if (start[i] < lo[i] || start[i] > hi[i]) return SABR_E_DOMAIN;
    if (feasible && !feasible(start, puser)) return SABR_E_DOMAIN;

    const double kInf = INFINITY;
    double* incumbent = malloc(sizeof(double) * dim);
    double* best_point = malloc(sizeof(double) * dim);
    memcpy(incumbent, start, sizeof(double) * dim);
    double v0 = f(incumbent, user);
    double incumbent_value = isnan(v0) ? kInf : v0;
    memcpy(best_point, incumbent, sizeof(double) * dim);
    double best_value = incumbent_value;
    long evals = 1;
    const int n_chains = sch->workers * sch->groups;
    chain_result* chains = calloc((size_t)n_chains, sizeof(chain_result));
    double* buf = malloc(sizeof(double) * (size_t)dim * 2 * (size_t)n_chains);
    double* x = malloc(sizeof(double) * dim);
    double* y = malloc(sizeof(double) * dim);
    for (int c = 0; c < n_chains; ++c) {
        chains[c].endpoint = buf + (size_t)c * 2 * dim;
        chains[c].best_point = buf + (size_t)c * 2 * dim + dim;
    }
    int64_t trace_len = 0;
    uint64_t level = 0;
    for (double temp = sch->t0; temp >= sch->t_min; temp *= sch->cooling, ++level) {
        if (evals >= sch->max_evals) break;
        const long remaining = sch->max_evals - evals;
        const long eval_cap = (remaining + n_chains - 1) / n_chains;
        for (int chain = 0; chain < n_chains; ++chain) {
            orc_xoshiro rng;
            orc_xoshiro_init(&rng, sch->seed, (level << 20) ^ (uint64_t)chain);
            chain_result* cr = &chains[chain];
            memcpy(cr->best_point, incumbent, sizeof(double) * dim);
            cr->best_value = incumbent_value;
            cr->evals = 0;
            memcpy(x, incumbent, sizeof(double) * dim);
            double fx = incumbent_value;
            for (int step = 0; step < sch->chain_length; ++step) {
                if (cr->evals >= eval_cap) break;
                propose(x, y, dim, temp, lo, hi, sch->t0, &rng);
                int ok = 1;
                for (int i = 0; i < dim; ++i)
                    if (y[i] < lo[i] || y[i] > hi[i]) ok = 0;
                if (ok && feasible && !feasible(y, puser)) ok = 0;
                if (!ok) continue;
                const double raw = f(y, user);
                const double fy = isnan(raw) ? kInf : raw;
                ++cr->evals;
                const int accept = fy <= fx || orc_xoshiro_uniform(&rng) < exp(-(fy - fx) / temp);
                if (accept) {
                    memcpy(x, y, sizeof(double) * dim);
                    fx = fy;
                    if (fx < cr->best_value) {
                        cr->best_value = fx;
                        memcpy(cr->best_point, x, sizeof(double) * dim);
                    }
                }
            }
            memcpy(cr->endpoint, x, sizeof(double) * dim);
            cr->endpoint_value = fx;
        }
        /* two-level reduction, annealer.cpp:141-159 */
        for (int group = 0; group < sch->groups; ++group) {
            int group_min = group * sch->workers;
            for (int p = group_min + 1; p < (group + 1) * sch->workers; ++p)
                if (chains[p].endpoint_value < chains[group_min].endpoint_value) group_min = p;
            if (chains[group_min].endpoint_value < incumbent_value) {
                incumbent_value = chains[group_min].endpoint_value;
                memcpy(incumbent, chains[group_min].endpoint, sizeof(double) * dim);
            }
        }
        for (int c = 0; c < n_chains; ++c) {
            evals += chains[c].evals;
            if (chains[c].best_value < best_value) {
                best_value = chains[c].best_value;
                memcpy(best_point, chains[c].best_point, sizeof(double) * dim);
            }
        }
        if (res->trace_t && trace_len < res->trace_capacity) {
            res->trace_t[trace_len] = temp;
            res->trace_f[trace_len] = incumbent_value;
        }
        ++trace_len;
    }
    memcpy(res->best_point, best_point, sizeof(double) * dim);
    res->best_value = best_value;
    res->evals = evals;
    res->trace_len = trace_len;
    free(incumbent);
    free(best_point);
    free(chains);
    free(buf);
    free(x);
    free(y);
    return SABR_OK;
}

typedef struct {
    int model;
    const sabr_surface* s;
    int64_t slice;
} cost_ctx;

static double cost_obj(const double* x, void* user) {
    const cost_ctx* c = (const cost_ctx*)user;
    if (c->model == SABR_MODEL_STATIC) return orc_cost_static(c->s, c->slice, x);
    return orc_cost_case1(c->s, x);
}

int orc_minimize_cost(int model, const sabr_surface* s, int64_t slice, const double* lo,
                      const double* hi, int dim, const sabr_schedule* sch, const double* start,
                      sabr_anneal_result* res) {
    cost_ctx c = {model, s, slice};
    return orc_minimize(cost_obj, &c, NULL, NULL, lo, hi, dim, sch, start, res);
}

static double sq(double x) { return x * x; }

/* The closed-form objectives of proj/tests/test_annealer.cpp */
static double builtin_obj(const double* x, void* user) {
    const int id = *(const int*)user;
    switch (id) {
        case SABR_OBJ_BOWL3: return sq(x[0] - 1.2) + sq(x[1] + 0.7) + sq(x[2] - 3.4);
        case SABR_OBJ_ROSENBROCK4: {
            double v = 0.0;
            for (int i = 0; i < 3; ++i) v += 100.0 * sq(x[i + 1] - sq(x[i])) + sq(1.0 - x[i]);
            return v;
        }
        case SABR_OBJ_SINQUAD2: return sq(x[0] - 0.3) + 3.0 * sq(x[1] + 2.1) + 0.1 * sin(7.0 * x[0]);
        case SABR_OBJ_SQUARE1: return sq(x[0]);
        case SABR_OBJ_COSBOWL2: return sq(x[0]) + sq(x[1]) + cos(3.0 * x[0]);
        case SABR_OBJ_CORNER2: return sq(x[0] - 2.0) + sq(x[1] - 2.0);
        case SABR_OBJ_NANRIGHT1: return x[0] > 0.5 ? NAN : sq(x[0] + 1.0);
    }
    return NAN;
}

static int pred_sum_le_1(const double* x, void* user) {
    (void)user;
    return x[0] + x[1] <= 1.0;
}

int orc_minimize_builtin(int objective, int predicate, const double* lo, const double* hi,
                         int dim, const sabr_schedule* sch, const double* start,
                         sabr_anneal_result* res) {
    int id = objective;
    return orc_minimize(builtin_obj, &id, predicate == SABR_PRED_SUM_LE_1 ? pred_sum_le_1 : NULL,
                        NULL, lo, hi, dim, sch, start, res);
}

double orc_builtin_value(int objective, const double* x) {
    int id = objective;
    return builtin_obj(x, &id);
}

/* Chains [chain_begin, chain_end) of one level, reduced with the reference's
 * scan order (strict '<', lowest chain first) into one record. */
int orc_level_record(int objective, int predicate, const double* lo, const double* hi, int dim,
                     const sabr_schedule* sch, const sabr_sa_state* st, uint64_t level,
                     double temp, int64_t chain_begin, int64_t chain_end,
                     sabr_level_record* out) {
    int id = objective;
    double x[SABR_MAX_DIM], y[SABR_MAX_DIM], bp[SABR_MAX_DIM];
    memset(out, 0, sizeof(*out));
    out->end_chain = out->best_chain = -1;
    for (int64_t chain = chain_begin; chain < chain_end; ++chain) {
        orc_xoshiro rng;
        orc_xoshiro_init(&rng, sch->seed, (level << 20) ^ (uint64_t)chain);
        memcpy(x, st->incumbent, sizeof(double) * dim);
        memcpy(bp, st->incumbent, sizeof(double) * dim);
        double fx = st->incumbent_value, bv = st->incumbent_value;
        long evals = 0;
        for (int step = 0; step < sch->chain_length; ++step) {
            if (evals >= st->eval_cap) break;
            propose(x, y, dim, temp, lo, hi, sch->t0, &rng);
            if (predicate == SABR_PRED_SUM_LE_1 && !(y[0] + y[1] <= 1.0)) continue;
            const double raw = builtin_obj(y, &id);
            const double fy = isnan(raw) ? INFINITY : raw;
            ++evals;
            if (fy <= fx || orc_xoshiro_uniform(&rng) < exp(-(fy - fx) / temp)) {
                memcpy(x, y, sizeof(double) * dim);
                fx = fy;
                if (fx < bv) {
                    bv = fx;
                    memcpy(bp, x, sizeof(double) * dim);
                }
            }
        }
        if (out->end_chain < 0 || fx < out->end_value) {
            out->end_chain = chain;
            out->end_value = fx;
            memcpy(out->end_point, x, sizeof(double) * dim);
        }
        if (out->best_chain < 0 || bv < out->best_value) {
            out->best_chain = chain;
            out->best_value = bv;
            memcpy(out->best_point, bp, sizeof(double) * dim);
        }
        out->evals += evals;
    }
    return SABR_OK;
}

/* --------------------------------------------------------- Monte Carlo --- */

typedef struct {
    int n;
    double *dt, *sqrt_dt, *nu, *rho, *srho;
    double beta;
    int lognormal;
} grid_t;

static void grid_free(grid_t* g) {
    free(g->dt);
    free(g->sqrt_dt);
    free(g->nu);
    free(g->rho);
    free(g->srho);
}

/* ModelDynamics::{nu_at, rho_at}, mc.cpp:213-229 with types.hpp param order */
static double model_nu_at(int model, const double* p, double t) {
    switch (model) {
        case SABR_MODEL_STATIC: return p[2];
        case SABR_MODEL_CASE1: return p[3] * exp(-p[5] * t);
        default: return c2_nu_at(p, t);
    }
}
static double model_rho_at(int model, const double* p, double t) {
    switch (model) {
        case SABR_MODEL_STATIC: return p[3];
        case SABR_MODEL_CASE1: return p[2] * exp(-p[4] * t);
        default: return c2_rho_at(p, t);
    }
}

/* ModelDynamics::from_* validation, mc.cpp:183-211 */
static int model_status(int model, const double* p) {
    switch (model) {
        case SABR_MODEL_STATIC: return static_valid(p) ? SABR_OK : SABR_E_DOMAIN;
        case SABR_MODEL_CASE1: return case1_valid(p) ? SABR_OK : SABR_E_DOMAIN;
        case SABR_MODEL_CASE2: {
            if (!(p[0] > 0) || !(p[1] >= 0 && p[1] <= 1) || !(p[8] >= 0 && p[9] >= 0) ||
                !(p[10] > 0))
                return SABR_E_DOMAIN;
            return orc_case2_feasible(p) ? SABR_OK : SABR_E_CONSTRAINT;
        }
    }
    return SABR_E_DOMAIN;
}

/* build_grid, mc.cpp:50-84 */
static int build_grid(int model, const double* p, double maturity, double dt, grid_t* g) {
    if (!(maturity > 0) || !(dt > 0)) return SABR_E_DOMAIN;
    const size_t full_steps = (size_t)floor(maturity / dt + 1e-9);
    if (full_steps == 0) return SABR_E_DOMAIN;
    const double rem = maturity - (double)full_steps * dt;
    const int extra = rem > 1e-12 * smax(maturity, 1.0);
    const int n = (int)full_steps + extra;
    g->n = n;
    g->dt = malloc(sizeof(double) * n);
    g->sqrt_dt = malloc(sizeof(double) * n);
    g->nu = malloc(sizeof(double) * n);
    g->rho = malloc(sizeof(double) * n);
    g->srho = malloc(sizeof(double) * n);
    g->beta = p[1];
    g->lognormal = g->beta == 1.0;
    for (size_t i = 0; i < full_steps; ++i) g->dt[i] = dt;
    if (extra) g->dt[n - 1] = rem;
    for (int i = 0; i < n; ++i) {
        /* node_time[i+1] = min((i+1)*dt, maturity), or maturity for the short step */
        const double t = (extra && i == n - 1) ? maturity : smin((double)(i + 1) * dt, maturity);
        const double nu = model_nu_at(model, p, t);
        const double rho = model_rho_at(model, p, t);
        g->sqrt_dt[i] = sqrt(g->dt[i]);
        g->nu[i] = nu;
        g->rho[i] = rho;
        g->srho[i] = sqrt(smax(0.0, 1.0 - rho * rho));
    }
    return SABR_OK;
}

/* box_muller on two given uniforms, mc.cpp:30-36 */
static void box_muller(double ua, double ub, double* z1, double* z2) {
    const double u1 = 1.0 - ua;
    const double u2 = ub;
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * ORC_PI * u2;
    *z1 = r * cos(theta);
    *z2 = r * sin(theta);
}

/* run_path (terminal observation only), mc.cpp:87-107.  rng_mode 0: the
 * block's sequential xoshiro stream; 1: Philox keyed by (seed, path, step). */
static double run_path(const grid_t* g, double forward0, double alpha0, int rng_mode,
                       orc_xoshiro* xo, uint64_t seed, uint64_t path) {
    double alpha = alpha0;
    double forward = forward0;
    for (int i = 0; i < g->n; ++i) {
        double ua, ub;
        if (rng_mode == SABR_RNG_XOSHIRO) {
            ua = orc_xoshiro_uniform(xo);
            ub = orc_xoshiro_uniform(xo);
        } else {
            orc_philox_uniform_pair(seed, path, (uint32_t)i, &ua, &ub);
        }
        double z1, z2;
        box_muller(ua, ub, &z1, &z2);
        const double nu = g->nu[i];
        const double dt = g->dt[i];
        const double sdt = g->sqrt_dt[i];
        const double alpha_next = alpha * exp(nu * z1 * sdt - 0.5 * nu * nu * dt);
        const double nu_hat = g->lognormal ? alpha : alpha * pow(forward, g->beta - 1.0);
        forward *= exp(nu_hat * (g->rho[i] * z1 + g->srho[i] * z2) * sdt -
                       0.5 * nu_hat * nu_hat * dt);
        alpha = alpha_next;
    }
    return forward;
}

/* SimulationPlan::validate, mc.cpp:161-166 */
static int plan_valid(const sabr_plan* p) {
    return p->num_paths >= 1 && p->dt > 0 && p->workers >= 1 && p->block_size >= 1 &&
           (p->rng == SABR_RNG_XOSHIRO || p->rng == SABR_RNG_PHILOX);
}

/* simulate_terminals -> simulate_observations, mc.cpp:110-139, :231-240
 * (serial; identical to reference::simulate_terminals, mc.cpp:322-343). */
int orc_simulate_terminals(int model, const double* params, double forward0, double alpha0,
                           double T, const sabr_plan* plan, double* out) {
    if (!plan_valid(plan)) return SABR_E_DOMAIN;
    int st = model_status(model, params);
    if (st != SABR_OK) return st;
    if (!(forward0 > 0) || alpha0 < 0) return SABR_E_DOMAIN;
    grid_t g;
    st = build_grid(model, params, T, plan->dt, &g);
    if (st != SABR_OK) return st;
    int bad = 0;
    if (plan->rng == SABR_RNG_XOSHIRO) {
        const uint64_t n_blocks = (plan->num_paths + plan->block_size - 1) / plan->block_size;
        for (uint64_t block = 0; block < n_blocks; ++block) {
            orc_xoshiro rng;
            orc_xoshiro_init(&rng, plan->seed, block);
            const uint64_t begin = block * plan->block_size;
            uint64_t end = begin + plan->block_size;
            if (end > plan->num_paths) end = plan->num_paths;
            for (uint64_t path = begin; path < end; ++path) {
                out[path] = run_path(&g, forward0, alpha0, SABR_RNG_XOSHIRO, &rng, 0, 0);
                if (!isfinite(out[path])) bad = 1;
            }
        }
    } else {
        for (uint64_t path = 0; path < plan->num_paths; ++path) {
            out[path] = run_path(&g, forward0, alpha0, SABR_RNG_PHILOX, NULL, plan->seed, path);
            if (!isfinite(out[path])) bad = 1;
        }
    }
    grid_free(&g);
    return bad ? SABR_E_RUNTIME : SABR_OK;
}

/* run_path with observation nodes, mc.cpp:87-107 (obs recorded after step
 * i+1 == node; node 0 is never recorded) */
static void run_path_obs(const grid_t* g, double forward0, double alpha0, int rng_mode,
                         orc_xoshiro* xo, uint64_t seed, uint64_t path, const int* nodes, int n_obs,
                         double* out) {
    double alpha = alpha0, forward = forward0;
    int next = 0;
    for (int i = 0; i < g->n; ++i) {
        double ua, ub;
        if (rng_mode == SABR_RNG_XOSHIRO) {
            ua = orc_xoshiro_uniform(xo);
            ub = orc_xoshiro_uniform(xo);
        } else {
            orc_philox_uniform_pair(seed, path, (uint32_t)i, &ua, &ub);
        }
        double z1, z2;
        box_muller(ua, ub, &z1, &z2);
        const double nu = g->nu[i], dt = g->dt[i], sdt = g->sqrt_dt[i];
        const double alpha_next = alpha * exp(nu * z1 * sdt - 0.5 * nu * nu * dt);
        const double nu_hat = g->lognormal ? alpha : alpha * pow(forward, g->beta - 1.0);
        forward *= exp(nu_hat * (g->rho[i] * z1 + g->srho[i] * z2) * sdt - 0.5 * nu_hat * nu_hat * dt);
        alpha = alpha_next;
        if (next < n_obs && nodes[next] == i + 1) out[next++] = forward;
    }
}

/* price_cliquet, mc.cpp:275-320 */
int orc_price_cliquet(int model, const double* params, double spot, double rate, double dividend,
                      double lf, double lc, double gf, double gc, const double* resets, int n_resets,
                      const sabr_plan* plan, double* value, double* se) {
    if (lf > lc || gf > gc || n_resets < 2) return SABR_E_DOMAIN;
    for (int i = 0; i < n_resets; ++i)
        if (resets[i] <= 0 || (i > 0 && resets[i] <= resets[i - 1])) return SABR_E_DOMAIN;
    if (!plan_valid(plan) || !(spot > 0)) return SABR_E_DOMAIN;
    int st = model_status(model, params);
    if (st != SABR_OK) return st;
    const double maturity = resets[n_resets - 1];
    const double forward0 = spot * exp((rate - dividend) * maturity);
    grid_t g;
    st = build_grid(model, params, maturity, plan->dt, &g);
    if (st != SABR_OK) return st;
    double* node_time = malloc(sizeof(double) * (g.n + 1));
    node_time[0] = 0.0;
    double acc = 0.0;
    for (int i = 0; i < g.n; ++i) {  /* node_time of build_grid, mc.cpp:59-68 */
        const int extra = (i == g.n - 1) && g.dt[i] != plan->dt;
        acc = extra ? maturity : smin((double)(i + 1) * plan->dt, maturity);
        node_time[i + 1] = acc;
    }
    int nodes[256];
    double disc[256];
    for (int k = 0; k < n_resets; ++k) {
        int best = 0;
        for (int j = 1; j <= g.n; ++j)
            if (fabs(node_time[j] - resets[k]) < fabs(node_time[best] - resets[k])) best = j;
        if (fabs(node_time[best] - resets[k]) > 0.5 * plan->dt + 1e-12 ||
            (k > 0 && best <= nodes[k - 1])) {
            free(node_time);
            grid_free(&g);
            return SABR_E_DOMAIN;
        }
        nodes[k] = best;
        disc[k] = exp(-(rate - dividend) * (maturity - node_time[best]));
    }
    const size_t n = plan->num_paths;
    double* rows = calloc(n * (size_t)n_resets, sizeof(double));
    int bad = 0;
    if (plan->rng == SABR_RNG_XOSHIRO) {
        const uint64_t n_blocks = (n + plan->block_size - 1) / plan->block_size;
        for (uint64_t b = 0; b < n_blocks; ++b) {
            orc_xoshiro rng;
            orc_xoshiro_init(&rng, plan->seed, b);
            const uint64_t begin = b * plan->block_size;
            const uint64_t end = begin + plan->block_size < n ? begin + plan->block_size : n;
            for (uint64_t p = begin; p < end; ++p)
                run_path_obs(&g, forward0, params[0], SABR_RNG_XOSHIRO, &rng, 0, 0, nodes, n_resets,
                             rows + p * n_resets);
        }
    } else {
        for (uint64_t p = 0; p < n; ++p)
            run_path_obs(&g, forward0, params[0], SABR_RNG_PHILOX, NULL, plan->seed, p, nodes, n_resets,
                         rows + p * n_resets);
    }
    for (size_t i = 0; i < n * (size_t)n_resets; ++i)
        if (!isfinite(rows[i])) bad = 1;
    const double discount = exp(-rate * maturity);
    double sum = 0.0, sum_sq = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double* row = rows + i * n_resets;
        double s = 0.0;
        for (int j = 1; j < n_resets; ++j) {
            const double s_prev = row[j - 1] * disc[j - 1];
            const double s_cur = row[j] * disc[j];
            s += sclamp((s_cur - s_prev) / s_prev, lf, lc);
        }
        const double v = discount * sclamp(s, gf, gc);
        sum += v;
        sum_sq += v * v;
    }
    const double mean = sum / (double)n;
    *value = mean;
    *se = sqrt(smax(0.0, (sum_sq - (double)n * mean * mean) / ((double)n - 1.0)) / (double)n);
    free(rows);
    free(node_time);
    grid_free(&g);
    return bad ? SABR_E_RUNTIME : SABR_OK;
}

/* price_european_batch + reduce_payoffs, mc.cpp:146-157, :249-273 */
int orc_price_european_batch(int model, const double* params, double spot,
                             const double* strikes, int64_t m, double rate, double dividend,
                             double T, const sabr_plan* plan, double* value, double* se) {
    if (!(spot > 0)) return SABR_E_DOMAIN;
    for (int64_t j = 0; j < m; ++j)
        if (strikes[j] <= 0) return SABR_E_DOMAIN;
    const double forward0 = spot * exp((rate - dividend) * T);
    double* term = malloc(sizeof(double) * plan->num_paths);
    const int st = orc_simulate_terminals(model, params, forward0, params[0], T, plan, term);
    if (st != SABR_OK) {
        free(term);
        return st;
    }
    const double discount = exp(-rate * T);
    const size_t n = plan->num_paths;
    for (int64_t j = 0; j < m; ++j) {
        double sum = 0.0, sum_sq = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double v = discount * smax(term[i] - strikes[j], 0.0);
            sum += v;
            sum_sq += v * v;
        }
        const double mean = sum / (double)n;
        const double var = smax(0.0, (sum_sq - (double)n * mean * mean) / ((double)n - 1.0));
        value[j] = mean;
        se[j] = sqrt(var / (double)n);
    }
    free(term);
    return SABR_OK;
}

/* black_scholes_call, black_scholes.cpp:20-35 */
double orc_black_scholes_call(double spot, double strike, double r, double y, double T,
                              double vol) {
    const double df_div = spot * exp(-y * T);
    const double df_k = strike * exp(-r * T);
    if (vol == 0.0) return smax(df_div - df_k, 0.0);
    const double sd = vol * sqrt(T);
    const double d1 = (log(spot / strike) + (r - y + 0.5 * vol * vol) * T) / sd;
    const double d2 = d1 - sd;
    return df_div * (0.5 * erfc(-d1 / ORC_SQRT2)) - df_k * (0.5 * erfc(-d2 / ORC_SQRT2));
}

/* implied_vol_from_price, black_scholes.cpp:37-69 (bounds checked by the caller's
 * orc_implied_vol_status): doubling bracket, then <= 200 Newton steps on vega
 * with the bisection fallback and the |diff| < 1e-10 exit. */
static double orc_norm_pdf(double x) { return exp(-0.5 * x * x) / sqrt(2.0 * ORC_PI); }

int orc_implied_vol_from_price(double price, double spot, double strike, double r, double y,
                               double T, double* vol_out) {
    if (spot <= 0 || strike <= 0 || T <= 0) return SABR_E_DOMAIN;
    const double lower = orc_black_scholes_call(spot, strike, r, y, T, 0.0);
    const double upper = spot * exp(-y * T);
    if (price <= lower || price >= upper) return SABR_E_DOMAIN;
    double lo = 0.0, hi = 1.0;
    while (orc_black_scholes_call(spot, strike, r, y, T, hi) < price) hi *= 2.0;
    double vol = 0.5 * (lo + hi);
    for (int it = 0; it < 200; ++it) {
        const double v = orc_black_scholes_call(spot, strike, r, y, T, vol);
        const double diff = v - price;
        if (fabs(diff) < 1e-10) break;
        if (diff > 0)
            hi = vol;
        else
            lo = vol;
        const double sd = vol * sqrt(T);
        const double d1 = (log(spot / strike) + (r - y + 0.5 * vol * vol) * T) / sd;
        const double vega = spot * exp(-y * T) * orc_norm_pdf(d1) * sqrt(T);
        double next = vol - diff / vega;
        if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
        vol = next;
    }
    *vol_out = vol;
    return SABR_OK;
}

/* case2_mc_cost, calibration.cpp:399-416 with market_prices, :277-287 */
int orc_cost_case2_mc(const sabr_surface* s, const double p[11], const sabr_plan* plan,
                      double* cost) {
    double sum = 0.0;
    for (int64_t i = 0; i < s->n_slices; ++i) {
        const int64_t q0 = s->quote_offset[i], q1 = s->quote_offset[i + 1];
        double* value = malloc(sizeof(double) * (size_t)(q1 - q0));
        double* se = malloc(sizeof(double) * (size_t)(q1 - q0));
        const int st = orc_price_european_batch(SABR_MODEL_CASE2, p, s->spot, s->strike + q0,
                                                q1 - q0, s->rate[i], s->dividend[i],
                                                s->maturity[i], plan, value, se);
        if (st != SABR_OK) {
            free(value);
            free(se);
            return st;
        }
        for (int64_t j = q0; j < q1; ++j) {
            const double market = orc_black_scholes_call(s->spot, s->strike[j], s->rate[i],
                                                         s->dividend[i], s->maturity[i], s->vol[j]);
            const double rel = (market - value[j - q0]) / market;
            sum += rel * rel;
        }
        free(value);
        free(se);
    }
    *cost = sum;
    return SABR_OK;
}
