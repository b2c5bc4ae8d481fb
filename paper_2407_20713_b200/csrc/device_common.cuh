// device_common.cuh — sm_100a device primitives of the SABR engine.
//
// RNG (reference streams + Philox), the asymptotic implied-vol building
// blocks and the level-merge rule shared by the host and the device.  Every
// function cites the reference line it reproduces (paths relative to
// /root/reference).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sabr_b200.h"

#define SABR_HD __host__ __device__ __forceinline__
#define SABR_D __device__ __forceinline__

namespace sabr_dev {

// ------------------------------------------------------------------ RNG ---

// splitmix64, proj/include/sabr/rng.hpp:7-12
SABR_HD uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

SABR_HD uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// 64-bit rotate by a compile-time K as two 32-bit funnel shifts (SHF.L.W):
// the generic form compiles to four shift/or instructions per rotate.
template <int K>
SABR_HD uint64_t rotl64c(uint64_t x) {
#ifdef __CUDA_ARCH__
    uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
    if constexpr (K >= 32) {
        const uint32_t t = lo;
        lo = hi;
        hi = t;
    }
    constexpr int k = K & 31;
    const uint32_t nhi = __funnelshift_l(lo, hi, k), nlo = __funnelshift_l(hi, lo, k);
    return (static_cast<uint64_t>(nhi) << 32) | nlo;
#else
    return rotl64(x, K);
#endif
}

// Xoshiro256pp, rng.hpp:16-43; state kept in four registers.
#ifdef __CUDA_ARCH__
// a ^ b ^ c as two LOP3 (one per 32-bit half)
__device__ __forceinline__ uint64_t xor3(uint64_t a, uint64_t b, uint64_t c) {
    uint32_t lo, hi;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;"
        : "=r"(lo)
        : "r"(static_cast<uint32_t>(a)), "r"(static_cast<uint32_t>(b)), "r"(static_cast<uint32_t>(c)));
    asm("lop3.b32 %0, %1, %2, %3, 0x96;"
        : "=r"(hi)
        : "r"(static_cast<uint32_t>(a >> 32)), "r"(static_cast<uint32_t>(b >> 32)), "r"(static_cast<uint32_t>(c >> 32)));
    return (static_cast<uint64_t>(hi) << 32) | lo;
}
#endif

struct Xoshiro {
    uint64_t s0, s1, s2, s3;

    // Xoshiro256pp(seed, stream), rng.hpp:19-23
    SABR_HD void init(uint64_t seed, uint64_t stream) {
        uint64_t sm = seed ^ (stream * 0xD2B74407B1CE6E93ull + 0x9E3779B97F4A7C15ull);
        s0 = splitmix64(sm);
        s1 = splitmix64(sm);
        s2 = splitmix64(sm);
        s3 = splitmix64(sm);
    }
    // the F2-linear state transition of next() without the output scrambler
    SABR_HD void advance() {
#ifdef __CUDA_ARCH__
        // s2' = s2^s0^t, s1' = s1^s2^s0, s0' = s0^s3^s1, s3' = s3^s1: one
        // three-input LOP3 per 32-bit half each (the C++ form shares s2^s0
        // and s3^s1 and costs two more)
        const uint64_t t = s1 << 17;
        const uint64_t n2 = xor3(s2, s0, t), n1 = xor3(s1, s2, s0), n0 = xor3(s0, s3, s1);
        s3 = rotl64c<45>(s3 ^ s1);
        s2 = n2;
        s1 = n1;
        s0 = n0;
#else
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl64c<45>(s3);
#endif
    }
    // next(), rng.hpp:29-39
    SABR_HD uint64_t next() {
        const uint64_t result = rotl64c<23>(s0 + s3) + s0;
        advance();
        return result;
    }
    // (n >> 11) * 2^-53 is computed as (n & ~0x7ff) * 2^-64: the masked value
    // has at most 53 significant bits, so its conversion is exact and the
    // products are the same doubles (one LOP3 instead of a 64-bit shift).
    static SABR_HD double top53(uint64_t n) { return static_cast<double>(n & ~0x7ffull); }
    // the uniform() that the next draw would return, without drawing it
    SABR_HD double peek_uniform() const { return top53(rotl64c<23>(s0 + s3) + s0) * 0x1.0p-64; }
    // the output next() would return (the raw 64-bit draw), without drawing it
    SABR_HD uint64_t peek() const { return rotl64c<23>(s0 + s3) + s0; }
    // 2 * uniform() - 1 of a raw draw n (sym() without the draw)
    static SABR_HD double sym_of(uint64_t n) { return fma(top53(n), 0x1.0p-63, -1.0); }
    // the next draw's 53 significant bits in place: uniform() = peek_bits() * 2^-64 exactly
    SABR_HD uint64_t peek_bits() const { return (rotl64c<23>(s0 + s3) + s0) & ~0x7ffull; }
    // advance() when p, in place and without selects: the eight 32-bit words
    // are updated by predicated instructions in an order that reads every old
    // word before it is overwritten (s1 first, s0 from s3 ^ s1 kept aside);
    // the select form (a copy advanced, then chosen) costs eight more ALU ops.
    SABR_HD void advance_if(bool p) {
#ifdef __CUDA_ARCH__
        uint32_t a0 = static_cast<uint32_t>(s0), b0 = static_cast<uint32_t>(s0 >> 32);
        uint32_t a1 = static_cast<uint32_t>(s1), b1 = static_cast<uint32_t>(s1 >> 32);
        uint32_t a2 = static_cast<uint32_t>(s2), b2 = static_cast<uint32_t>(s2 >> 32);
        uint32_t a3 = static_cast<uint32_t>(s3), b3 = static_cast<uint32_t>(s3 >> 32);
        asm("{\n\t.reg .pred q;\n\t.reg .b32 tl, th, xl, xh;\n\t"
            "setp.ne.u32 q, %8, 0;\n\t"
            "shl.b32 tl, %2, 17;\n\t"                 // t = s1 << 17
            "shf.l.clamp.b32 th, %2, %3, 17;\n\t"
            "xor.b32 xl, %6, %2;\n\t"                  // x = s3 ^ s1
            "xor.b32 xh, %7, %3;\n\t"
            "@q lop3.b32 %2, %2, %4, %0, 0x96;\n\t"  // s1 ^= s2 ^ s0
            "@q lop3.b32 %3, %3, %5, %1, 0x96;\n\t"
            "@q lop3.b32 %4, %4, %0, tl, 0x96;\n\t"  // s2 ^= s0 ^ t
            "@q lop3.b32 %5, %5, %1, th, 0x96;\n\t"
            "@q xor.b32 %0, %0, xl;\n\t"              // s0 ^= s3 ^ s1
            "@q xor.b32 %1, %1, xh;\n\t"
            "@q shf.l.wrap.b32 %6, xl, xh, 13;\n\t"   // s3 = rotl(s3 ^ s1, 45)
            "@q shf.l.wrap.b32 %7, xh, xl, 13;\n\t"
            "}"
            : "+r"(a0), "+r"(b0), "+r"(a1), "+r"(b1), "+r"(a2), "+r"(b2), "+r"(a3), "+r"(b3)
            : "r"(static_cast<uint32_t>(p)));
        s0 = (static_cast<uint64_t>(b0) << 32) | a0;
        s1 = (static_cast<uint64_t>(b1) << 32) | a1;
        s2 = (static_cast<uint64_t>(b2) << 32) | a2;
        s3 = (static_cast<uint64_t>(b3) << 32) | a3;
#else
        if (p) advance();
#endif
    }
    // uniform(), rng.hpp:42: (next() >> 11) * 2^-53 (exact conversion)
    SABR_HD double uniform() { return top53(next()) * 0x1.0p-64; }
    // 2*uniform() - 1 (annealer.cpp:66) in one exact FMA: (n >> 11) * 2^-52
    // is exact and the difference with 1 is representable, so this equals
    // the reference's RN(RN(2u) - 1) bit for bit.
    SABR_HD double sym() { return fma(top53(next()), 0x1.0p-63, -1.0); }

    // state <- M^k state, where x^k mod P(x) = sum_i poly_i x^i (256 bits,
    // host-computed; see xoshiro_jump.cpp).  Branch-free masked accumulate.
    SABR_HD void jump(const uint64_t poly[4]) {
        uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 1
        for (int w = 0; w < 4; ++w) {
            const uint64_t word = poly[w];
#pragma unroll 8
            for (int b = 0; b < 64; ++b) {
                const uint64_t m = 0ull - ((word >> b) & 1ull);
                a0 ^= s0 & m;
                a1 ^= s1 & m;
                a2 ^= s2 & m;
                a3 ^= s3 & m;
                advance();
            }
        }
        s0 = a0;
        s1 = a1;
        s2 = a2;
        s3 = a3;
    }
};

// Philox4x32-10, counter (path lo, path hi, step, 0), key = seed.  The CPU
// twin is oracle/sabr_oracle.c:orc_philox4x32.
SABR_D void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key,
                          uint32_t out[4]) {
    uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// the pair's two raw 64-bit draws (philox_uniform_pair = their top53 * 2^-64)
SABR_D void philox_bits_pair(uint64_t seed, uint64_t path, uint32_t step, uint64_t& a, uint64_t& b) {
    uint32_t x[4];
    philox4x32_10(static_cast<uint32_t>(path), static_cast<uint32_t>(path >> 32), step, 0u, seed, x);
    a = (static_cast<uint64_t>(x[0]) << 32) | x[1];
    b = (static_cast<uint64_t>(x[2]) << 32) | x[3];
}

SABR_D void philox_uniform_pair(uint64_t seed, uint64_t path, uint32_t step, double& ua,
                                double& ub) {
    uint32_t x[4];
    philox4x32_10(static_cast<uint32_t>(path), static_cast<uint32_t>(path >> 32), step, 0u, seed, x);
    const uint64_t a = (static_cast<uint64_t>(x[0]) << 32) | x[1];
    const uint64_t b = (static_cast<uint64_t>(x[2]) << 32) | x[3];
    ua = Xoshiro::top53(a) * 0x1.0p-64;
    ub = Xoshiro::top53(b) * 0x1.0p-64;
}

// ------------------------------------------------------------ fast exp ---
// exp(x) = 2^(k/128) * e^r, |r| <= ln2/256: k from one FMA with the 1.5*2^52
// shift trick, 2^(i/128) from a 128-entry double-double table (i = k mod 128,
// staged in shared memory by the caller), e^r - 1 by a degree-5 polynomial
// (truncation < 6e-19), 2^(k>>7) applied by an integer add to the exponent.
// ~0.51 ulp like glibc's exp; 11 FP64 ops and 5 64-bit constants instead of
// libdevice's 16 FP64 ops and ~11 materialised constants.  Branch-free (a
// branch would give every inlined call its own reconvergence region and stop
// the scheduler interleaving independent exps): |x| > 700 saturates to
// +inf / +0 (exp(700) = 1e304 only feeds non-finite detection), NaN -> NaN.
// table entry i = {RN(2^(i/128)), RN(2^(i/128) - hi)}: built on the host in
// long double (kernels_mc.cu: exp_table_host()).
constexpr int kExpTableSize = 128;

// The table replicated across the shared-memory bank groups: entry i of copy
// c at [kExpRep * i + c], and a lane reads copy (lane & 7) (the caller passes
// tab + (lane & 7) and STRIDE = kExpRep).  The eight lanes of a quarter-warp,
// one LDS.128 wavefront, then never meet in a bank: random arguments no
// longer serialise the lookup (8.9-way conflicts on the shared table, ncu).
constexpr int kExpRep = 8;

// exp_tab without the saturation test: valid for |x| <= 700 only (callers
// that can bound the argument on the host use it and save the compare/select).
template <int STRIDE = 1>
SABR_D double exp_tab_unsat(double x, const double2* __restrict__ tab) {
    constexpr double kInvLn2N = 0x1.71547652b82fep7;  // 128 / ln 2
    constexpr double kShift = 0x1.8p52;
    constexpr double kLn2NHi = 0x1.62e42fefa39efp-8;  // ln2/128 = hi + lo (FMA reduction)
    constexpr double kLn2NLo = 0x1.abc9e3b39803fp-63;
    const double z = fma(x, kInvLn2N, kShift);
    const double kd = z - kShift;
    const int k = static_cast<int>(__double2loint(z));
    double r = fma(kd, -kLn2NHi, x);
    r = fma(kd, -kLn2NLo, r);
    // e^r - 1 = r + r^2/2 + r^3/6 + r^4/24 + r^5/120
    const double r2 = r * r;
    const double q = fma(fma(r, 1.0 / 120, 1.0 / 24), r2, fma(r, 1.0 / 6, 0.5));
    const double p = fma(q, r2, r);
    const double2 t = tab[(k & 127) * STRIDE];
    const double v = t.x + fma(t.x, p, t.y);
    // scale by 2^(k >> 7): add to the exponent field (result stays normal for |x| <= 700)
    return __hiloint2double(__double2hiint(v) + ((k >> 7) << 20), __double2loint(v));
}

template <int STRIDE = 1>
SABR_D double exp_tab(double x, const double2* __restrict__ tab) {
    const double res = exp_tab_unsat<STRIDE>(x, tab);
    // NaN fails the test and flows through the arithmetic into res
    const double sat = x > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
    return fabs(x) > 700.0 ? sat : res;
}

// exp for the Monte Carlo candidate step (r02): exp_tab without the ln2/128
// low-part correction and with one polynomial term fewer (e^r - 1 = r + r^2
// (1/2 + r/6 + r^2/24), |r| <= ln2/256): relative error <= 1.3e-15 for
// |x| <= 20 (the dropped terms: r^5/120 <= 1.2e-15, |k| ln2lo <= 5e-16),
// two FP64 instructions fewer per candidate-step.  nu_hat = exp(arg) scales
// one log-Euler increment, so this moves F_T by ~1e-15 relative (the MC
// parity bar is 1e-12); the saturation and NaN behaviour are
// exp_tab's.  F_T itself keeps exp_tab.
template <int STRIDE = 1>
SABR_D double exp_mc(double x, const double2* __restrict__ tab) {
    constexpr double kInvLn2N = 0x1.71547652b82fep7;  // 128 / ln 2
    constexpr double kShift = 0x1.8p52;
    constexpr double kLn2NHi = 0x1.62e42fefa39efp-8;  // ln2/128 (rounded)
    const double z = fma(x, kInvLn2N, kShift);
    const double kd = z - kShift;
    const int k = static_cast<int>(__double2loint(z));
    const double r = fma(kd, -kLn2NHi, x);
    const double r2 = r * r;
    const double q = fma(fma(r, 1.0 / 24, 1.0 / 6), r, 0.5);
    const double p = fma(q, r2, r);
    const double2 t = tab[(k & 127) * STRIDE];
    const double v = t.x + fma(t.x, p, t.y);
    const double res = __hiloint2double(__double2hiint(v) + ((k >> 7) << 20), __double2loint(v));
    const double sat = x > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
    return fabs(x) > 700.0 ? sat : res;
}

// case2_mc_cost's sum over one candidate's quotes, calibration.cpp:410-413:
// the reference's sequential order; 8 quotes' loads and divisions are
// independent and issued together (C5: 600 quotes per candidate)
SABR_D double mc_quote_cost(const double* __restrict__ v, const double* __restrict__ market, int nq) {
    double sum = 0.0;
    int q = 0;
    for (; q + 8 <= nq; q += 8) {
        double rel[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rel[u] = (market[q + u] - v[q + u]) / market[q + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) sum += rel[u] * rel[u];
    }
    for (; q < nq; ++q) {
        const double rel = (market[q] - v[q]) / market[q];
        sum += rel * rel;
    }
    return sum;
}

// ----------------------------------------------------------- Metropolis ---
// annealer.cpp:125-126: accept iff fy <= fx || u < exp(-(fy - fx) / T), with
// u = uniform() drawn only when fy > fx.  With tau = -ln u the test is
// q < tau, q = (fy - fx) / T, and tau depends only on the chain's stream, not
// on the objective, so it is computed off the critical path in FP32 (one
// I2F.F32, one MUFU.LG2) and the comparison certified with a margin:
//   |tau_f - tau| <= 2^-18 + 2^-22 tau (2^-24 relative rounding of the 53-bit
//   draw, lg2.approx's 2^-22 absolute error, the FADD/FMUL roundings),
//   |q_f - q| <= 2^-23 q (q_f = RN_f32((fy - fx) * RN(1/T)), RN(1/T) 1 ulp),
// so |q_f - tau_f| > 2^-15 (1 + tau_f) decides q < tau exactly, and with
// margin ~1.5e-5 relative the glibc exp's own rounding cannot flip it either.
// Otherwise (probability ~3e-5 per uphill step) the caller decides with
// metropolis_exact: the reference's division and a libdevice exp.  tau_f is
// capped at 745: u = 0 (m = 0) accepts iff exp(-q) > 0, i.e. q < 745.13..., and
// the cap's margin band sends q near 745 to the exact test.  q = +inf (fy =
// +inf) rejects; q = NaN cannot occur uphill (fy > fx excludes fx = +inf).
SABR_D float neg_log_uniform(uint64_t m) {  // m = peek_bits(): u = m * 2^-64
    const float mf = __ull2float_rn(m);
    float lg;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(mf));  // -inf for m = 0
    return fminf((64.0f - lg) * 0.693147182f, 745.0f);
}
struct MetroFast {
    bool accept, unsure;
};
SABR_D MetroFast metropolis_fast(double fy, double fx, double inv_temp, float tau) {
    const bool up = !(fy <= fx);
    const float qf = __double2float_rn((fy - fx) * inv_temp);
    const float diff = qf - tau;
    const bool clear = fabsf(diff) > fmaf(tau, 0x1p-15f, 0x1p-15f);
    return MetroFast{!up || (qf < tau), up && !clear};
}
SABR_D bool metropolis_exact(double fy, double fx, double temp, uint64_t m) {
    const double u = static_cast<double>(m) * 0x1.0p-64;
    return u < exp(-((fy - fx) / temp));
}

// ---------------------------------------------------- table log / sqrt ---
// Bit casts usable on host and device (the host builds of these functions are
// the accuracy checks of tools/mathtab_check.cpp).
SABR_HD uint64_t dbits(double x) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    __builtin_memcpy(&u, &x, 8);
    return u;
#endif
}
SABR_HD double bitsd(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    __builtin_memcpy(&x, &u, 8);
    return x;
#endif
}

// log(x) for positive normal x: x = 2^k z with z in [0.6875, 1.375) (so z is
// near 1 when x is), z in one of 128 intervals with centre c:
// log x = k ln2 - log(invc) + log1p(r), r = z*invc - 1 (one FMA), |r| < 2^-7,
// log1p by its degree-8 Taylor polynomial (truncation < 2^-60 |r|).  Table
// entry i = {invc = RN(1/c), -log(invc) as hi (on a 2^-42 grid, so k ln2_hi +
// hi is exact) + lo} (host long double,
// kernels_mc.cu: log_table_host()); the two intervals around 1 (kLogOne - 1,
// kLogOne) have invc = 1, -log(invc) = 0, so r = z - 1 exactly and nothing
// cancels as log x -> 0.  <= 1 ulp (0.72, tools/mathtab_check.cpp) with the
// series to r^7 (r^8/8 < 2^-60 here; r02: the r^8 term dropped); 15 FP64
// ops, no branch (libdevice log: 31 FP64 ops, 104 instructions).
constexpr int kLogTableSize = 128;
constexpr int kLogOne = 80;  // the interval that starts at z = 1: (bits(1) - bits(0.6875)) >> 45

SABR_HD double log_tab(double x, const double4* __restrict__ tab) {
    constexpr uint64_t kOff = 0x3fe6000000000000ull;  // 0.6875
    constexpr double kLn2Hi = 0x1.62e42fefa3800p-1;   // 11 trailing zero bits: k*kLn2Hi exact
    constexpr double kLn2Lo = 0x1.ef35793c76730p-45;
    const uint64_t ix = dbits(x);
    const uint64_t tmp = ix - kOff;
    const int i = static_cast<int>((tmp >> 45) & (kLogTableSize - 1));
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const double z = bitsd(ix - (tmp & (0xfffull << 52)));
    const double4 e = tab[i];
    const double r = fma(z, e.x, -1.0);
    const double kd = static_cast<double>(k);
    const double t1 = fma(kd, kLn2Hi, e.y);
    const double t2 = t1 + r;
    const double lo = fma(kd, kLn2Lo, e.z) + ((t1 - t2) + r);
    const double r2 = r * r;
    const double p = fma(fma(fma(fma(fma(fma(1.0 / 7, r, -1.0 / 6), r, 1.0 / 5), r, -1.0 / 4), r, 1.0 / 3), r, -0.5),
                         r2, lo);
    return t2 + p;
}

// sqrt(a) for a >= 0 (finite): MUFU.RSQ64H seed, one Goldschmidt step and a
// final residual correction: the step takes the ~2^-23 seed to ~2^-46, the
// correction (with the residual a - s^2 formed exactly by an FMA) to full
// precision, 0.5 ulp (tools/mathtab_check.cpp; r02: the second Goldschmidt
// step was redundant); libdevice's IEEE sqrt has a slow-path branch and 24
// FP64 ops.  sqrt(0) = 0.
SABR_HD double sqrt_pos(double a) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
#else
    // host model of the hardware seed: 1/sqrt(a) truncated to 23 bits
    const double y = bitsd(dbits(1.0 / __builtin_sqrt(a)) & ~((1ull << 29) - 1));
#endif
    double s = a * y, h = 0.5 * y;
    const double r = fma(-s, h, 0.5);
    s = fma(s, r, s);
    h = fma(h, r, h);
    const double d = fma(-s, s, a);
    s = fma(d, h, s);
    return a > 0.0 ? s : 0.0;
}

// (sin 2 pi u, cos 2 pi u) for u in [0, 1): 2 pi u = (pi/64)(k + f) with
// x = 128 u (exact), k = rint(x), f = x - k in [-1/2, 1/2] (exact); table
// entry k mod 128 = {sin(pi k/64), cos(pi k/64)} (host long double,
// kernels_mc.cu: sincos_table_host()); t = (pi/64) f in double-double
// precision, sin t and cos t - 1 by Taylor polynomials to t^7 / t^6 (r02;
// truncation < 1e-20
// for |t| <= pi/128); recombined by the angle-addition formulas.
// <= 1 ulp (tools/mathtab_check.cpp); branch-free (libdevice sincospi: 96
// instructions).
constexpr int kSinCosTableSize = 128;

SABR_HD void sincos_2pi(double u, const double2* __restrict__ tab, double& s, double& c) {
    constexpr double kPi64Hi = 0x1.921fb54442d18p-5;   // RN(pi/64)
    constexpr double kPi64Lo = 0x1.1a62633145c07p-59;  // pi/64 - kPi64Hi
    constexpr double kShift = 0x1.8p52;
    const double x = u * 128.0;
    const double kd = (x + kShift) - kShift;  // rint for 0 <= x < 2^51
    const double f = x - kd;
    const int k = static_cast<int>(kd) & (kSinCosTableSize - 1);
    const double t = fma(f, kPi64Hi, f * kPi64Lo);
    const double t2 = t * t;
    const double ps = fma(fma(t2, -1.0 / 5040, 1.0 / 120), t2, -1.0 / 6);
    const double st = fma(t * t2, ps, t);
    const double pc = fma(fma(t2, -1.0 / 720, 1.0 / 24), t2, -0.5);
    const double cm1 = t2 * pc;
    const double2 e = tab[k];
    s = e.x + fma(e.x, cm1, e.y * st);
    c = e.y + fma(e.y, cm1, -(e.x * st));
}

// Box-Muller on two uniforms, proj/src/mc.cpp:30-36.  theta = 2*pi*u2 is
// evaluated as sincospi(2*u2) (2*u2 is exact), i.e. without the rounding of
// the 2*pi product; differences are below 1e-15 absolute in z.
SABR_D void box_muller(double ua, double ub, double& z1, double& z2) {
    const double u1 = 1.0 - ua;
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * ub, &s, &c);
    z1 = r * c;
    z2 = r * s;
}

// The same with the table log, sqrt_pos and the table sincos (the MC path
// loops): u1 = 1 - U lies in (2^-53, 1], a positive normal, -2 log(u1) >= 0.
SABR_D void box_muller_tab(double ua, double ub, const double4* __restrict__ logtab,
                           const double2* __restrict__ sctab, double& z1, double& z2) {
    const double u1 = 1.0 - ua;
    const double r = sqrt_pos(-2.0 * log_tab(u1, logtab));
    double s, c;
    sincos_2pi(ub, sctab, s, c);
    z1 = r * c;
    z2 = r * s;
}

// Box-Muller for the FP32 MC path (mc.cpp:30-36) on two raw draws, on the
// MUFU only: u1 = 1 - U1 from the integer (~m1 = 2^64 - 1 - m1 with m1 the
// draw's 53 significant bits: in float this is 2^64 - m1 rounded, never 0,
// and exactly 2^64 -> u1 = 1 for U1 = 0), r = sqrt(-2 ln2 lg2 u1), theta =
// 2 pi U2 taken to [-pi, pi) for sin/cos.approx.  Absolute errors ~1e-6 in
// the normals (lg2/sin/cos.approx ~2^-21), far inside the FP32 path's 2e-5
// price tolerance; one LG2, one SQRT, one SIN, one COS and one I2F instead of
// libm's logf/sqrtf/sincospif (~150 instructions per path-step with their
// range reductions and slow-path calls).
SABR_D void box_muller_f32_bits(uint64_t n1, uint64_t n2, float& z1, float& z2) {
    const uint64_t m1 = n1 & ~0x7ffull;
    float lg, r, sn, cs;
    // lg2 of u1 itself (in [2^-53, 1]), not of the 2^64-scaled integer: the
    // result is near 0 when u1 is near 1 (small r), where float resolves it
    // finely; near 64 its ulp (2^-17) made -2 ln u1 coarse by 1e-5 (measured:
    // 8e-5 worst per-path error, 1.7e-6 with this form)
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(__ull2float_rn(~m1) * 0x1.0p-64f));
    const float w = -1.38629436f * lg;  // -2 ln u1 >= 0
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(w));
    // U2 taken to [-1/2, 1/2) without a conversion (r02, one XU instruction
    // fewer): its top 23 bits with the top one flipped are the mantissa of a
    // float in [1, 2), which minus 1.5 (exactly) is U2 or U2 - 1 truncated to
    // 2^-23; the half-step 2^-24 folded into the angle's FMA centres the
    // grid, so the angle is within 2 pi 2^-24 of 2 pi U2
    const float v2 = __uint_as_float(static_cast<uint32_t>(n2 >> 41) ^ 0x3fc00000u) - 1.5f;
    const float t = fmaf(v2, 6.28318531f, 6.28318531f * 0x1.0p-24f);  // 2 pi U2 in [-pi, pi)
    asm("sin.approx.ftz.f32 %0, %1;" : "=f"(sn) : "f"(t));
    asm("cos.approx.ftz.f32 %0, %1;" : "=f"(cs) : "f"(t));
    z1 = r * cs;
    z2 = r * sn;
}

// ------------------------------------------------------------ analytics ---

// Round-to-nearest primitives that the compiler may not contract into FMAs:
// the Case I closed forms cancel catastrophically just above the series
// switch (x = decay*T in [0.25, ~1]: up to 6e3x for f_eta2), so they are
// evaluated with the reference's exact operation order and roundings.
#ifdef __CUDA_ARCH__
#define SABR_ADD(a, b) __dadd_rn((a), (b))
#define SABR_SUB(a, b) __dsub_rn((a), (b))
#define SABR_MUL(a, b) __dmul_rn((a), (b))
#define SABR_DIV(a, b) __ddiv_rn((a), (b))
#else
#define SABR_ADD(a, b) ((a) + (b))
#define SABR_SUB(a, b) ((a) - (b))
#define SABR_MUL(a, b) ((a) * (b))
#define SABR_DIV(a, b) ((a) / (b))
#endif

// Taylor tables of the scaled Case I functions, analytics.cpp:23-39, as
// fully unrolled Horner evaluations (analytics.cpp:41-45).  The series (used
// for x < 0.25, where nothing cancels: every term is < 0.25^i of the first)
// is evaluated with one FMA per coefficient on the device - half the FP64
// instructions of the reference's multiply-then-add, and at least as
// accurate; the cancelling closed forms above the switch keep the
// reference's exact operation order (SABR_* below).
template <int N>
SABR_HD double horner(const double (&c)[N], double x) {
    double acc = 0.0;
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
#ifdef __CUDA_ARCH__
        acc = fma(acc, x, c[i]);
#else
        acc = SABR_ADD(SABR_MUL(acc, x), c[i]);
#endif
    }
    return acc;
}

SABR_HD double series_nu1(double x) {
    constexpr double c[14] = {
        1.0, -1.0 / 4, 1.0 / 20, -1.0 / 120, 1.0 / 840, -1.0 / 6720, 1.0 / 60480,
        -1.0 / 604800, 1.0 / 6652800, -1.0 / 79833600, 1.0 / 1037836800,
        -1.0 / 14529715200.0, 1.0 / 217945728000.0, -1.0 / 3487131648000.0};
    return horner(c, x);
}
SABR_HD double series_nu2(double x) {
    constexpr double c[14] = {
        1.0, -1.0 / 2, 3.0 / 20, -1.0 / 30, 1.0 / 168, -1.0 / 1120, 1.0 / 8640,
        -1.0 / 75600, 1.0 / 739200, -1.0 / 7983360, 1.0 / 94348800,
        -1.0 / 1210809600, 1.0 / 16765056000.0, -1.0 / 249080832000.0};
    return horner(c, x);
}
SABR_HD double series_eta1(double x) {
    constexpr double c[14] = {
        1.0, -1.0 / 3, 1.0 / 12, -1.0 / 60, 1.0 / 360, -1.0 / 2520, 1.0 / 20160,
        -1.0 / 181440, 1.0 / 1814400, -1.0 / 19958400, 1.0 / 239500800,
        -1.0 / 3113510400.0, 1.0 / 43589145600.0, -1.0 / 653837184000.0};
    return horner(c, x);
}
SABR_HD double series_eta2(double x) {
    constexpr double c[14] = {
        1.0, -3.0 / 5, 7.0 / 30, -1.0 / 14, 31.0 / 1680, -1.0 / 240,
        127.0 / 151200, -17.0 / 110880, 73.0 / 2851200, -31.0 / 7862400,
        2047.0 / 3632428800.0, -1.0 / 13305600, 8191.0 / 871782912000.0,
        -5461.0 / 4940103168000.0};
    return horner(c, x);
}

// dyn_coeffs_case1 (analytics.cpp:207-215 with f_nu1..f_eta2 :47-67), same
// operation order and roundings as the reference; exp(-x) is shared by the
// two functions of one argument (the reference evaluates it twice, same value).
SABR_HD void dyn_coeffs_case1(double rho0, double nu0, double a, double b, double T,
                              double& nu1_sq, double& nu2_sq, double& eta1, double& eta2_sq) {
    constexpr double kXSwitch = 0.25;  // analytics.cpp:21
    const double xb = SABR_MUL(SABR_MUL(2.0, b), T);
    const double xab = SABR_MUL(SABR_ADD(a, b), T);
    const double nn = SABR_MUL(nu0, nu0);
    const double nr = SABR_MUL(nu0, rho0);
    double f1, f2, g1, g2;
    if (xb < kXSwitch) {
        f1 = series_nu1(xb);
        f2 = series_nu2(xb);
    } else {
        const double e = exp(-xb);
        const double x2 = SABR_MUL(xb, xb);
        const double c6 = SABR_DIV(6.0, SABR_MUL(x2, xb));
        // 6/(x^3) * (x*x/2 - x + 1 - e)
        // x*x/2 as a multiply by 0.5: halving is exact, so the bits equal the reference division
        f1 = SABR_MUL(c6, SABR_SUB(SABR_ADD(SABR_SUB(SABR_MUL(x2, 0.5), xb), 1.0), e));
        // 6/(x^3) * (2*(e-1) + x*(e+1))
        f2 = SABR_MUL(c6, SABR_ADD(SABR_MUL(2.0, SABR_SUB(e, 1.0)), SABR_MUL(xb, SABR_ADD(e, 1.0))));
    }
    if (xab < kXSwitch) {
        g1 = series_eta1(xab);
        g2 = series_eta2(xab);
    } else {
        const double e = exp(-xab);
        const double x2 = SABR_MUL(xab, xab);
        // 2/(x*x) * (e - (1 - x))
        g1 = SABR_MUL(SABR_DIV(2.0, x2), SABR_SUB(e, SABR_SUB(1.0, xab)));
        // 3/(x*x*x*x) * (e*e - 8*e + 7 + 2*x*(x - 3))
        const double x4 = SABR_MUL(SABR_MUL(x2, xab), xab);
        const double poly = SABR_ADD(SABR_ADD(SABR_SUB(SABR_MUL(e, e), SABR_MUL(8.0, e)), 7.0),
                                     SABR_MUL(SABR_MUL(2.0, xab), SABR_SUB(xab, 3.0)));
        g2 = SABR_MUL(SABR_DIV(3.0, x4), poly);
    }
    nu1_sq = SABR_MUL(nn, f1);
    nu2_sq = SABR_MUL(nn, f2);
    eta1 = SABR_MUL(nr, g1);
    eta2_sq = SABR_MUL(SABR_MUL(nr, nr), g2);
}

// The maturity-dependent part of Eq. 7 / Eq. 8 hoisted per (candidate,
// slice): sigma(K) = (c0 + a1*lm + a2*lm^2) * inv_omega with lm = ln(K/f).
struct SmileTerms {
    double c0, a1, a2, inv_omega;
};

// 1/x for positive, finite, normal x: MUFU.RCP64H seed + two Newton steps
// (<= 1 ulp; branch-free, unlike the IEEE division's special-case path).
SABR_HD double fast_rcp(double x) {
#ifdef __CUDA_ARCH__
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
#else
    return 1.0 / x;
#endif
}

// static_implied_vol, analytics.cpp:183-205 (everything that does not depend
// on the strike).  pw = pow(f, 1-beta).
SABR_HD SmileTerms static_terms(double alpha, double beta, double nu, double rho, double pw,
                                double T) {
    const double one_m_beta = 1.0 - beta;
    const double omega = pw * fast_rcp(alpha);
    const double inv_omega = alpha * fast_rcp(pw);
    const double rnw = rho * nu * omega;
    const double nw = nu * omega;
    const double rr = 2.0 - 3.0 * rho * rho;
    SmileTerms t;
    t.a1 = -0.5 * (one_m_beta - rnw);
    t.a2 = (one_m_beta * one_m_beta + 3.0 * (one_m_beta - rnw) + rr * nw * nw) * (1.0 / 12.0);
    const double b = one_m_beta * one_m_beta * (inv_omega * inv_omega) * (1.0 / 24.0) +
                     beta * rho * nu * inv_omega * 0.25 + rr * nu * nu * (1.0 / 24.0);
    t.c0 = 1.0 + b * T;
    t.inv_omega = inv_omega;
    return t;
}

// The factored cost's terms: static_terms / dynamic_terms folded into
// x = (C0, A1, A2) = (1 + B T, A1, A2) / omega and regrouped in powers of
// 1/omega (q = (1-beta)/omega; static: p = q - rho nu, Case I: p = q - eta1):
//     A1/omega = -p/2
//     A2/omega = static: ((1-beta) q + 3 p + (2 - 3 rho^2) nu^2 omega) / 12
//                Case I: (1-beta) q / 12 + p / 4 + (4 nu1^2 + 3 (eta2^2 - 3 eta1^2)) omega / 24
//     B        = static: q^2/24 + beta rho nu / (4 omega) + (2 - 3 rho^2) nu^2 / 24
//                Case I: q^2/24 + beta eta1 / (4 omega) + (2 nu2^2 - 3 eta2^2) / 24
//     C0       = 1/omega + (1/omega) B T
// with one reciprocal of alpha f^(1-beta) for both omega and 1/omega.  Each
// term is within a few ulp of the reference's value; the factored cost's own
// conditioning dominates.  The static form with its constants folded into the
// slice factor is kernels_sa.cu static_qterms_f; the Case I form on the scaled
// functionals is dynamic_quad_terms_k below.

// The Case I terms of the factored cost written on the
// scaled functionals of a slice (r02),
//     Af1 = nu0^2/6 f_nu1,  Ef2 = nu0^2/12 f_nu2,  dg1 = nu0 rho0/4 f_eta1 = eta1/4,
//     bg2 = (nu0 rho0)^2/8 f_eta2 = eta2^2/8,
// so that with q = (1-beta)/omega
//     A1/omega = 2 dg1 - q/2
//     A2/omega = k/24 omega - dg1 + q (1/4 + (1-beta)/12),  k/24 = Af1 + bg2 - 6 dg1^2
//     B        = q^2/24 + beta dg1 / omega + Ef2 - bg2
//     C0       = 1/omega + (1/omega) B T.
// The closed forms produce the scaled functionals directly: each chain's
// constant (nu0^2/6, ...) is folded into its scale factor (case1_scales), so
// the slice costs no separate multiplications by nu0, rho0 and 1/24.  Each term
// is within a few ulp of the reference's (dynamic_implied_vol,
// analytics.cpp:291-312); every Case I path uses these functions, so the
// kernel variants agree bit for bit, and with beta = 1 (q = 0 exactly) the
// general form reduces term by term to dynamic_quad_terms_b1.
SABR_HD void dynamic_quad_terms_k(double Af1, double Ef2, double dg1, double bg2, double beta, double inv,
                                  double omega, double T, double& c0, double& a1, double& a2) {
    const double omb = 1.0 - beta;
    const double q = omb * inv;
    const double k24 = fma(-6.0 * dg1, dg1, Af1 + bg2);
    a1 = fma(-0.5, q, dg1 + dg1);
    a2 = fma(k24, omega, fma(q, fma(omb, 1.0 / 12.0, 0.25), -dg1));
    const double B = fma(beta * dg1, inv, fma(q * (1.0 / 24.0), q, Ef2 - bg2));
    c0 = fma(inv, B * T, inv);
}
// beta = 1: 1/omega = alpha, omega = rcp(alpha), q = 0
SABR_HD void dynamic_quad_terms_b1(double Af1, double Ef2, double dg1, double bg2, double inv, double omega,
                                   double T, double& c0, double& a1, double& a2) {
    const double k24 = fma(-6.0 * dg1, dg1, Af1 + bg2);
    a1 = dg1 + dg1;
    a2 = fma(k24, omega, -dg1);
    const double B = fma(dg1, inv, Ef2 - bg2);
    c0 = fma(inv, B * T, inv);
}

#ifdef __CUDACC__
// The Taylor tables of series_nu1 .. series_eta2 as one 64-double block
// (4 series x 16, two trailing zeros each), for a shared-memory copy: FP64
// instructions take no immediate or constant-bank operands, so unrolled
// Horner loops over compile-time tables rematerialise every coefficient with
// two uniform moves per use; from shared memory one LDS.128 brings two.
constexpr int kSeriesStride = 16;
static __constant__ double kCase1Series[4 * kSeriesStride] = {
    1.0, -1.0 / 4, 1.0 / 20, -1.0 / 120, 1.0 / 840, -1.0 / 6720, 1.0 / 60480, -1.0 / 604800,
    1.0 / 6652800, -1.0 / 79833600, 1.0 / 1037836800, -1.0 / 14529715200.0, 1.0 / 217945728000.0,
    -1.0 / 3487131648000.0, 0.0, 0.0,
    1.0, -1.0 / 2, 3.0 / 20, -1.0 / 30, 1.0 / 168, -1.0 / 1120, 1.0 / 8640, -1.0 / 75600,
    1.0 / 739200, -1.0 / 7983360, 1.0 / 94348800, -1.0 / 1210809600, 1.0 / 16765056000.0,
    -1.0 / 249080832000.0, 0.0, 0.0,
    1.0, -1.0 / 3, 1.0 / 12, -1.0 / 60, 1.0 / 360, -1.0 / 2520, 1.0 / 20160, -1.0 / 181440,
    1.0 / 1814400, -1.0 / 19958400, 1.0 / 239500800, -1.0 / 3113510400.0, 1.0 / 43589145600.0,
    -1.0 / 653837184000.0, 0.0, 0.0,
    1.0, -3.0 / 5, 7.0 / 30, -1.0 / 14, 31.0 / 1680, -1.0 / 240, 127.0 / 151200, -17.0 / 110880,
    73.0 / 2851200, -31.0 / 7862400, 2047.0 / 3632428800.0, -1.0 / 13305600, 8191.0 / 871782912000.0,
    -5461.0 / 4940103168000.0, 0.0, 0.0};

// Horner over the shared-memory copy (ser: 4 x kSeriesStride doubles).
__device__ __forceinline__ double horner_s(const double* __restrict__ ser, int fn, double x) {
    const double2* c = reinterpret_cast<const double2*>(ser + fn * kSeriesStride);
    double acc = 0.0;
#pragma unroll
    for (int k = 6; k >= 0; --k) {
        const double2 cc = c[k];
        acc = fma(fma(acc, x, cc.y), x, cc.x);
    }
    return acc;
}

// The two functionals of one argument (f_nu1/f_nu2 at x = 2bT: PAIR 0;
// f_eta1/f_eta2 at x = (a+b)T: PAIR 1), analytics.cpp:47-67, in the
// arithmetic of dyn_coeffs_case1_fast.
template <int PAIR>
__device__ __forceinline__ void case1_series_pair(double x, const double* __restrict__ ser, double& f,
                                                  double& g) {
    f = horner_s(ser, 2 * PAIR, x);
    g = horner_s(ser, 2 * PAIR + 1, x);
}

// The closed forms of one functional pair (f_nu1/f_nu2 at x = 2bT: PAIR 0;
// f_eta1/f_eta2 at x = (a+b)T: PAIR 1), analytics.cpp:46-67, with their
// scale factors supplied (sa, sb within a few ulp
// of the quotients times the chain's constants, case1_scales): PAIR 0 takes
// sa ~ nu0^2 / x^3 and sb ~ nu0^2 / (2 x^3), PAIR 1 sa ~ nu0 rho0 / (2 x^2) and
// sb ~ 3 (nu0 rho0)^2 / (8 x^4).  The brackets are the reference's
// (analytics.cpp:46-67) operation for operation; where one of its products is
// exact (x*x/2, 2*(e-1), 8*e, 2*x*(x-3) = 2*RN(x*(x-3))) the product and the
// following sum are one FMA, which rounds once, as the reference's sum does.
template <int PAIR, int STRIDE = 1>
__device__ __forceinline__ void case1_closed_pair_r(double x, double sa, double sb,
                                                    const double2* __restrict__ tab, double& f, double& g) {
    // exp(-x) for x >= 0.25 (never NaN: x = 2bT or (a+b)T from the box);
    // past x = 700 the clamp's e ~ 1e-304 leaves every bracket the double it
    // is with e = 0 (each bracket holds a term >= x - 1), so exp_tab's
    // saturation selects are not needed
    const double e = exp_tab_unsat<STRIDE>(fmax(-x, -700.0), tab);
    if constexpr (PAIR == 0) {
        const double x2 = SABR_MUL(x, x);
        // x*x/2 - x + 1 - e
        f = SABR_MUL(sa, SABR_SUB(SABR_ADD(fma(x2, 0.5, -x), 1.0), e));
        // 2*(e-1) + x*(e+1)
        g = SABR_MUL(sb, fma(2.0, SABR_SUB(e, 1.0), SABR_MUL(x, SABR_ADD(e, 1.0))));
    } else {
        // e - (1 - x)
        f = SABR_MUL(sa, SABR_SUB(e, SABR_SUB(1.0, x)));
        // e*e - 8*e + 7 + 2*x*(x-3)
        const double poly = fma(2.0, SABR_MUL(x, SABR_SUB(x, 3.0)), SABR_ADD(fma(-8.0, e, SABR_MUL(e, e)), 7.0));
        g = SABR_MUL(sb, poly);
    }
}

// One functional pair for C chains: when every chain of the thread takes the
// same branch (the rule late in a schedule, when the chains cluster), their
// evaluations share one branch body and interleave (C-fold ILP); mixed
// threads evaluate chain by chain.  Per-chain results do not depend on C.
// The closed forms take their scale factors from sa, sb; the series values
// are multiplied by ca, cb (the chains' constants, case1_series_consts).
template <int PAIR, int C, int STRIDE = 1>
__device__ __forceinline__ void case1_pair_n(const double (&x)[C], const double* __restrict__ ser,
                                             const double2* __restrict__ tab, double (&f)[C], double (&g)[C],
                                             const double (&sa)[C], const double (&sb)[C],
                                             const double (&ca)[C], const double (&cb)[C]) {
    constexpr double kXSwitch = 0.25;  // analytics.cpp:21
    bool all_series = true, all_closed = true;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        all_series &= x[c] < kXSwitch;
        all_closed &= !(x[c] < kXSwitch);
    }
    if (all_series) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            case1_series_pair<PAIR>(x[c], ser, f[c], g[c]);
            f[c] *= ca[c];
            g[c] *= cb[c];
        }
    } else if (all_closed) {
#pragma unroll
        for (int c = 0; c < C; ++c) case1_closed_pair_r<PAIR, STRIDE>(x[c], sa[c], sb[c], tab, f[c], g[c]);
    } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (x[c] < kXSwitch) {
                case1_series_pair<PAIR>(x[c], ser, f[c], g[c]);
                f[c] *= ca[c];
                g[c] *= cb[c];
            } else {
                case1_closed_pair_r<PAIR, STRIDE>(x[c], sa[c], sb[c], tab, f[c], g[c]);
            }
        }
    }
}

// dyn_coeffs_case1 for the factored objectives: the series from shared
// memory (horner_s), the reciprocals as MUFU + Newton (<= 1 ulp from the
// reference's quotients; they scale the cancelling brackets, they are not
// inside them) and exp by table (exp_tab, ~0.5 ulp).  The brackets keep the
// reference's operation order and roundings.
// One vector's four scaled functionals of a slice (dynamic_quad_terms_k):
// sc = the per-slice scale factors and cs = the chain constants of
// case1_scales.
__device__ __forceinline__ void case1_functionals(double a, double b, double T, const double (&sc)[4],
                                                  const double (&cs)[4], const double* __restrict__ ser,
                                                  const double2* __restrict__ tab, double& Af1, double& Ef2,
                                                  double& dg1, double& bg2) {
    const double xb[1] = {SABR_MUL(SABR_MUL(2.0, b), T)};
    const double xab[1] = {SABR_MUL(SABR_ADD(a, b), T)};
    const double s0[1] = {sc[0]}, s1[1] = {sc[1]}, s2[1] = {sc[2]}, s3[1] = {sc[3]};
    const double c0[1] = {cs[0]}, c1[1] = {cs[1]}, c2[1] = {cs[2]}, c3[1] = {cs[3]};
    double F1[1], F2[1], G1[1], G2[1];
    case1_pair_n<0, 1, 1>(xb, ser, tab, F1, F2, s0, s1, c0, c1);
    case1_pair_n<1, 1, 1>(xab, ser, tab, G1, G2, s2, s3, c2, c3);
    Af1 = F1[0];
    Ef2 = F2[0];
    dg1 = G1[0];
    bg2 = G2[0];
}
#endif

// dynamic_implied_vol, analytics.cpp:291-312 (strike-independent part).
SABR_HD SmileTerms dynamic_terms(double nu1_sq, double nu2_sq, double eta1, double eta2_sq,
                                 double alpha, double beta, double pw, double T) {
    const double one_m_beta = 1.0 - beta;
    const double omega = pw * fast_rcp(alpha);
    const double inv_omega = alpha * fast_rcp(pw);
    const double e1w = eta1 * omega;
    SmileTerms t;
    t.a1 = 0.5 * (beta - 1.0) + 0.5 * e1w;
    t.a2 = one_m_beta * one_m_beta * (1.0 / 12.0) + (one_m_beta - e1w) * 0.25 +
           (4.0 * nu1_sq + 3.0 * (eta2_sq - 3.0 * eta1 * eta1)) * omega * omega * (1.0 / 24.0);
    const double b = one_m_beta * one_m_beta * (inv_omega * inv_omega) * (1.0 / 24.0) +
                     beta * eta1 * inv_omega * 0.25 + (2.0 * nu2_sq - 3.0 * eta2_sq) * (1.0 / 24.0);
    t.c0 = 1.0 + b * T;
    t.inv_omega = inv_omega;
    return t;
}

SABR_HD double smile_vol(const SmileTerms& t, double lm, double lm2) {
    return (t.c0 + t.a1 * lm + t.a2 * lm2) * t.inv_omega;
}

// CaseIIParams::rho_at / nu_at, analytics.cpp:138-143.
// p = {alpha,beta,rho0,q_rho,d_rho,nu0,q_nu,d_nu,a,b,horizon}
SABR_HD double case2_rho_at(const double* p, double t) {
    return (p[2] + p[3] * t) * exp(-p[8] * t) + p[4];
}
SABR_HD double case2_nu_at(const double* p, double t) {
    return (p[5] + p[6] * t) * exp(-p[9] * t) + p[7];
}

// CaseIIParams::validate as a predicate (case2_feasible), analytics.cpp:145-175,
// calibration.cpp:161-168: the identical 256-node grid on (0, horizon] plus
// the two stationary points, with the same 1e-9 rho tolerance.
SABR_HD bool case2_feasible(const double* p) {
    const double alpha = p[0], beta = p[1], a = p[8], b = p[9], horizon = p[10];
    if (!(alpha > 0) || !(beta >= 0 && beta <= 1) || !(a >= 0 && b >= 0) || !(horizon > 0))
        return false;
    constexpr double kLo = -1 - 1e-9, kHi = 1 + 1e-9;
    bool ok = true;
    for (int i = 1; i <= 256; ++i) {
        const double t = horizon * i / 256;
        const double r = case2_rho_at(p, t);
        ok = ok && !(r < kLo || r > kHi) && !(case2_nu_at(p, t) <= 0);
    }
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
    return ok;
}

// case2_feasible by one warp: the 256 grid nodes split over the lanes (8
// each), lane 0 adds the scalar checks and the two stationary points; the
// verdict is the AND over the warp (order-free, so identical to the serial
// predicate).  Every lane must pass the same p.
SABR_D bool case2_feasible_warp(const double* p) {
    const int lane = threadIdx.x & 31;
    const double alpha = p[0], beta = p[1], a = p[8], b = p[9], horizon = p[10];
    constexpr double kLo = -1 - 1e-9, kHi = 1 + 1e-9;
    bool ok = (alpha > 0) && (beta >= 0 && beta <= 1) && (a >= 0 && b >= 0) && (horizon > 0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = 1 + lane + 32 * j;
        const double t = horizon * i / 256;
        const double r = case2_rho_at(p, t);
        ok = ok && !(r < kLo || r > kHi) && !(case2_nu_at(p, t) <= 0);
    }
    if (lane == 0) {
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
    return __all_sync(0xffffffffu, ok);
}

// ------------------------------------------------------ level merge rule ---

// (value, global chain index) lexicographic order: strict '<' on the value
// with the lowest chain winning ties reproduces the sequential scans of
// proj/src/annealer.cpp:141-159 for any split of the chains.
SABR_HD bool lex_less(double v, int64_t i, double w, int64_t j) {
    return v < w || (v == w && i < j);
}

// One level's cross-rank merge (annealer.cpp:141-160) applied to the state;
// identical on host (CPU tests, sabr_merge_level_records) and device.
SABR_HD void merge_level(sabr_sa_state* st, const sabr_level_record* rec, int64_t nranks,
                         int64_t n_chains, int64_t max_evals, int64_t levels_total, int dim,
                         double* trace_f) {
    int64_t e = -1, b = -1, evals = 0;
    for (int64_t r = 0; r < nranks; ++r) {
        if (rec[r].end_chain >= 0 &&
            (e < 0 || lex_less(rec[r].end_value, rec[r].end_chain, rec[e].end_value, rec[e].end_chain)))
            e = r;
        if (rec[r].best_chain >= 0 &&
            (b < 0 ||
             lex_less(rec[r].best_value, rec[r].best_chain, rec[b].best_value, rec[b].best_chain)))
            b = r;
        evals += rec[r].evals;
    }
    if (e >= 0 && rec[e].end_value < st->incumbent_value) {
        st->incumbent_value = rec[e].end_value;
        for (int i = 0; i < dim; ++i) st->incumbent[i] = rec[e].end_point[i];
    }
    if (b >= 0 && rec[b].best_value < st->best_value) {
        st->best_value = rec[b].best_value;
        for (int i = 0; i < dim; ++i) st->best[i] = rec[b].best_point[i];
    }
    st->evals += evals;
    if (trace_f) *trace_f = st->incumbent_value;
    st->levels_run += 1;
    if (st->levels_run >= levels_total || st->evals >= max_evals) {
        st->done = 1;
    } else {
        const int64_t remaining = max_evals - st->evals;
        st->eval_cap = (remaining + n_chains - 1) / n_chains;
    }
}

}  // namespace sabr_dev
