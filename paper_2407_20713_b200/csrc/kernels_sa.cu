// kernels_sa.cu — synchronous parallel simulated annealing on sm_100a.
//
// One thread = one Markov chain (proj/src/annealer.cpp:107-139).  A launch
// runs one temperature level for all of this rank's chains: chain state
// (point, value, best point, xoshiro256++ state) lives in registers, the
// market grid of the objective is staged once per CTA into shared memory, and
// the level-end reductions of annealer.cpp:141-159 (per-group endpoint
// minimum, best-ever, eval count) are a deterministic (value, chain-index)
// arg-min done in-kernel: warp shuffles, then one CTA record, then the last
// CTA to finish (ticket) reduces the CTA records and - on a single rank -
// applies the merge to the device-resident annealer state.  The host never
// synchronises inside the level loop.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <math_constants.h>

#include "device_common.cuh"
#include "kernels.hpp"
#include "pdl.cuh"
#include "slice_qr.hpp"

namespace sabr_gpu {

using namespace sabr_dev;

namespace {

constexpr int kThreads = 128;
constexpr size_t kSmemStageLimit = 96 * 1024;

// Thread-per-chain level kernel: 64-thread CTAs, 11 per SM (22 warps, <= 88
// registers).  1e5 chains = 1563 CTAs fit one wave on 148 SMs with at most
// 22 warps per SM (128-thread CTAs: 6 per SM, 24 warps on the busiest SMs
// and only 80 registers).
constexpr int kLevelThreads = 64;
constexpr int kLevelMinCtas = 11;

// Per-quote market data as one 32-byte record (two LDS.128 per quote).
struct __align__(16) Quote {
    double lm, lm2, mkt, inv_mkt;
};

struct Grid {
    int ns;
    const double* T;
    const double* lnf_hi;
    const double* lnf_lo;
    const int32_t* qoff;
    const Quote* q;
    const double2* tab;  // exp_tab table in shared memory
};

// Every kernel stages the 2 KB exp table into shared memory (stage_exp +
// __syncthreads) before the first exp_tab.
__device__ __forceinline__ void stage_exp(const SurfaceView& sv, double2* tab_s) {
    for (int i = threadIdx.x; i < kExpTableSize; i += blockDim.x) tab_s[i] = sv.exptab[i];
}

__host__ __device__ inline size_t stage_bytes(int ns, int nq) {
    return static_cast<size_t>(nq) * sizeof(Quote) + 3 * sizeof(double) * ns +
           sizeof(int32_t) * (ns + 1) + 16;
}

// Cooperative copy of the market grid into shared memory ("staged once").
// SMEM is a compile-time choice so the quote reads compile to LDS (a runtime
// smem/global choice would force generic LD + 64-bit address arithmetic).
template <bool SMEM>
__device__ Grid stage_grid(const SurfaceView& sv, unsigned char* smem) {
    Grid g;
    g.ns = sv.n_slices;
    if constexpr (!SMEM) {  // grid too large for shared memory: read through L1
        g.T = sv.T;
        g.lnf_hi = sv.lnf_hi;
        g.lnf_lo = sv.lnf_lo;
        g.qoff = sv.qoff;
        g.q = reinterpret_cast<const Quote*>(sv.quotes);
        return g;
    }
    Quote* q = reinterpret_cast<Quote*>(smem);
    double* d = reinterpret_cast<double*>(q + sv.n_quotes);
    int32_t* o = reinterpret_cast<int32_t*>(d + 3 * sv.n_slices);
    const Quote* src = reinterpret_cast<const Quote*>(sv.quotes);
    for (int i = threadIdx.x; i < sv.n_quotes; i += blockDim.x) q[i] = src[i];
    for (int i = threadIdx.x; i < sv.n_slices; i += blockDim.x) {
        d[i] = sv.T[i];
        d[sv.n_slices + i] = sv.lnf_hi[i];
        d[2 * sv.n_slices + i] = sv.lnf_lo[i];
    }
    for (int i = threadIdx.x; i <= sv.n_slices; i += blockDim.x) o[i] = sv.qoff[i];
    __syncthreads();
    g.q = q;
    g.T = d;
    g.lnf_hi = d + sv.n_slices;
    g.lnf_lo = d + 2 * sv.n_slices;
    g.qoff = o;
    return g;
}

// f^(1-beta) = exp((1-beta) ln f) with ln f carried in double-double, so the
// result is as accurate as a correctly rounded exp (pow in analytics.cpp:191).
// SAT = false: |(1-beta) ln f| <= 700 is guaranteed by the host (FAST kernels).
template <bool SAT = true, int STRIDE = 1>
__device__ __forceinline__ double pow_fwd(double omb, double lnf_hi, double lnf_lo,
                                          const double2* tab) {
    const double y = omb * lnf_hi;
    const double err = fma(omb, lnf_hi, -y) + omb * lnf_lo;
    const double e = SAT ? exp_tab<STRIDE>(y, tab) : exp_tab_unsat<STRIDE>(y, tab);
    return fma(e, err, e);
}

__device__ __forceinline__ double quote_rel(const SmileTerms& t, const Quote& qq) {
    const double sigma = smile_vol(t, qq.lm, qq.lm2);
    return (qq.mkt - sigma) * qq.inv_mkt;
}

// Sum of squared relative errors over one slice, calibration.cpp:253-267.
// Four interleaved partial sums (quotes j mod 4) break the serial FMA chain
// of the reference's left-to-right sum: the dependency latency of a single
// accumulator was the kernel's top stall; the reassociation moves the result
// by ~1 ulp of the cost.
__device__ __forceinline__ double slice_cost(const SmileTerms& t, const Quote* q, int q0,
                                             int q1) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = q0;
    for (; j + 4 <= q1; j += 4) {
        const double r0 = quote_rel(t, q[j]), r1 = quote_rel(t, q[j + 1]);
        const double r2 = quote_rel(t, q[j + 2]), r3 = quote_rel(t, q[j + 3]);
        s0 = fma(r0, r0, s0);
        s1 = fma(r1, r1, s1);
        s2 = fma(r2, r2, s2);
        s3 = fma(r3, r3, s3);
    }
    for (; j < q1; ++j) {
        const double r = quote_rel(t, q[j]);
        s0 = fma(r, r, s0);
    }
    return (s0 + s1) + (s2 + s3);
}

// Objective of calibrate_static_T1: full vector {alpha, beta, nu, rho} on the
// (single) slice of the view.  calibration.cpp:300-306, analytics.cpp:183-205.
__device__ __forceinline__ double static_cost(const double* v, const Grid& g) {
    const double pw = pow_fwd(1.0 - v[1], g.lnf_hi[0], g.lnf_lo[0], g.tab);
    const SmileTerms t = static_terms(v[0], v[1], v[2], v[3], pw, g.T[0]);
    return slice_cost(t, g.q, g.qoff[0], g.qoff[1]);
}

// Objective of calibrate_dynamic_case1_T1: {alpha,beta,rho0,nu0,a,b} summed
// over slices in order.  calibration.cpp:339-349, analytics.cpp:207-215, :291-312.
__device__ __forceinline__ double case1_cost(const double* v, const Grid& g) {
    double sum = 0.0;
    const double omb = 1.0 - v[1];
    for (int i = 0; i < g.ns; ++i) {
        const double T = g.T[i];
        double n1, n2, e1, e2;
        dyn_coeffs_case1(v[2], v[3], v[4], v[5], T, n1, n2, e1, e2);
        const double pw = pow_fwd(omb, g.lnf_hi[i], g.lnf_lo[i], g.tab);
        const SmileTerms t = dynamic_terms(n1, n2, e1, e2, v[0], v[1], pw, T);
        sum += slice_cost(t, g.q, g.qoff[i], g.qoff[i + 1]);
    }
    return sum;
}

// ------------------------------------ padded quad grid (shared memory) ---
// The objectives of the SA level kernel and the cost batch read the market
// grid from shared memory as quad records: quotes 4k..4k+3 of a slice are
// one 96-byte record {ln(K/f)[4], ln^2(K/f)[4], 1/market[4]}, each slice
// padded to whole quads, so one quad is six LDS.128 at immediate offsets of
// one base pointer and the per-quote work is four FP64 instructions:
//     s = C0 + A1*lm + A2*lm2   (C0, A1, A2 = c0, a1, a2 times 1/omega)
//     r = 1 - s*(1/market)      (= (market - sigma)/market, calibration.cpp:262)
//     acc += r*r
// The last, partial quad of a slice is evaluated on the zero padding and its
// padding lanes are discarded (predicated accumulate), so the padding never
// enters a sum.  One extra zero quad ends the grid: the quad loop prefetches
// the record after the one it computes.
struct QuadRec {
    double2 lm01, lm23, sq01, sq23, inv01, inv23;
};

struct PGrid {
    int ns;
    const double* T;
    const double* lnf_hi;
    const double* lnf_lo;
    const int32_t* p0;  // [ns] first quad of slice s
    const int32_t* nq;  // [ns] quotes of slice s
    const QuadRec* rec;
    const double2* tab;
};

__host__ __device__ inline int grid_quads(int ns, int nq) { return (nq + 3 * ns + 3) / 4 + 1; }

__host__ __device__ inline size_t pstage_bytes(int ns, int nq) {
    return sizeof(QuadRec) * grid_quads(ns, nq) + 3 * sizeof(double) * ns + 2 * sizeof(int32_t) * ns + 16;
}

__device__ PGrid stage_pgrid(const SurfaceView& sv, unsigned char* smem) {
    const int ns = sv.n_slices, nqd = grid_quads(ns, sv.n_quotes);
    QuadRec* rec = reinterpret_cast<QuadRec*>(smem);
    double* d = reinterpret_cast<double*>(rec + nqd);
    int32_t* p0 = reinterpret_cast<int32_t*>(d + 3 * ns);
    int32_t* nq = p0 + ns;
    double* flat = reinterpret_cast<double*>(rec);
    const Quote* src = reinterpret_cast<const Quote*>(sv.quotes);
    int p = 0;  // quad index
    for (int s = 0; s < ns; ++s) {
        const int q0 = sv.qoff[s], n = sv.qoff[s + 1] - q0, n4 = (n + 3) & ~3;
        for (int k = threadIdx.x; k < n4; k += blockDim.x) {
            const bool real = k < n;
            const Quote q = real ? src[q0 + k] : Quote{0.0, 0.0, 0.0, 0.0};
            double* r = flat + 12 * (p + (k >> 2)) + (k & 3);
            r[0] = q.lm;
            r[4] = q.lm2;
            r[8] = q.inv_mkt;
        }
        if (threadIdx.x == 0) {
            p0[s] = p;
            nq[s] = n;
            d[s] = sv.T[s];
            d[ns + s] = sv.lnf_hi[s];
            d[2 * ns + s] = sv.lnf_lo[s];
        }
        p += n4 >> 2;
    }
    for (int k = threadIdx.x; k < 12 * (nqd - p); k += blockDim.x) flat[12 * p + k] = 0.0;
    __syncthreads();
    PGrid g;
    g.ns = ns;
    g.T = d;
    g.lnf_hi = d + ns;
    g.lnf_lo = d + 2 * ns;
    g.p0 = p0;
    g.nq = nq;
    g.rec = rec;
    g.tab = nullptr;
    return g;
}

struct QuadTerms {
    double c0, a1, a2;
};

__device__ __forceinline__ QuadTerms quad_terms(const SmileTerms& t) {
    return QuadTerms{t.c0 * t.inv_omega, t.a1 * t.inv_omega, t.a2 * t.inv_omega};
}

__device__ __forceinline__ double quad_rel(const QuadTerms& t, double lm, double lm2, double inv) {
    return fma(-fma(t.a2, lm2, fma(t.a1, lm, t.c0)), inv, 1.0);
}

// Sum of squared relative errors over one slice (calibration.cpp:253-267) for
// C candidates at once: one set of quote loads feeds all C.  Four partial
// sums per candidate by quote index mod 4: the dependency latency of a single
// accumulator was the kernel's top stall; the reassociation moves the result
// by ~1 ulp of the cost.  Each candidate's arithmetic and summation order do
// not depend on C (the one- and two-chain kernels produce identical values).
// The next quad's record is loaded while the current one is computed.
template <int C>
__device__ __forceinline__ void quad_cost_n(const QuadTerms (&t)[C], const QuadRec* __restrict__ r,
                                            int n, double (&out)[C]) {
    double acc[C][4];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.0;
    QuadRec cur = r[0];
    const int full = n >> 2;
#pragma unroll 1
    for (int k = 0; k < full; ++k) {
        const QuadRec nxt = r[k + 1];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const double r0 = quad_rel(t[c], cur.lm01.x, cur.sq01.x, cur.inv01.x);
            const double r1 = quad_rel(t[c], cur.lm01.y, cur.sq01.y, cur.inv01.y);
            const double r2 = quad_rel(t[c], cur.lm23.x, cur.sq23.x, cur.inv23.x);
            const double r3 = quad_rel(t[c], cur.lm23.y, cur.sq23.y, cur.inv23.y);
            acc[c][0] = fma(r0, r0, acc[c][0]);
            acc[c][1] = fma(r1, r1, acc[c][1]);
            acc[c][2] = fma(r2, r2, acc[c][2]);
            acc[c][3] = fma(r3, r3, acc[c][3]);
        }
        cur = nxt;
    }
    const int rem = n & 3;
    if (rem) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const double r0 = quad_rel(t[c], cur.lm01.x, cur.sq01.x, cur.inv01.x);
            const double r1 = quad_rel(t[c], cur.lm01.y, cur.sq01.y, cur.inv01.y);
            const double r2 = quad_rel(t[c], cur.lm23.x, cur.sq23.x, cur.inv23.x);
            acc[c][0] = fma(r0, r0, acc[c][0]);
            if (rem > 1) acc[c][1] = fma(r1, r1, acc[c][1]);
            if (rem > 2) acc[c][2] = fma(r2, r2, acc[c][2]);
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = (acc[c][0] + acc[c][1]) + (acc[c][2] + acc[c][3]);
}

__device__ __forceinline__ double pslice_cost(const SmileTerms& st, const PGrid& g, int s) {
    const QuadTerms t[1] = {quad_terms(st)};
    double out[1];
    quad_cost_n<1>(t, g.rec + g.p0[s], g.nq[s], out);
    return out[0];
}

__device__ __forceinline__ double static_cost(const double* v, const PGrid& g) {
    const double pw = pow_fwd(1.0 - v[1], g.lnf_hi[0], g.lnf_lo[0], g.tab);
    const SmileTerms t = static_terms(v[0], v[1], v[2], v[3], pw, g.T[0]);
    return pslice_cost(t, g, 0);
}

__device__ __forceinline__ double case1_cost(const double* v, const PGrid& g) {
    double sum = 0.0;
    const double omb = 1.0 - v[1];
    for (int i = 0; i < g.ns; ++i) {
        const double T = g.T[i];
        double n1, n2, e1, e2;
        dyn_coeffs_case1(v[2], v[3], v[4], v[5], T, n1, n2, e1, e2);
        const double pw = pow_fwd(omb, g.lnf_hi[i], g.lnf_lo[i], g.tab);
        const SmileTerms t = dynamic_terms(n1, n2, e1, e2, v[0], v[1], pw, T);
        sum += pslice_cost(t, g, i);
    }
    return sum;
}

// ------------------------------------- C chains per thread (shared loads) ---
// The single slice of a static objective, hoisted into registers for the
// whole chain loop.
struct StaticSlice {
    double lnf_hi, lnf_lo, T;
    const QuadRec* rec;
    int nq;
};

__device__ __forceinline__ StaticSlice static_slice(const PGrid& g) {
    return StaticSlice{g.lnf_hi[0], g.lnf_lo[0], g.T[0], g.rec + g.p0[0], g.nq[0]};
}

template <int C, int DIMF, bool FAST, int STRIDE = 1>
__device__ __forceinline__ void static_cost_n(const double (&v)[C][DIMF], const StaticSlice& sl,
                                              const double2* tab, double (&out)[C]) {
    QuadTerms t[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const double pw = pow_fwd<!FAST, STRIDE>(1.0 - v[c][1], sl.lnf_hi, sl.lnf_lo, tab);
        t[c] = quad_terms(static_terms(v[c][0], v[c][1], v[c][2], v[c][3], pw, sl.T));
    }
    quad_cost_n<C>(t, sl.rec, sl.nq, out);
}

template <int C, int DIMF>
__device__ __forceinline__ void case1_cost_n(const double (&v)[C][DIMF], const PGrid& g,
                                             double (&out)[C]) {
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = 0.0;
    for (int i = 0; i < g.ns; ++i) {
        const double T = g.T[i];
        QuadTerms t[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double n1, n2, e1, e2;
            dyn_coeffs_case1(v[c][2], v[c][3], v[c][4], v[c][5], T, n1, n2, e1, e2);
            const double pw = pow_fwd(1.0 - v[c][1], g.lnf_hi[i], g.lnf_lo[i], g.tab);
            t[c] = quad_terms(dynamic_terms(n1, n2, e1, e2, v[c][0], v[c][1], pw, T));
        }
        double s[C];
        quad_cost_n<C>(t, g.rec + g.p0[i], g.nq[i], s);
#pragma unroll
        for (int c = 0; c < C; ++c) out[c] += s[c];
    }
}

// ------------------------------------------- factored slice cost (QR) ---
// The default objective of the SA and cost kernels (slice_qr.hpp): a slice's
// sum of squared relative errors is ||R (C0, A1, A2, -1)||^2 with the slice's
// 4x4 factor R, computed on the host in binary128.  Nine FP64 instructions per
// slice replace the four per quote; the grid a CTA stages is kQrStride + 3
// doubles per slice.
struct QGrid {
    int ns;
    const double* T;
    const double* lnf_hi;
    const double* lnf_lo;
    const double* R;    // [ns][kQrStride], 16-byte aligned
    const double* ser;  // [4][kSeriesStride] Case I series tables (horner_s)
    const double2* tab;
    const double* iT;   // [4][ns] 1/T^2, 1/T^3, 1/T^4 and 1/T (Case I: the closed forms'
                        // scale factors 6/(2bT)^3 = 6/(2b)^3 * 1/T^3, ..., case1_cost_n)
};

__host__ __device__ inline size_t qstage_bytes(int ns) {
    return sizeof(double) * (4 * kSeriesStride + static_cast<size_t>(kQrStride + 7) * ns);
}

__device__ QGrid stage_qgrid(const SurfaceView& sv, unsigned char* smem) {
    const int ns = sv.n_slices;
    double* ser = reinterpret_cast<double*>(smem);
    double* R = ser + 4 * kSeriesStride;
    double* d = R + kQrStride * ns;
    for (int k = threadIdx.x; k < 4 * kSeriesStride; k += blockDim.x) ser[k] = kCase1Series[k];
    for (int k = threadIdx.x; k < kQrStride * ns; k += blockDim.x) R[k] = sv.qr[k];
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        d[i] = sv.T[i];
        d[ns + i] = sv.lnf_hi[i];
        d[2 * ns + i] = sv.lnf_lo[i];
        const double it = 1.0 / sv.T[i], it2 = it * it;
        d[3 * ns + i] = it2;
        d[4 * ns + i] = it2 * it;
        d[5 * ns + i] = it2 * it2;
        d[6 * ns + i] = it;
    }
    __syncthreads();
    QGrid g;
    g.ns = ns;
    g.R = R;
    g.ser = ser;
    g.T = d;
    g.lnf_hi = d + ns;
    g.lnf_lo = d + 2 * ns;
    g.iT = d + 3 * ns;
    g.tab = nullptr;
    return g;
}

// One slice's factor in registers (the static objective's only slice).
struct QrFactor {
    double r00, r01, r02, r03, r11, r12, r13, r22, r23, r33sq;
};

__device__ __forceinline__ QrFactor load_qr(const double* R) {
    const double2* p = reinterpret_cast<const double2*>(R);
    const double2 a = p[0], b = p[1], c = p[2], d = p[3], e = p[4];
    return QrFactor{a.x, a.y, b.x, b.y, c.x, c.y, d.x, d.y, e.x, e.y};
}

__device__ __forceinline__ double qr_cost(const QuadTerms& t, const QrFactor& f) {
    const double u0 = fma(f.r02, t.a2, fma(f.r01, t.a1, fma(f.r00, t.c0, -f.r03)));
    const double u1 = fma(f.r12, t.a2, fma(f.r11, t.a1, -f.r13));
    const double u2 = fma(f.r22, t.a2, -f.r23);
    return fma(u0, u0, fma(u1, u1, fma(u2, u2, f.r33sq)));
}

struct QrSlice {  // the static objective's slice, hoisted into registers
    double lnf_hi, lnf_lo, T24, T4;  // T/24, T/4
    QrFactor f;                      // R with columns 1, 2 scaled by -1/2, 1/12 (static_qterms_f)
};

// The static slice with the constants of the static terms folded in (r02):
// A1/omega = -p/2 and A2/omega = X/12 enter ||R v||^2 through R's columns 1
// and 2 (scaled once per CTA: -1/2 exactly, 1/12 within an ulp), and B T
// is formed directly with T/24 and T/4: three FP64 instructions fewer per eval.
__device__ __forceinline__ QrSlice qr_slice(const QGrid& g) {
    QrFactor f = load_qr(g.R);
    f.r01 *= -0.5;
    f.r11 *= -0.5;
    f.r02 *= (1.0 / 12.0);
    f.r12 *= (1.0 / 12.0);
    f.r22 *= (1.0 / 12.0);
    const double T = g.T[0];
    return QrSlice{g.lnf_hi[0], g.lnf_lo[0], T * (1.0 / 24.0), T * 0.25, f};
}

// The static terms (device_common.cuh: the factored cost's terms) on the
// folded slice: (C0, p, X) for qr_cost on the folded factor
__device__ __forceinline__ QuadTerms static_qterms_f(const double* v, double pw, const QrSlice& sl) {
    const double alpha = v[0], beta = v[1], nu = v[2], rho = v[3];  // the static vector (alpha, beta, nu, rho)
    const double omb = 1.0 - beta;
    const double r = fast_rcp(alpha * pw);
    const double inv = alpha * (alpha * r);  // 1/omega
    const double omega = pw * (pw * r);
    const double rn = rho * nu;
    const double q = omb * inv;
    const double p = q - rn;
    const double rrn2 = fma(-3.0 * rho, rho, 2.0) * (nu * nu);
    QuadTerms t;
    t.a1 = p;
    t.a2 = fma(rrn2, omega, fma(3.0, p, omb * q));
    const double BT = fma(q * sl.T24, q, fma((sl.T4 * beta) * rn, inv, rrn2 * sl.T24));
    t.c0 = fma(inv, BT, inv);
    return t;
}

__device__ __forceinline__ double static_cost(const double* v, const QGrid& g) {
    const QrSlice sl = qr_slice(g);
    const double pw = pow_fwd(1.0 - v[1], sl.lnf_hi, sl.lnf_lo, g.tab);
    return qr_cost(static_qterms_f(v, pw, sl), sl.f);
}

// Per-vector constants of the Case I closed forms' scale factors (r02): with
// the CTA's 1/T^3, 1/T^2, 1/T^4 per slice, P1/T^3 = nu0^2/6 * 6/x^3 (x = 2bT),
// Q1/T^2 = nu0 rho0/4 * 2/x^2 and Q2/T^4 = (nu0 rho0)^2/8 * 3/x^4 (x = (a+b)T)
// within a few ulp: the closed forms then yield the scaled functionals of
// dynamic_quad_terms_k.  Only the closed-form branch (x >= 0.25, so b > 0 and
// a + b > 0) uses them.
__device__ __forceinline__ void case1_scales(double nu0, double rho0, double a, double b, double& P1, double& Q1,
                                             double& Q2) {
    const double rb = fast_rcp(SABR_MUL(2.0, b)), rab = fast_rcp(SABR_ADD(a, b));
    const double nr = nu0 * rho0, rab2 = rab * rab;
    P1 = (nu0 * nu0) * (rb * (rb * rb));
    Q1 = (0.5 * nr) * rab2;
    Q2 = (0.375 * (nr * nr)) * (rab2 * rab2);
}
// the series branch's constants: nu0^2/6, nu0^2/12, nu0 rho0/4, (nu0 rho0)^2/8
__device__ __forceinline__ void case1_series_consts(double nu0, double rho0, double (&c)[4]) {
    const double nn = nu0 * nu0, nr = nu0 * rho0;
    c[0] = nn * (1.0 / 6.0);
    c[1] = 0.5 * c[0];
    c[2] = 0.25 * nr;
    c[3] = 0.125 * (nr * nr);
}
// the four scale factors of slice i (g.iT: 1/T^2, 1/T^3, 1/T^4 blocks)
__device__ __forceinline__ void case1_slice_scales(double P1, double Q1, double Q2, double iT2, double iT3,
                                                   double iT4, double (&sc)[4]) {
    sc[0] = P1 * iT3;
    sc[1] = 0.5 * sc[0];
    sc[2] = Q1 * iT2;
    sc[3] = Q2 * iT4;
}

// The Case I objective of one vector (case1_cost_n's arithmetic, bit for bit).
__device__ __forceinline__ double case1_cost(const double* v, const QGrid& g) {
    double sum = 0.0;
    const double omb = 1.0 - v[1];
    double P1, Q1, Q2, cs[4];
    case1_scales(v[3], v[2], v[4], v[5], P1, Q1, Q2);
    case1_series_consts(v[3], v[2], cs);
    const double ia = fast_rcp(v[0]);
    for (int i = 0; i < g.ns; ++i) {
        const double T = g.T[i];
        double sc[4], Af1, Ef2, dg1, bg2;
        case1_slice_scales(P1, Q1, Q2, g.iT[i], g.iT[g.ns + i], g.iT[2 * g.ns + i], sc);
        case1_functionals(v[4], v[5], T, sc, cs, g.ser, g.tab, Af1, Ef2, dg1, bg2);
        const double pw = pow_fwd(omb, g.lnf_hi[i], g.lnf_lo[i], g.tab);
        QuadTerms t;
        dynamic_quad_terms_k(Af1, Ef2, dg1, bg2, v[1], v[0] * fast_rcp(pw), pw * ia, T, t.c0, t.a1, t.a2);
        sum += qr_cost(t, load_qr(g.R + kQrStride * i));
    }
    return sum;
}


template <int C, int DIMF, bool FAST, int STRIDE = 1>
__device__ __forceinline__ void static_cost_n(const double (&v)[C][DIMF], const QrSlice& sl,
                                              const double2* tab, double (&out)[C]) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const double pw = pow_fwd<!FAST, STRIDE>(1.0 - v[c][1], sl.lnf_hi, sl.lnf_lo, tab);
        out[c] = qr_cost(static_qterms_f(v[c], pw, sl), sl.f);
    }
}

// pw_fixed: when beta is not searched, f_i^(1-beta) per slice, computed once
// per CTA with the same pow_fwd (so the values are the ones each chain would
// compute); nullptr when beta is free.
// slices whose f^(1-beta) a CTA keeps when beta is not searched (pw_fixed)
constexpr int kMaxPwSlices = 64;

// BETA1: beta is held at exactly 1 (C3), f^(1-beta) = 1 (dynamic_quad_terms_b1).
template <int C, int DIMF, int STRIDE = 1, bool BETA1 = false>
__device__ __forceinline__ void case1_cost_n(const double (&v)[C][DIMF], const QGrid& g,
                                             double (&out)[C], const double* pw_fixed = nullptr,
                                             const double2* tab = nullptr) {
    if (STRIDE == 1) tab = g.tab;
    // Reciprocals shared by the slices (r02): the closed forms scale their
    // brackets by 6/x^3 (x = 2bT), 2/x^2 and 3/x^4 (x = (a+b)T); with
    // 1/x = 1/(2b) * 1/T and 1/((a+b)T) = 1/(a+b) * 1/T (1/T staged per CTA)
    // two reciprocals per chain replace three per slice.  1/omega =
    // alpha * rcp(f^(1-beta)) and omega = f^(1-beta) * rcp(alpha): one
    // reciprocal of alpha per chain, and with beta fixed the CTA's
    // rcp(f^(1-beta)) per slice.  Each factor is within a few ulp of the
    // per-slice quotient; it scales a cancelling bracket, it is not inside
    // one (the brackets keep the reference's operations, analytics.cpp:47-67).
    // per chain, slice-independent: 2b, a+b, the scale-factor constants
    // (case1_scales) and rcp(alpha)
    double b2[C], ab[C], P1[C], Q1[C], Q2[C], ia[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        b2[c] = SABR_MUL(2.0, v[c][5]);
        ab[c] = SABR_ADD(v[c][4], v[c][5]);
        case1_scales(v[c][3], v[c][2], v[c][4], v[c][5], P1[c], Q1[c], Q2[c]);
        ia[c] = fast_rcp(v[c][0]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = 0.0;
    for (int i = 0; i < g.ns; ++i) {
        const double T = g.T[i], iT2 = g.iT[i], iT3 = g.iT[g.ns + i], iT4 = g.iT[2 * g.ns + i];
        const QrFactor f = load_qr(g.R + kQrStride * i);
        // dyn_coeffs_case1_fast for the C chains, branch bodies shared
        double xb[C], xab[C], sa0[C], sb0[C], sa1[C], sb1[C], f1[C], f2[C], g1[C], g2[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            xb[c] = SABR_MUL(b2[c], T);
            xab[c] = SABR_MUL(ab[c], T);
            double sc[4];
            case1_slice_scales(P1[c], Q1[c], Q2[c], iT2, iT3, iT4, sc);
            sa0[c] = sc[0];
            sb0[c] = sc[1];
            sa1[c] = sc[2];
            sb1[c] = sc[3];
        }
        // both functional pairs of every chain in the closed-form regime (the
        // rule on C3's surfaces): one straight-line block, 2C independent
        // dependency chains (ILP) instead of two branch regions of C
        bool all_closed = true;
#pragma unroll
        for (int c = 0; c < C; ++c) all_closed &= !(xb[c] < 0.25) & !(xab[c] < 0.25);
        if (all_closed) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                case1_closed_pair_r<0, STRIDE>(xb[c], sa0[c], sb0[c], tab, f1[c], f2[c]);
                case1_closed_pair_r<1, STRIDE>(xab[c], sa1[c], sb1[c], tab, g1[c], g2[c]);
            }
        } else {
            double ca0[C], cb0[C], ca1[C], cb1[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                double cs[4];
                case1_series_consts(v[c][3], v[c][2], cs);
                ca0[c] = cs[0];
                cb0[c] = cs[1];
                ca1[c] = cs[2];
                cb1[c] = cs[3];
            }
            case1_pair_n<0, C, STRIDE>(xb, g.ser, tab, f1, f2, sa0, sb0, ca0, cb0);
            case1_pair_n<1, C, STRIDE>(xab, g.ser, tab, g1, g2, sa1, sb1, ca1, cb1);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            QuadTerms t;
            if constexpr (BETA1) {
                dynamic_quad_terms_b1(f1[c], f2[c], g1[c], g2[c], v[c][0], ia[c], T, t.c0, t.a1, t.a2);
            } else {
                double pw, ipw;
                if (pw_fixed) {
                    pw = pw_fixed[i];
                    ipw = pw_fixed[kMaxPwSlices + i];
                } else {
                    pw = pow_fwd<true, STRIDE>(1.0 - v[c][1], g.lnf_hi[i], g.lnf_lo[i], tab);
                    ipw = fast_rcp(pw);
                }
                dynamic_quad_terms_k(f1[c], f2[c], g1[c], g2[c], v[c][1], v[c][0] * ipw, pw * ia[c], T, t.c0, t.a1,
                                     t.a2);
            }
            out[c] += qr_cost(t, f);
        }
    }
}

// Objective grid of the SA / cost kernels (GK): kGridQR the factored slices
// (default), kGridQuads the padded per-quote grid in shared memory
// (SABR_SA_COST=quotes), kGridL1 the AoS per-quote grid read through L1 (a
// per-quote grid too large for shared memory).
constexpr int kGridL1 = 0;
constexpr int kGridQuads = 1;
constexpr int kGridQR = 2;

template <int GK>
using ObjGrid = std::conditional_t<GK == kGridQR, QGrid, std::conditional_t<GK == kGridQuads, PGrid, Grid>>;

template <int GK>
__device__ __forceinline__ ObjGrid<GK> stage_obj(const SurfaceView& sv, unsigned char* smem) {
    if constexpr (GK == kGridQR) return stage_qgrid(sv, smem);
    else if constexpr (GK == kGridQuads) return stage_pgrid(sv, smem);
    else return stage_grid<false>(sv, smem);
}

__device__ __forceinline__ double sq(double x) { return x * x; }

// The closed-form objectives of proj/tests/test_annealer.cpp.
__device__ double builtin_value(int id, const double* x) {
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
        case SABR_OBJ_NANRIGHT1: return x[0] > 0.5 ? CUDART_NAN : sq(x[0] + 1.0);
    }
    return CUDART_NAN;
}

template <int KIND, class G>
__device__ __forceinline__ double objective(const double* v, const G& g, int builtin) {
    if constexpr (KIND == OBJ_STATIC) return static_cost(v, g);
    else if constexpr (KIND == OBJ_CASE1) return case1_cost(v, g);
    else return builtin_value(builtin, v);
}

// SearchSpace::is_feasible minus contains() (a clamped proposal is always in
// the box): the optional predicate (test_annealer.cpp:108-121).
__device__ __forceinline__ bool predicate_ok(int pred, const double* y) {
    if (pred == SABR_PRED_SUM_LE_1) return y[0] + y[1] <= 1.0;
    return true;
}

// ------------------------------------------------------- reductions ---
struct ArgMin {
    double v;
    int64_t i;
    int32_t blk;
};

__device__ __forceinline__ void argmin_combine(ArgMin& a, const ArgMin& b) {
    if (lex_less(b.v, b.i, a.v, a.i)) a = b;
}

__device__ __forceinline__ ArgMin warp_argmin(ArgMin a) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        ArgMin o;
        o.v = __shfl_down_sync(0xffffffffu, a.v, off);
        o.i = __shfl_down_sync(0xffffffffu, a.i, off);
        o.blk = __shfl_down_sync(0xffffffffu, a.blk, off);
        argmin_combine(a, o);
    }
    return a;
}

__device__ __forceinline__ long long warp_sum(long long x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    return x;
}

template <int NT>
struct RedShared {
    static constexpr int kW = NT / 32;
    ArgMin e[kW], b[kW];
    long long n[kW];
    ArgMin e_win, b_win;
    long long n_tot;
    int is_last;
};

// Block-wide (endpoint, best) arg-min and eval sum; result valid in `rs`
// after the call for all threads.
template <int NT>
__device__ void block_reduce(RedShared<NT>& rs, ArgMin e, ArgMin b, long long n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    e = warp_argmin(e);
    b = warp_argmin(b);
    n = warp_sum(n);
    if (lane == 0) {
        rs.e[warp] = e;
        rs.b[warp] = b;
        rs.n[warp] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ArgMin ee = rs.e[0], bb = rs.b[0];
        long long nn = rs.n[0];
        for (int w = 1; w < RedShared<NT>::kW; ++w) {
            argmin_combine(ee, rs.e[w]);
            argmin_combine(bb, rs.b[w]);
            nn += rs.n[w];
        }
        rs.e_win = ee;
        rs.b_win = bb;
        rs.n_tot = nn;
    }
    __syncthreads();
}

// One CTA record of the level-end reduction: written by thread 0, then the
// ticket; returns true (all threads) in the last CTA of the grid.
template <int NT, int DIMF>
__device__ bool publish_block_record(RedShared<NT>& rs, sabr_level_record& rec,
                                     const SaLevelArgs& a) {
    if (threadIdx.x == 0) {
        rec.end_value = rs.e_win.v;
        rec.end_chain = rs.e_win.i == LLONG_MAX ? -1 : rs.e_win.i;
        rec.best_value = rs.b_win.v;
        rec.best_chain = rs.b_win.i == LLONG_MAX ? -1 : rs.b_win.i;
        rec.evals = rs.n_tot;
        a.block_recs[blockIdx.x] = rec;
        a.block_sum[blockIdx.x] = BlockSummary{rec.end_value, rec.end_chain, rec.best_value, rec.best_chain,
                                               rec.evals, 0};
        __threadfence();
        const unsigned t = atomicAdd(a.ticket, 1u);
        rs.is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return rs.is_last != 0;
}

// The fused cross-rank exchange of one level record (thread 0 of the last
// CTA): store it into this rank's slot of every rank's mailbox (peer memory
// over NVLink / NVSwitch; the own mailbox is local), fence system-wide, raise
// the slot's epoch, wait until every slot of the own mailbox carries this
// level's epoch, then apply merge_level to the records in rank order - the
// all-gather and the merge of the NCCL path (sa_merge_kernel) without leaving
// the level kernel.  A 20 s timeout turns a lost peer into an error (run
// stopped, peer_error set) instead of a hang.
__device__ __noinline__ void peer_exchange_and_merge(const SaLevelArgs& a, const sabr_level_record& out,
                                                     int64_t level, int dim) {
    const unsigned long long epoch = a.epoch_base + static_cast<unsigned long long>(level) + 1ull;
    const int par = static_cast<int>(epoch & 1ull);
    for (int r = 0; r < a.nranks; ++r) a.peer_boxes[r]->rec[par][a.my_rank] = out;
    __threadfence_system();
    // system-scope atomics: the mailboxes are written by other GPUs
    for (int r = 0; r < a.nranks; ++r)
        atomicExch_system(&a.peer_boxes[r]->epoch[par][a.my_rank], epoch);
    PeerMailbox* own = a.peer_boxes[a.my_rank];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < a.nranks; ++r) {
        for (;;) {
            unsigned long long seen;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(seen) : "l"(&own->epoch[par][r]) : "memory");
            if (seen >= epoch) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 20000000000ull) {  // 20 s
                atomicExch(a.peer_error, 1);
                a.state->done = 1;
                return;
            }
            __nanosleep(100);
        }
    }
    __threadfence_system();
    sabr_level_record recs[kMaxPeerRanks];
    for (int r = 0; r < a.nranks; ++r) {
        const volatile sabr_level_record* src = &own->rec[par][r];
        recs[r].end_value = src->end_value;
        recs[r].end_chain = src->end_chain;
        recs[r].best_value = src->best_value;
        recs[r].best_chain = src->best_chain;
        recs[r].evals = src->evals;
        for (int i = 0; i < SABR_MAX_DIM; ++i) {
            recs[r].end_point[i] = src->end_point[i];
            recs[r].best_point[i] = src->best_point[i];
        }
    }
    merge_level(a.state, recs, a.nranks, a.n_chains, a.max_evals, a.levels_total, dim, a.trace_f + level);
}

// Last CTA: reduce the CTA records of this rank into the rank record and, on
// a single rank, merge it into the annealer state (annealer.cpp:141-159).
// Four records in flight per thread: the scan is L2-latency bound.
template <int NT, int DIMF>
__device__ void reduce_block_records(RedShared<NT>& rs, const SaLevelArgs& a, int64_t level) {
    __threadfence();
    ArgMin ee{CUDART_INF, LLONG_MAX, -1}, bb{CUDART_INF, LLONG_MAX, -1};
    long long nn = 0;
    const int nrec = static_cast<int>(gridDim.x);
    // 16 summaries in flight per thread: the scan is L2-latency bound and
    // runs in one CTA while the rest of the GPU is idle
    constexpr int U = 16;
    for (int k0 = threadIdx.x; k0 < nrec; k0 += U * NT) {
        double4 v[U];
        long long n[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * NT;
            v[u] = make_double4(CUDART_INF, __longlong_as_double(-1ll), CUDART_INF, __longlong_as_double(-1ll));
            n[u] = 0;
            if (k < nrec) {
                const double4* p = reinterpret_cast<const double4*>(a.block_sum + k);
                const double2 lo = __ldcg(reinterpret_cast<const double2*>(p));
                const double2 hi = __ldcg(reinterpret_cast<const double2*>(p) + 1);
                v[u] = make_double4(lo.x, lo.y, hi.x, hi.y);
                n[u] = __ldcg(&a.block_sum[k].evals);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * NT;
            const long long ei = __double_as_longlong(v[u].y), bi = __double_as_longlong(v[u].w);
            if (ei >= 0) argmin_combine(ee, ArgMin{v[u].x, ei, k});
            if (bi >= 0) argmin_combine(bb, ArgMin{v[u].z, bi, k});
            nn += n[u];
        }
    }
    block_reduce(rs, ee, bb, nn);
    if (threadIdx.x == 0) {
        sabr_level_record out;
        out.end_value = rs.e_win.v;
        out.end_chain = rs.e_win.blk >= 0 ? rs.e_win.i : -1;
        out.best_value = rs.b_win.v;
        out.best_chain = rs.b_win.blk >= 0 ? rs.b_win.i : -1;
        out.evals = rs.n_tot;
        out._pad = 0;
        for (int i = 0; i < SABR_MAX_DIM; ++i) {
            out.end_point[i] = rs.e_win.blk >= 0 && i < DIMF
                                   ? __ldcg(&a.block_recs[rs.e_win.blk].end_point[i]) : 0.0;
            out.best_point[i] = rs.b_win.blk >= 0 && i < DIMF
                                    ? __ldcg(&a.block_recs[rs.b_win.blk].best_point[i]) : 0.0;
        }
        *a.rank_rec = out;
        *a.ticket = 0u;
        if (a.nranks == 1) {
            merge_level(a.state, &out, 1, a.n_chains, a.max_evals, a.levels_total, DIMF,
                        a.trace_f + level);
        } else if (a.peer_boxes != nullptr) {
            peer_exchange_and_merge(a, out, level, DIMF);
        }
    }
}

// griddepcontrol (sm_90+): pdl_trigger / pdl_wait, pdl.cuh

// --------------------------------------------------------- level kernel ---
// propose, annealer.cpp:60-74, for one coordinate: bit-identical to the
// reference (2u - 1 via Xoshiro::sym, the reflections use the host-doubled
// bounds, no FMA contraction).
__device__ __forceinline__ double propose_coord(double x, double step_scale, double lo, double hi,
                                                double lo2, double hi2, Xoshiro& rng) {
    double v = __dadd_rn(x, __dmul_rn(step_scale, rng.sym()));
    if (v > hi) v = __dsub_rn(hi2, v);
    if (v < lo) v = __dsub_rn(lo2, v);
    return (v < lo) ? lo : (hi < v) ? hi : v;
}

// propose_coord when the host has shown (sa_fast_path) that, for every
// x in [lo, hi] and |step| <= range, one reflection lands inside the box:
// then the reference's second reflection and its clamp never fire, and the
// coordinate is one of {v, 2hi - v, 2lo - v} (two compares, no clamp).
__device__ __forceinline__ double propose_coord_fast(double x, double step_scale, double lo, double hi,
                                                     double lo2, double hi2, Xoshiro& rng) {
    const double v = __dadd_rn(x, __dmul_rn(step_scale, rng.sym()));
    const double rh = __dsub_rn(hi2, v), rl = __dsub_rn(lo2, v);
    return (v > hi) ? rh : (v < lo) ? rl : v;
}

// One temperature level of this rank's chains (annealer.cpp:99-161).
// ALLFREE (the FAST variant): every coordinate is searched (no mask test),
// one reflection always lands in the box (propose_coord_fast) and every
// forward has |ln f| <= 700 (unsaturated exp in pow_fwd) - see sa_fast_path.
template <int KIND, int DIMF, bool ALLFREE, int GK>
__global__ void __launch_bounds__(kLevelThreads, kLevelMinCtas)
    sa_level_kernel(const __grid_constant__ SurfaceView sv, const __grid_constant__ SaLevelArgs a,
                    const int64_t level, const double temp, const double inv_temp) {
    constexpr int NT = kLevelThreads;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ RedShared<NT> rs;
    __shared__ sabr_level_record rec;
    __shared__ double2 tab_s[kExpTableSize];
    // the chain-best point is written only on improvement and read once at
    // the end: it lives in shared memory (column per thread), not registers
    __shared__ double bp_s[DIMF][NT];

    sabr_sa_state* st = a.state;
    if (st->done) return;  // early-stopped run (max_evals): uniform exit

    stage_exp(sv, tab_s);
    ObjGrid<GK> g{};
    if constexpr (KIND != OBJ_BUILTIN) g = stage_obj<GK>(sv, smem);
    __syncthreads();
    g.tab = tab_s;

    const int64_t local = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
    const bool active = local < a.n_local;
    const int64_t chain = a.chain_begin + local;

    double* const bp = &bp_s[0][threadIdx.x];  // bp[i * NT] = dim i
    double x[DIMF], y[DIMF];
#pragma unroll
    for (int i = 0; i < DIMF; ++i) {
        x[i] = st->incumbent[i];
        bp[i * NT] = x[i];
    }
    double fx = st->incumbent_value;
    double bv = fx;
    int ev = 0;

    if (active) {
        // per-level eval cap (annealer.cpp:102-104) as a step count bound
        const long long cap64 = st->eval_cap;
        const int cap = cap64 < a.chain_length ? static_cast<int>(cap64 < 0 ? 0 : cap64) : a.chain_length;
        // substream keyed by (seed, level, chain): annealer.cpp:112-115
        Xoshiro rng;
        rng.init(a.seed, (static_cast<uint64_t>(level) << 20) ^ static_cast<uint64_t>(chain));
        const double ratio = temp / a.t0;
        const double scale = (ratio < 1.0) ? ratio : 1.0;  // std::min(1.0, T/t0), annealer.cpp:62
        double step_scale[DIMF];
#pragma unroll
        for (int i = 0; i < DIMF; ++i) step_scale[i] = __dmul_rn(a.range[i], scale);
        for (int step = 0; step < a.chain_length; ++step) {
            if (ev >= cap) break;  // annealer.cpp:120
#pragma unroll
            for (int i = 0; i < DIMF; ++i) {
                if (ALLFREE)
                    y[i] = propose_coord_fast(x[i], step_scale[i], a.lo[i], a.hi[i], a.lo2[i], a.hi2[i], rng);
                else if ((a.free_mask >> i) & 1u)
                    y[i] = propose_coord(x[i], step_scale[i], a.lo[i], a.hi[i], a.lo2[i], a.hi2[i], rng);
                else
                    y[i] = x[i];
            }
            if (!predicate_ok(a.predicate, y)) continue;  // annealer.cpp:122
            double fy = objective<KIND>(y, g, a.builtin);
            if (isnan(fy)) fy = CUDART_INF;  // safe_eval, annealer.cpp:84-87
            ++ev;
            // Metropolis, annealer.cpp:125-126 (uniform drawn only when fy > fx).
            // (fy - fx) / T as (fy - fx) * RN(1/T) (<= 1 ulp from the IEEE
            // quotient: the decision boundary moves by ~1e-16 relative, the
            // size of the reference's own exp rounding).
            bool accept = fy <= fx;
            if (!accept) {
                const uint64_t m = rng.peek_bits();
                rng.advance();
                float tau = neg_log_uniform(m);
                if (metropolis_fast(fy, fx, inv_temp, tau).unsure)
                    tau = metropolis_exact(fy, fx, temp, m) ? CUDART_INF_F : -CUDART_INF_F;
                accept = metropolis_fast(fy, fx, inv_temp, tau).accept;
            }
            if (accept) {
#pragma unroll
                for (int i = 0; i < DIMF; ++i) x[i] = y[i];
                fx = fy;
                if (fx < bv) {
                    bv = fx;
#pragma unroll
                    for (int i = 0; i < DIMF; ++i) bp[i * NT] = x[i];
                }
            }
        }
    }

    // ---- level-end reduction (annealer.cpp:141-159) ----
    ArgMin e{active ? fx : CUDART_INF, active ? chain : LLONG_MAX, static_cast<int32_t>(blockIdx.x)};
    ArgMin b{active ? bv : CUDART_INF, active ? chain : LLONG_MAX, static_cast<int32_t>(blockIdx.x)};
    block_reduce(rs, e, b, static_cast<long long>(ev));
    if (active && chain == rs.e_win.i) {
#pragma unroll
        for (int i = 0; i < DIMF; ++i) rec.end_point[i] = x[i];
    }
    if (active && chain == rs.b_win.i) {
#pragma unroll
        for (int i = 0; i < DIMF; ++i) rec.best_point[i] = bp[i * NT];
    }
    __syncthreads();
    if (!publish_block_record<NT, DIMF>(rs, rec, a)) return;
    reduce_block_records<NT, DIMF>(rs, a, level);
}

// The same level with C chains per thread (model objectives, grid in shared
// memory, no predicate), with a branch-free Metropolis step and programmatic
// dependent launch.  With C = 2 the chains of a thread step in lockstep and
// share the grid loads, the loop control and the constants, and their
// independent dependency chains interleave (ILP).  A CTA of kLevelThreads / C
// threads covers kLevelThreads chains (thread t owns chains t, t + NT, ...
// of the CTA's range), so the per-CTA records are those of sa_level_kernel.
// Each chain's arithmetic is that of sa_level_kernel: the kernels produce
// identical trajectories.  C = 2 (default): 32-thread CTAs; C = 1
// (SABR_SA_CPT=1, factored grid only): 64-thread CTAs.  1e5 chains: 1563
// CTAs, 11 per SM, in one wave either way.
constexpr int kPairMinCtas = 11;
// threads per CTA and CTAs per SM (launch bound) of the C-chain level kernel:
// C = 1, 2 cover kLevelThreads chains per CTA; C = 3 (SABR_SA_CPT=3, A/B)
// uses one warp of 96 chains and 8 CTAs per SM (<= 255 registers)
// kCase1Rep (A/B, off): Case I with two chains per thread in two-warp CTAs of
// 128 chains, 6 per SM at 168 registers, which leaves each CTA room for the
// 8-copy bank-replicated exp table (11 one-warp CTAs per SM cannot hold it).
// Its 8 exp lookups per eval then stop conflicting (ncu: 14.9M -> 0.08M excess
// shared wavefronts per level), but the kernel is bound by FP64 dependency
// latency and C3 ran 1.3% slower (1.867e10 -> 1.843e10 evals/s), so the
// one-warp CTAs with one table copy stay.
constexpr bool kCase1Rep = false;
template <int KIND, int C>
constexpr int level_nt() {
    return C == 3 ? 32 : (kCase1Rep && KIND == OBJ_CASE1 && C == 2) ? 64 : kLevelThreads / C;
}
template <int KIND, int C>
constexpr int level_min_ctas() {
    return C == 3 ? 8 : (kCase1Rep && KIND == OBJ_CASE1 && C == 2) ? 6 : kPairMinCtas;
}
// copies of the bank-replicated exp table (device_common.cuh: kExpRep) per
// objective in the C-chain level kernel
template <int KIND>
constexpr int rep_copies() { return kExpRep; }

// The chains of one CTA for one level (annealer.cpp:107-139) and the CTA's
// level-end arg-min (annealer.cpp:141-159): on return (all threads) rs holds
// the CTA's (endpoint, best) winners and eval count, rec their points.
// Shared by the per-level kernel and the single-CTA persistent kernel.
// PIPE (ALLFREE only): the RNG is software-pipelined - the draws of step s + 1
// are generated while step s's objective runs, for both Metropolis outcomes,
// and selected once fy is known.  That takes the xoshiro chain off the
// critical path at the price of ~8 instructions per chain-step: a gain for
// the latency-bound one-CTA run (C1: one warp per SM), a loss for the
// issue-bound full-GPU level kernel (C2: -3.6%).
// FIXM (with ALLFREE false): a compile-time mask of fixed coordinates, every
// other coordinate searched with the one-reflection propose (a.fast_free);
// Case I with beta fixed, the C3 configuration, uses FIXM = 2.
template <int KIND, int DIMF, bool ALLFREE, int GK, int C, int NT, bool PIPE = false, int FIXM = 0,
          bool B1 = false>
__device__ __forceinline__ void run_level_chains(const SaLevelArgs& a, const ObjGrid<GK>& g,
                                                 const double2* tab_s, const double2* tab_lane,
                                                 const double* pw_fixed,
                                                 const sabr_sa_state* st, const double temp,
                                                 const double inv_temp, const bool (&active)[C],
                                                 const int64_t (&chain)[C], Xoshiro (&rng)[C],
                                                 double (&bp_s)[C][DIMF][NT], RedShared<NT>& rs,
                                                 sabr_level_record& rec) {
    double x[C][DIMF], y[C][DIMF], fx[C], bv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
        for (int i = 0; i < DIMF; ++i) {
            x[c][i] = st->incumbent[i];
            bp_s[c][i][threadIdx.x] = x[c][i];
        }
        fx[c] = bv[c] = st->incumbent_value;
    }
    int steps = 0;
    if (active[0]) {  // chain c > 0 active implies chain 0 active
        const long long cap64 = st->eval_cap;
        steps = cap64 < a.chain_length ? static_cast<int>(cap64 < 0 ? 0 : cap64) : a.chain_length;
        const double ratio = temp / a.t0;
        const double scale = (ratio < 1.0) ? ratio : 1.0;
        double step_scale[DIMF];
#pragma unroll
        for (int i = 0; i < DIMF; ++i) step_scale[i] = __dmul_rn(a.range[i], scale);
        std::conditional_t<GK == kGridQR, QrSlice, StaticSlice> sl{};
        if constexpr (KIND == OBJ_STATIC) {
            if constexpr (GK == kGridQR) sl = qr_slice(g);
            else sl = static_slice(g);
        }
        // PIPE: ws holds this step's proposal draws as 2u - 1, cand the
        // Metropolis candidate o_{p+D} and rng the state that produces it;
        // step s computes o_{p+D+1} .. o_{p+2D} (rng ends at S_{p+2D}), and
        // once fy is known, step s + 1 takes o_{p+D+1 ..} when the candidate
        // was consumed (fy > fx) and o_{p+D ..} otherwise.
        constexpr uint32_t kFull = (1u << DIMF) - 1u;
        constexpr bool kFastProp = ALLFREE || FIXM != 0;
        constexpr uint32_t kFree = ALLFREE ? kFull : (kFull & ~static_cast<uint32_t>(FIXM));
        constexpr int kDraws = __builtin_popcount(kFree);  // draws per step on the fast path
        constexpr bool kPipe = PIPE && kFastProp;
        double ws[C][kPipe ? DIMF : 1];
        uint64_t cand[C];
        if constexpr (kPipe) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
#pragma unroll
                for (int i = 0; i < DIMF; ++i)
                    if ((kFree >> i) & 1u) ws[c][i] = rng[c].sym();
                cand[c] = rng[c].peek();
            }
        }
        for (int step = 0; step < steps; ++step) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
#pragma unroll
                for (int i = 0; i < DIMF; ++i) {
                    if (kFastProp && !((kFree >> i) & 1u)) {
                        y[c][i] = x[c][i];  // fixed coordinate (FIXM)
                    } else if (kPipe) {
                        const double v = __dadd_rn(x[c][i], __dmul_rn(step_scale[i], ws[c][i]));
                        const double rh = __dsub_rn(a.hi2[i], v), rl = __dsub_rn(a.lo2[i], v);
                        y[c][i] = (v > a.hi[i]) ? rh : (v < a.lo[i]) ? rl : v;
                    } else if (kFastProp)
                        y[c][i] = propose_coord_fast(x[c][i], step_scale[i], a.lo[i], a.hi[i], a.lo2[i],
                                                     a.hi2[i], rng[c]);
                    else if ((a.free_mask >> i) & 1u)
                        y[c][i] = propose_coord(x[c][i], step_scale[i], a.lo[i], a.hi[i], a.lo2[i],
                                                a.hi2[i], rng[c]);
                    else
                        y[c][i] = x[c][i];
                }
            }
            // the Metropolis draw of this step (used only when fy > fx) and
            // its -ln u: they depend on the stream alone, so they are ready
            // before the objective is (metropolis_fast)
            uint64_t mbits[C];
            float tau[C];
            double nsym[C][kPipe ? kDraws + 1 : 1];  // PIPE: 2u - 1 of o_{p+D} .. o_{p+2D}
#pragma unroll
            for (int c = 0; c < C; ++c) {
                mbits[c] = kPipe ? cand[c] & ~0x7ffull : rng[c].peek_bits();
                tau[c] = neg_log_uniform(mbits[c]);
                if constexpr (kPipe) {
                    nsym[c][0] = Xoshiro::sym_of(cand[c]);
                    rng[c].advance();  // past the candidate
#pragma unroll
                    for (int j = 1; j <= kDraws; ++j)
                        nsym[c][j] = Xoshiro::sym_of(j < kDraws ? rng[c].next() : rng[c].peek());
                }
            }
            double fy[C];
            if constexpr (KIND == OBJ_STATIC) {
                if (tab_lane) static_cost_n<C, DIMF, ALLFREE, rep_copies<KIND>()>(y, sl, tab_lane, fy);
                else static_cost_n<C, DIMF, ALLFREE>(y, sl, tab_s, fy);
            } else if constexpr (GK == kGridQR) {
                if (tab_lane) case1_cost_n<C, DIMF, rep_copies<KIND>(), B1>(y, g, fy, pw_fixed, tab_lane);
                else case1_cost_n<C, DIMF, 1, B1>(y, g, fy, pw_fixed);
            }
            else case1_cost_n<C, DIMF>(y, g, fy);
            // Metropolis (annealer.cpp:125-126) without a branch: the FP32
            // certificate decides (metropolis_fast); the draw is committed
            // (the stream advanced) only when fy > fx, as the reference draws
            // it.  The rare undecided comparison takes the exact test, whose
            // verdict goes back into tau (+inf: accept, -inf: reject), so the
            // decision stays one FP32 compare after the rare branch and no
            // predicate lives across it.
            bool unsure = false;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (isnan(fy[c])) fy[c] = CUDART_INF;
                unsure |= metropolis_fast(fy[c], fx[c], inv_temp, tau[c]).unsure;
                const bool up = !(fy[c] <= fx[c]);
                if constexpr (kPipe) {
#pragma unroll
                    for (int i = 0; i < DIMF; ++i) {
                        if (!((kFree >> i) & 1u)) continue;
                        const int r = __popc(kFree & ((1u << i) - 1u));  // the draw's slot (constant)
                        ws[c][i] = up ? nsym[c][r + 1] : nsym[c][r];
                    }
                    rng[c].advance_if(up);  // S_{p+2D} -> S_{p+2D+1} when the draw was consumed
                    cand[c] = rng[c].peek();
                } else {
                    rng[c].advance_if(up);
                }
            }
            if (unsure) {
#pragma unroll
                for (int c = 0; c < C; ++c)
                    if (metropolis_fast(fy[c], fx[c], inv_temp, tau[c]).unsure)
                        tau[c] = metropolis_exact(fy[c], fx[c], temp, mbits[c]) ? CUDART_INF_F : -CUDART_INF_F;
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const bool accept = metropolis_fast(fy[c], fx[c], inv_temp, tau[c]).accept;
                const bool better = accept && fy[c] < bv[c];
#pragma unroll
                for (int i = 0; i < DIMF; ++i) x[c][i] = accept ? y[c][i] : x[c][i];
                fx[c] = accept ? fy[c] : fx[c];
                bv[c] = better ? fy[c] : bv[c];
                if (better) {
#pragma unroll
                    for (int i = 0; i < DIMF; ++i) bp_s[c][i][threadIdx.x] = y[c][i];
                }
            }
        }
    }

    // ---- level-end reduction (annealer.cpp:141-159) ----
    ArgMin e{CUDART_INF, LLONG_MAX, static_cast<int32_t>(blockIdx.x)};
    ArgMin b{CUDART_INF, LLONG_MAX, static_cast<int32_t>(blockIdx.x)};
    long long ev = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (!active[c]) continue;
        argmin_combine(e, ArgMin{fx[c], chain[c], static_cast<int32_t>(blockIdx.x)});
        argmin_combine(b, ArgMin{bv[c], chain[c], static_cast<int32_t>(blockIdx.x)});
        ev += steps;
    }
    block_reduce(rs, e, b, ev);
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (active[c] && chain[c] == rs.e_win.i) {
#pragma unroll
            for (int i = 0; i < DIMF; ++i) rec.end_point[i] = x[c][i];
        }
        if (active[c] && chain[c] == rs.b_win.i) {
#pragma unroll
            for (int i = 0; i < DIMF; ++i) rec.best_point[i] = bp_s[c][i][threadIdx.x];
        }
    }
    __syncthreads();
}

// B1 (with FIXM bit 1): beta held at exactly 1 (SaLevelArgs::beta_one), the
// Case I objective without f^(1-beta) (case1_cost_n BETA1)
template <int KIND, int DIMF, bool ALLFREE, int GK, int C, int FIXM = 0, bool PIPE = false, bool B1 = false>
__global__ void __launch_bounds__(level_nt<KIND, C>(), level_min_ctas<KIND, C>())
    sa_level_multi_kernel(const __grid_constant__ SurfaceView sv, const __grid_constant__ SaLevelArgs a,
                          const int64_t level, const double temp, const double inv_temp) {
    constexpr int NT = level_nt<KIND, C>();
    // the static objective's pow reads the bank-replicated exp table (Case I:
    // one copy, kCase1Rep)
    constexpr bool kRep = GK == kGridQR && (KIND == OBJ_STATIC || (kCase1Rep && KIND == OBJ_CASE1 && C == 2));
    constexpr int kRepN = rep_copies<KIND>();
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ RedShared<NT> rs;
    __shared__ sabr_level_record rec;
    __shared__ double2 tab_s[kExpTableSize];
    __shared__ double2 tabr_s[kRep ? kExpTableSize * kRepN : 1];
    __shared__ double bp_s[C][DIMF][NT];

    sabr_sa_state* st = a.state;
    // Programmatic dependent launch: the next level's grid may start as soon
    // as SMs free up; everything before pdl_wait() (table and grid staging,
    // the chains' stream seeding) does not depend on the previous level and
    // overlaps its tail (the last CTA's merge).  Nothing written by the
    // previous level is read before pdl_wait().
    pdl_trigger();
    stage_exp(sv, tab_s);
    if constexpr (kRep)
        for (int i = threadIdx.x; i < kExpTableSize * kRepN; i += NT) tabr_s[i] = sv.exptab[i / kRepN];
    ObjGrid<GK> g = stage_obj<GK>(sv, smem);
    __syncthreads();
    g.tab = tab_s;
    const double2* tab_lane = kRep ? tabr_s + (threadIdx.x & (kRepN - 1)) : nullptr;

    bool active[C];
    int64_t chain[C];
    Xoshiro rng[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int64_t local = static_cast<int64_t>(blockIdx.x) * (NT * C) + c * NT + threadIdx.x;
        active[c] = local < a.n_local;
        chain[c] = a.chain_begin + local;
        // substream keyed by (seed, level, chain): annealer.cpp:112-115
        rng[c].init(a.seed, (static_cast<uint64_t>(level) << 20) ^ static_cast<uint64_t>(chain[c]));
    }
    pdl_wait();
    if (st->done) return;  // early-stopped run (max_evals): uniform exit
    // Case I with beta not searched: f_i^(1-beta) is one value per slice
    __shared__ double pw_s[2 * kMaxPwSlices];  // f_i^(1-beta), then rcp(f_i^(1-beta))
    const double* pw_fixed = nullptr;
    if constexpr (KIND == OBJ_CASE1 && GK == kGridQR) {
        if (!((a.free_mask >> 1) & 1u) && g.ns <= kMaxPwSlices) {
            const double omb = 1.0 - st->incumbent[1];
            for (int i = threadIdx.x; i < g.ns; i += NT) {
                pw_s[i] = pow_fwd(omb, g.lnf_hi[i], g.lnf_lo[i], g.tab);
                pw_s[kMaxPwSlices + i] = fast_rcp(pw_s[i]);
            }
            __syncthreads();
            pw_fixed = pw_s;
        }
    }
    run_level_chains<KIND, DIMF, ALLFREE, GK, C, NT, PIPE, FIXM, B1>(a, g, tab_s, tab_lane, pw_fixed, st, temp,
                                                                     inv_temp, active, chain, rng, bp_s, rs, rec);
    if (!publish_block_record<NT, DIMF>(rs, rec, a)) return;
    reduce_block_records<NT, DIMF>(rs, a, level);
}

// Every level of a run whose chains fit one CTA (C1: 32 chains), on one rank,
// in one launch: the per-level launch, the grid-level record scan and the
// level-to-level dependency (8.3 us per level at C1) collapse into a
// __syncthreads.  Per level: the same chains and arg-min as
// sa_level_multi_kernel, then thread 0 applies merge_level to the CTA record
// (what reduce_block_records does for a one-CTA grid).  temps[level] is the
// host's schedule (annealer.cpp:99, repeated multiplication), 1/T as the host
// computes it.  Identical trajectories to the per-level kernels.
template <int KIND, int DIMF, bool ALLFREE, int GK, int C>
__global__ void __launch_bounds__(kLevelThreads / C, 1)
    sa_run_small_kernel(const __grid_constant__ SurfaceView sv, const __grid_constant__ SaLevelArgs a,
                        const double* __restrict__ temps, const int64_t n_levels) {
    constexpr int NT = kLevelThreads / C;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ RedShared<NT> rs;
    __shared__ sabr_level_record rec;
    __shared__ double2 tab_s[kExpTableSize];
    __shared__ double bp_s[C][DIMF][NT];
    __shared__ double pw_s[2 * kMaxPwSlices];  // f_i^(1-beta), then rcp(f_i^(1-beta))
    sabr_sa_state* st = a.state;
    stage_exp(sv, tab_s);
    ObjGrid<GK> g = stage_obj<GK>(sv, smem);
    __syncthreads();
    g.tab = tab_s;
    bool active[C];
    int64_t chain[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int64_t local = static_cast<int64_t>(c) * NT + threadIdx.x;
        active[c] = local < a.n_local;
        chain[c] = a.chain_begin + local;
    }
    const double* pw_fixed = nullptr;
    if constexpr (KIND == OBJ_CASE1 && GK == kGridQR) {
        if (!((a.free_mask >> 1) & 1u) && g.ns <= kMaxPwSlices) {  // beta not searched: constant
            const double omb = 1.0 - st->incumbent[1];
            for (int i = threadIdx.x; i < g.ns; i += NT) {
                pw_s[i] = pow_fwd(omb, g.lnf_hi[i], g.lnf_lo[i], g.tab);
                pw_s[kMaxPwSlices + i] = fast_rcp(pw_s[i]);
            }
            __syncthreads();
            pw_fixed = pw_s;
        }
    }
    for (int64_t level = 0; level < n_levels; ++level) {
        if (st->done) break;  // block-uniform (merge_level's writes are behind the __syncthreads)
        const double temp = temps[level];
        const double inv_temp = 1.0 / temp;
        Xoshiro rng[C];
#pragma unroll
        for (int c = 0; c < C; ++c)
            rng[c].init(a.seed, (static_cast<uint64_t>(level) << 20) ^ static_cast<uint64_t>(chain[c]));
        run_level_chains<KIND, DIMF, ALLFREE, GK, C, NT, true>(a, g, tab_s, nullptr, pw_fixed, st, temp,
                                                               inv_temp, active, chain, rng, bp_s, rs, rec);
        if (threadIdx.x == 0) {
            sabr_level_record out;
            const bool e_ok = rs.e_win.i != LLONG_MAX, b_ok = rs.b_win.i != LLONG_MAX;
            out.end_value = rs.e_win.v;
            out.end_chain = e_ok ? rs.e_win.i : -1;
            out.best_value = rs.b_win.v;
            out.best_chain = b_ok ? rs.b_win.i : -1;
            out.evals = rs.n_tot;
            out._pad = 0;
            for (int i = 0; i < SABR_MAX_DIM; ++i) {
                out.end_point[i] = e_ok && i < DIMF ? rec.end_point[i] : 0.0;
                out.best_point[i] = b_ok && i < DIMF ? rec.best_point[i] : 0.0;
            }
            merge_level(st, &out, 1, a.n_chains, a.max_evals, a.levels_total, DIMF, a.trace_f + level);
        }
        __syncthreads();
    }
}

__global__ void sa_merge_kernel(const SaLevelArgs a, const sabr_level_record* recs,
                                const int64_t level) {
    if (a.state->done) return;
    merge_level(a.state, recs, a.nranks, a.n_chains, a.max_evals, a.levels_total, a.dim_full,
                a.trace_f + level);
}

template <int KIND, int DIMF, int GK>
__global__ void sa_start_kernel(const __grid_constant__ SurfaceView sv, const SaLevelArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double2 tab_s[kExpTableSize];
    stage_exp(sv, tab_s);
    ObjGrid<GK> g{};
    if constexpr (KIND != OBJ_BUILTIN) g = stage_obj<GK>(sv, smem);
    __syncthreads();
    g.tab = tab_s;
    if (threadIdx.x != 0) return;
    double x[DIMF];
    for (int i = 0; i < DIMF; ++i) x[i] = a.state->incumbent[i];
    double v = objective<KIND>(x, g, a.builtin);
    if (isnan(v)) v = CUDART_INF;
    a.state->incumbent_value = v;
    a.state->best_value = v;
}

// The SA objective on a batch of full parameter vectors (same code path).
template <int KIND, int DIMF, int GK>
__global__ void __launch_bounds__(kThreads)
    cost_batch_kernel(const __grid_constant__ SurfaceView sv, const double* __restrict__ params,
                      const int64_t n, double* __restrict__ cost) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double2 tab_s[kExpTableSize];
    stage_exp(sv, tab_s);
    ObjGrid<GK> g = stage_obj<GK>(sv, smem);
    __syncthreads();
    g.tab = tab_s;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    if (i >= n) return;
    double v[DIMF];
#pragma unroll
    for (int k = 0; k < DIMF; ++k) v[k] = params[i * DIMF + k];
    cost[i] = objective<KIND>(v, g, 0);
}

// Model vols for every quote of the view (report rows, calibration.cpp:180-194).
template <int KIND, int DIMF, bool SMEM>
__global__ void vol_batch_kernel(const __grid_constant__ SurfaceView sv, const double* __restrict__ params,
                                 const int64_t n, double* __restrict__ vols) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double2 tab_s[kExpTableSize];
    stage_exp(sv, tab_s);
    Grid g = stage_grid<SMEM>(sv, smem);
    __syncthreads();
    g.tab = tab_s;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v[DIMF];
#pragma unroll
    for (int k = 0; k < DIMF; ++k) v[k] = params[i * DIMF + k];
    const int nq = g.qoff[g.ns];
    const double omb = 1.0 - v[1];
    for (int s = 0; s < g.ns; ++s) {
        const double pw = pow_fwd(omb, g.lnf_hi[s], g.lnf_lo[s], g.tab);
        SmileTerms t;
        if constexpr (KIND == OBJ_STATIC) {
            t = static_terms(v[0], v[1], v[2], v[3], pw, g.T[s]);
        } else {
            double n1, n2, e1, e2;
            dyn_coeffs_case1(v[2], v[3], v[4], v[5], g.T[s], n1, n2, e1, e2);
            t = dynamic_terms(n1, n2, e1, e2, v[0], v[1], pw, g.T[s]);
        }
        for (int j = g.qoff[s]; j < g.qoff[s + 1]; ++j)
            vols[i * nq + j] = smile_vol(t, g.q[j].lm, g.q[j].lm2);
    }
}

__global__ void case2_feasible_kernel(const double* __restrict__ params, const int64_t n,
                                      uint8_t* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) p[k] = params[i * 11 + k];
    out[i] = case2_feasible(p) ? 1 : 0;
}


// ------------------------------------------------------- T_II chain kernels ---
// propose, annealer.cpp:60-74, over the full vector (fixed dims untouched;
// uniforms drawn for free dims in order, as the reference's search vector).
__device__ __forceinline__ void propose_full(const double* x, double* y, const double* lo,
                                             const double* hi, const double* range,
                                             uint32_t mask, double scale, Xoshiro& rng) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if ((mask >> i) & 1u) {
            const double u = rng.uniform();
            const double stp = __dmul_rn(__dmul_rn(range[i], scale), __dsub_rn(__dmul_rn(2.0, u), 1.0));
            double v = __dadd_rn(x[i], stp);
            if (v > hi[i]) v = __dsub_rn(__dmul_rn(2.0, hi[i]), v);
            if (v < lo[i]) v = __dsub_rn(__dmul_rn(2.0, lo[i]), v);
            y[i] = (v < lo[i]) ? lo[i] : (hi[i] < v) ? hi[i] : v;
        } else {
            y[i] = x[i];
        }
    }
}

__device__ __forceinline__ void load_rng(Xoshiro& r, const uint64_t* s) {
    r.s0 = s[0];
    r.s1 = s[1];
    r.s2 = s[2];
    r.s3 = s[3];
}
__device__ __forceinline__ void store_rng(const Xoshiro& r, uint64_t* s) {
    s[0] = r.s0;
    s[1] = r.s1;
    s[2] = r.s2;
    s[3] = r.s3;
}

__global__ void t2_level_init_kernel(T2Chain* __restrict__ chains, const sabr_sa_state* st,
                                     const T2StepArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.n_local || st->done) return;
    T2Chain& ch = chains[c];
    for (int i = 0; i < SABR_MAX_DIM; ++i) ch.x[i] = ch.bp[i] = ch.y[i] = st->incumbent[i];
    ch.fx = ch.bv = st->incumbent_value;
    ch.evals = 0;
    ch.active = 0;
    Xoshiro r;
    r.init(a.seed, (static_cast<uint64_t>(a.level) << 20) ^ static_cast<uint64_t>(a.chain_begin + c));
    store_rng(r, ch.rng);
}

// One warp per chain: lane 0 proposes (its stored stream), the warp shares
// the proposal and evaluates the 256-node feasibility grid together.
constexpr int kProposeChainsPerCta = 4;

__global__ void __launch_bounds__(32 * kProposeChainsPerCta)
    t2_propose_kernel(T2Chain* __restrict__ chains, const sabr_sa_state* st, const T2StepArgs a,
                      double* __restrict__ alpha0, double* __restrict__ beta, uint8_t* __restrict__ active) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x * kProposeChainsPerCta + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= a.n_local) return;  // warp-uniform
    T2Chain& ch = chains[c];
    if (st->done || ch.evals >= st->eval_cap) {  // annealer.cpp:120
        if (lane == 0) {
            ch.active = 0;
            active[c] = 0;
        }
        return;
    }
    double y[11];
    if (lane == 0) {
        Xoshiro r;
        load_rng(r, ch.rng);
        const double ratio = a.temp / a.t0;
        const double scale = (ratio < 1.0) ? ratio : 1.0;
        double x[10];
        for (int i = 0; i < 10; ++i) x[i] = ch.x[i];
        propose_full(x, y, a.lo, a.hi, a.range, a.free_mask, scale, r);
        store_rng(r, ch.rng);
    }
#pragma unroll
    for (int i = 0; i < 10; ++i) y[i] = __shfl_sync(0xffffffffu, y[i], 0);
    y[10] = a.horizon;
    // SearchSpace::is_feasible -> case2_feasible (calibration.cpp:467-469)
    const bool ok = case2_feasible_warp(y);
    if (lane == 0) {
        for (int i = 0; i < 10; ++i) ch.y[i] = y[i];
        ch.active = ok ? 1 : 0;
        active[c] = ok ? 1 : 0;
        alpha0[c] = y[0];
        beta[c] = y[1];
    }
}

// coef[i][c] (step-major, cand_stride columns); inactive and padding
// candidates get zero coefficients (simulated harmlessly, never priced).
// One candidate's FP32 row for mc_tile_kernel_f32 (kernels_mc.cu): the
// coefficients {nu sqrt(dt), nu^2 dt / 2, rho sqrt(dt), srho sqrt(dt)} scaled
// by log2(e) with the drift negated, {c1, -c2, rs, ss}; pairs: the
// pair-interleaved layout of the packed FP32x2 kernel, per pair of
// candidates {c1 c1' -c2 -c2'} {rs rs' ss ss'}.
__device__ __forceinline__ void put_coef32(float4* __restrict__ coef32, int64_t step, int c, int cand_stride,
                                           int pairs, const double4 v) {
    constexpr double L = 1.4426950408889634;
    const float a = static_cast<float>(v.x * L), b = static_cast<float>(-v.y * L);
    const float r = static_cast<float>(v.z * L), q = static_cast<float>(v.w * L);
    if (!pairs) {
        coef32[step * cand_stride + c] = make_float4(a, b, r, q);
        return;
    }
    float* row = reinterpret_cast<float*>(coef32 + step * cand_stride + (c & ~1));
    const int h = c & 1;
    row[h] = a;
    row[2 + h] = b;
    row[4 + h] = r;
    row[6 + h] = q;
}

// idx: the compacted candidate list (t2_compact_kernel): candidate c of the
// launch is chain idx[c] (-1: no candidate); n_live: the list's length - a
// launch that starts past it writes nothing (its MC blocks all exit).
__global__ void t2_coef_kernel(const T2Chain* __restrict__ chains, const int32_t* __restrict__ idx,
                               const int32_t* __restrict__ n_live, const int32_t c0,
                               const int32_t n_local, const int32_t cand_stride,
                               const double* __restrict__ t_end, const double* __restrict__ dt,
                               const double* __restrict__ sdt, const int64_t total_steps,
                               double4* __restrict__ coef, float4* __restrict__ coef32,
                               const int pairs) {
    pdl_wait();
    pdl_trigger();
    if (c0 >= *n_live) return;  // uniform
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(cand_stride) * total_steps) return;
    const int c = static_cast<int>(t % cand_stride);
    const int64_t i = t / cand_stride;
    const int32_t chain = c < n_local ? idx[c0 + c] : -1;
    if (chain < 0) {
        if (coef32) put_coef32(coef32, i, c, cand_stride, pairs, make_double4(0.0, 0.0, 0.0, 0.0));
        else coef[t] = make_double4(0.0, 0.0, 0.0, 0.0);
        return;
    }
    const T2Chain& ch = chains[chain];
    double p[11];
    for (int k = 0; k < 10; ++k) p[k] = ch.y[k];
    const double tt = t_end[i];
    const double nu = case2_nu_at(p, tt);    // nu, rho at the step END, mc.cpp:69-82
    const double rho = case2_rho_at(p, tt);
    const double q = 1.0 - rho * rho;
    const double srho = sqrt((0.0 < q) ? q : 0.0);
    const double s = sdt[i];
    const double4 v = make_double4(nu * s, 0.5 * nu * nu * dt[i], rho * s, srho * s);
    if (coef32) put_coef32(coef32, i, c, cand_stride, pairs, v);
    else coef[t] = v;
}

// The step's candidates compacted (feasible proposals first, in chain
// order): the MC launches then fill every CB-candidate group of a thread with
// live work instead of simulating the infeasible proposals' zero rows (C5 in
// the default box: ~45% of proposals).  A candidate's price does not depend
// on its position in the batch (kernels_mc.cu), so results are unchanged.
// One CTA: each thread scans a contiguous segment, then a CTA-wide scan of
// the segment counts.
constexpr int kCompactThreads = 1024;
__global__ void __launch_bounds__(kCompactThreads)
    t2_compact_kernel(const uint8_t* __restrict__ active, const double* __restrict__ alpha0,
                      const double* __restrict__ beta, const int32_t n, int32_t* __restrict__ idx,
                      double* __restrict__ alpha0_c, double* __restrict__ beta_c, uint8_t* __restrict__ active_c,
                      int32_t* __restrict__ n_live, int* __restrict__ bad_c) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t warp_tot[kCompactThreads / 32];
    const int seg = (n + kCompactThreads - 1) / kCompactThreads;
    const int b = threadIdx.x * seg, e = min(n, b + seg);
    int cnt = 0;
    for (int c = b; c < e; ++c) cnt += active[c] != 0;
    // exclusive scan over the CTA: warp shuffles, then the warp totals
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = warp_tot[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += v;
        }
        warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    int k = incl - cnt + (warp > 0 ? warp_tot[warp - 1] : 0);
    for (int c = b; c < e; ++c) {
        if (active[c] == 0) continue;
        idx[k] = c;
        alpha0_c[k] = alpha0[c];
        beta_c[k] = beta[c];
        active_c[k] = 1;
        ++k;
    }
    const int total = warp_tot[kCompactThreads / 32 - 1];
    for (int c = total + threadIdx.x; c < n; c += kCompactThreads) {
        idx[c] = -1;
        alpha0_c[c] = 1.0;
        beta_c[c] = 1.0;
        active_c[c] = 0;
    }
    if (threadIdx.x == 0) *n_live = total;
    // the step's non-finite flags reset here rather than by a memset, which
    // would break the PDL chain of the step's kernels
    for (int c = threadIdx.x; c < n; c += kCompactThreads) bad_c[c] = 0;
}

// The compacted candidates' costs and non-finite flags back to their chains.
__global__ void t2_scatter_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ n_live,
                                  const double* __restrict__ cost_c, const int* __restrict__ bad_c,
                                  double* __restrict__ cost, int* __restrict__ bad) {
    pdl_wait();
    pdl_trigger();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= *n_live) return;
    const int c = idx[k];
    cost[c] = cost_c[k];
    bad[c] |= bad_c[k];
}

// Metropolis for one chain's evaluated proposal (annealer.cpp:122-133)
__device__ __forceinline__ void t2_accept_one(T2Chain& ch, double fy, const T2StepArgs& a) {
    if (isnan(fy)) fy = CUDART_INF;
    ch.evals += 1;
    bool accept = fy <= ch.fx;
    if (!accept) {
        Xoshiro r;
        load_rng(r, ch.rng);
        accept = r.uniform() < exp(-(fy - ch.fx) / a.temp);
        store_rng(r, ch.rng);
    }
    if (accept) {
        for (int i = 0; i < 10; ++i) ch.x[i] = ch.y[i];
        ch.fx = fy;
        if (fy < ch.bv) {
            ch.bv = fy;
            for (int i = 0; i < 10; ++i) ch.bp[i] = ch.y[i];
        }
    }
}

__global__ void t2_accept_kernel(T2Chain* __restrict__ chains, const T2StepArgs a,
                                 const double* __restrict__ cost, const int* __restrict__ bad,
                                 int* __restrict__ nonfinite) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.n_local) return;
    T2Chain& ch = chains[c];
    if (!ch.active) return;
    if (bad[c]) atomicOr(nonfinite, 1);
    t2_accept_one(ch, cost[c], a);
}

// A step whose candidates are one MC launch (r02): the candidate's cost
// (mc_cost_kernel's sum), its chain (t2_scatter) and the Metropolis test
// (t2_accept) in one kernel, two launches fewer per SA step.  One warp per
// compacted candidate: the lanes load the quotes and form the relative errors
// side by side, then every lane adds their squares in quote order from warp
// broadcasts, sum = fma(rel, rel, sum) - mc_quote_cost's contracted sum, bit
// for bit - and lane 0 runs the Metropolis test.
constexpr int kFinishWarps = 4;
__global__ void __launch_bounds__(32 * kFinishWarps)
    t2_finish_kernel(T2Chain* __restrict__ chains, const T2StepArgs a, const int32_t* __restrict__ idx,
                     const int32_t* __restrict__ n_live, const double* __restrict__ values, const int32_t nq,
                     const double* __restrict__ market, const int* __restrict__ bad_c, int* __restrict__ nonfinite) {
    pdl_wait();
    pdl_trigger();
    const int k = blockIdx.x * kFinishWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (k >= *n_live) return;  // warp-uniform
    const double* v = values + static_cast<int64_t>(k) * nq;
    double sum = 0.0;
    for (int q0 = 0; q0 < nq; q0 += 32) {
        const int q = q0 + lane;
        const double rel = q < nq ? (market[q] - v[q]) / market[q] : 0.0;
        const int n = min(32, nq - q0);
        for (int j = 0; j < n; ++j) {
            const double r = __shfl_sync(0xffffffffu, rel, j);
            sum = fma(r, r, sum);
        }
    }
    if (lane != 0) return;
    T2Chain& ch = chains[idx[k]];
    if (bad_c[k]) atomicOr(nonfinite, 1);
    t2_accept_one(ch, sum, a);
}

__global__ void __launch_bounds__(kThreads)
    t2_level_end_kernel(const T2Chain* __restrict__ chains, const SaLevelArgs a, const int64_t level) {
    __shared__ RedShared<kThreads> rs;
    __shared__ sabr_level_record rec;
    if (a.state->done) return;
    const int64_t local = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const bool active = local < a.n_local;
    const int64_t chain = a.chain_begin + local;
    const T2Chain* ch = active ? chains + local : nullptr;
    ArgMin e{active ? ch->fx : CUDART_INF, active ? chain : LLONG_MAX, static_cast<int32_t>(blockIdx.x)};
    ArgMin b{active ? ch->bv : CUDART_INF, active ? chain : LLONG_MAX, static_cast<int32_t>(blockIdx.x)};
    block_reduce(rs, e, b, active ? ch->evals : 0);
    if (active && chain == rs.e_win.i)
        for (int i = 0; i < SABR_MAX_DIM; ++i) rec.end_point[i] = ch->x[i];
    if (active && chain == rs.b_win.i)
        for (int i = 0; i < SABR_MAX_DIM; ++i) rec.best_point[i] = ch->bp[i];
    __syncthreads();
    if (!publish_block_record<kThreads, SABR_MAX_DIM>(rs, rec, a)) return;
    reduce_block_records<kThreads, SABR_MAX_DIM>(rs, a, level);
}

// Shared-memory bytes of the staged grid (0 and *use_smem = 0: read the AoS
// grid through L1).  `padded`: the SoA layout of the SA / cost objectives.
size_t smem_for(const SurfaceView& sv, int* use_smem, bool padded = false) {
    const size_t b = padded ? pstage_bytes(sv.n_slices, sv.n_quotes) : stage_bytes(sv.n_slices, sv.n_quotes);
    *use_smem = b <= kSmemStageLimit;
    return *use_smem ? b : 0;
}

template <class K>
cudaError_t set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(bytes));
    return cudaSuccess;
}

// Run `body(kernel_ptr, smem_bytes)` with the SMEM variant the view supports:
// the padded grid staged in shared memory, or (too large) the AoS grid read
// through L1.  (Kernel-parameter/constant-bank grids were tried: sm_100a FP64
// instructions take no constant-bank operands, so they only add registers.)
// SABR_SA_COST=quotes selects the per-quote objectives (A/B checks).
bool qr_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SABR_SA_COST");
        return !(e && std::string(e) == "quotes");
    }();
    return on;
}

// The objective grid of a model view: the factored slices when the view has
// them, else the padded per-quote grid in shared memory, else the AoS grid
// through L1.  *smem = the dynamic shared memory it stages.
int grid_kind(const SurfaceView& sv, size_t* smem) {
    if (sv.qr != nullptr && qr_enabled() && qstage_bytes(sv.n_slices) <= kSmemStageLimit) {
        *smem = qstage_bytes(sv.n_slices);
        return kGridQR;
    }
    int use = 0;
    *smem = smem_for(sv, &use, true);
    return use ? kGridQuads : kGridL1;
}

template <int GK>
using GridTag = std::integral_constant<int, GK>;

template <int KIND, class Pick, class Body>
cudaError_t dispatch_grid(const SurfaceView& sv, Pick&& pick, Body&& body) {
    if constexpr (KIND == OBJ_BUILTIN) {
        return body(pick(GridTag<kGridQuads>{}), size_t(0));
    } else {
        size_t smem = 0;
        switch (grid_kind(sv, &smem)) {
            case kGridQR: return body(pick(GridTag<kGridQR>{}), smem);
            case kGridQuads: return body(pick(GridTag<kGridQuads>{}), smem);
            default: return body(pick(GridTag<kGridL1>{}), size_t(0));
        }
    }
}

// Chains per thread of the model-objective level kernel: SABR_SA_CPT=1, 2 or
// 3; SABR_SA_CPT=0 selects the general one-chain kernel sa_level_kernel (A/B
// checks).  -1 when unset: the default per objective (level_t).
int chains_per_thread() {
    static const int c = [] {
        const char* e = std::getenv("SABR_SA_CPT");
        if (!e) return -1;
        const int v = std::atoi(e);
        return v == 0 || v == 1 || v == 3 ? v : 2;
    }();
    return c;
}

// SABR_SA_PDL=0 launches the level kernels without programmatic dependent launch.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SABR_SA_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

bool pipe_enabled() {  // SABR_SA_PIPE=1: software-pipelined RNG in the C3 level kernel (A/B)
    static const bool on = [] {
        const char* e = std::getenv("SABR_SA_PIPE");
        return e && std::atoi(e) == 1;
    }();
    return on;
}

template <int KIND, int DIMF>
cudaError_t level_t(const SurfaceView& sv, const SaLevelArgs& a, int64_t level, double temp,
                    cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((a.n_local + kLevelThreads - 1) / kLevelThreads);
    const bool all_free = a.fast != 0 && a.free_mask == (1u << DIMF) - 1u &&
                          (KIND == OBJ_BUILTIN || sv.max_abs_lnf <= 700.0);
    const double inv_temp = 1.0 / temp;
    auto run = [&](auto k, size_t smem) {
        cudaError_t e = set_smem(k, smem);
        if (e != cudaSuccess) return e;
        k<<<grid, kLevelThreads, smem, s>>>(sv, a, level, temp, inv_temp);
        return cudaGetLastError();
    };
    if constexpr (KIND != OBJ_BUILTIN) {
        size_t smem = 0;
        const int gk = grid_kind(sv, &smem);
        // default: three chains per thread for the static objective (one warp
        // of 96 chains per CTA: C2 7.28e10 -> 7.47e10 evals/s), two for Case I
        // (three: 1.53e10 -> 1.34e10) and for the per-quote grid
        const int cpt = chains_per_thread() >= 0 ? chains_per_thread()
                                                 : (KIND == OBJ_STATIC && gk == kGridQR ? 3 : 2);
        if ((gk == kGridQR && cpt > 0) || (gk == kGridQuads && cpt == 2)) {
            using K = decltype(&sa_level_multi_kernel<KIND, DIMF, true, kGridQR, 2>);
            const K kq2[2] = {sa_level_multi_kernel<KIND, DIMF, false, kGridQR, 2>,
                              sa_level_multi_kernel<KIND, DIMF, true, kGridQR, 2>};
            const K kq1[2] = {sa_level_multi_kernel<KIND, DIMF, false, kGridQR, 1>,
                              sa_level_multi_kernel<KIND, DIMF, true, kGridQR, 1>};
            const K kp2[2] = {sa_level_multi_kernel<KIND, DIMF, false, kGridQuads, 2>,
                              sa_level_multi_kernel<KIND, DIMF, true, kGridQuads, 2>};
            const K kq3[2] = {sa_level_multi_kernel<KIND, DIMF, false, kGridQR, 3>,
                              sa_level_multi_kernel<KIND, DIMF, true, kGridQR, 3>};
            K k = (gk == kGridQR ? (cpt == 1 ? kq1 : cpt == 3 ? kq3 : kq2) : kp2)[all_free ? 1 : 0];
            // Case I with beta fixed (C3): the one-reflection propose on the
            // searched dims, beta held (FIXM = bit 1); SABR_SA_PIPE=1 adds the
            // software-pipelined RNG (A/B)
            if constexpr (KIND == OBJ_CASE1 && DIMF == 6) {
                if (gk == kGridQR && cpt == 2 && !all_free && a.fast_free != 0 &&
                    a.free_mask == ((1u << DIMF) - 1u & ~2u))
                    k = pipe_enabled() ? sa_level_multi_kernel<KIND, DIMF, false, kGridQR, 2, 2, true>
                        : a.beta_one     ? sa_level_multi_kernel<KIND, DIMF, false, kGridQR, 2, 2, false, true>
                                         : sa_level_multi_kernel<KIND, DIMF, false, kGridQR, 2, 2, false>;
            }
            const int ntc = gk == kGridQR && cpt == 3 ? 3 : (gk == kGridQR && cpt == 1 ? 1 : 2);
            const unsigned threads = static_cast<unsigned>(ntc == 3 ? level_nt<KIND, 3>()
                                                           : ntc == 1 ? level_nt<KIND, 1>() : level_nt<KIND, 2>());
            const unsigned grid = static_cast<unsigned>((a.n_local + threads * ntc - 1) / (threads * ntc));
            cudaError_t e = set_smem(k, smem);
            if (e != cudaSuccess) return e;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, k, sv, a, level, temp, inv_temp);
        }
    }
    if (all_free)
        return dispatch_grid<KIND>(
            sv, [](auto smem) { return sa_level_kernel<KIND, DIMF, true, decltype(smem)::value>; }, run);
    return dispatch_grid<KIND>(
        sv, [](auto smem) { return sa_level_kernel<KIND, DIMF, false, decltype(smem)::value>; }, run);
}

// SABR_SA_PERSIST=0 disables the one-launch path for one-CTA runs (A/B checks).
bool persist_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SABR_SA_PERSIST");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

template <int KIND, int DIMF>
cudaError_t run_small_t(const SurfaceView& sv, const SaLevelArgs& a, const double* temps, int64_t n_levels,
                        cudaStream_t s) {
    constexpr int C = 1;
    if constexpr (KIND == OBJ_BUILTIN) {
        return cudaErrorNotSupported;
    } else {
        size_t smem = 0;
        if (!persist_enabled() || a.nranks != 1 || a.n_local > kLevelThreads / C || grid_kind(sv, &smem) != kGridQR)
            return cudaErrorNotSupported;
        if (temps == nullptr) return cudaSuccess;  // eligibility query
        const bool all_free = a.fast != 0 && a.free_mask == (1u << DIMF) - 1u && sv.max_abs_lnf <= 700.0;
        auto k = all_free ? sa_run_small_kernel<KIND, DIMF, true, kGridQR, C>
                          : sa_run_small_kernel<KIND, DIMF, false, kGridQR, C>;
        cudaError_t e = set_smem(k, smem);
        if (e != cudaSuccess) return e;
        k<<<1, kLevelThreads / C, smem, s>>>(sv, a, temps, n_levels);
        return cudaGetLastError();
    }
}

template <int KIND, int DIMF>
cudaError_t start_t(const SurfaceView& sv, const SaLevelArgs& a, cudaStream_t s) {
    return dispatch_grid<KIND>(
        sv, [](auto smem) { return sa_start_kernel<KIND, DIMF, decltype(smem)::value>; },
        [&](auto k, size_t smem) {
            cudaError_t e = set_smem(k, smem);
            if (e != cudaSuccess) return e;
            k<<<1, 32, smem, s>>>(sv, a);
            return cudaGetLastError();
        });
}

template <int KIND, int DIMF>
cudaError_t cost_t(const SurfaceView& sv, const double* params, int64_t n, double* cost,
                   cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((n + kThreads - 1) / kThreads);
    return dispatch_grid<KIND>(
        sv, [](auto smem) { return cost_batch_kernel<KIND, DIMF, decltype(smem)::value>; },
        [&](auto k, size_t smem) {
            cudaError_t e = set_smem(k, smem);
            if (e != cudaSuccess) return e;
            k<<<grid, kThreads, smem, s>>>(sv, params, n, cost);
            return cudaGetLastError();
        });
}

template <int KIND, int DIMF>
cudaError_t vol_t(const SurfaceView& sv, const double* params, int64_t n, double* vols,
                  cudaStream_t s) {
    int use = 0;
    const size_t smem = smem_for(sv, &use);
    const unsigned grid = static_cast<unsigned>((n + 63) / 64);
    if (use) {
        auto k = vol_batch_kernel<KIND, DIMF, true>;
        cudaError_t e = set_smem(k, smem);
        if (e != cudaSuccess) return e;
        k<<<grid, 64, smem, s>>>(sv, params, n, vols);
    } else {
        vol_batch_kernel<KIND, DIMF, false><<<grid, 64, 0, s>>>(sv, params, n, vols);
    }
    return cudaGetLastError();
}

}  // namespace

int sa_block_threads() { return kLevelThreads; }
int t2_block_threads() { return kThreads; }

#define SABR_DISPATCH(kind, dim, CALL)                                       \
    do {                                                                     \
        if (kind == OBJ_STATIC) return CALL(OBJ_STATIC, 4);                  \
        if (kind == OBJ_CASE1) return CALL(OBJ_CASE1, 6);                    \
        switch (dim) {                                                       \
            case 1: return CALL(OBJ_BUILTIN, 1);                             \
            case 2: return CALL(OBJ_BUILTIN, 2);                             \
            case 3: return CALL(OBJ_BUILTIN, 3);                             \
            case 4: return CALL(OBJ_BUILTIN, 4);                             \
        }                                                                    \
        return cudaErrorInvalidValue;                                        \
    } while (0)

cudaError_t launch_sa_level(int kind, const SurfaceView& sv, const SaLevelArgs& a, int64_t level,
                            double temp, cudaStream_t s) {
#define CALL(K, D) level_t<K, D>(sv, a, level, temp, s)
    SABR_DISPATCH(kind, a.dim_full, CALL);
#undef CALL
}

cudaError_t launch_sa_run_small(int kind, const SurfaceView& sv, const SaLevelArgs& a, const double* temps,
                                int64_t n_levels, cudaStream_t s) {
#define CALL(K, D) run_small_t<K, D>(sv, a, temps, n_levels, s)
    SABR_DISPATCH(kind, a.dim_full, CALL);
#undef CALL
}

cudaError_t launch_sa_start(int kind, const SurfaceView& sv, const SaLevelArgs& a,
                            cudaStream_t s) {
#define CALL(K, D) start_t<K, D>(sv, a, s)
    SABR_DISPATCH(kind, a.dim_full, CALL);
#undef CALL
}

namespace {
__global__ void peer_hello_kernel(PeerMailbox* const* boxes, int nranks, int my_rank, unsigned long long magic) {
    for (int r = 0; r < nranks; ++r) atomicExch_system(&boxes[r]->hello[my_rank], magic);
    __threadfence_system();
}
}  // namespace

cudaError_t launch_peer_hello(PeerMailbox* const* boxes, int nranks, int my_rank, unsigned long long magic,
                              cudaStream_t s) {
    peer_hello_kernel<<<1, 1, 0, s>>>(boxes, nranks, my_rank, magic);
    return cudaGetLastError();
}

cudaError_t launch_sa_merge(const SaLevelArgs& a, const sabr_level_record* recs, int64_t level,
                            cudaStream_t s) {
    sa_merge_kernel<<<1, 1, 0, s>>>(a, recs, level);
    return cudaGetLastError();
}

cudaError_t launch_cost_batch(int kind, const SurfaceView& sv, const double* params,
                              int32_t dim_full, int64_t n, double* cost, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (kind == OBJ_STATIC && dim_full == 4) return cost_t<OBJ_STATIC, 4>(sv, params, n, cost, s);
    if (kind == OBJ_CASE1 && dim_full == 6) return cost_t<OBJ_CASE1, 6>(sv, params, n, cost, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_vol_batch(int kind, const SurfaceView& sv, const double* params,
                             int32_t dim_full, int64_t n, double* vols, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (kind == OBJ_STATIC && dim_full == 4) return vol_t<OBJ_STATIC, 4>(sv, params, n, vols, s);
    if (kind == OBJ_CASE1 && dim_full == 6) return vol_t<OBJ_CASE1, 6>(sv, params, n, vols, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_case2_feasible(const double* params, int64_t n, uint8_t* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    case2_feasible_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(params, n, out);
    return cudaGetLastError();
}

cudaError_t launch_t2_level_init(T2Chain* chains, const sabr_sa_state* st, const T2StepArgs& a,
                                 cudaStream_t s) {
    if (a.n_local <= 0) return cudaSuccess;
    t2_level_init_kernel<<<(a.n_local + 127) / 128, 128, 0, s>>>(chains, st, a);
    return cudaGetLastError();
}

cudaError_t launch_t2_propose(T2Chain* chains, const sabr_sa_state* st, const T2StepArgs& a,
                              double* alpha0, double* beta, uint8_t* active, cudaStream_t s) {
    if (a.n_local <= 0) return cudaSuccess;
    return launch_pdl(t2_propose_kernel, dim3((a.n_local + kProposeChainsPerCta - 1) / kProposeChainsPerCta),
                      dim3(32 * kProposeChainsPerCta), 0, s, chains, st, a, alpha0, beta, active);
}

cudaError_t launch_t2_coef(const T2Chain* chains, const int32_t* idx, const int32_t* n_live, int32_t c0,
                           int32_t n_local, int32_t cand_stride, const double* t_end, const double* dt,
                           const double* sdt, int64_t total_steps, void* coef, int fp32,
                           cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(cand_stride) * total_steps;
    if (n <= 0) return cudaSuccess;
    return launch_pdl(t2_coef_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, chains, idx,
                      n_live, c0, n_local, cand_stride, t_end, dt, sdt, total_steps,
                      fp32 ? nullptr : static_cast<double4*>(coef), fp32 ? static_cast<float4*>(coef) : nullptr,
                      static_cast<int>(fp32 == 2));
}

cudaError_t launch_t2_compact(const uint8_t* active, const double* alpha0, const double* beta, int32_t n,
                              int32_t* idx, double* alpha0_c, double* beta_c, uint8_t* active_c,
                              int32_t* n_live, int* bad_c, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    return launch_pdl(t2_compact_kernel, dim3(1), dim3(kCompactThreads), 0, s, active, alpha0, beta, n, idx,
                      alpha0_c, beta_c, active_c, n_live, bad_c);
}

cudaError_t launch_t2_scatter(const int32_t* idx, const int32_t* n_live, int32_t n, const double* cost_c,
                              const int* bad_c, double* cost, int* bad, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    return launch_pdl(t2_scatter_kernel, dim3((n + 255) / 256), dim3(256), 0, s, idx, n_live, cost_c, bad_c, cost,
                      bad);
}

cudaError_t launch_t2_accept(T2Chain* chains, const T2StepArgs& a, const double* cost,
                             const int* bad, int* nonfinite, cudaStream_t s) {
    if (a.n_local <= 0) return cudaSuccess;
    return launch_pdl(t2_accept_kernel, dim3((a.n_local + 127) / 128), dim3(128), 0, s, chains, a, cost, bad,
                      nonfinite);
}

cudaError_t launch_t2_finish(T2Chain* chains, const T2StepArgs& a, const int32_t* idx, const int32_t* n_live,
                             const double* values, int32_t nq, const double* market, const int* bad_c,
                             int* nonfinite, cudaStream_t s) {
    if (a.n_local <= 0) return cudaSuccess;
    return launch_pdl(t2_finish_kernel, dim3((a.n_local + kFinishWarps - 1) / kFinishWarps), dim3(32 * kFinishWarps),
                      0, s, chains, a, idx, n_live, values, nq, market, bad_c, nonfinite);
}

cudaError_t launch_t2_level_end(const T2Chain* chains, const SaLevelArgs& a, int64_t level,
                                cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, (a.n_local + kThreads - 1) / kThreads));
    t2_level_end_kernel<<<grid, kThreads, 0, s>>>(chains, a, level);
    return cudaGetLastError();
}

}  // namespace sabr_gpu
