// kernels_mc.cu — fused log-Euler SABR Monte Carlo on sm_100a.
//
// One thread simulates `ppt` consecutive paths of one maturity slice for a
// group of CB candidate parameter sets at once: the two uniforms and the
// Box-Muller normals of a path-step are drawn once and shared by all CB
// candidates (the reference's common random numbers: every candidate and
// every slice restarts the same streams, calibration.cpp:404-409, mc.cpp:127).
// Per candidate the scheme is the reference log-Euler step (mc.cpp:87-107)
// carried in log space for the forward (one exp per candidate-step; F_T =
// F_0 exp(sum)).  Payoffs are reduced in-kernel (warp shuffles -> per-warp
// shared accumulators -> one partial per 128*ppt-path tile); a second kernel
// sums the tiles in fixed order.  The reduction tree depends only on
// (num_paths, ppt), so a candidate's price is a pure function of its
// parameters and the plan - never of the batch it was launched in.
#include <math_constants.h>

#include "device_common.cuh"
#include "kernels_mc.hpp"
#include "pdl.cuh"

namespace sabr_gpu {

using namespace sabr_dev;

namespace {

constexpr int kWarps = kMcThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    return v;
}

// Per-warp payoff sums by a shared-memory transpose (both tile kernels, r02): each
// lane writes its discounted payoffs and their squares for 16 (candidate,
// quote, moment) columns as one row of a [32][17] tile; then the two
// half-warps each sum 16 rows of one column and meet with one shuffle.  Per
// value that is one STS, one LDS and one DADD, where two 5-level warp_sum
// trees cost ten shuffles and five DADD; the order (lanes 0-15 and 16-31 in
// four interleaved partial sums each, then the halves) is fixed, so a price
// still depends only on (num_paths, ppt).
constexpr int kTrCols = 16;
constexpr int kTrStride = kTrCols + 1;  // 64-bit rows 17 doubles apart: no bank conflicts

__device__ __forceinline__ void tr_flush(double* __restrict__ tb, double* __restrict__ accw, int base,
                                         int ncols, int lane) {
    __syncwarp();
    const int col = lane & (kTrCols - 1), r0 = lane & kTrCols;  // rows 0-15 or 16-31
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < kTrCols; r += 4) {
        s0 += tb[(r0 + r) * kTrStride + col];
        s1 += tb[(r0 + r + 1) * kTrStride + col];
        s2 += tb[(r0 + r + 2) * kTrStride + col];
        s3 += tb[(r0 + r + 3) * kTrStride + col];
    }
    double s = (s0 + s1) + (s2 + s3);
    const double o = __shfl_xor_sync(0xffffffffu, s, kTrCols);
    s = (lane < kTrCols) ? s + o : o + s;  // the same sum on both halves
    if (lane < ncols) accw[base + lane] += s;
    __syncwarp();
}

// Discounted call payoffs of one path for every (candidate, quote), mc.cpp:265-269,
// added to the warp's accumulators accw[(cc * mq + j) * 2 + {0, 1}].
template <int CB>
__device__ __forceinline__ void payoff_sums_tr(const double (&F)[CB], bool live, uint32_t act_mask,
                                               const double* __restrict__ K, int mq, double disc,
                                               double* __restrict__ tb, double* __restrict__ accw,
                                               int lane) {
    double* row = tb + lane * kTrStride;
    int col = 0, base = 0;
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {
        const bool on = live && ((act_mask >> cc) & 1u);
        for (int j = 0; j < mq; ++j) {
            const double d = F[cc] - __ldg(K + j);
            const double v = on ? disc * ((d < 0.0) ? 0.0 : d) : 0.0;
            row[col] = v;
            row[col + 1] = v * v;
            col += 2;
            if (col == kTrCols) {
                tr_flush(tb, accw, base, kTrCols, lane);
                base += kTrCols;
                col = 0;
            }
        }
    }
    if (col > 0) tr_flush(tb, accw, base, col, lane);
}

// CONST: every slice of the launch has time-invariant step rows (McSlice::
// const_coef): the first row and dt serve every step, no per-step loads.  A
// separate instantiation, so the general kernel's code is unchanged.
template <int CB, bool CONST>
__global__ void __launch_bounds__(kMcThreads, 4) mc_tile_kernel(const __grid_constant__ McParams P) {
    extern __shared__ __align__(16) double acc[];  // [kWarps][CB][mq][2], then [kWarps][32][kTrStride]

    int64_t idx = blockIdx.x;
    const int tile = P.tile_begin + static_cast<int>(idx % P.tile_count);
    idx /= P.tile_count;
    // slice-major over candidate groups, longest slices first (slice_order:
    // slice indices by descending step count), so the longest blocks start in
    // the first waves and the launch ends on short ones
    const int g = static_cast<int>(idx % P.n_groups);
    const int sr = static_cast<int>(idx / P.n_groups);
    const int s = P.slice_order != nullptr ? P.slice_order[sr] : sr;
    const McSlice sl = P.slices[s];
    const int c0 = g * CB;
    const int mq = sl.q_end - sl.q_begin;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // the exp table replicated across the bank groups (device_common.cuh,
    // kExpRep): the CB exp lookups per path-step index it with path-dependent
    // arguments, and a lane reads its own copy - no conflicts (ncu r01: 2.65x
    // the ideal shared wavefronts, short_scoreboard the second stall)
    __shared__ double2 tab[kExpTableSize * kExpRep];
    __shared__ double4 ltab[kLogTableSize];
    __shared__ double2 sctab[kSinCosTableSize];
    for (int i = threadIdx.x; i < kExpTableSize * kExpRep; i += kMcThreads) tab[i] = P.exptab[i / kExpRep];
    for (int i = threadIdx.x; i < kLogTableSize; i += kMcThreads) ltab[i] = P.logtab[i];
    for (int i = threadIdx.x; i < kSinCosTableSize; i += kMcThreads) sctab[i] = P.sctab[i];
    const double2* tab_lane = tab + (lane & (kExpRep - 1));
    // the table staging does not depend on this step's candidates: it
    // overlaps the preceding kernel under PDL (pdl.cuh).  (The jump-ahead
    // ahead of the wait too, as in the FP32 kernel, cost the time-varying
    // 8-candidate instantiation 16 B more stack and C5 FP64 2.5%.)
    pdl_wait();

    // Per candidate: ln(alpha) and (beta - 1).  Every candidate is carried in
    // log space, F = F0 exp(x), alpha = exp(la):
    //   nu_hat = alpha F^(beta-1) = exp(la + (beta-1)(ln F0 + x))   (mc.cpp:99-100)
    //   la    += nu z1 sqrt(dt) - nu^2 dt / 2                         (mc.cpp:97-98)
    //   x     += nu_hat (rho z1 + srho z2) sqrt(dt) - nu_hat^2 dt / 2  (mc.cpp:101-102)
    // Inactive / padding candidates have zero coefficients and are skipped in
    // the payoffs: no per-candidate branch in the step loop.
    uint32_t act_mask = 0;
    double la0[CB], bm1[CB];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {
        const int c = c0 + cc;
        const bool act = c < P.n_cand && (P.active == nullptr || P.active[c] != 0);
        act_mask |= act ? (1u << cc) : 0u;
        la0[cc] = act ? log(P.alpha0[c]) : 0.0;
        bm1[cc] = act ? P.beta[c] - 1.0 : 0.0;
    }
    if (act_mask == 0) return;  // block-uniform
    __syncthreads();            // exp table staged

    const bool reduce = P.partials != nullptr;
    if (reduce) {
        for (int i = threadIdx.x; i < kWarps * CB * mq * 2; i += kMcThreads) acc[i] = 0.0;
        __syncthreads();
    }

    const uint64_t tile_paths = static_cast<uint64_t>(kMcThreads) * P.ppt;
    const uint64_t p0 = static_cast<uint64_t>(tile) * tile_paths + static_cast<uint64_t>(threadIdx.x) * P.ppt;

    Xoshiro rng;
    if (P.rng == SABR_RNG_XOSHIRO && p0 < P.num_paths) {
        // block b of the plan, mc.cpp:126-127; jump to this thread's first path
        rng.init(P.seed, p0 / P.block_size);
        const uint64_t k = (p0 % P.block_size) / P.ppt;
        const uint64_t* poly = P.jump + 4 * (sl.jump_off + static_cast<int64_t>(k));
        uint64_t pl[4] = {poly[0], poly[1], poly[2], poly[3]};
        rng.jump(pl);
    }

    const int64_t cstride = P.cand_stride;
    const StepCoef* __restrict__ crow0 = P.coef + static_cast<int64_t>(sl.step_off) * cstride + c0;
    const double* __restrict__ hdt = P.hdt + sl.step_off;
    const double lnf0 = sl.lnf0;

    for (int k = 0; k < P.ppt; ++k) {
        const uint64_t path = p0 + k;
        const bool live = path < P.num_paths;
        double la[CB], x[CB];
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
            la[cc] = la0[cc];
            x[cc] = 0.0;
        }
        if (live) {
            // normals of step i (box_muller, mc.cpp:30-36) from the path's stream
            auto normals = [&](int i, double& z1, double& z2) {
                double ua, ub;
                if (P.rng == SABR_RNG_XOSHIRO) {
                    ua = rng.uniform();
                    ub = rng.uniform();
                } else {
                    philox_uniform_pair(P.seed, path, static_cast<uint32_t>(i), ua, ub);
                }
                box_muller_tab(ua, ub, ltab, sctab, z1, z2);
            };
            // all candidates' log-Euler step with the shared normals; each
            // candidate's coefficients of the NEXT step are loaded right after
            // its current ones are used (rolling prefetch: the L1 latency of
            // these uniform loads was the top stall, long_scoreboard)
            double2 qa[CB], qb[CB];
            auto load_row = [&](const StepCoef* row, int cc) {
                qa[cc] = __ldg(reinterpret_cast<const double2*>(row + cc));
                qb[cc] = __ldg(reinterpret_cast<const double2*>(row + cc) + 1);
            };
            auto advance_all = [&](double h, double z1, double z2, const StepCoef* next) {
#pragma unroll
                for (int cc = 0; cc < CB; ++cc) {
                    // beta == 1 (mc.cpp:99-100: nu_hat = alpha): bm1 = 0 exactly,
                    // so the fma returns la exactly for any finite x - no select
                    const double arg = fma(bm1[cc], lnf0 + x[cc], la[cc]);
                    const double nh = exp_mc<kExpRep>(arg, tab_lane);
                    la[cc] += fma(qa[cc].x, z1, -qa[cc].y);
                    const double u = fma(qb[cc].y, z2, qb[cc].x * z1);
                    x[cc] = fma(nh, fma(-nh, h, u), x[cc]);
                    if (next != nullptr) load_row(next, cc);
                }
            };
            // software pipeline: the (serial) Box-Muller chain of step i+1 is
            // independent of the candidate updates of step i, so both sit in
            // one basic block; the draw order is the reference's (2 per step)
            // and the last step is peeled so consecutive paths of a thread
            // continue the block stream exactly.
            const StepCoef* crow = crow0;
#pragma unroll
            for (int cc = 0; cc < CB; ++cc) load_row(crow, cc);
            double h = __ldg(hdt);
            double z1, z2;
            normals(0, z1, z2);
            const int n = sl.n_steps;
            if constexpr (CONST) {
                for (int i = 0; i + 1 < n; ++i) {
                    double n1, n2;
                    normals(i + 1, n1, n2);
                    advance_all(h, z1, z2, nullptr);
                    z1 = n1;
                    z2 = n2;
                }
            } else {
                for (int i = 0; i + 1 < n; ++i) {
                    double n1, n2;
                    normals(i + 1, n1, n2);
                    const double hn = __ldg(hdt + i + 1);
                    crow += cstride;
                    advance_all(h, z1, z2, crow);
                    h = hn;
                    z1 = n1;
                    z2 = n2;
                }
            }
            advance_all(h, z1, z2, nullptr);
        }
        double F[CB];
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
            F[cc] = sl.forward0 * exp_tab<kExpRep>(x[cc], tab_lane);
            if (live && ((act_mask >> cc) & 1u) && !isfinite(F[cc])) atomicOr(P.bad + c0 + cc, 1);  // mc.cpp:133-138
        }
        if (P.terminals != nullptr && live) P.terminals[path] = F[0];
        if (!reduce) continue;
        // discounted call payoffs, mc.cpp:265-269, summed over the warp
        payoff_sums_tr<CB>(F, live, act_mask, P.strikes + sl.q_begin, mq, sl.discount,
                           acc + kWarps * CB * mq * 2 + warp * 32 * kTrStride, acc + warp * CB * mq * 2, lane);
    }
    if (!reduce) return;
    __syncthreads();
    // warps in fixed order -> one partial per (candidate, quote, tile)
    for (int t = threadIdx.x; t < CB * mq; t += kMcThreads) {
        const int cc = t / mq, j = t % mq;
        if (c0 + cc >= P.n_cand) continue;
        double s1 = 0.0, s2 = 0.0;
        for (int w = 0; w < kWarps; ++w) {
            s1 += acc[((w * CB + cc) * mq + j) * 2];
            s2 += acc[((w * CB + cc) * mq + j) * 2 + 1];
        }
        double* out = P.partials +
                      ((static_cast<int64_t>(tile) * P.n_cand + c0 + cc) * P.n_quotes + sl.q_begin + j) * 2;
        out[0] = s1;
        out[1] = s2;
    }
}

// The FP32 fast path (SABR_FP32): the same streams, the reference's log-Euler
// step in FP32 state, one MUFU ex2 per candidate-step; F_T and the payoff
// sums in FP64.  r02: the state is carried in base-2 logarithms,
//   A = log2(alpha) + (beta - 1) log2(F0)   (so nu_hat = 2^(A + (beta-1) Y))
//   Y = log2(F / F0),
// with the coefficients pre-scaled by log2(e) (kernels_sa.cu t2_coef_kernel,
// engine.cu set_coefficients), so a candidate-step is
//   nu_hat = ex2(fma(beta - 1, Y, A));  A += c1 z1 - c2;
//   Y += nu_hat (rs z1 + ss z2 - nu_hat h)
// and two candidates share every instruction but the ex2 as packed FP32x2
// (FFMA2 / FADD2 / FMUL2, the normals as broadcast operands): 4.5 instead of
// 10 instructions per candidate-step.  CB >= 2 reads the pair-interleaved
// coefficient rows (McParams::coef32_pairs): per pair and step
// {c1 c1' -c2 -c2'} {rs rs' ss ss'}; CB = 1 reads {c1 -c2 rs ss}.
// CTAs per SM of the FP32 kernel: its packed state fits 76 (time-invariant
// rows) / 95 registers without spills in the step loop at CB <= 8, so 6 / 5
// CTAs (24 / 20 warps per SM) hide the MUFU and FFMA2 latencies (r02: at 4
// CTAs ncu showed 1.4 eligible warps per scheduler, "wait" the top stall);
// at CB = 16, 4 (time-invariant, SMQ) / 5 (time-varying, WQ + KSM)
template <int CB, bool CONST>
constexpr int f32_min_ctas() { return CB <= 8 ? (CONST ? 6 : 5) : (CONST ? 4 : 5); }

// one float4 of shared memory, re-read at every use (asm volatile: the
// compiler may not keep it in registers across the step loop)
__device__ __forceinline__ float4 lds_f4(const float4* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
    return v;
}

template <int CB, bool CONST>
__global__ void __launch_bounds__(kMcThreads, f32_min_ctas<CB, CONST>())
    mc_tile_kernel_f32(const __grid_constant__ McParams P) {
    extern __shared__ __align__(16) double acc[];  // [kWarps][CB][mq][2], then [kWarps][32][kTrStride]
    constexpr int NP = (CB + 1) / 2;                // candidate pairs (CB = 1: one, its odd half idle)

    int64_t idx = blockIdx.x;
    const int tile = P.tile_begin + static_cast<int>(idx % P.tile_count);
    idx /= P.tile_count;
    // slice-major over candidate groups, longest slices first (slice_order:
    // slice indices by descending step count), so the longest blocks start in
    // the first waves and the launch ends on short ones
    const int g = static_cast<int>(idx % P.n_groups);
    const int sr = static_cast<int>(idx / P.n_groups);
    const int s = P.slice_order != nullptr ? P.slice_order[sr] : sr;
    const McSlice sl = P.slices[s];
    const int c0 = g * CB;
    const int mq = sl.q_end - sl.q_begin;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t tile_paths = static_cast<uint64_t>(kMcThreads) * P.ppt;
    const uint64_t p0 = static_cast<uint64_t>(tile) * tile_paths + static_cast<uint64_t>(threadIdx.x) * P.ppt;

    Xoshiro rng{};  // zero state for a path past num_paths (WQ runs its step loop too)
    if (P.rng == SABR_RNG_XOSHIRO && p0 < P.num_paths) {
        rng.init(P.seed, p0 / P.block_size);
        const uint64_t k = (p0 % P.block_size) / P.ppt;
        const uint64_t* poly = P.jump + 4 * (sl.jump_off + static_cast<int64_t>(k));
        uint64_t pl[4] = {poly[0], poly[1], poly[2], poly[3]};
        rng.jump(pl);
    }
    // the streams' jump-ahead does not depend on this step's candidates: it
    // overlaps the preceding kernel under PDL (pdl.cuh)
    pdl_wait();

    uint32_t act_mask = 0;
    float2 a0[NP], bm1[NP];
#pragma unroll
    for (int cc = 0; cc < 2 * NP; ++cc) {
        const int c = c0 + cc;
        const bool act = cc < CB && c < P.n_cand && (P.active == nullptr || P.active[c] != 0);
        act_mask |= act ? (1u << cc) : 0u;
        const double b1 = act ? P.beta[c] - 1.0 : 0.0;
        const float a = act ? static_cast<float>((log(P.alpha0[c]) + b1 * sl.lnf0) * 1.4426950408889634) : 0.0f;
        if (cc & 1) {
            a0[cc >> 1].y = a;
            bm1[cc >> 1].y = static_cast<float>(b1);
        } else {
            a0[cc >> 1].x = a;
            bm1[cc >> 1].x = static_cast<float>(b1);
        }
    }
    if (act_mask == 0) return;  // block-uniform
    // 16 candidates with time-varying rows: the per-pair constants in shared
    // memory too (KSM), read where used instead of holding 32 registers, so
    // the kernel fits 96 registers and 5 CTAs per SM (C5 FP32 +7%; in the
    // time-invariant instantiation the same move cost registers elsewhere)
    constexpr bool KSM = !CONST && CB >= 16;
    __shared__ float2 ksh[2][KSM ? NP : 1];  // [0] A at x = 0, [1] beta - 1
    if constexpr (KSM) {
        if (threadIdx.x == 0) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                ksh[0][p] = a0[p];
                ksh[1][p] = bm1[p];
            }
        }
        __syncthreads();
    }

    const bool reduce = P.partials != nullptr;
    double* tb = acc + kWarps * CB * mq * 2 + warp * 32 * kTrStride;
    if (reduce) {
        for (int i = threadIdx.x; i < kWarps * CB * mq * 2; i += kMcThreads) acc[i] = 0.0;
        __syncthreads();
    }


    // coefficient rows as float4: CB >= 2 two per pair (pair layout), CB = 1 one
    constexpr int NQ = CB >= 2 ? 2 * NP : 1;
    const int64_t rstride = P.cand_stride;  // float4s per step row (CB >= 2: cand_stride is even)
    const float4* __restrict__ crow0 = P.coef32 + static_cast<int64_t>(sl.step_off) * rstride + c0;
    const double* __restrict__ hdt = P.hdt + sl.step_off;
    // SMQ (time-invariant rows at 16 candidates): the block's one coefficient
    // row lives in shared memory and is read (broadcast) at every step instead
    // of holding 64 registers: fewer spills at 128 registers, C4 FP32 +1.8%
    // (more CTAs per SM still spill: 5 CTAs at 96 registers ran 42% slower)
    constexpr bool SMQ = CONST && CB >= 16;
    __shared__ float4 qsh[SMQ ? NQ : 1];
    // WQ (time-varying rows at 16 candidates): each warp stages the next
    // step's row in a shared double buffer (lane l < NQ loads element l), and
    // every lane reads it from there: one float4 of prefetch per lane instead
    // of the two 64-register row buffers
    constexpr bool WQ = !CONST && CB >= 16;
    __shared__ float4 wq[WQ ? kWarps : 1][2][WQ ? NQ : 1];
    int wbuf = 0;
    if constexpr (SMQ) {
        if (threadIdx.x < NQ) qsh[threadIdx.x] = crow0[threadIdx.x];
        __syncthreads();
    }

    for (int k = 0; k < P.ppt; ++k) {
        const uint64_t path = p0 + k;
        const bool live = path < P.num_paths;
        float2 A[NP], Y[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            A[p] = KSM ? ksh[0][p] : a0[p];
            Y[p] = make_float2(0.0f, 0.0f);
        }
        // WQ: every lane runs the step loop (its __syncwarp needs the whole warp);
        // a path past num_paths is simulated on an unused stream and never priced
        if (live || WQ) {
            auto normals = [&](int i, float& z1, float& z2) {
                uint64_t na, nb;  // the step's two draws, in the reference's order
                if (P.rng == SABR_RNG_XOSHIRO) {
                    na = rng.next();
                    nb = rng.next();
                } else {
                    philox_bits_pair(P.seed, path, static_cast<uint32_t>(i), na, nb);
                }
                box_muller_f32_bits(na, nb, z1, z2);  // box_muller, mc.cpp:30-36
            };
            // q[2p] = {c1, c1', -c2, -c2'}, q[2p+1] = {rs, rs', ss, ss'} (CB = 1: q[0] = {c1, -c2, rs, ss})
            auto advance_all = [&](float nh_scale, const float4 (&q)[NQ], float z1, float z2) {
                const float2 Z1 = make_float2(z1, z1), Z2 = make_float2(z2, z2);
                const float2 H = make_float2(nh_scale, nh_scale);  // -h log2(e)
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    float2 c1, nc2, rs, ss;
                    if constexpr (SMQ || WQ) {
                        const float4* src = SMQ ? qsh : wq[WQ ? warp : 0][wbuf];
                        const float4 qa = lds_f4(src + 2 * p), qb = lds_f4(src + 2 * p + 1);
                        c1 = make_float2(qa.x, qa.y);
                        nc2 = make_float2(qa.z, qa.w);
                        rs = make_float2(qb.x, qb.y);
                        ss = make_float2(qb.z, qb.w);
                    } else if constexpr (CB >= 2) {
                        c1 = make_float2(q[2 * p].x, q[2 * p].y);
                        nc2 = make_float2(q[2 * p].z, q[2 * p].w);
                        rs = make_float2(q[2 * p + 1].x, q[2 * p + 1].y);
                        ss = make_float2(q[2 * p + 1].z, q[2 * p + 1].w);
                    } else {
                        c1 = make_float2(q[0].x, 0.0f);
                        nc2 = make_float2(q[0].y, 0.0f);
                        rs = make_float2(q[0].z, 0.0f);
                        ss = make_float2(q[0].w, 0.0f);
                    }
                    float2 b1;
                    if constexpr (KSM) {
                        float x, y;
                        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                                     : "=f"(x), "=f"(y)
                                     : "r"(static_cast<unsigned>(__cvta_generic_to_shared(&ksh[1][p]))));
                        b1 = make_float2(x, y);
                    } else {
                        b1 = bm1[p];
                    }
                    const float2 arg = __ffma2_rn(b1, Y[p], A[p]);
                    float2 nh;  // 2^arg, MUFU.EX2 (flush-to-zero: no denormal rescaling)
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(nh.x) : "f"(arg.x));
                    if constexpr (CB >= 2) asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(nh.y) : "f"(arg.y));
                    else nh.y = 0.0f;
                    A[p] = __fadd2_rn(__ffma2_rn(c1, Z1, A[p]), nc2);
                    const float2 u = __ffma2_rn(ss, Z2, __fmul2_rn(rs, Z1));
                    Y[p] = __ffma2_rn(nh, __ffma2_rn(nh, H, u), Y[p]);
                }
            };
            auto load = [&](float4 (&q)[NQ], const float4* row) {
#pragma unroll
                for (int i = 0; i < NQ; ++i) q[i] = __ldg(row + i);
            };
            float4 q[NQ], qn[NQ];
            const float4* crow = crow0;
            if constexpr (!SMQ && !WQ) load(qn, crow);
            float hn = static_cast<float>(-__ldg(hdt) * 1.4426950408889634);
            float z1, z2;
            normals(0, z1, z2);
            const int n = sl.n_steps;
            if constexpr (CONST) {  // time-invariant rows (McSlice::const_coef): loaded once
#pragma unroll 2
                for (int i = 0; i + 1 < n; ++i) {
                    float n1, n2;
                    normals(i + 1, n1, n2);
                    advance_all(hn, qn, z1, z2);
                    z1 = n1;
                    z2 = n2;
                }
                advance_all(hn, qn, z1, z2);
            } else if constexpr (WQ) {
                if (lane < NQ) wq[warp][0][lane] = __ldg(crow0 + lane);
                wbuf = 0;
                __syncwarp();
                float h = hn;
                for (int i = 0; i + 1 < n; ++i) {
                    const float4 pf = lane < NQ ? __ldg(crow0 + static_cast<int64_t>(i + 1) * rstride + lane)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                    hn = static_cast<float>(-__ldg(hdt + i + 1) * 1.4426950408889634);
                    float n1, n2;
                    normals(i + 1, n1, n2);
                    advance_all(h, qn, z1, z2);
                    if (lane < NQ) wq[warp][wbuf ^ 1][lane] = pf;
                    __syncwarp();
                    wbuf ^= 1;
                    h = hn;
                    z1 = n1;
                    z2 = n2;
                }
                advance_all(h, qn, z1, z2);
                __syncwarp();  // the last reads before the next path re-stages buffer 0
            } else {
            // unrolled by 2 so the q <- qn rotation is register renaming;
            // step i+1's row is loaded while step i computes
#pragma unroll 2
            for (int i = 0; i + 1 < n; ++i) {
#pragma unroll
                for (int t = 0; t < NQ; ++t) q[t] = qn[t];
                const float h = hn;
                crow += rstride;
                load(qn, crow);
                hn = static_cast<float>(-__ldg(hdt + i + 1) * 1.4426950408889634);
                float n1, n2;
                normals(i + 1, n1, n2);
                advance_all(h, q, z1, z2);
                z1 = n1;
                z2 = n2;
            }
            advance_all(hn, qn, z1, z2);
            }
        }
        double F[CB];
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
            const float y = (cc & 1) ? Y[cc >> 1].y : Y[cc >> 1].x;
            F[cc] = sl.forward0 * exp2(static_cast<double>(y));
            if (live && ((act_mask >> cc) & 1u) && !isfinite(F[cc])) atomicOr(P.bad + c0 + cc, 1);
        }
        if (P.terminals != nullptr && live) P.terminals[path] = F[0];
        if (!reduce) continue;
        payoff_sums_tr<CB>(F, live, act_mask, P.strikes + sl.q_begin, mq, sl.discount, tb,
                           acc + warp * CB * mq * 2, lane);
    }
    if (!reduce) return;
    __syncthreads();
    for (int t = threadIdx.x; t < CB * mq; t += kMcThreads) {
        const int cc = t / mq, j = t % mq;
        if (c0 + cc >= P.n_cand) continue;
        double s1 = 0.0, s2 = 0.0;
        for (int w = 0; w < kWarps; ++w) {
            s1 += acc[((w * CB + cc) * mq + j) * 2];
            s2 += acc[((w * CB + cc) * mq + j) * 2 + 1];
        }
        double* out = P.partials +
                      ((static_cast<int64_t>(tile) * P.n_cand + c0 + cc) * P.n_quotes + sl.q_begin + j) * 2;
        out[0] = s1;
        out[1] = s2;
    }
}

// price_cliquet (mc.cpp:275-320): the path is observed at the reset nodes
// (run_path records F after step i+1 == node, mc.cpp:104-105) and the payoff
// sum_j clamp((S_j - S_{j-1}) / S_{j-1}, local) -> clamp(., global) is
// accumulated on the fly (mc.cpp:308-318); discounted payoffs reduced as in
// the European tile kernel (one partial per tile).
__global__ void __launch_bounds__(kMcThreads) mc_cliquet_kernel(const __grid_constant__ McParams P,
                                                                 const __grid_constant__ CliquetSpecDev C) {
    __shared__ double acc[kWarps][2];
    __shared__ double2 tab[kExpTableSize];
    __shared__ double4 ltab[kLogTableSize];
    __shared__ double2 sctab[kSinCosTableSize];
    for (int i = threadIdx.x; i < kExpTableSize; i += kMcThreads) tab[i] = P.exptab[i];
    for (int i = threadIdx.x; i < kLogTableSize; i += kMcThreads) ltab[i] = P.logtab[i];
    for (int i = threadIdx.x; i < kSinCosTableSize; i += kMcThreads) sctab[i] = P.sctab[i];
    if (threadIdx.x < kWarps * 2) (&acc[0][0])[threadIdx.x] = 0.0;
    __syncthreads();
    const int tile = blockIdx.x;
    const McSlice sl = P.slices[0];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool logn = P.beta[0] == 1.0;
    const double bm1 = P.beta[0] - 1.0;
    const double la0 = log(P.alpha0[0]);
    const uint64_t p0 = static_cast<uint64_t>(tile) * kMcThreads * P.ppt + static_cast<uint64_t>(threadIdx.x) * P.ppt;
    Xoshiro rng;
    if (P.rng == SABR_RNG_XOSHIRO && p0 < P.num_paths) {
        rng.init(P.seed, p0 / P.block_size);
        const uint64_t* poly = P.jump + 4 * (sl.jump_off + static_cast<int64_t>((p0 % P.block_size) / P.ppt));
        uint64_t pl[4] = {poly[0], poly[1], poly[2], poly[3]};
        rng.jump(pl);
    }
    // an observation at node 0 is never recorded by run_path: the reference
    // then observes nothing at all (mc.cpp:104), all observations stay 0
    const bool none = C.n_obs > 0 && C.obs_node[0] == 0;
    for (int k = 0; k < P.ppt; ++k) {
        const uint64_t path = p0 + k;
        const bool live = path < P.num_paths;
        double v = 0.0;
        if (live) {
            double la = la0, x = 0.0, s_prev = 0.0, strip = 0.0;
            bool finite = true;
            int next = 0;
            if (none) {
                // all rows 0: ret = (0 - 0) / 0 for every pair
                for (int j = 1; j < C.n_obs; ++j) {
                    const double ret = (0.0 - 0.0) / 0.0;
                    strip += (ret < C.local_floor) ? C.local_floor : (C.local_cap < ret) ? C.local_cap : ret;
                }
                next = C.n_obs;  // still draw the whole path: later paths continue the stream
            }
            for (int i = 0; i < sl.n_steps; ++i) {
                double ua, ub;
                if (P.rng == SABR_RNG_XOSHIRO) {
                    ua = rng.uniform();
                    ub = rng.uniform();
                } else {
                    philox_uniform_pair(P.seed, path, static_cast<uint32_t>(i), ua, ub);
                }
                double z1, z2;
                box_muller_tab(ua, ub, ltab, sctab, z1, z2);
                const StepCoef q = P.coef[sl.step_off + i];
                const double nh = exp_mc(logn ? la : fma(bm1, sl.lnf0 + x, la), tab);
                la += fma(q.c1, z1, -q.c2);
                const double u = fma(q.ss, z2, q.rs * z1);
                x = fma(nh, fma(-nh, __ldg(P.hdt + sl.step_off + i), u), x);
                if (next < C.n_obs && C.obs_node[next] == i + 1) {
                    const double F = sl.forward0 * exp_tab(x, tab);
                    finite = finite && isfinite(F);
                    const double s_cur = F * C.obs_discount[next];
                    if (next > 0) {
                        const double ret = (s_cur - s_prev) / s_prev;
                        strip += (ret < C.local_floor) ? C.local_floor : (C.local_cap < ret) ? C.local_cap : ret;
                    }
                    s_prev = s_cur;
                    ++next;
                }
            }
            if (!finite) atomicOr(P.bad, 1);  // mc.cpp:133-138
            const double g = (strip < C.global_floor) ? C.global_floor : (C.global_cap < strip) ? C.global_cap : strip;
            v = sl.discount * g;
        }
        const double s1 = warp_sum(v);
        const double s2 = warp_sum(v * v);
        if (lane == 0) {
            acc[warp][0] += s1;
            acc[warp][1] += s2;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s1 = 0.0, s2 = 0.0;
        for (int w = 0; w < kWarps; ++w) {
            s1 += acc[w][0];
            s2 += acc[w][1];
        }
        P.partials[static_cast<int64_t>(tile) * 2] = s1;
        P.partials[static_cast<int64_t>(tile) * 2 + 1] = s2;
    }
}

// reduce_payoffs (mc.cpp:146-157) over the tiles.  Block (X, G): threadIdx.x
// picks one of X consecutive (candidate, quote) columns (coalesced: the
// partials are tile-major), threadIdx.y one of G tile groups; group y sums
// tiles y, y + G, y + 2G, ... in order, then the G group sums are added in
// group order.  G depends only on n_tiles (a function of num_paths and ppt),
// so a price is still a pure function of the plan.  r02: with one thread per
// column (G = 1) C4's 672 columns ran as 6 CTAs walking 782 tiles each, 88 us
// per SA step, latency-bound; G = 32 spreads the walk over 32x the threads
// (a single-candidate price of 2^24 paths: 32768 tiles, G = 256).
constexpr int kReduceThreads = 256;
__host__ __device__ inline int reduce_groups(int n_tiles) {
    int g = 1;
    while (g < kReduceThreads && g * 2 * 24 <= n_tiles) g *= 2;  // >= 24 tiles per group
    return g;
}

__global__ void __launch_bounds__(kReduceThreads) mc_reduce_kernel(const McParams P, double* __restrict__ value,
                                                                   double* __restrict__ std_error) {
    __shared__ double2 part[kReduceThreads];
    pdl_wait();
    pdl_trigger();
    const int G = blockDim.y, X = blockDim.x;
    const int64_t ncol = static_cast<int64_t>(P.n_cand) * P.n_quotes;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * X + threadIdx.x;
    const bool on = t < ncol && (P.active == nullptr || P.active[t / P.n_quotes] != 0);
    const int64_t stride = ncol * 2;
    double s1 = 0.0, s2 = 0.0;
    if (on) {
        const double* p = P.partials + t * 2;
        int k = threadIdx.y;
        // 8 tiles' loads in flight per round trip, the additions in tile order
        for (; k + 7 * G < P.n_tiles; k += 8 * G) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const double2*>(p + (k + u * G) * stride);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                s1 += v[u].x;
                s2 += v[u].y;
            }
        }
        for (; k < P.n_tiles; k += G) {
            const double2 v = *reinterpret_cast<const double2*>(p + k * stride);
            s1 += v.x;
            s2 += v.y;
        }
    }
    if (G > 1) {
        part[threadIdx.y * X + threadIdx.x] = make_double2(s1, s2);
        __syncthreads();
        if (threadIdx.y != 0) return;
        s1 = 0.0;
        s2 = 0.0;
        for (int y = 0; y < G; ++y) {
            const double2 v = part[y * X + threadIdx.x];
            s1 += v.x;
            s2 += v.y;
        }
    }
    if (!on) return;
    const double n = static_cast<double>(P.num_paths);
    const double mean = s1 / n;
    const double q = (s2 - n * mean * mean) / (n - 1.0);
    const double var = (0.0 < q) ? q : 0.0;
    value[t] = mean;
    if (std_error) std_error[t] = sqrt(var / n);
}

// case2_mc_cost, calibration.cpp:410-413: sum over slices and quotes in order.
__global__ void mc_cost_kernel(const McParams P, const double* __restrict__ value,
                               const double* __restrict__ market, double* __restrict__ cost) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P.n_cand) return;
    if (P.active != nullptr && P.active[c] == 0) return;
    cost[c] = mc_quote_cost(value + static_cast<int64_t>(c) * P.n_quotes, market, P.n_quotes);
}


template <int CB>
cudaError_t tiles_t(const McParams& p, cudaStream_t s) {
    const int mq = p.max_q;
    // the warps' payoff transpose tiles follow the accumulators (payoff_sums_tr)
    const size_t smem = p.partials ? (static_cast<size_t>(kWarps) * CB * mq * 2 +
                                      static_cast<size_t>(kWarps) * 32 * kTrStride) * sizeof(double)
                                   : 0;
    bool cst = p.n_slices > 0;
    for (int i = 0; i < p.n_slices; ++i) cst = cst && p.host_slices != nullptr && p.host_slices[i].const_coef;
    auto k = p.fp32 ? (cst ? mc_tile_kernel_f32<CB, true> : mc_tile_kernel_f32<CB, false>)
                    : (cst ? mc_tile_kernel<CB, true> : mc_tile_kernel<CB, false>);
    // the FP64 kernel's 22 KB of static tables leave 26 KB of dynamic shared
    // memory by default: opt in to the size this launch needs
    if (smem > 16 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    McParams q = p;
    if (q.tile_count <= 0) {
        q.tile_begin = 0;
        q.tile_count = q.n_tiles;
    }
    const int n_groups = (q.n_cand + CB - 1) / CB;
    q.n_groups = n_groups;
    const int64_t blocks = static_cast<int64_t>(q.tile_count) * q.n_slices * n_groups;
    if (blocks <= 0) return cudaSuccess;
    return launch_pdl(k, dim3(static_cast<unsigned>(blocks)), dim3(kMcThreads), smem, s, q);
}

}  // namespace

// Shared memory of one tile CTA at CB candidates and max_q quotes per slice:
// the warps' payoff accumulators and transpose tiles (dynamic) plus, in FP64,
// the exp / log / sincos tables (static), against the 227 KB a CTA can opt in
// to.  The largest CB that fits, 0 when even one candidate does not.
int mc_max_cand_block(int max_q, bool fp32) {
    constexpr size_t kLimit = 227 * 1024;
    const size_t tables = fp32 ? 0
                               : sizeof(double2) * kExpTableSize * kExpRep + sizeof(double4) * kLogTableSize +
                                     sizeof(double2) * kSinCosTableSize;
    for (int cb : {16, 8, 4, 2, 1}) {
        const size_t dyn = (static_cast<size_t>(kWarps) * cb * max_q * 2 + static_cast<size_t>(kWarps) * 32 * kTrStride) *
                           sizeof(double);
        if (tables + dyn + 1024 <= kLimit) return cb;
    }
    return 0;
}

cudaError_t launch_mc_tiles(const McParams& p, int cand_block, cudaStream_t s) {
    switch (cand_block) {
        case 1: return tiles_t<1>(p, s);
        case 2: return tiles_t<2>(p, s);
        case 4: return tiles_t<4>(p, s);
        case 8: return tiles_t<8>(p, s);
        case 16: return tiles_t<16>(p, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_mc_cliquet(const McParams& p, const CliquetSpecDev& spec, cudaStream_t s) {
    if (p.n_tiles <= 0) return cudaSuccess;
    mc_cliquet_kernel<<<static_cast<unsigned>(p.n_tiles), kMcThreads, 0, s>>>(p, spec);
    return cudaGetLastError();
}

// {RN(2^(i/128)), RN(2^(i/128) - hi)} from x86 long double (64-bit mantissa):
// the table behind exp_tab, accurate to ~2^-64 relative.
const double2* exp_table_host() {
    static double2 table[kExpTableSize];
    static bool built = false;
    if (!built) {
        for (int i = 0; i < kExpTableSize; ++i) {
            const long double v = exp2l(static_cast<long double>(i) / kExpTableSize);
            const double hi = static_cast<double>(v);
            table[i] = make_double2(hi, static_cast<double>(v - static_cast<long double>(hi)));
        }
        built = true;
    }
    return table;
}

// {RN(1/c_i), -log(RN(1/c_i)) as hi + lo} for the 128 intervals of log_tab
// (device_common.cuh), c_i the interval centre; x86 long double.
const double4* log_table_host() {
    static double4 table[kLogTableSize];
    static bool built = false;
    if (!built) {
        for (int i = 0; i < kLogTableSize; ++i) {
            const double c = bitsd(0x3fe6000000000000ull + (static_cast<uint64_t>(i) << 45) + (1ull << 44));
            // the two intervals around 1 use invc = 1 exactly: r = z - 1 is then
        // exact and nothing cancels as log x -> 0
        const double invc = (i == kLogOne - 1 || i == kLogOne) ? 1.0
                                                                : static_cast<double>(1.0L / static_cast<long double>(c));
            const long double nl = -logl(static_cast<long double>(invc));
            // hi on a 2^-42 grid: k*ln2_hi + hi is then exact for every |k| < 2^10
        const double hi = static_cast<double>(roundl(nl * 0x1.0p42L) * 0x1.0p-42L);
            table[i] = make_double4(invc, hi, static_cast<double>(nl - static_cast<long double>(hi)), 0.0);
        }
        built = true;
    }
    return table;
}

// {sin(pi k/64), cos(pi k/64)}, k = 0..127, for sincos_2pi (device_common.cuh).
const double2* sincos_table_host() {
    static double2 table[kSinCosTableSize];
    static bool built = false;
    if (!built) {
        const long double pi = 3.141592653589793238462643383279502884L;
        for (int k = 0; k < kSinCosTableSize; ++k)
            table[k] = make_double2(static_cast<double>(sinl(pi * k / 64)), static_cast<double>(cosl(pi * k / 64)));
        built = true;
    }
    return table;
}

cudaError_t launch_mc_reduce(const McParams& p, double* value, double* std_error,
                             const double* market, double* cost, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(p.n_cand) * p.n_quotes;
    if (n > 0) {
        const int G = reduce_groups(p.n_tiles), X = kReduceThreads / G;
        cudaError_t e = launch_pdl(mc_reduce_kernel, dim3(static_cast<unsigned>((n + X - 1) / X)), dim3(X, G), 0, s,
                                   p, value, std_error);
        if (e != cudaSuccess) return e;
    }
    if (cost != nullptr && p.n_cand > 0) {
        return launch_pdl(mc_cost_kernel, dim3((p.n_cand + 127) / 128), dim3(128), 0, s, p, value, market, cost);
    }
    return cudaSuccess;
}

}  // namespace sabr_gpu
