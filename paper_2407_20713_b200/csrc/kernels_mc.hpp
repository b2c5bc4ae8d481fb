// kernels_mc.hpp — host-visible interface of the log-Euler Monte Carlo kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sabr_gpu {

// One maturity slice of a Monte Carlo launch.  Steps of slice s occupy
// [step_off, step_off + n_steps) of the per-candidate coefficient rows.
struct McSlice {
    int32_t n_steps;
    int32_t step_off;
    int32_t q_begin;   // strikes [q_begin, q_end) of the launch's strike list
    int32_t q_end;
    int64_t jump_off;  // xoshiro mode: first polynomial of this slice's jump table
    double forward0;   // S*exp((r-y)T), mc.cpp:258
    double lnf0;       // log(forward0)
    double discount;   // exp(-rT), mc.cpp:262
    int32_t const_coef;  // every step row of this slice equals its first (time-invariant
                         // dynamics on a uniform grid): the FP64 kernel loads it once
    int32_t _pad;
};

// Per-step, per-candidate log-Euler coefficients (mc.cpp:97-102) for the
// grid of build_grid (mc.cpp:50-84):
//   c1 = nu(t_end)*sqrt(dt), c2 = nu^2*dt/2, rs = rho*sqrt(dt), ss = srho*sqrt(dt)
struct __align__(16) StepCoef {
    double c1, c2, rs, ss;
};

struct McParams {
    int32_t n_slices;
    int32_t n_cand;
    int32_t n_quotes;       // total strikes over slices
    int32_t max_q;          // largest strike count of one slice
    int32_t n_tiles;        // path tiles per (candidate, slice)
    int32_t tile_begin;     // this launch simulates tiles [tile_begin, tile_begin + tile_count)
    int32_t tile_count;     // (<= 0: all n_tiles); T_II path sharding over ranks
    int32_t n_groups;       // candidate groups of the launch (set by launch_mc_tiles)
    const int32_t* slice_order;  // [n_slices] block order of the slices (null: 0, 1, ...)
    int32_t ppt;            // paths per thread (consecutive, same RNG block)
    int32_t rng;            // sabr_rng
    int64_t total_steps;    // row length of coef / hdt
    uint64_t num_paths;
    uint64_t block_size;
    uint64_t seed;
    const McSlice* slices;  // [n_slices]
    const McSlice* host_slices;  // [n_slices] host copy (launch-time choices), or null
    const double* alpha0;   // [n_cand]
    const double* beta;     // [n_cand]
    const uint8_t* active;  // [n_cand] or null: inactive candidates (zero coefficients)
                            // are simulated harmlessly and skipped in the payoffs
    int32_t cand_stride;    // candidates per coefficient row (n_cand rounded up to CB)
    const StepCoef* coef;   // [total_steps][cand_stride] (step-major; padding = 0)
    const double* hdt;      // [total_steps] dt/2
    const double* strikes;  // [n_quotes]
    const uint64_t* jump;   // xoshiro jump polynomials, 4 words each
    double* partials;       // [n_tiles][n_cand][n_quotes][2] (sum, sum of squares; tile-major so a
                            // rank's tile range is one contiguous slab) or null
    double* terminals;      // [num_paths] (n_cand == 1, n_slices == 1) or null
    int* bad;               // [n_cand] non-finite flag
    const double2* exptab;  // [128] 2^(i/128) double-double (exp_tab, device_common.cuh)
    const double4* logtab;  // [128] log_tab entries (Box-Muller's log, device_common.cuh)
    const double2* sctab;   // [128] sincos_2pi entries (Box-Muller's angle)
    int32_t fp32;           // SABR_FP32: the FP32/MUFU path loop (coef32 instead of coef)
    const float4* coef32;   // [total_steps][cand_stride] FP32 {c1, -c2, rs, ss} * log2(e); launches with
                            // CB >= 2 read it pair-interleaved (kernels_sa.cu put_coef32)
};

// The exp_tab and log_tab tables, built once on the host in long double.
const double2* exp_table_host();
const double4* log_table_host();
const double2* sincos_table_host();

// price_cliquet (mc.cpp:275-320): observation nodes (step counts) and their
// F -> S factors exp(-(r-y)(T - t_node)).
constexpr int kMaxCliquetObs = 128;
struct CliquetSpecDev {
    int32_t n_obs;
    int32_t obs_node[kMaxCliquetObs];
    double obs_discount[kMaxCliquetObs];
    double local_floor, local_cap, global_floor, global_cap;
};

// One candidate, one slice (McParams with n_cand = n_slices = 1, no strikes):
// per-path clamped return strip, tile partials of (sum, sum of squares).
cudaError_t launch_mc_cliquet(const McParams& p, const CliquetSpecDev& spec, cudaStream_t s);

constexpr int kMcThreads = 128;

// Simulate + fused payoff reduction per tile (price_european_batch,
// mc.cpp:249-273) or terminal write (simulate_terminals, mc.cpp:231-240).
cudaError_t launch_mc_tiles(const McParams& p, int cand_block, cudaStream_t s);
// the largest candidate block (16, 8, 4, 2, 1) whose tile CTA fits in shared
// memory at max_q quotes per slice; 0 when none does
int mc_max_cand_block(int max_q, bool fp32);

// Final fixed-order reduction over tiles -> value/std_error per (cand, quote)
// (reduce_payoffs, mc.cpp:146-157); optional cost per candidate against
// market prices (case2_mc_cost, calibration.cpp:399-416).
cudaError_t launch_mc_reduce(const McParams& p, double* value, double* std_error,
                             const double* market, double* cost, cudaStream_t s);

}  // namespace sabr_gpu
