// kernels.hpp — host-visible launchers of the sm_100a kernels (internal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sabr_b200.h"

namespace sabr_gpu {

// Market grid in device memory (SoA, one contiguous allocation).  For the
// static T_I objective the view covers the calibrated slice only.
struct SurfaceView {
    int32_t n_slices;
    int32_t n_quotes;
    const double* T;       // [n_slices] maturity
    const double* lnf_hi;  // [n_slices] ln(forward), double-double
    const double* lnf_lo;  // [n_slices]
    const int32_t* qoff;   // [n_slices+1]
    // [n_quotes] x {lm = ln(K/f) (std::log(strike/forward), the reference
    // expression, evaluated on the host), lm*lm, market value, 1/market}
    const double* quotes;
    // [n_slices][kQrStride]: each slice's cost as a 4x4 quadratic form
    // (slice_qr.hpp), nullptr when the view has none
    const double* qr;
    const double2* exptab;  // [128] exp_tab table (device_common.cuh), staged per CTA
    double max_abs_lnf;     // max_i |ln f_i| (host-side bound for the unsaturated exp)
};

enum ObjectiveKind : int32_t {
    OBJ_STATIC = 0,   // cost_individual o static_implied_vol       calibration.cpp:300-306
    OBJ_CASE1 = 1,    // sum_i cost_individual o dynamic_implied_vol calibration.cpp:339-349
    OBJ_BUILTIN = 2,  // test_annealer.cpp closed forms
};

// The arg-min part of a CTA's level record, contiguous per CTA so the last
// CTA's reduction reads three 16-byte vectors per record (the points stay in
// the full sabr_level_record and are read for the two winners only).
struct __align__(16) BlockSummary {
    double end_value;
    long long end_chain;
    double best_value;
    long long best_chain;
    long long evals;
    long long pad;
};

// Per-rank mailbox of the fused peer exchange (sabr_ctx_enable_peer_exchange):
// every rank's last CTA stores its level record into slot [level parity][its
// rank] of every rank's mailbox over NVLink / NVSwitch peer memory, then
// raises the slot's epoch; a rank merges once all epochs of its own mailbox
// show the level.  Two parities: a rank can be at most one level ahead of a
// slower peer (its next merge needs the peer's next record), so a record is
// never overwritten before the slower peer has read it.
constexpr int kMaxPeerRanks = 16;
struct PeerMailbox {
    sabr_level_record rec[2][kMaxPeerRanks];
    unsigned long long epoch[2][kMaxPeerRanks];
    unsigned long long hello[kMaxPeerRanks];  // handshake at enable time
};

// Handshake of sabr_ctx_enable_peer_exchange: write `magic` into slot
// [my_rank] of every rank's mailbox (peer stores), fenced system-wide.
cudaError_t launch_peer_hello(PeerMailbox* const* boxes, int nranks, int my_rank, unsigned long long magic,
                              cudaStream_t s);

struct SaLevelArgs {
    double lo[SABR_MAX_DIM];
    double hi[SABR_MAX_DIM];
    double range[SABR_MAX_DIM];  // hi - lo (annealer.cpp:65)
    double lo2[SABR_MAX_DIM];    // 2*lo, 2*hi (the reflections of annealer.cpp:68-71,
    double hi2[SABR_MAX_DIM];    // rounded on the host exactly as the reference does)
    uint32_t free_mask;          // bit i: full-vector dim i is searched
    int32_t dim_full;
    int32_t chain_length;
    int32_t builtin;             // sabr_builtin_objective when OBJ_BUILTIN
    int32_t predicate;           // SABR_PRED_*
    int32_t nranks;
    int32_t fast;                // all dims free and one reflection always lands in the box
    int32_t fast_free;           // one reflection always lands in the box for every searched dim
    int32_t beta_one;            // Case I: beta (dim 1) not searched and held at exactly 1
    double t0;
    uint64_t seed;
    int64_t chain_begin;         // global index of this rank's first chain
    int64_t n_local;             // chains on this rank
    int64_t n_chains;            // global chain count
    int64_t max_evals;
    int64_t levels_total;
    sabr_sa_state* state;        // device
    sabr_level_record* block_recs;  // [grid] scratch
    BlockSummary* block_sum;        // [grid] scratch (arg-min fields of block_recs)
    sabr_level_record* rank_rec;    // [1] this rank's record (NCCL send buffer)
    unsigned int* ticket;           // [1] zero-initialised
    PeerMailbox* const* peer_boxes; // [nranks] mailboxes (peer pointers) or null: fused exchange
    int32_t my_rank;                // this rank (peer exchange)
    unsigned long long epoch_base;  // level l publishes epoch epoch_base + l + 1
    int* peer_error;                // set when the exchange timed out
    double* trace_f;                // [levels_total] device
};

// Launch one temperature level (proj/src/annealer.cpp:99-161).  With nranks==1
// the merge into `state` happens inside the kernel's last block.
cudaError_t launch_sa_level(int kind, const SurfaceView& sv, const SaLevelArgs& a, int64_t level,
                            double temp, cudaStream_t s);
// Merge `nranks` gathered records into the state (multi-rank path).
cudaError_t launch_sa_merge(const SaLevelArgs& a, const sabr_level_record* recs, int64_t level,
                            cudaStream_t s);
// Evaluate the objective at state->incumbent and seed incumbent/best values.
// All levels of a one-CTA, one-rank run in one launch (sa_run_small_kernel);
// cudaErrorNotSupported when the run does not qualify (then launch per level).
// temps == nullptr: only report whether it qualifies.
cudaError_t launch_sa_run_small(int kind, const SurfaceView& sv, const SaLevelArgs& a, const double* temps,
                                int64_t n_levels, cudaStream_t s);
cudaError_t launch_sa_start(int kind, const SurfaceView& sv, const SaLevelArgs& a,
                            cudaStream_t s);
// cost[i] of full parameter vectors params[i*dim_full ..].
cudaError_t launch_cost_batch(int kind, const SurfaceView& sv, const double* params,
                              int32_t dim_full, int64_t n, double* cost, cudaStream_t s);
// model vols[i*n_quotes + j] for all quotes of the view.
cudaError_t launch_vol_batch(int kind, const SurfaceView& sv, const double* params,
                             int32_t dim_full, int64_t n, double* vols, cudaStream_t s);
cudaError_t launch_case2_feasible(const double* params, int64_t n, uint8_t* out,
                                  cudaStream_t s);

int sa_block_threads();   // threads per CTA of the T_I level kernel (one record each)
int t2_block_threads();   // threads per CTA of t2_level_end

// ----------------------------------------------------------- T_II chains ---
// Chain state of the Monte Carlo objective annealer, kept in HBM between the
// per-step kernels (propose -> coefficients -> MC -> Metropolis).
struct T2Chain {
    double x[SABR_MAX_DIM];   // current point (full parameter vector)
    double y[SABR_MAX_DIM];   // proposal of this step
    double bp[SABR_MAX_DIM];  // chain best point
    double fx, bv;
    uint64_t rng[4];          // xoshiro256++ state, keyed (seed, level<<20 ^ chain)
    long long evals;
    int32_t active;           // proposal of this step is feasible and evaluated
    int32_t pad;
};

struct T2StepArgs {
    double lo[SABR_MAX_DIM], hi[SABR_MAX_DIM], range[SABR_MAX_DIM];
    uint32_t free_mask;
    int32_t n_local;
    double t0, temp, horizon;
    uint64_t seed;
    int64_t chain_begin;
    int64_t level;
};

// one MC launch per step: cost + scatter + Metropolis in one kernel (t2_finish_kernel)
cudaError_t launch_t2_finish(T2Chain* chains, const T2StepArgs& a, const int32_t* idx, const int32_t* n_live,
                             const double* values, int32_t nq, const double* market, const int* bad_c,
                             int* nonfinite, cudaStream_t s);
cudaError_t launch_t2_level_init(T2Chain* chains, const sabr_sa_state* st, const T2StepArgs& a,
                                 cudaStream_t s);
// propose + feasibility (analytics.cpp:145-175 on the grid), writes the MC
// candidate arrays (alpha0, beta, active) for this step.
cudaError_t launch_t2_propose(T2Chain* chains, const sabr_sa_state* st, const T2StepArgs& a,
                              double* alpha0, double* beta, uint8_t* active, cudaStream_t s);
// per (candidate, step) coefficients of build_grid (mc.cpp:69-82) on device
cudaError_t launch_t2_coef(const T2Chain* chains, const int32_t* idx, const int32_t* n_live, int32_t c0,
                           int32_t n_local, int32_t cand_stride, const double* t_end, const double* dt,
                           const double* sdt, int64_t total_steps, void* coef, int fp32 /* 0 FP64, 1 FP32, 2 FP32 pair-interleaved */,
                           cudaStream_t s);
// the step's feasible candidates compacted (t2_compact_kernel; bad_c, the
// compacted non-finite flags, zeroed), and their costs / non-finite flags
// scattered back to their chains
cudaError_t launch_t2_compact(const uint8_t* active, const double* alpha0, const double* beta, int32_t n,
                              int32_t* idx, double* alpha0_c, double* beta_c, uint8_t* active_c,
                              int32_t* n_live, int* bad_c, cudaStream_t s);
cudaError_t launch_t2_scatter(const int32_t* idx, const int32_t* n_live, int32_t n, const double* cost_c,
                              const int* bad_c, double* cost, int* bad, cudaStream_t s);
// Metropolis (annealer.cpp:123-134) with the MC costs of this step
cudaError_t launch_t2_accept(T2Chain* chains, const T2StepArgs& a, const double* cost,
                             const int* bad, int* nonfinite, cudaStream_t s);
// level-end reduction of the chains into the annealer state (as sa_level)
cudaError_t launch_t2_level_end(const T2Chain* chains, const SaLevelArgs& a, int64_t level,
                                cudaStream_t s);

// ---- batched Black-Scholes (black_scholes.cpp:20-69), kernels_bs.cu ----
enum BsStatus : int32_t {
    BS_OK = 0,
    BS_E_INPUTS = 1,  // "black_scholes_call: spot, strike, maturity must be positive"
    BS_E_VOL = 2,     // "black_scholes_call: vol must be nonnegative"
    BS_E_BOUNDS = 3,  // "implied_vol_from_price: price outside no-arbitrage bounds"
};
cudaError_t launch_bs_call(int64_t n, const double* spot, const double* strike, const double* r, const double* y,
                           const double* T, const double* vol, double* out, int32_t* status, cudaStream_t s);
cudaError_t launch_implied_vol(int64_t n, const double* price, const double* spot, const double* strike,
                               const double* r, const double* y, const double* T, double* out, int32_t* status,
                               cudaStream_t s);

}  // namespace sabr_gpu
