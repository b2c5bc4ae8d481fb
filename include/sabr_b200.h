/*
 * sabr_b200.h — the C-ABI drop-in boundary of the B200 SABR calibration engine.
 *
 * Every entry point below replaces one reference interface of
 * arxiv/paper_2407_20713 (the CPU C++ engine under proj/), cited as
 * `proj/...:line`.  The ABI is plain C: caller-owned arrays, sizes as 64-bit
 * integers, no exceptions and no C++ or torch types.  Errors are returned as a
 * sabr_status whose value maps 1:1 onto the exception type the reference
 * throws (proj/include/sabr/types.hpp:10-15, std::domain_error,
 * std::out_of_range, std::runtime_error); the message of the last failing call
 * on the calling thread is available from sabr_last_error().
 *
 * Layering:  Python / C++ callers  ->  this ABI  ->  C++ host
 * (ParamSpace, validation, SA level loop, NCCL)  ->  sm_100a kernels.
 */
#ifndef SABR_B200_H
#define SABR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SABR_API __attribute__((visibility("default")))
#else
#define SABR_API
#endif

/* ---- status codes (exception mapping) --------------------------------- */
typedef enum sabr_status {
    SABR_OK = 0,
    SABR_E_DOMAIN = 1,       /* std::domain_error                          */
    SABR_E_OUT_OF_RANGE = 2, /* std::out_of_range (bad slice index, .at()) */
    SABR_E_CONSTRAINT = 3,   /* sabr::constraint_error (types.hpp:10-15)   */
    SABR_E_RUNTIME = 4,      /* std::runtime_error (non-finite MC path)    */
    SABR_E_CUDA = 5,         /* CUDA runtime failure / no device           */
    SABR_E_NCCL = 6,         /* NCCL failure                               */
    SABR_E_INVALID = 7,      /* bad ABI argument (null pointer, capacity)  */
    SABR_E_LOGIC = 8         /* std::logic_error / anything else           */
} sabr_status;

typedef enum sabr_model {
    SABR_MODEL_STATIC = 0, /* StaticSabrParams {alpha,beta,nu,rho}        types.hpp:19-26  */
    SABR_MODEL_CASE1 = 1,  /* CaseIParams {alpha,beta,rho0,nu0,a,b}        types.hpp:30-41  */
    SABR_MODEL_CASE2 = 2   /* CaseIIParams {alpha,beta,rho0,q_rho,d_rho,nu0,q_nu,d_nu,a,b,horizon}
                              types.hpp:48-60 */
} sabr_model;

/* Monte Carlo random stream.  XOSHIRO reproduces the reference streams
 * exactly: block b of `block_size` paths uses Xoshiro256pp(seed, b)
 * (proj/src/mc.cpp:126-127) consumed path after path; the GPU reaches path p
 * of a block by an F2-linear jump of 2*n_steps*p draws.  PHILOX is the
 * counter-based stream keyed by (seed) with counter (step, path); its CPU
 * restatement lives in oracle/. */
typedef enum sabr_rng { SABR_RNG_XOSHIRO = 0, SABR_RNG_PHILOX = 1 } sabr_rng;

/* ---- value types ------------------------------------------------------- */

/* VolSurface (proj/include/sabr/calibration.hpp:16-37) in SoA form.
 * Slice i owns quotes [quote_offset[i], quote_offset[i+1]). */
typedef struct sabr_surface {
    double spot;
    int64_t n_slices;
    const double* maturity;      /* [n_slices] */
    const double* rate;          /* [n_slices] decimal */
    const double* dividend;      /* [n_slices] decimal */
    const int64_t* quote_offset; /* [n_slices+1] */
    const double* strike;        /* [total quotes] absolute */
    const double* vol;           /* [total quotes] decimal */
} sabr_surface;

/* AnnealingSchedule (proj/include/sabr/annealer.hpp:17-29). */
typedef struct sabr_schedule {
    double t0;
    double cooling;
    int32_t chain_length;
    int32_t workers;
    int32_t groups;
    int32_t omp_threads; /* accepted, ignored: results never depend on it */
    double t_min;
    int64_t max_evals;
    uint64_t seed;
} sabr_schedule;

/* Arithmetic of the Monte Carlo path loop.  FP64 is the reference's
 * precision and the parity path.  FP32 is the opt-in fast path: the same
 * streams and the same log-Euler scheme with FP32 state and MUFU exp2 per
 * candidate-step (normals from FP32 library functions, payoff sums in FP64);
 * prices agree with FP64 on identical streams to ~1e-5 relative. */
typedef enum sabr_precision { SABR_FP64 = 0, SABR_FP32 = 1 } sabr_precision;

/* SimulationPlan (proj/include/sabr/mc.hpp:12-20) plus the stream choice. */
typedef struct sabr_plan {
    uint64_t num_paths;
    double dt;
    uint64_t seed;
    int32_t workers; /* accepted, validated, ignored */
    int32_t rng;     /* sabr_rng */
    uint64_t block_size;
    int32_t precision; /* sabr_precision */
    int32_t _pad;
} sabr_plan;

/* BoundsOverrides / FixedParams (calibration.hpp:77-79). */
typedef struct sabr_bounds {
    int64_t n;
    const char* const* names;
    const double* lo;
    const double* hi;
} sabr_bounds;

typedef struct sabr_fixed {
    int64_t n;
    const char* const* names;
    const double* values;
} sabr_fixed;

/* ReportRow (calibration.hpp:39-45). */
typedef struct sabr_report_row {
    double maturity;
    double strike;
    double market;
    double model;
    double rel_error;
} sabr_report_row;

#define SABR_MAX_PARAMS 16
#define SABR_NAME_LEN 16

/* CalibrationReport (calibration.hpp:47-59).  `rows` and the trace arrays are
 * caller-owned; n_rows / trace_len report how many were written (the call
 * fails with SABR_E_INVALID if a capacity is too small). Parameters are listed
 * in std::map order (sorted by name), as the reference report holds them. */
typedef struct sabr_report {
    char model[SABR_NAME_LEN];
    char technique[SABR_NAME_LEN];
    char quantity[SABR_NAME_LEN];
    int64_t n_params;
    char param_names[SABR_MAX_PARAMS][SABR_NAME_LEN];
    double param_values[SABR_MAX_PARAMS];
    double final_cost;
    double mean_rel_error;
    double max_rel_error;
    double wall_seconds;
    int64_t evals;
    uint64_t seed;
    sabr_report_row* rows;
    int64_t rows_capacity;
    int64_t n_rows;
    /* temperature trace of the annealer (AnnealResult::temperature_trace,
     * annealer.hpp:43-48); optional (null/0 = not requested). */
    double* trace_t;
    double* trace_f;
    int64_t trace_capacity;
    int64_t trace_len;
} sabr_report;

/* AnnealResult (annealer.hpp:43-48). */
typedef struct sabr_anneal_result {
    double* best_point; /* [dim] caller-owned */
    double best_value;
    int64_t evals;
    double* trace_t;
    double* trace_f;
    int64_t trace_capacity;
    int64_t trace_len;
} sabr_anneal_result;

/* Device timing of the last call on a context (CUDA events on the context
 * stream).  `kernel_ms` is the summed duration of the dominant kernel family
 * (SA level kernels for T_I, MC kernels for T_II/pricing). */
typedef struct sabr_timing {
    double total_ms;
    double kernel_ms;
    int64_t kernel_launches;
    int64_t total_launches;
    double units;         /* cost-evals or path-steps processed by the dominant kernels */
    double path_steps;    /* MC path-steps simulated (0 for T_I)                        */
} sabr_timing;

typedef struct sabr_ctx sabr_ctx;

/* ---- library / context -------------------------------------------------- */
SABR_API const char* sabr_last_error(void);
SABR_API const char* sabr_version(void);

/* One context per process per GPU.  `stream` may be 0 (context owns a
 * stream) or a cudaStream_t the caller wants the kernels launched on. */
SABR_API sabr_status sabr_ctx_create(int32_t device, void* stream, sabr_ctx** out);
SABR_API void sabr_ctx_destroy(sabr_ctx* ctx);
SABR_API sabr_status sabr_ctx_set_profiling(sabr_ctx* ctx, int32_t on);
SABR_API sabr_status sabr_ctx_last_timing(sabr_ctx* ctx, sabr_timing* out);

/* Multi-GPU: chains are split contiguously over `nranks` contexts (one per
 * process per GPU); the per-temperature-level exchange (the two-level group
 * reduction of proj/src/annealer.cpp:141-159) is one ncclAllGather of a
 * fixed-size record per rank.  sabr_comm_unique_id is called on rank 0 and
 * the 128 bytes are broadcast by the caller (torch.distributed, MPI, ...). */
SABR_API sabr_status sabr_comm_unique_id(uint8_t out[128]);
SABR_API sabr_status sabr_ctx_init_comm(sabr_ctx* ctx, const uint8_t uid[128],
                                        int32_t rank, int32_t nranks);

/* The same rank decomposition with the per-level record exchange done by the
 * caller on the host instead of NCCL (a non-NCCL transport, or several ranks
 * sharing one GPU in tests).  Once per temperature level the engine calls
 * fn(user, send, recv, bytes): send = this rank's `bytes`, recv = nranks *
 * `bytes` in rank order (an all-gather), both host memory; fn returns 0 on
 * success.  Results are identical to the NCCL path and to a single rank. */
typedef int (*sabr_allgather_fn)(void* user, const void* send, void* recv, int64_t bytes);
SABR_API sabr_status sabr_ctx_init_host_exchange(sabr_ctx* ctx, int32_t rank, int32_t nranks,
                                                 sabr_allgather_fn fn, void* user);

/* Fused peer-memory exchange for the T_I calibrators (after init_comm or
 * init_host_exchange, which carry the one-time exchange of CUDA IPC handles):
 * the last CTA of each rank's level kernel stores the 240-byte level record
 * into every rank's mailbox over NVLink / NVSwitch peer memory, waits for the
 * peers' records and merges them itself - no NCCL call, no separate merge
 * kernel per level.  Needs peer access between the ranks' GPUs (or ranks on
 * one GPU) and at most 16 ranks; results are identical to the other
 * transports.  Other calibrators keep using the transport. */
SABR_API sabr_status sabr_ctx_enable_peer_exchange(sabr_ctx* ctx);
/* Back to the transport for every calibrator (e.g. when another rank could
 * not enable the peer exchange: all ranks must use the same path). */
SABR_API sabr_status sabr_ctx_disable_peer_exchange(sabr_ctx* ctx);

/* ---- calibration (proj/include/sabr/calibration.hpp) -------------------- */

/* calibrate_static_T1, calibration.hpp:82-85 / proj/src/calibration.cpp:289-323 */
SABR_API sabr_status sabr_calibrate_static_T1(sabr_ctx* ctx, const sabr_surface* surface,
                                              int64_t slice, const sabr_bounds* bounds,
                                              const sabr_schedule* schedule,
                                              const sabr_fixed* fixed, sabr_report* report);

/* calibrate_static_T1 on n slices of one surface at once: reports[i] is
 * exactly what sabr_calibrate_static_T1(ctx, surface, slices[i], ...) returns.
 * Replaces a caller's loop over slices (e.g. proj/tools/sabr_cli.cpp:70 run
 * per slice).  On a single-rank context the slices' annealers run side by
 * side on up to 8 streams (child contexts of ctx, created on first use, one
 * host thread each, each running its share of the slices in order), so the
 * level kernels of independent slices share the SMs (a C2 slice's level grid
 * alone holds 7 of the 10 one-warp CTAs an SM can run);
 * the child streams are ordered after ctx's stream and ctx's stream after
 * them.  Multi-rank contexts with the peer exchange enabled do the same (each
 * child gets its own peer mailboxes, set up over ctx's transport; collective:
 * every rank makes the same call); with the per-level transport all-gather the
 * slices run one after another.  The first failing slice's status is
 * returned (its message in sabr_last_error). */
SABR_API sabr_status sabr_calibrate_static_T1_slices(sabr_ctx* ctx, const sabr_surface* surface,
                                                     const int64_t* slices, int64_t n,
                                                     const sabr_bounds* bounds,
                                                     const sabr_schedule* schedule,
                                                     const sabr_fixed* fixed, sabr_report* reports);

/* calibrate_dynamic_case1_T1, calibration.hpp:88-91 / calibration.cpp:325-365 */
SABR_API sabr_status sabr_calibrate_dynamic_case1_T1(sabr_ctx* ctx,
                                                     const sabr_surface* surface,
                                                     const sabr_bounds* bounds,
                                                     const sabr_schedule* schedule,
                                                     const sabr_fixed* fixed,
                                                     sabr_report* report);

/* calibrate_case2_T2, calibration.hpp:97-104 / calibration.cpp:450-481.
 * report_plan and start_override may be null. */
SABR_API sabr_status sabr_calibrate_case2_T2(sabr_ctx* ctx, const sabr_surface* surface,
                                             const sabr_bounds* bounds,
                                             const sabr_schedule* schedule,
                                             const sabr_plan* plan, const sabr_fixed* fixed,
                                             const sabr_plan* report_plan,
                                             const double* start_override,
                                             int64_t start_len, sabr_report* report);

/* calibrate_case2_formula, calibration.hpp:108-111 / calibration.cpp:483-534 */
SABR_API sabr_status sabr_calibrate_case2_formula(sabr_ctx* ctx, const sabr_surface* surface,
                                                  const sabr_bounds* bounds,
                                                  const sabr_schedule* schedule,
                                                  const sabr_fixed* fixed,
                                                  sabr_report* report);

/* evaluate_case1 (calibration.hpp:121, calibration.cpp:367-393); p = CaseIParams[6] */
SABR_API sabr_status sabr_evaluate_case1(sabr_ctx* ctx, const sabr_surface* surface,
                                         const double* p, sabr_report* report);

/* evaluate_case2_prices (calibration.hpp:122-124, calibration.cpp:420-448);
 * p = CaseIIParams[11] (horizon last). */
SABR_API sabr_status sabr_evaluate_case2_prices(sabr_ctx* ctx, const sabr_surface* surface,
                                                const double* p, const sabr_plan* plan,
                                                sabr_report* report);

/* ---- batched objective (the SA cost function on the GPU) ---------------- */

/* cost[i] = objective of full parameter vector params[i*dim .. ]:
 *   STATIC (dim 4): cost_individual(surface, slice, static_implied_vol)
 *                   calibration.cpp:253-267 with :300-306
 *   CASE1  (dim 6): sum over slices, calibration.cpp:339-349 (slice must be -1)
 *   CASE2  (dim 11 incl. horizon): case2_mc_cost, calibration.cpp:399-416
 *                   (needs `plan`; infeasible vectors raise SABR_E_CONSTRAINT)
 *   SABR_OBJECTIVE_CASE2_FORMULA (dim 11): the calibrate_case2_formula
 *                   objective, calibration.cpp:497-520 (dyn_coeffs_case2 with
 *                   8-node Gauss-Legendre + Black-Scholes per quote; 1e10 when
 *                   a formula vol leaves its validity range) */
#define SABR_OBJECTIVE_CASE2_FORMULA 3
SABR_API sabr_status sabr_cost_batch(sabr_ctx* ctx, int32_t model, const sabr_surface* surface,
                                     int64_t slice, const double* params, int64_t n,
                                     const sabr_plan* plan, double* cost);

/* Per-quote model vols for a batch of parameter vectors (static: the slice
 * only; case1 and case2: all quotes). vols[i*n_quotes + j].
 * analytics.cpp:183-205, :291-312; case2 rows are 11 wide (horizon last) and
 * use dyn_coeffs_case2 with its default 64 Gauss-Legendre nodes
 * (analytics.hpp:25-26), as the smile command does (sabr_cli.cpp:234-243). */
SABR_API sabr_status sabr_implied_vol_batch(sabr_ctx* ctx, int32_t model,
                                            const sabr_surface* surface, int64_t slice,
                                            const double* params, int64_t n, double* vols);

/* CaseIIParams::validate as a predicate (analytics.cpp:145-175 via
 * case2_feasible, calibration.cpp:161-168).  params: n x 11 (horizon last). */
SABR_API sabr_status sabr_case2_feasible_batch(sabr_ctx* ctx, const double* params,
                                               int64_t n, uint8_t* feasible);

/* ---- Monte Carlo (proj/include/sabr/mc.hpp) ----------------------------- */

/* mc::simulate_terminals, mc.hpp:66-69 / mc.cpp:231-240.  F_T[num_paths]. */
SABR_API sabr_status sabr_mc_simulate_terminals(sabr_ctx* ctx, int32_t model,
                                                const double* params, double forward0,
                                                double alpha0, double maturity,
                                                const sabr_plan* plan, double* terminals);

/* mc::price_european_batch, mc.hpp:75-80 / mc.cpp:249-273 */
SABR_API sabr_status sabr_mc_price_european_batch(sabr_ctx* ctx, int32_t model,
                                                  const double* params, double spot,
                                                  const double* strikes, int64_t n_strikes,
                                                  double rate, double dividend,
                                                  double maturity, const sabr_plan* plan,
                                                  double* value, double* std_error);

/* mc::price_cliquet, mc.hpp:82-84 / mc.cpp:275-320.  resets[n_resets]. */
SABR_API sabr_status sabr_mc_price_cliquet(sabr_ctx* ctx, int32_t model, const double* params,
                                           double spot, double rate, double dividend,
                                           double local_floor, double local_cap,
                                           double global_floor, double global_cap,
                                           const double* reset_dates, int64_t n_resets,
                                           const sabr_plan* plan, double* value,
                                           double* std_error);

/* ---- annealer on built-in device objectives ------------------------------
 * minimize (annealer.hpp:53-57, annealer.cpp:76-167) with the objective one of
 * the closed-form test functions of proj/tests/test_annealer.cpp, so the
 * annealer's own unit tests run unchanged against the GPU driver.  The
 * optional predicate is SABR_PRED_SUM_LE_1 (x0 + x1 <= 1, test_annealer.cpp:108-121). */
typedef enum sabr_builtin_objective {
    SABR_OBJ_BOWL3 = 0,      /* (x0-1.2)^2+(x1+0.7)^2+(x2-3.4)^2      test_annealer.cpp:30-32 */
    SABR_OBJ_ROSENBROCK4 = 1,/* 4-d Rosenbrock                         :43-48  */
    SABR_OBJ_SINQUAD2 = 2,   /* (x0-.3)^2+3(x1+2.1)^2+.1 sin(7x0)      :62-64  */
    SABR_OBJ_SQUARE1 = 3,    /* x0^2                                   :84-87  */
    SABR_OBJ_COSBOWL2 = 4,   /* x0^2+x1^2+cos(3x0)                     :97-99  */
    SABR_OBJ_CORNER2 = 5,    /* (x0-2)^2+(x1-2)^2                      :114-117 */
    SABR_OBJ_NANRIGHT1 = 6   /* NaN for x0>0.5 else (x0+1)^2           :124-128 */
} sabr_builtin_objective;

#define SABR_PRED_NONE 0
#define SABR_PRED_SUM_LE_1 1

SABR_API sabr_status sabr_minimize_builtin(sabr_ctx* ctx, int32_t objective, int32_t predicate,
                                           const double* lower, const double* upper,
                                           int64_t dim, const sabr_schedule* schedule,
                                           const double* start, sabr_anneal_result* result);

/* ---- host-side helpers (no GPU needed) ----------------------------------- */

/* Deterministic merge of per-rank level records (the cross-GPU half of the
 * reduction at annealer.cpp:141-159).  Exposed so the multi-rank logic can be
 * exercised on CPU-only hosts.  records: nranks x sabr_level_record. */
#define SABR_MAX_DIM 12
typedef struct sabr_level_record {
    double end_value;
    int64_t end_chain; /* global chain index, -1 = none */
    double best_value;
    int64_t best_chain;
    int64_t evals;
    int64_t _pad;
    double end_point[SABR_MAX_DIM];
    double best_point[SABR_MAX_DIM];
} sabr_level_record;

typedef struct sabr_sa_state {
    double incumbent[SABR_MAX_DIM];
    double incumbent_value;
    double best[SABR_MAX_DIM];
    double best_value;
    int64_t evals;
    int64_t eval_cap;
    int64_t done;
    int64_t levels_run;
} sabr_sa_state;

/* Applies one level: merges `nranks` records in rank order (strict '<',
 * lowest global chain index wins ties), updates incumbent/best/evals and the
 * next level's eval cap; returns the new incumbent value in *trace_f. */
SABR_API sabr_status sabr_merge_level_records(sabr_sa_state* state,
                                              const sabr_level_record* records,
                                              int64_t nranks, int64_t n_chains,
                                              int64_t max_evals, int64_t levels_total,
                                              double* trace_f);

/* Surface CSV loader (io::parse_surface, proj/src/io.cpp:68-161): two calls,
 * first with null arrays to get the sizes. */
SABR_API sabr_status sabr_surface_csv_dims(const char* path, int64_t* n_slices,
                                           int64_t* n_quotes);
SABR_API sabr_status sabr_surface_csv_read(const char* path, double* spot, double* maturity,
                                           double* rate, double* dividend,
                                           int64_t* quote_offset, double* strike, double* vol);

/* Diagnostics: measured FP64 FMA-pipe peak of the context's GPU in TFLOP/s
 * (8 independent DFMA chains per thread, 8 CTAs of 256 threads per SM) - the
 * roofline denominator of the FP64-bound kernels. */
SABR_API sabr_status sabr_bench_fp64_peak(sabr_ctx* ctx, double* tflops);
/* Diagnostics: measured MUFU (XU pipe) ex2.approx.f32 throughput in 1e12
 * ops/s - the roofline denominator of the FP32 MC path's transcendentals. */
SABR_API sabr_status sabr_bench_mufu_peak(sabr_ctx* ctx, double* tops);

/* Black-Scholes call (black_scholes.hpp:7-9), used for the T_II market side. */
SABR_API sabr_status sabr_black_scholes_call(double spot, double strike, double rate,
                                             double dividend, double maturity, double vol,
                                             double* price);

/* Batched black_scholes_call / implied_vol_from_price (black_scholes.hpp:7-14,
 * black_scholes.cpp:20-69) on the device, one contract per element (SoA,
 * caller-owned host arrays of length n).  The reference's scalar functions
 * throw std::domain_error; here the first rejected element in index order
 * returns SABR_E_DOMAIN with the reference's message (the outputs are then
 * unspecified).  implied_vol keeps the reference's bracket + safeguarded
 * Newton iteration (|BS(vol) - price| < 1e-10 or 200 steps). */
SABR_API sabr_status sabr_black_scholes_call_batch(sabr_ctx* ctx, int64_t n, const double* spot,
                                                   const double* strike, const double* rate,
                                                   const double* dividend, const double* maturity,
                                                   const double* vol, double* price);
SABR_API sabr_status sabr_implied_vol_from_price_batch(sabr_ctx* ctx, int64_t n, const double* price,
                                                       const double* spot, const double* strike,
                                                       const double* rate, const double* dividend,
                                                       const double* maturity, double* vol);

#ifdef __cplusplus
}
#endif

#endif /* SABR_B200_H */
