/*
 * oracle/sabr_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the hot path of arxiv/paper_2407_20713 (the CPU C++
 * SABR engine under /root/reference/proj): RNG, the asymptotic implied vols
 * and cost functions, the synchronous parallel annealer, the log-Euler Monte
 * Carlo engine and the Case II feasibility predicate.  Every function cites
 * the reference lines it restates.  Two Monte Carlo streams are restated: the
 * reference's own xoshiro256++ block streams (bit-identical to the reference
 * on the same libm) and the counter-based Philox4x32-10 stream the GPU engine
 * offers as SABR_RNG_PHILOX (identical streams to the GPU).
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * compiled reference (oracle/_ref/libsabr_ref.so) and against the golden
 * vectors in tests/golden/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.
 */
#ifndef SABR_ORACLE_H
#define SABR_ORACLE_H

#include <stdint.h>

#include "../include/sabr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* RNG (proj/include/sabr/rng.hpp:7-43) */
typedef struct { uint64_t s[4]; } orc_xoshiro;
void orc_xoshiro_init(orc_xoshiro* g, uint64_t seed, uint64_t stream);
uint64_t orc_xoshiro_next(orc_xoshiro* g);
double orc_xoshiro_uniform(orc_xoshiro* g);
/* Philox4x32-10, key = seed, counter = (path_lo, path_hi, step, 0). */
void orc_philox4x32(const uint32_t ctr[4], uint64_t key, uint32_t out[4]);
void orc_philox_uniform_pair(uint64_t seed, uint64_t path, uint32_t step, double* u_a,
                             double* u_b);

/* Analytics (proj/src/analytics.cpp) */
double orc_static_implied_vol(const double p[4], double strike, double forward, double T);
void orc_dyn_coeffs_case1(const double p[6], double T, double out[4]);
double orc_dynamic_implied_vol(const double c[4], double alpha, double beta, double strike,
                               double forward, double T);
double orc_forward(const sabr_surface* s, int64_t slice);
int orc_case2_feasible(const double p[11]);

/* Cost functions (proj/src/calibration.cpp:253-275, :300-306, :339-349) */
double orc_cost_static(const sabr_surface* s, int64_t slice, const double p[4]);
double orc_cost_case1(const sabr_surface* s, const double p[6]);
/* dyn_coeffs_case2 (analytics.cpp:255-289, p feasible) and the
 * calibrate_case2_formula objective (calibration.cpp:497-520) */
void orc_dyn_coeffs_case2(const double p[11], double T, int nodes, double out[4]);
double orc_cost_case2_formula(const sabr_surface* s, const double p[11]);
/* |cost change| when exp/pow in the analytics move by one ulp (test bound). */
double orc_cost_sensitivity(int model, const sabr_surface* s, int64_t slice, const double* p);

/* Annealer (proj/src/annealer.cpp:60-167) on a C objective. */
typedef double (*orc_objective)(const double* x, void* user);
typedef int (*orc_predicate)(const double* x, void* user);
int orc_minimize(orc_objective f, void* user, orc_predicate feasible, void* puser,
                 const double* lo, const double* hi, int dim, const sabr_schedule* sch,
                 const double* start, sabr_anneal_result* res);
/* Convenience: the T_I objectives over the full parameter vector. */
int orc_minimize_cost(int model, const sabr_surface* s, int64_t slice, const double* lo,
                      const double* hi, int dim, const sabr_schedule* sch, const double* start,
                      sabr_anneal_result* res);
int orc_minimize_builtin(int objective, int predicate, const double* lo, const double* hi,
                         int dim, const sabr_schedule* sch, const double* start,
                         sabr_anneal_result* res);

/* One temperature level of chains [chain_begin, chain_end) from `st`
 * (annealer.cpp:107-139) reduced to one record (the per-rank half of
 * annealer.cpp:141-159): the multi-rank decomposition the GPU engine uses.
 * objective: a sabr_builtin_objective; returns SABR_OK. */
int orc_level_record(int objective, int predicate, const double* lo, const double* hi, int dim,
                     const sabr_schedule* sch, const sabr_sa_state* st, uint64_t level,
                     double temp, int64_t chain_begin, int64_t chain_end,
                     sabr_level_record* out);
double orc_builtin_value(int objective, const double* x);

/* Monte Carlo (proj/src/mc.cpp:30-273).  model/params as in sabr_b200.h. */
int orc_simulate_terminals(int model, const double* params, double forward0, double alpha0,
                           double T, const sabr_plan* plan, double* out);
int orc_price_european_batch(int model, const double* params, double spot,
                             const double* strikes, int64_t m, double rate, double dividend,
                             double T, const sabr_plan* plan, double* value, double* se);
int orc_implied_vol_from_price(double price, double spot, double strike, double r, double y,
                               double T, double* vol_out);
double orc_black_scholes_call(double spot, double strike, double r, double y, double T,
                              double vol);
/* price_cliquet, mc.cpp:275-320 */
int orc_price_cliquet(int model, const double* params, double spot, double rate, double dividend,
                      double lf, double lc, double gf, double gc, const double* resets, int n_resets,
                      const sabr_plan* plan, double* value, double* se);
/* case2_mc_cost (calibration.cpp:399-416); params 11 (horizon last). */
int orc_cost_case2_mc(const sabr_surface* s, const double p[11], const sabr_plan* plan,
                      double* cost);

#ifdef __cplusplus
}
#endif

#endif
