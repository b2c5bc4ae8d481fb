// engine.cu — the C-ABI of include/sabr_b200.h: context, validation in the
// reference's order, the T_I annealer driver (device-resident level loop),
// Monte Carlo pricing drivers and report assembly.  All numerical work runs in
// the sm_100a kernels; the host only validates, lays out and launches.
#include <dlfcn.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>

#include "device_common.cuh"
#include "engine.hpp"
#include "kernels_c2f.hpp"
#include "slice_qr.hpp"
#include "xoshiro_jump.hpp"

#include <functional>

// NCCL is loaded at run time (the one torch already mapped, else the system
// library), so the engine has no link-time NCCL dependency.
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclChar = 0 };

namespace sabr_gpu {

namespace {

thread_local std::string g_last_error;

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.handle = h;
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.handle || !api.getUniqueId || !api.commInitRank || !api.allGather)
        fail(SABR_E_NCCL, "NCCL (libnccl.so.2) could not be loaded");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != 0) {
        const char* msg = nccl().getErrorString ? nccl().getErrorString(r) : "";
        fail(SABR_E_NCCL, std::string(what) + ": " + msg);
    }
}

template <class F>
sabr_status guarded(F&& f) {
    try {
        f();
        return SABR_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return SABR_E_OUT_OF_RANGE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SABR_E_LOGIC;
    }
}

struct CtxLock {
    sabr_ctx* ctx;
    std::lock_guard<std::mutex> lock;
    explicit CtxLock(sabr_ctx* c) : ctx(c), lock(check(c)->mu) {
        check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
    }
    static sabr_ctx* check(sabr_ctx* c) {
        if (!c) fail(SABR_E_INVALID, "context is null");
        return c;
    }
};

void sync(sabr_ctx* ctx) { check_cuda(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize"); }

void copy_name(char* dst, const std::string& s) {
    std::memset(dst, 0, SABR_NAME_LEN);
    std::strncpy(dst, s.c_str(), SABR_NAME_LEN - 1);
}

struct Row {
    double maturity, strike, market, model, rel_error;
};

struct Report {
    std::string model, technique, quantity;
    std::map<std::string, double> params;
    double final_cost = 0.0;
    std::vector<Row> rows;
    double mean_rel_error = 0.0, max_rel_error = 0.0, wall_seconds = 0.0;
    int64_t evals = 0;
    uint64_t seed = 0;
    std::vector<double> trace_t, trace_f;

    // fill_aggregates, calibration.cpp:170-178
    void aggregates() {
        double sum = 0.0, mx = 0.0;
        for (const auto& r : rows) {
            sum += r.rel_error;
            mx = std::max(mx, r.rel_error);
        }
        mean_rel_error = rows.empty() ? 0.0 : sum / rows.size();
        max_rel_error = mx;
    }
    void write(sabr_report* out) const {
        if (!out) fail(SABR_E_INVALID, "report is null");
        copy_name(out->model, model);
        copy_name(out->technique, technique);
        copy_name(out->quantity, quantity);
        out->n_params = 0;
        for (const auto& kv : params) {
            if (out->n_params >= SABR_MAX_PARAMS) break;
            copy_name(out->param_names[out->n_params], kv.first);
            out->param_values[out->n_params] = kv.second;
            ++out->n_params;
        }
        out->final_cost = final_cost;
        out->mean_rel_error = mean_rel_error;
        out->max_rel_error = max_rel_error;
        out->wall_seconds = wall_seconds;
        out->evals = evals;
        out->seed = seed;
        out->n_rows = static_cast<int64_t>(rows.size());
        if (out->rows) {
            if (out->rows_capacity < out->n_rows) fail(SABR_E_INVALID, "report: rows capacity too small");
            for (size_t i = 0; i < rows.size(); ++i)
                out->rows[i] = {rows[i].maturity, rows[i].strike, rows[i].market, rows[i].model,
                                rows[i].rel_error};
        }
        out->trace_len = static_cast<int64_t>(trace_f.size());
        if (out->trace_t && out->trace_f && out->trace_capacity > 0) {
            const size_t n = std::min(trace_f.size(), static_cast<size_t>(out->trace_capacity));
            for (size_t i = 0; i < n; ++i) {
                out->trace_t[i] = trace_t[i];
                out->trace_f[i] = trace_f[i];
            }
        }
    }
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------- T_I annealer ---
// True when every dim is free and, for every x in [lo, hi] and every step of
// propose (annealer.cpp:60-74), the first reflection already lands in
// [lo, hi].  The step is s = RN(RN(range*scale) * sym) with scale <= 1 and
// sym = 2u - 1 in [-1, 1 - 2^-52], so -range <= s <= RN(range*(1 - 2^-52))
// and (rounding is monotone) v = RN(x + s) lies in
// [RN(lo - range), RN(hi + RN(range*(1 - 2^-52)))]; if 2hi - v >= lo and
// 2lo - v <= hi hold at those extremes, the reference's second reflection and
// its clamp never change the value, and the level kernels use
// propose_coord_fast (same bits, fewer compares).
// free_only: the property for the searched dims (fixed dims never move)
bool single_reflection(const SaLevelArgs& a, int dim_full, bool free_only = false) {
    static const bool enabled = [] {  // SABR_SA_FAST=0: general propose (A/B checks)
        const char* e = std::getenv("SABR_SA_FAST");
        return !(e && std::atoi(e) == 0);
    }();
    if (!enabled) return false;
    for (int i = 0; i < dim_full; ++i) {
        if (!((a.free_mask >> i) & 1u)) {
            if (free_only) continue;
            return false;
        }
        const double vmax = a.hi[i] + a.range[i] * (1.0 - 0x1.0p-52), vmin = a.lo[i] - a.range[i];
        if (!std::isfinite(vmax) || !std::isfinite(vmin) || !std::isfinite(a.hi2[i]) ||
            !std::isfinite(a.lo2[i]))
            return false;
        if (!(a.hi2[i] - vmax >= a.lo[i]) || !(a.lo2[i] - vmin <= a.hi[i])) return false;
    }
    return true;
}

struct T1Out {
    std::vector<double> best_full;
    double best_value = 0.0;
    int64_t evals = 0;
    std::vector<double> trace_t, trace_f;
};

// minimize (annealer.cpp:76-167) for a device objective; `start_full` is the
// full parameter vector (fixed entries at their values), only dims in
// free_mask are searched.
using StartFn = std::function<cudaError_t(const SaLevelArgs&)>;
using LevelFn = std::function<cudaError_t(const SaLevelArgs&, int64_t, double)>;
using RunAllFn = std::function<cudaError_t(const SaLevelArgs&, const double*, int64_t)>;

// The device-resident level loop shared by every T_I-style objective:
// `start` seeds incumbent/best values on the device, `level` launches one
// temperature level (whose last CTA merges, or which writes the rank record
// for the NCCL merge).  `records` = CTA records one level kernel writes.
// All ranks' exchange modes must agree (one all-gather, also a barrier).
void mode_consensus(sabr_ctx* ctx, uint64_t mine) {
    auto* dsend = static_cast<uint64_t*>(dev_buf(ctx, "mode_send", sizeof(uint64_t)));
    auto* drecv = static_cast<uint64_t*>(dev_buf(ctx, "mode_recv", sizeof(uint64_t) * ctx->nranks));
    check_cuda(cudaMemcpyAsync(dsend, &mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream), "H2D mode");
    allgather(ctx, dsend, drecv, sizeof(uint64_t));
    std::vector<uint64_t> modes(ctx->nranks);
    check_cuda(cudaMemcpyAsync(modes.data(), drecv, sizeof(uint64_t) * ctx->nranks, cudaMemcpyDeviceToHost,
                               ctx->stream), "D2H modes");
    sync(ctx);
    for (int r = 0; r < ctx->nranks; ++r)
        if (modes[r] != mine)
            fail(SABR_E_INVALID, "exchange mode differs between ranks (enable/disable the peer exchange on "
                                 "every rank)");
}

T1Out run_sa_generic(sabr_ctx* ctx, int dim_full, uint32_t free_mask, const std::vector<double>& lo,
                     const std::vector<double>& hi, const std::vector<double>& start_full,
                     const sabr_schedule& sch, bool start_ok, int64_t records,
                     const StartFn& start, const LevelFn& level_fn, int builtin, int pred,
                     bool use_peer = false, const RunAllFn& run_all = nullptr,
                     bool skips_infeasible = false) {
    validate_schedule(sch);
    // SearchSpace::validate, annealer.cpp:48-58
    if (free_mask == 0) fail(SABR_E_DOMAIN, "SearchSpace: bounds must be nonempty and equal-sized");
    for (int i = 0; i < dim_full; ++i)
        if (((free_mask >> i) & 1u) && !(lo[i] < hi[i]))
            fail(SABR_E_DOMAIN, "SearchSpace: lower must be strictly below upper");
    bool feasible = true;
    for (int i = 0; i < dim_full; ++i)
        if (((free_mask >> i) & 1u) && (start_full[i] < lo[i] || start_full[i] > hi[i])) feasible = false;
    if (pred == SABR_PRED_SUM_LE_1 && !(start_full[0] + start_full[1] <= 1.0)) feasible = false;
    if (!feasible || !start_ok) fail(SABR_E_DOMAIN, "annealer: start point is infeasible");

    const std::vector<double> temps = temperatures(sch, pred == SABR_PRED_NONE && !skips_infeasible ? level_cap_all_evals(sch) : -1);
    const int64_t L = static_cast<int64_t>(temps.size());
    const int64_t n_chains = static_cast<int64_t>(sch.workers) * sch.groups;
    const int64_t begin = ctx->rank * n_chains / ctx->nranks;
    const int64_t end = (ctx->rank + 1) * n_chains / ctx->nranks;

    sabr_sa_state st{};
    for (int i = 0; i < dim_full; ++i) st.incumbent[i] = st.best[i] = start_full[i];
    st.evals = 1;
    st.done = (L == 0 || st.evals >= sch.max_evals) ? 1 : 0;
    st.eval_cap = st.done ? 0 : (sch.max_evals - st.evals + n_chains - 1) / n_chains;

    const int64_t grid = std::max<int64_t>(1, records);
    SaLevelArgs a{};
    for (int i = 0; i < dim_full; ++i) {
        a.lo[i] = lo[i];
        a.hi[i] = hi[i];
        a.range[i] = hi[i] - lo[i];
        a.lo2[i] = 2.0 * lo[i];
        a.hi2[i] = 2.0 * hi[i];
    }
    a.free_mask = free_mask;
    a.fast = single_reflection(a, dim_full) ? 1 : 0;
    a.fast_free = single_reflection(a, dim_full, true) ? 1 : 0;
    a.beta_one = (dim_full > 1 && !((free_mask >> 1) & 1u) && start_full[1] == 1.0) ? 1 : 0;
    a.dim_full = dim_full;
    a.chain_length = sch.chain_length;
    a.builtin = builtin;
    a.predicate = pred;
    a.nranks = ctx->nranks;
    a.t0 = sch.t0;
    a.seed = sch.seed;
    a.chain_begin = begin;
    a.n_local = end - begin;
    a.n_chains = n_chains;
    a.max_evals = sch.max_evals;
    a.levels_total = L;
    a.state = static_cast<sabr_sa_state*>(dev_buf(ctx, "sa_state", sizeof(sabr_sa_state)));
    a.block_recs = static_cast<sabr_level_record*>(
        dev_buf(ctx, "sa_block_recs", sizeof(sabr_level_record) * grid));
    a.block_sum = static_cast<BlockSummary*>(dev_buf(ctx, "sa_block_sum", sizeof(BlockSummary) * grid));
    a.rank_rec = static_cast<sabr_level_record*>(dev_buf(ctx, "sa_rank_rec", sizeof(sabr_level_record)));
    auto* recv = static_cast<sabr_level_record*>(
        dev_buf(ctx, "sa_recv_recs", sizeof(sabr_level_record) * ctx->nranks));
    a.ticket = static_cast<unsigned int*>(dev_buf(ctx, "sa_ticket", sizeof(unsigned int)));
    a.trace_f = static_cast<double*>(dev_buf(ctx, "sa_trace", sizeof(double) * std::max<int64_t>(1, L)));
    check_cuda(cudaMemcpyAsync(a.state, &st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream), "H2D state");
    check_cuda(cudaMemsetAsync(a.ticket, 0, sizeof(unsigned int), ctx->stream), "memset ticket");
    if (a.n_local == 0) {  // a rank without chains contributes an empty record every level
        sabr_level_record empty{};
        empty.end_chain = empty.best_chain = -1;
        check_cuda(cudaMemcpyAsync(a.rank_rec, &empty, sizeof(empty), cudaMemcpyHostToDevice, ctx->stream),
                   "H2D record");
    }
    check_cuda(start(a), "sa_start");

    // fused peer exchange (all ranks decide alike: every rank has chains iff n_chains >= nranks)
    const bool peer = ctx->peer && ctx->nranks > 1 && n_chains >= ctx->nranks && use_peer;
    // Every rank must run the same exchange mode: a rank on the peer
    // mailboxes and a rank in the per-level all-gather would wait on each
    // other.  One all-gather of the mode byte over the transport, which
    // doubles as a barrier before level 0, so the mailbox timeout below
    // starts with every rank inside the run.  (A child context of
    // sabr_calibrate_static_T1_slices borrows its parent's transport; the
    // parent ran this check for all of them before the children started.)
    if (ctx->nranks > 1 && !ctx->child) mode_consensus(ctx, peer ? 1u : 0u);
    if (peer) {
        a.peer_boxes = ctx->peer_boxes;
        a.my_rank = ctx->rank;
        a.epoch_base = ctx->peer_epoch;
        a.peer_error = ctx->peer_error;
        ctx->peer_epoch += static_cast<unsigned long long>(L);
        // a timeout of an earlier run must not fail this one
        check_cuda(cudaMemsetAsync(ctx->peer_error, 0, sizeof(int), ctx->stream), "memset peer error");
    }

    Timer timer(ctx);
    timer.start();
    int64_t launched = 0;
    auto* done_flag = static_cast<int64_t*>(ctx->pinned);
    int64_t first_level = 0;
    if (run_all && L > 0 && a.n_local > 0 && ctx->nranks == 1 && run_all(a, nullptr, L) == cudaSuccess) {
        // one launch for every level (a one-CTA run)
        const double* temps_dev = upload(ctx, "sa_temps", temps);
        timer.before();
        check_cuda(run_all(a, temps_dev, L), "sa_run_small");
        timer.after();
        ++launched;
        first_level = L;
    }
    for (int64_t level = first_level; level < L; ++level) {
        NvtxRange nvtx_level("sabr.level");
        if (a.n_local > 0) {
            timer.before();
            check_cuda(level_fn(a, level, temps[level]), "sa_level");
            timer.after();
            ++launched;
        }
        if (ctx->nranks > 1 && !peer) {
            allgather(ctx, a.rank_rec, recv, sizeof(sabr_level_record));
            check_cuda(launch_sa_merge(a, recv, level, ctx->stream), "sa_merge");
        }
        if ((level & 31) == 31 && level + 1 < L) {  // early stop on max_evals
            check_cuda(cudaMemcpyAsync(done_flag, &a.state->done, sizeof(int64_t),
                                       cudaMemcpyDeviceToHost, ctx->stream), "D2H done");
            sync(ctx);
            if (*done_flag) break;
        }
    }
    sabr_sa_state out{};
    check_cuda(cudaMemcpyAsync(&out, a.state, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream), "D2H state");
    sync(ctx);
    timer.stop(static_cast<double>(out.evals - 1), 0.0, launched, launched);
    if (peer) {
        int err = 0;
        check_cuda(cudaMemcpy(&err, ctx->peer_error, sizeof(int), cudaMemcpyDeviceToHost), "D2H peer error");
        if (err) fail(SABR_E_NCCL, "peer exchange: a rank's level record did not arrive within 20 s");
    }

    T1Out r;
    r.best_full.assign(out.best, out.best + dim_full);
    r.best_value = out.best_value;
    r.evals = out.evals;
    r.trace_f.resize(out.levels_run);
    if (out.levels_run > 0) {
        check_cuda(cudaMemcpy(r.trace_f.data(), a.trace_f, sizeof(double) * out.levels_run,
                              cudaMemcpyDeviceToHost), "D2H trace");
    }
    r.trace_t.assign(temps.begin(), temps.begin() + out.levels_run);
    return r;
}

// minimize (annealer.cpp:76-167) for the thread-per-chain objectives.
T1Out run_sa_t1(sabr_ctx* ctx, int kind, const SurfaceView& sv, int dim_full, uint32_t free_mask,
                const std::vector<double>& lo, const std::vector<double>& hi,
                const std::vector<double>& start_full, const sabr_schedule& sch, int builtin,
                int pred) {
    const int64_t n_chains = static_cast<int64_t>(sch.workers) * sch.groups;
    const int64_t n_local = (ctx->rank + 1) * n_chains / ctx->nranks - ctx->rank * n_chains / ctx->nranks;
    const int threads = sa_block_threads();
    const int64_t records = (n_local + threads - 1) / threads;
    cudaStream_t s = ctx->stream;
    return run_sa_generic(
        ctx, dim_full, free_mask, lo, hi, start_full, sch, true, records,
        [&](const SaLevelArgs& a) { return launch_sa_start(kind, sv, a, s); },
        [&](const SaLevelArgs& a, int64_t level, double temp) {
            return launch_sa_level(kind, sv, a, level, temp, s);
        },
        builtin, pred, /*use_peer=*/true,
        [&](const SaLevelArgs& a, const double* temps, int64_t n_levels) {
            return launch_sa_run_small(kind, sv, a, temps, n_levels, s);
        });
}

// GaussLegendreRule(n), proj/src/quadrature.cpp:13-33 (same Newton iteration,
// same nodes/weights to the last bit).
void gauss_legendre(int n, double* nodes, double* weights) {
    constexpr double kPi = 3.14159265358979323846;
    const int m = (n + 1) / 2;
    for (int i = 0; i < m; ++i) {
        double x = std::cos(kPi * (i + 0.75) / (n + 0.5));
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
            if (std::abs(dx) < 1e-15) break;
        }
        nodes[i] = -x;
        nodes[n - 1 - i] = x;
        weights[i] = weights[n - 1 - i] = 2.0 / ((1.0 - x * x) * pp * pp);
    }
}

// Device view of the calibrate_case2_formula objective (calibration.cpp:483-520).
C2fView make_c2f_view(sabr_ctx* ctx, const HostSurface& s, const std::vector<double>& market,
                      double horizon, int gl_n = 8) {
    if (s.n() > static_cast<size_t>(kMaxC2fSlices))
        fail(SABR_E_DOMAIN, "calibrate_case2_formula: at most 64 slices on the device");
    std::vector<C2fSlice> sl(s.n());
    std::vector<C2fQuote> q(s.total_quotes());
    for (size_t i = 0; i < s.n(); ++i) {
        const double f = s.forward(i);
        sl[i] = {s.T[i], std::sqrt(s.T[i]), f, s.r[i] - s.y[i]};
        for (int64_t j = s.off[i]; j < s.off[i + 1]; ++j) {
            const double lm = std::log(s.K[j] / f);
            q[j] = {lm, lm * lm, std::log(s.spot / s.K[j]), s.spot * std::exp(-s.y[i] * s.T[i]),
                    s.K[j] * std::exp(-s.r[i] * s.T[i]), market[j], 1.0 / market[j],
                    static_cast<int32_t>(i), 0};
        }
    }
    C2fView v{};
    v.ns = static_cast<int32_t>(s.n());
    v.nq = static_cast<int32_t>(s.total_quotes());
    v.sl = upload(ctx, "c2f_slices", sl);
    v.q = upload(ctx, "c2f_quotes", q);
    v.horizon = horizon;
    v.gl_n = gl_n;  // dyn_coeffs_case2(p, T, 8), calibration.cpp:506 (64: the default, model vols)
    gauss_legendre(v.gl_n, v.gl_x, v.gl_w);
    v.exptab = exp_table_device(ctx);
    return v;
}

std::vector<double> c2f_costs(sabr_ctx* ctx, const C2fView& v, const std::vector<double>& params11) {
    const int64_t n = static_cast<int64_t>(params11.size()) / 11;
    std::vector<double> out(n);
    if (n == 0) return out;
    double* dp = upload(ctx, "c2f_params", params11);
    double* dc = static_cast<double*>(dev_buf(ctx, "c2f_cost", sizeof(double) * n));
    check_cuda(launch_c2f_cost(v, dp, n, dc, ctx->stream), "c2f_cost");
    check_cuda(cudaMemcpyAsync(out.data(), dc, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream),
               "D2H cost");
    sync(ctx);
    return out;
}

// Objective value(s) of full vectors on the device.
std::vector<double> device_costs(sabr_ctx* ctx, int kind, const SurfaceView& sv,
                                 const std::vector<double>& params, int dim) {
    const int64_t n = static_cast<int64_t>(params.size()) / dim;
    std::vector<double> out(n);
    if (n == 0) return out;
    double* dp = upload(ctx, "cost_params", params);
    double* dc = static_cast<double*>(dev_buf(ctx, "cost_out", sizeof(double) * n));
    check_cuda(launch_cost_batch(kind, sv, dp, dim, n, dc, ctx->stream), "cost_batch");
    check_cuda(cudaMemcpyAsync(out.data(), dc, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream),
               "D2H cost");
    sync(ctx);
    return out;
}

std::vector<double> device_vols(sabr_ctx* ctx, int kind, const SurfaceView& sv,
                                const std::vector<double>& params, int dim, int64_t nq) {
    const int64_t n = static_cast<int64_t>(params.size()) / dim;
    std::vector<double> out(n * nq);
    if (n == 0 || nq == 0) return out;
    double* dp = upload(ctx, "vol_params", params);
    double* dv = static_cast<double*>(dev_buf(ctx, "vol_out", sizeof(double) * n * nq));
    check_cuda(launch_vol_batch(kind, sv, dp, dim, n, dv, ctx->stream), "vol_batch");
    check_cuda(cudaMemcpyAsync(out.data(), dv, sizeof(double) * n * nq, cudaMemcpyDeviceToHost, ctx->stream),
               "D2H vols");
    sync(ctx);
    return out;
}

// The box of a T_I search must stay inside the model domain: the reference
// would raise the model's domain_error (or abort inside its OpenMP region)
// at the first proposal outside it; we reject such boxes up front.
void check_box(int model, const ParamSpace& ps) {
    const size_t d = ps.defs.size();
    std::vector<double> corner(d);
    for (int pass = 0; pass < 2; ++pass) {
        for (size_t i = 0; i < d; ++i)
            corner[i] = ps.is_free[i] ? (pass == 0 ? ps.defs[i].lo : ps.defs[i].hi) : ps.fixed_values[i];
        if (model == SABR_MODEL_STATIC) validate_static(corner.data());
        else validate_case1(corner.data());
    }
}

std::vector<double> market_prices(const HostSurface& s) {
    std::vector<double> m(s.total_quotes());
    for (size_t i = 0; i < s.n(); ++i)
        for (int64_t j = s.off[i]; j < s.off[i + 1]; ++j)
            m[j] = black_scholes_call(s.spot, s.K[j], s.r[i], s.y[i], s.T[i], s.vol[j]);
    return m;
}

Report evaluate_case1_impl(sabr_ctx* ctx, const HostSurface& surface, const double* p) {
    surface.validate();
    Report rep{"case1", "T_I", "vol"};
    rep.params = {{"alpha", p[0]}, {"beta", p[1]}, {"rho0", p[2]}, {"nu0", p[3]}, {"a", p[4]}, {"b", p[5]}};
    validate_case1(p);
    for (size_t i = 0; i < surface.n(); ++i) {
        surface.forward(i);
        require(surface.T[i] > 0, "dyn_coeffs_case1: maturity must be positive");
    }
    const SurfaceView sv = make_view(ctx, "view_case1", surface, nullptr);
    const std::vector<double> pv(p, p + 6);
    const auto vols = device_vols(ctx, OBJ_CASE1, sv, pv, 6, static_cast<int64_t>(surface.total_quotes()));
    for (size_t i = 0; i < surface.n(); ++i)
        for (int64_t j = surface.off[i]; j < surface.off[i + 1]; ++j)
            rep.rows.push_back({surface.T[i], surface.K[j], surface.vol[j], vols[j],
                                std::abs(surface.vol[j] - vols[j]) / surface.vol[j]});
    rep.aggregates();
    rep.final_cost = device_costs(ctx, OBJ_CASE1, sv, pv, 6)[0];
    return rep;
}

Report evaluate_case2_impl(sabr_ctx* ctx, const HostSurface& surface, const double* p,
                           const sabr_plan& plan) {
    surface.validate();
    Report rep{"case2", "T_II", "price"};
    rep.params = {{"alpha", p[0]}, {"beta", p[1]}, {"rho0", p[2]}, {"q_rho", p[3]},
                  {"d_rho", p[4]}, {"nu0", p[5]},  {"q_nu", p[6]}, {"d_nu", p[7]},
                  {"a", p[8]},     {"b", p[9]}};
    rep.seed = plan.seed;
    const auto market = market_prices(surface);
    validate_case2(p);
    std::vector<double> value, se;
    mc_price_single(ctx, SABR_MODEL_CASE2, p, surface.spot, surface.T, surface.r, surface.y,
                    surface.off, surface.K, plan, value, se);
    for (size_t i = 0; i < surface.n(); ++i)
        for (int64_t j = surface.off[i]; j < surface.off[i + 1]; ++j)
            rep.rows.push_back({surface.T[i], surface.K[j], market[j], value[j],
                                std::abs(market[j] - value[j]) / market[j]});
    rep.aggregates();
    rep.final_cost = 0.0;
    for (const auto& r : rep.rows) rep.final_cost += r.rel_error * r.rel_error;
    return rep;
}


// ------------------------------------------------------- surface CSV IO ---
std::vector<std::string> split(const std::string& line, char sep) {
    std::vector<std::string> out;
    std::string cur;
    for (const char c : line) {
        if (c == sep) {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += c;
        }
    }
    out.push_back(cur);
    return out;
}

[[noreturn]] void parse_fail(const std::string& what, long line = -1) {
    fail(SABR_E_RUNTIME, line >= 0 ? what + " (line " + std::to_string(line) + ")" : what);
}

double parse_number(const std::string& token, long line) {
    double value{};
    const char* first = token.data();
    const char* last = token.data() + token.size();
    const auto res = std::from_chars(first, last, value);
    if (res.ec != std::errc{} || res.ptr != last) parse_fail("not a number: '" + token + "'", line);
    return value;
}

// io::parse_surface (proj/src/io.cpp:50-161): grammar, percent conversion
// and validation with the same messages.
HostSurface parse_surface(const std::string& path) {
    std::ifstream in(path);
    if (!in) parse_fail("cannot open " + path);
    std::ostringstream text;
    text << in.rdbuf();
    std::istringstream lines(text.str());
    double spot = 0.0;
    bool saw_spot = false, saw_mode = false, percent = false;
    struct Sl {
        double T, r, y;
        std::vector<std::pair<double, double>> q;
    };
    std::vector<Sl> slices;
    std::string line;
    long lineno = 0;
    while (std::getline(lines, line)) {
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty() || line[0] == '#') continue;
        const auto f = split(line, ',');
        const std::string& key = f[0];
        if (key == "spot") {
            if (f.size() != 2) parse_fail("spot expects one value", lineno);
            spot = parse_number(f[1], lineno);
            saw_spot = true;
        } else if (key == "label" || key == "date") {
            if (f.size() != 2) parse_fail(key + " expects one value", lineno);
        } else if (key == "strikes") {
            if (f.size() != 2) parse_fail("strikes expects one value", lineno);
            if (f[1] == "percent") percent = true;
            else if (f[1] == "absolute") percent = false;
            else parse_fail("strikes must be 'percent' or 'absolute'", lineno);
            saw_mode = true;
        } else if (key == "slice") {
            if (f.size() != 4) parse_fail("slice expects maturity,rate,dividend", lineno);
            slices.push_back({parse_number(f[1], lineno), parse_number(f[2], lineno),
                              parse_number(f[3], lineno), {}});
        } else {
            if (f.size() != 2) parse_fail("quote row expects strike,vol", lineno);
            if (slices.empty()) parse_fail("quote row before any slice header", lineno);
            slices.back().q.push_back({parse_number(f[0], lineno), parse_number(f[1], lineno)});
        }
    }
    if (!saw_spot) parse_fail("missing spot header");
    if (!saw_mode) parse_fail("missing strikes header");
    if (slices.empty()) parse_fail("no slices");
    HostSurface s;
    s.spot = spot;
    s.off = {0};
    for (const auto& sl : slices) {
        s.T.push_back(sl.T);
        s.r.push_back(sl.r / 100.0);
        s.y.push_back(sl.y / 100.0);
        for (const auto& [k, v] : sl.q) {
            s.K.push_back(percent ? k / 100.0 * spot : k);
            s.vol.push_back(v / 100.0);
        }
        s.off.push_back(static_cast<int64_t>(s.K.size()));
    }
    try {
        s.validate();
    } catch (const Error& e) {
        parse_fail(std::string(e.what()) + " in " + path);
    }
    return s;
}

}  // namespace

// ======================================================= shared helpers ===
void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SABR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Host-built per-step coefficients (one candidate) for the chosen path-loop
// arithmetic: FP64 rows, plus their FP32 copy for SABR_FP32.
void set_coefficients(sabr_ctx* ctx, McParams& P, const std::vector<StepCoef>& coef, int precision) {
    P.coef = upload(ctx, "mc_coef", coef);
    P.fp32 = precision == SABR_FP32 ? 1 : 0;
    P.coef32 = nullptr;
    if (P.fp32) {  // {c1, -c2, rs, ss} * log2(e): mc_tile_kernel_f32's base-2 state (one candidate)
        constexpr double kLog2e = 1.4426950408889634;
        std::vector<float4> c32(coef.size());
        for (size_t i = 0; i < coef.size(); ++i)
            c32[i] = make_float4(static_cast<float>(coef[i].c1 * kLog2e), static_cast<float>(-coef[i].c2 * kLog2e),
                                 static_cast<float>(coef[i].rs * kLog2e), static_cast<float>(coef[i].ss * kLog2e));
        P.coef32 = upload(ctx, "mc_coef32", c32);
    }
}

const double2* exp_table_device(sabr_ctx* ctx) {
    auto it = ctx->bufs.find("exptab");
    if (it != ctx->bufs.end()) return static_cast<const double2*>(it->second.first);
    const double2* host = exp_table_host();
    return upload(ctx, "exptab", std::vector<double2>(host, host + sabr_dev::kExpTableSize));
}

const double2* sincos_table_device(sabr_ctx* ctx) {
    auto it = ctx->bufs.find("sctab");
    if (it != ctx->bufs.end()) return static_cast<const double2*>(it->second.first);
    const double2* host = sincos_table_host();
    return upload(ctx, "sctab", std::vector<double2>(host, host + sabr_dev::kSinCosTableSize));
}

const double4* log_table_device(sabr_ctx* ctx) {
    auto it = ctx->bufs.find("logtab");
    if (it != ctx->bufs.end()) return static_cast<const double4*>(it->second.first);
    const double4* host = log_table_host();
    return upload(ctx, "logtab", std::vector<double4>(host, host + sabr_dev::kLogTableSize));
}

void* dev_buf(sabr_ctx* ctx, const std::string& key, size_t bytes) {
    auto& slot = ctx->bufs[key];
    if (slot.second < bytes) {
        if (slot.first) {
            check_cuda(cudaStreamSynchronize(ctx->stream), "sync before realloc");
            cudaFree(slot.first);
            slot = {nullptr, 0};
        }
        void* p = nullptr;
        const size_t cap = std::max<size_t>(bytes, 256);
        check_cuda(cudaMalloc(&p, cap), "cudaMalloc");
        slot = {p, cap};
    }
    return slot.first;
}

Timer::Timer(sabr_ctx* c) : ctx(c) {}
void Timer::start() {
    t0 = std::chrono::steady_clock::now();
    ctx->kev_used = 0;
    if (ctx->profiling) check_cuda(cudaEventRecord(ctx->ev0, ctx->stream), "event record");
}
void Timer::before() {
    sampling = ctx->profiling && (calls++ % kSample == 0);
    if (!sampling) return;
    if (ctx->kev_used + 2 > ctx->kev.size()) {
        for (int i = 0; i < 256; ++i) {
            cudaEvent_t e;
            check_cuda(cudaEventCreate(&e), "event create");
            ctx->kev.push_back(e);
        }
    }
    check_cuda(cudaEventRecord(ctx->kev[ctx->kev_used++], ctx->stream), "event record");
}
void Timer::after() {
    if (!sampling) return;
    check_cuda(cudaEventRecord(ctx->kev[ctx->kev_used++], ctx->stream), "event record");
}
void Timer::stop(double units, double path_steps, int64_t kernel_launches, int64_t total_launches) {
    sabr_timing& t = ctx->timing;
    t.units = units;
    t.path_steps = path_steps;
    t.kernel_launches = kernel_launches;
    t.total_launches = total_launches;
    if (ctx->profiling) {
        check_cuda(cudaEventRecord(ctx->ev1, ctx->stream), "event record");
        check_cuda(cudaEventSynchronize(ctx->ev1), "event sync");
        float ms = 0.f;
        check_cuda(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "event elapsed");
        t.total_ms = ms;
        double kms = 0.0;
        size_t pairs = 0;
        for (size_t i = 0; i + 1 < ctx->kev_used; i += 2, ++pairs) {
            float k = 0.f;
            check_cuda(cudaEventElapsedTime(&k, ctx->kev[i], ctx->kev[i + 1]), "event elapsed");
            kms += k;
        }
        t.kernel_ms = pairs ? kms / pairs * static_cast<double>(calls) : ms;
    } else {
        t.total_ms = t.kernel_ms = 1e3 * seconds_since(t0);
    }
}

void allgather(sabr_ctx* ctx, const void* send, void* recv, size_t bytes) {
    if (ctx->nranks <= 1) {
        if (send != recv)
            check_cuda(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
        return;
    }
    if (ctx->exchange) {  // host transport: D2H, caller's all-gather, H2D
        std::vector<unsigned char> hs(bytes), hr(bytes * static_cast<size_t>(ctx->nranks));
        check_cuda(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H record");
        check_cuda(cudaStreamSynchronize(ctx->stream), "sync");
        if (ctx->exchange(ctx->exchange_user, hs.data(), hr.data(), static_cast<int64_t>(bytes)) != 0)
            fail(SABR_E_NCCL, "host exchange: the all-gather callback failed");
        check_cuda(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, ctx->stream), "H2D records");
        check_cuda(cudaStreamSynchronize(ctx->stream), "sync");
        return;
    }
    nccl_check(nccl().allGather(send, recv, bytes, ncclChar, static_cast<ncclComm_t>(ctx->comm),
                                ctx->stream),
               "ncclAllGather");
}

SurfaceView make_view(sabr_ctx* ctx, const std::string& key, const HostSurface& s,
                      const std::vector<double>* market) {
    const int ns = static_cast<int>(s.n());
    const int nq = static_cast<int>(s.total_quotes());
    // layout: quotes (16-byte aligned records) first, then the slices' QR
    // factors (slice_qr.hpp), then T, ln f (hi, lo)
    const size_t qr_off = 4 * static_cast<size_t>(nq);
    std::vector<double> d(qr_off + static_cast<size_t>(kQrStride) * ns + 3 * ns);
    std::vector<int32_t> qoff(ns + 1);
    double* sd = d.data() + qr_off + static_cast<size_t>(kQrStride) * ns;
    std::vector<double> lms, mkts;
    for (int i = 0; i < ns; ++i) {
        const double f = s.forward(i);
        const double lf = std::log(f);
        sd[i] = s.T[i];
        sd[ns + i] = lf;
        sd[2 * ns + i] = static_cast<double>(std::log(static_cast<long double>(f)) - static_cast<long double>(lf));
        qoff[i] = static_cast<int32_t>(s.off[i]);
        for (int64_t j = s.off[i]; j < s.off[i + 1]; ++j) {
            const double m = market ? (*market)[j] : s.vol[j];
            if (m == 0) fail(SABR_E_DOMAIN, "cost: zero market value");  // calibration.cpp:261
            const double lm = std::log(s.K[j] / f);  // analytics.cpp:203
            double* q = d.data() + 4 * j;
            q[0] = lm;
            q[1] = lm * lm;
            q[2] = m;
            q[3] = 1.0 / m;
        }
        lms.clear();
        mkts.clear();
        for (int64_t j = s.off[i]; j < s.off[i + 1]; ++j) {
            lms.push_back(d[4 * j]);
            mkts.push_back(d[4 * j + 2]);
        }
        slice_qr_factor(lms.data(), mkts.data(), static_cast<int64_t>(lms.size()),
                        d.data() + qr_off + static_cast<size_t>(kQrStride) * i);
    }
    qoff[ns] = nq;
    double* dd = upload(ctx, key + "_d", d);
    int32_t* dq = upload(ctx, key + "_q", qoff);
    SurfaceView v;
    v.n_slices = ns;
    v.n_quotes = nq;
    v.quotes = dd;
    v.qr = dd + qr_off;
    v.T = dd + qr_off + static_cast<size_t>(kQrStride) * ns;
    v.lnf_hi = v.T + ns;
    v.lnf_lo = v.T + 2 * ns;
    v.qoff = dq;
    v.exptab = exp_table_device(ctx);
    v.max_abs_lnf = 0.0;
    for (int i = 0; i < ns; ++i) v.max_abs_lnf = std::max(v.max_abs_lnf, std::fabs(sd[ns + i]));
    return v;
}

// build_grid, proj/src/mc.cpp:50-84 (same errors)
HostGrid build_grid(double maturity, double dt) {
    if (maturity <= 0) fail(SABR_E_DOMAIN, "mc: maturity must be positive");
    if (dt <= 0) fail(SABR_E_DOMAIN, "mc: dt must be positive");
    const auto full_steps = static_cast<size_t>(std::floor(maturity / dt + 1e-9));
    if (full_steps == 0) fail(SABR_E_DOMAIN, "mc: maturity shorter than one time step");
    HostGrid g;
    for (size_t i = 0; i < full_steps; ++i) {
        g.dt.push_back(dt);
        g.t_end.push_back(std::min((i + 1) * dt, maturity));
    }
    const double rem = maturity - full_steps * dt;
    if (rem > 1e-12 * std::max(maturity, 1.0)) {
        g.dt.push_back(rem);
        g.t_end.push_back(maturity);
    }
    for (double h : g.dt) g.sdt.push_back(std::sqrt(h));
    return g;
}

double model_nu_at(int model, const double* p, double t) {
    switch (model) {
        case SABR_MODEL_STATIC: return p[2];
        case SABR_MODEL_CASE1: return p[3] * std::exp(-p[5] * t);
        default: return (p[5] + p[6] * t) * std::exp(-p[9] * t) + p[7];
    }
}
double model_rho_at(int model, const double* p, double t) {
    switch (model) {
        case SABR_MODEL_STATIC: return p[3];
        case SABR_MODEL_CASE1: return p[2] * std::exp(-p[4] * t);
        default: return (p[2] + p[3] * t) * std::exp(-p[8] * t) + p[4];
    }
}

// CaseIIParams::validate with its messages (analytics.cpp:145-175).
void validate_case2(const double* p) {
    validate_case2_domain(p);
    const double horizon = p[10];
    std::vector<double> ts;
    for (int i = 1; i <= 256; ++i) ts.push_back(horizon * i / 256);
    if (p[8] > 0 && p[3] != 0) {
        const double t = 1.0 / p[8] - p[2] / p[3];
        if (t > 0 && t <= horizon) ts.push_back(t);
    }
    if (p[9] > 0 && p[6] != 0) {
        const double t = 1.0 / p[9] - p[5] / p[6];
        if (t > 0 && t <= horizon) ts.push_back(t);
    }
    for (double t : ts) {
        const double r = model_rho_at(SABR_MODEL_CASE2, p, t);
        if (r < -1 - 1e-9 || r > 1 + 1e-9)
            fail(SABR_E_CONSTRAINT, "CaseIIParams: rho(t) outside [-1,1] at t = " + std::to_string(t));
        if (model_nu_at(SABR_MODEL_CASE2, p, t) <= 0)
            fail(SABR_E_CONSTRAINT, "CaseIIParams: nu(t) not positive at t = " + std::to_string(t));
    }
}

bool case2_feasible_host(const double* p) {
    try {
        validate_case2(p);
        return true;
    } catch (const Error&) {
        return false;
    }
}

void validate_model(int model, const double* p) {
    if (!p) fail(SABR_E_INVALID, "params is null");
    switch (model) {
        case SABR_MODEL_STATIC: validate_static(p); return;
        case SABR_MODEL_CASE1: validate_case1(p); return;
        case SABR_MODEL_CASE2: validate_case2(p); return;
    }
    fail(SABR_E_DOMAIN, "unknown model");
}

// Paths per thread: a function of the plan alone (it fixes the payoff
// reduction tree, so prices never depend on the batch or the GPU count).
// Large plans amortise the xoshiro jump over 4 consecutive paths; plans
// below 2^18 paths keep one path per thread so even a single candidate fills
// the 148 SMs.
int choose_ppt(const sabr_plan& plan) {
    if (plan.num_paths < (1ull << 18)) return 1;
    if (plan.rng == SABR_RNG_PHILOX) return 4;
    for (int p : {4, 2})
        if (plan.block_size % p == 0) return p;
    return 1;
}

// every step of the grid has the same dt (no short last step)
bool uniform_grid(const HostGrid& g) {
    for (size_t i = 1; i < g.dt.size(); ++i)
        if (std::memcmp(&g.dt[i], &g.dt[0], sizeof(double)) != 0 || std::memcmp(&g.sdt[i], &g.sdt[0], sizeof(double)) != 0)
            return false;
    return true;
}

std::vector<uint64_t> mc_layout(sabr_ctx* ctx, const sabr_plan& plan, int ppt,
                                const std::vector<HostGrid>& grids, McJob& job) {
    std::vector<uint64_t> jump;
    job.total_steps = 0;
    const uint64_t in_block = std::min<uint64_t>(plan.block_size, plan.num_paths);
    const uint64_t count = (in_block + ppt - 1) / ppt;
    for (size_t s = 0; s < grids.size(); ++s) {
        McSlice& sl = job.slices[s];
        sl.n_steps = static_cast<int32_t>(grids[s].dt.size());
        sl.step_off = static_cast<int32_t>(job.total_steps);
        job.total_steps += sl.n_steps;
        for (double h : grids[s].dt) job.hdt.push_back(0.5 * h);
        sl.jump_off = 0;
        if (plan.rng == SABR_RNG_XOSHIRO) {
            const uint64_t draws = 2ull * sl.n_steps * ppt;
            auto key = std::make_pair(draws, count);
            auto it = ctx->jump_cache.find(key);
            if (it == ctx->jump_cache.end())
                it = ctx->jump_cache.emplace(key, xoshiro_jump_table(draws, count)).first;
            sl.jump_off = static_cast<int64_t>(jump.size() / 4);
            jump.insert(jump.end(), it->second.begin(), it->second.end());
        }
    }
    if (jump.empty()) jump.assign(4, 0);
    return jump;
}

void mc_price_single(sabr_ctx* ctx, int model, const double* params, double spot,
                     const std::vector<double>& maturity, const std::vector<double>& rate,
                     const std::vector<double>& dividend, const std::vector<int64_t>& qoff,
                     const std::vector<double>& strikes, const sabr_plan& plan,
                     std::vector<double>& value, std::vector<double>& se) {
    validate_plan(plan);
    const size_t ns = maturity.size();
    std::vector<HostGrid> grids;
    for (size_t s = 0; s < ns; ++s) grids.push_back(build_grid(maturity[s], plan.dt));
    const double alpha0 = params[0];
    const int ppt = choose_ppt(plan);
    McJob job;
    job.slices.resize(ns);
    const auto jump = mc_layout(ctx, plan, ppt, grids, job);
    std::vector<StepCoef> coef;
    coef.reserve(job.total_steps);
    for (size_t s = 0; s < ns; ++s) {
        McSlice& sl = job.slices[s];
        sl.q_begin = static_cast<int32_t>(qoff[s]);
        sl.q_end = static_cast<int32_t>(qoff[s + 1]);
        job.max_q = std::max(job.max_q, sl.q_end - sl.q_begin);
        // forward0 inline as in mc.cpp:258, discount mc.cpp:262
        sl.forward0 = spot * std::exp((rate[s] - dividend[s]) * maturity[s]);
        if (!(sl.forward0 > 0) || alpha0 < 0)
            fail(SABR_E_DOMAIN, "mc: forward0 must be positive and alpha0 nonnegative");
        sl.lnf0 = std::log(sl.forward0);
        sl.discount = std::exp(-rate[s] * maturity[s]);
        const HostGrid& g = grids[s];
        const size_t first = coef.size();
        for (size_t i = 0; i < g.dt.size(); ++i) {
            const double nu = model_nu_at(model, params, g.t_end[i]);
            const double rho = model_rho_at(model, params, g.t_end[i]);
            const double srho = std::sqrt(std::max(0.0, 1.0 - rho * rho));
            coef.push_back({nu * g.sdt[i], 0.5 * nu * nu * g.dt[i], rho * g.sdt[i], srho * g.sdt[i]});
        }
        sl.const_coef = uniform_grid(g) && std::all_of(coef.begin() + first, coef.end(), [&](const StepCoef& c) {
                            return std::memcmp(&c, &coef[first], sizeof(StepCoef)) == 0;
                        });
    }
    const int nq = static_cast<int>(strikes.size());
    McParams P{};
    P.n_slices = static_cast<int32_t>(ns);
    P.n_cand = 1;
    P.n_quotes = nq;
    P.max_q = job.max_q;
    P.ppt = ppt;
    P.n_tiles = static_cast<int32_t>((plan.num_paths + static_cast<uint64_t>(kMcThreads) * ppt - 1) /
                                     (static_cast<uint64_t>(kMcThreads) * ppt));
    P.rng = plan.rng;
    P.total_steps = job.total_steps;
    P.num_paths = plan.num_paths;
    P.block_size = plan.block_size;
    P.seed = plan.seed;
    P.slices = upload(ctx, "mc_slices", job.slices);
    P.host_slices = job.slices.data();
    const double beta = params[1];
    P.alpha0 = upload(ctx, "mc_alpha0", std::vector<double>{alpha0});
    P.beta = upload(ctx, "mc_beta", std::vector<double>{beta});
    P.active = nullptr;
    set_coefficients(ctx, P, coef, plan.precision);
    P.cand_stride = 1;
    P.hdt = upload(ctx, "mc_hdt", job.hdt);
    P.strikes = upload(ctx, "mc_strikes", strikes);
    P.jump = upload(ctx, "mc_jump", jump);
    P.exptab = exp_table_device(ctx);
    P.logtab = log_table_device(ctx);
    P.sctab = sincos_table_device(ctx);
    P.partials = static_cast<double*>(
        dev_buf(ctx, "mc_partials", sizeof(double) * 2 * static_cast<size_t>(nq) * P.n_tiles));
    P.terminals = nullptr;
    P.bad = static_cast<int*>(dev_buf(ctx, "mc_bad", sizeof(int)));
    check_cuda(cudaMemsetAsync(P.bad, 0, sizeof(int), ctx->stream), "memset bad");
    double* dv = static_cast<double*>(dev_buf(ctx, "mc_value", sizeof(double) * nq));
    double* ds = static_cast<double*>(dev_buf(ctx, "mc_se", sizeof(double) * nq));
    if (mc_max_cand_block(P.max_q, P.fp32 != 0) == 0)
        fail(SABR_E_RUNTIME, "price_european_batch: too many strikes in one slice for the MC tile kernel");
    Timer timer(ctx);
    timer.start();
    timer.before();
    check_cuda(launch_mc_tiles(P, 1, ctx->stream), "mc_tiles");
    timer.after();
    check_cuda(launch_mc_reduce(P, dv, ds, nullptr, nullptr, ctx->stream), "mc_reduce");
    value.resize(nq);
    se.resize(nq);
    int bad = 0;
    check_cuda(cudaMemcpyAsync(value.data(), dv, sizeof(double) * nq, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    check_cuda(cudaMemcpyAsync(se.data(), ds, sizeof(double) * nq, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    check_cuda(cudaMemcpyAsync(&bad, P.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync(ctx);
    timer.stop(static_cast<double>(plan.num_paths) * job.total_steps,
               static_cast<double>(plan.num_paths) * job.total_steps, 1, 2);
    if (bad) fail(SABR_E_RUNTIME, "mc: non-finite path value (scheme unstable for these inputs)");
}

}  // namespace sabr_gpu

using namespace sabr_gpu;

// =============================================================== C-ABI ===
extern "C" {

SABR_API const char* sabr_last_error(void) { return g_last_error.c_str(); }

SABR_API const char* sabr_version(void) { return "sabr_b200 0.1 (sm_100a)"; }

SABR_API sabr_status sabr_ctx_create(int32_t device, void* stream, sabr_ctx** out) {
    return guarded([&] {
        if (!out) fail(SABR_E_INVALID, "out is null");
        *out = nullptr;
        int n = 0;
        check_cuda(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n)
            fail(SABR_E_CUDA, "no CUDA device " + std::to_string(device) + " (" + std::to_string(n) + " visible)");
        check_cuda(cudaSetDevice(device), "cudaSetDevice");
        auto* c = new sabr_ctx();
        c->device = device;
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
        } else {
            check_cuda(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream create");
            c->own_stream = true;
        }
        check_cuda(cudaMallocHost(&c->pinned, 4096), "cudaMallocHost");
        check_cuda(cudaEventCreate(&c->ev0), "event create");
        check_cuda(cudaEventCreate(&c->ev1), "event create");
        *out = c;
    });
}

SABR_API void sabr_ctx_destroy(sabr_ctx* ctx) {
    if (!ctx) return;
    for (sabr_ctx* c : ctx->children) {
        c->comm = nullptr;  // borrowed from ctx
        sabr_ctx_destroy(c);
    }
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->bufs)
        if (kv.second.first) cudaFree(kv.second.first);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (auto e : ctx->kev) cudaEventDestroy(e);
    for (void* p : ctx->peer_opened) cudaIpcCloseMemHandle(p);
    if (ctx->peer_box) cudaFree(ctx->peer_box);
    if (ctx->comm && nccl().commDestroy) nccl().commDestroy(static_cast<ncclComm_t>(ctx->comm));
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

SABR_API sabr_status sabr_ctx_set_profiling(sabr_ctx* ctx, int32_t on) {
    return guarded([&] {
        CtxLock l(ctx);
        ctx->profiling = on != 0;
    });
}

SABR_API sabr_status sabr_ctx_last_timing(sabr_ctx* ctx, sabr_timing* out) {
    return guarded([&] {
        CtxLock l(ctx);
        if (!out) fail(SABR_E_INVALID, "out is null");
        *out = ctx->timing;
    });
}

SABR_API sabr_status sabr_comm_unique_id(uint8_t out[128]) {
    return guarded([&] {
        ncclUniqueId id;
        nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, id.internal, 128);
    });
}

SABR_API sabr_status sabr_ctx_init_host_exchange(sabr_ctx* ctx, int32_t rank, int32_t nranks,
                                                 sabr_allgather_fn fn, void* user) {
    return guarded([&] {
        CtxLock l(ctx);
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(SABR_E_INVALID, "bad rank/nranks");
        if (nranks > 1 && !fn) fail(SABR_E_INVALID, "exchange callback is null");
        ctx->rank = rank;
        ctx->nranks = nranks;
        ctx->exchange = nranks > 1 ? fn : nullptr;
        ctx->exchange_user = user;
    });
}

SABR_API sabr_status sabr_ctx_enable_peer_exchange(sabr_ctx* ctx) {
    return guarded([&] {
        CtxLock l(ctx);
        if (ctx->nranks <= 1) return;  // nothing to exchange
        if (ctx->nranks > kMaxPeerRanks) fail(SABR_E_INVALID, "peer exchange: at most 16 ranks");
        if (!ctx->comm && !ctx->exchange) fail(SABR_E_INVALID, "peer exchange: initialise a transport first");
        if (ctx->peer) return;
        PeerMailbox* box = nullptr;
        check_cuda(cudaMalloc(&box, sizeof(PeerMailbox)), "cudaMalloc mailbox");
        check_cuda(cudaMemset(box, 0, sizeof(PeerMailbox)), "memset mailbox");
        cudaIpcMemHandle_t h;
        check_cuda(cudaIpcGetMemHandle(&h, box), "cudaIpcGetMemHandle");
        // one all-gather of the 64-byte handles over the existing transport
        auto* dsend = static_cast<unsigned char*>(dev_buf(ctx, "peer_h_send", sizeof(h)));
        auto* drecv = static_cast<unsigned char*>(dev_buf(ctx, "peer_h_recv", sizeof(h) * ctx->nranks));
        check_cuda(cudaMemcpyAsync(dsend, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream), "H2D handle");
        allgather(ctx, dsend, drecv, sizeof(h));
        std::vector<cudaIpcMemHandle_t> all(ctx->nranks);
        check_cuda(cudaMemcpyAsync(all.data(), drecv, sizeof(h) * ctx->nranks, cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H handles");
        sync(ctx);
        std::vector<PeerMailbox*> ptrs(ctx->nranks, nullptr);
        for (int r = 0; r < ctx->nranks; ++r) {
            if (r == ctx->rank) {
                ptrs[r] = box;
                continue;
            }
            void* p = nullptr;
            check_cuda(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            ctx->peer_opened.push_back(p);
            ptrs[r] = static_cast<PeerMailbox*>(p);
        }
        ctx->peer_boxes = upload(ctx, "peer_boxes", ptrs);
        ctx->peer_error = static_cast<int*>(dev_buf(ctx, "peer_error", sizeof(int)));
        check_cuda(cudaMemsetAsync(ctx->peer_error, 0, sizeof(int), ctx->stream), "memset");
        // handshake: every rank's peer stores must arrive in every mailbox
        // before the level kernels rely on them
        const unsigned long long magic = 0x5AB200C0FFEE0000ull + static_cast<unsigned long long>(ctx->rank);
        check_cuda(launch_peer_hello(ctx->peer_boxes, ctx->nranks, ctx->rank, magic, ctx->stream), "peer hello");
        sync(ctx);
        allgather(ctx, dsend, drecv, sizeof(h));  // a barrier over the transport
        sync(ctx);
        std::vector<unsigned long long> hello(kMaxPeerRanks);
        check_cuda(cudaMemcpy(hello.data(), box->hello, sizeof(unsigned long long) * kMaxPeerRanks,
                              cudaMemcpyDeviceToHost), "D2H hello");
        for (int r = 0; r < ctx->nranks; ++r)
            if (hello[r] != 0x5AB200C0FFEE0000ull + static_cast<unsigned long long>(r))
                fail(SABR_E_NCCL, "peer exchange: a peer's stores did not reach this rank's mailbox");
        ctx->peer_box = box;
        ctx->peer = true;
    });
}

// Collective, like enable: a barrier over the transport (no rank can still be
// storing into a mailbox: runs are synchronous calls and every rank reaches
// this point), then the peers' mappings are closed and the own mailbox freed.
SABR_API sabr_status sabr_ctx_disable_peer_exchange(sabr_ctx* ctx) {
    return guarded([&] {
        CtxLock l(ctx);
        if (!ctx->peer) return;
        auto* dsend = static_cast<unsigned char*>(dev_buf(ctx, "peer_h_send", sizeof(cudaIpcMemHandle_t)));
        auto* drecv = static_cast<unsigned char*>(
            dev_buf(ctx, "peer_h_recv", sizeof(cudaIpcMemHandle_t) * ctx->nranks));
        allgather(ctx, dsend, drecv, sizeof(cudaIpcMemHandle_t));
        sync(ctx);
        for (void* p : ctx->peer_opened) cudaIpcCloseMemHandle(p);
        ctx->peer_opened.clear();
        if (ctx->peer_box) cudaFree(ctx->peer_box);
        ctx->peer_box = nullptr;
        ctx->peer_boxes = nullptr;
        ctx->peer = false;
    });
}

SABR_API sabr_status sabr_ctx_init_comm(sabr_ctx* ctx, const uint8_t uid[128], int32_t rank,
                                        int32_t nranks) {
    return guarded([&] {
        CtxLock l(ctx);
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(SABR_E_INVALID, "bad rank/nranks");
        if (nranks == 1) {
            ctx->rank = 0;
            ctx->nranks = 1;
            return;
        }
        ncclUniqueId id;
        std::memcpy(id.internal, uid, 128);
        ncclComm_t comm = nullptr;
        nccl_check(nccl().commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
        ctx->comm = comm;
        ctx->rank = rank;
        ctx->nranks = nranks;
    });
}

// calibrate_static_T1, proj/src/calibration.cpp:289-323
// the body of sabr_calibrate_static_T1 for a caller that holds ctx's lock
static sabr_status sabr_calibrate_static_T1_locked(sabr_ctx* ctx, const sabr_surface* surface_in,
                                                   int64_t slice_in, const sabr_bounds* bounds,
                                                   const sabr_schedule* schedule, const sabr_fixed* fixed,
                                                   sabr_report* report) {
    return guarded([&] {
        NvtxRange nvtx("sabr.calibrate_static_T1");
        if (!schedule) fail(SABR_E_INVALID, "schedule is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        surface.validate();
        const auto t0 = std::chrono::steady_clock::now();
        if (slice_in < 0) surface.at(static_cast<size_t>(-1));
        const size_t slice = static_cast<size_t>(slice_in);
        const ParamSpace ps(static_defs(), bounds_from_abi(bounds), fixed_from_abi(fixed),
                            atm_vol_guess(surface, slice));
        if (surface.quotes(slice) < ps.free_ix.size())
            fail(SABR_E_DOMAIN, "calibrate_static_T1: fewer quotes than free parameters");
        const HostSurface one = surface.slice_only(slice);
        const SurfaceView sv = make_view(ctx, "view_static", one, nullptr);

        Report rep{"static", "T_I", "vol"};
        std::vector<double> best_full;
        if (ps.free_ix.empty()) {  // run_or_evaluate, calibration.cpp:208-214
            best_full = ps.full({});
            validate_static(best_full.data());
            rep.final_cost = device_costs(ctx, OBJ_STATIC, sv, best_full, 4)[0];
            rep.evals = 1;
        } else {
            const auto start = ps.full(ps.start_point());
            validate_static(start.data());
            check_box(SABR_MODEL_STATIC, ps);
            std::vector<double> lo(4), hi(4);
            for (int i = 0; i < 4; ++i) {
                lo[i] = ps.defs[i].lo;
                hi[i] = ps.defs[i].hi;
            }
            const T1Out r = run_sa_t1(ctx, OBJ_STATIC, sv, 4, ps.free_mask(), lo, hi, start, *schedule,
                                      0, SABR_PRED_NONE);
            best_full = r.best_full;
            rep.final_cost = r.best_value;
            rep.evals = r.evals;
            rep.trace_t = r.trace_t;
            rep.trace_f = r.trace_f;
        }
        rep.params = ps.named(best_full);
        rep.seed = schedule->seed;
        const auto vols = device_vols(ctx, OBJ_STATIC, sv, best_full, 4,
                                      static_cast<int64_t>(one.total_quotes()));
        for (size_t j = 0; j < one.total_quotes(); ++j)
            rep.rows.push_back({one.T[0], one.K[j], one.vol[j], vols[j],
                                std::abs(one.vol[j] - vols[j]) / one.vol[j]});
        rep.aggregates();
        rep.wall_seconds = seconds_since(t0);
        rep.write(report);
    });
}

SABR_API sabr_status sabr_calibrate_static_T1(sabr_ctx* ctx, const sabr_surface* surface_in,
                                              int64_t slice_in, const sabr_bounds* bounds,
                                              const sabr_schedule* schedule,
                                              const sabr_fixed* fixed, sabr_report* report) {
    sabr_status s = SABR_OK;
    const sabr_status g = guarded([&] {
        CtxLock l(ctx);
        s = sabr_calibrate_static_T1_locked(ctx, surface_in, slice_in, bounds, schedule, fixed, report);
    });
    return g != SABR_OK ? g : s;
}

// calibrate_static_T1 over several slices (a caller's loop over slices,
// proj/tools/sabr_cli.cpp:70).  Single rank: one child context (own stream)
// and one host thread per slice, so independent slices' level kernels are
// co-resident (C2: 7.7e10 -> 9.6e10 cost-evals/s over the four EUR/USD
// slices, tools/slices_concurrent_probe.py); each slice runs exactly the code
// of sabr_calibrate_static_T1, so the reports are the same.
SABR_API sabr_status sabr_calibrate_static_T1_slices(sabr_ctx* ctx, const sabr_surface* surface,
                                                     const int64_t* slices, int64_t n,
                                                     const sabr_bounds* bounds,
                                                     const sabr_schedule* schedule,
                                                     const sabr_fixed* fixed, sabr_report* reports) {
    std::vector<sabr_status> st;
    std::vector<std::string> msg;
    const sabr_status s0 = guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.calibrate_static_T1_slices");
        if (n < 0 || (n > 0 && (!slices || !reports))) fail(SABR_E_INVALID, "slices / reports are null");
        st.assign(static_cast<size_t>(n), SABR_OK);
        msg.assign(static_cast<size_t>(n), std::string());
        if (n == 0) return;
        const auto t0 = std::chrono::steady_clock::now();
        // side by side: one rank, or ranks exchanging through peer mailboxes
        // (each child its own, so no run touches the shared transport); the
        // per-level transport all-gather serves one run at a time
        const bool side_by_side =
            n > 1 && (ctx->nranks == 1 || (ctx->peer && schedule != nullptr &&
                                           static_cast<int64_t>(schedule->workers) * schedule->groups >= ctx->nranks));
        if (!side_by_side) {
            sabr_timing sum{};
            for (int64_t i = 0; i < n; ++i) {
                st[i] = sabr_calibrate_static_T1_locked(ctx, surface, slices[i], bounds, schedule, fixed,
                                                        reports + i);
                if (st[i] != SABR_OK) {
                    msg[i] = g_last_error;
                    break;
                }
                sum.units += ctx->timing.units;
                sum.kernel_ms += ctx->timing.kernel_ms;
                sum.kernel_launches += ctx->timing.kernel_launches;
                sum.total_launches += ctx->timing.total_launches;
            }
            sum.total_ms = 1e3 * seconds_since(t0);
            ctx->timing = sum;
            return;
        }
        // at most kMaxSideBySide streams: worker w runs slices w, w + W, ...
        // in order (the same order on every rank)
        constexpr int64_t kMaxSideBySide = 8;
        const int64_t W = std::min(n, kMaxSideBySide);
        while (ctx->children.size() < static_cast<size_t>(W)) {
            sabr_ctx* c = nullptr;
            if (sabr_ctx_create(ctx->device, nullptr, &c) != SABR_OK) fail(SABR_E_CUDA, g_last_error);
            c->child = true;
            ctx->children.push_back(c);
        }
        if (ctx->nranks > 1) {
            // the children borrow the transport for their mailbox set-up only
            // (collective: every rank enables child 0, 1, ... in this order),
            // then one mode check on the parent is the barrier before level 0
            for (int64_t w = 0; w < W; ++w) {
                sabr_ctx* c = ctx->children[w];
                c->rank = ctx->rank;
                c->nranks = ctx->nranks;
                c->comm = ctx->comm;
                c->exchange = ctx->exchange;
                c->exchange_user = ctx->exchange_user;
                if (!c->peer && sabr_ctx_enable_peer_exchange(c) != SABR_OK) fail(SABR_E_NCCL, g_last_error);
            }
            mode_consensus(ctx, 2u);
        }
        // the children start after ctx's stream's prior work
        check_cuda(cudaEventRecord(ctx->ev0, ctx->stream), "event record");
        for (int64_t w = 0; w < W; ++w) {
            ctx->children[w]->profiling = ctx->profiling;
            check_cuda(cudaStreamWaitEvent(ctx->children[w]->stream, ctx->ev0, 0), "stream wait");
        }
        std::vector<sabr_timing> tm(static_cast<size_t>(n));
        std::vector<std::thread> th;
        th.reserve(static_cast<size_t>(W));
        for (int64_t w = 0; w < W; ++w)
            th.emplace_back([&, w] {
                sabr_ctx* c = ctx->children[w];
                for (int64_t i = w; i < n; i += W) {
                    st[i] = sabr_calibrate_static_T1(c, surface, slices[i], bounds, schedule, fixed, reports + i);
                    tm[i] = c->timing;
                    if (st[i] != SABR_OK) {
                        msg[i] = g_last_error;
                        break;
                    }
                }
            });
        for (auto& t : th) t.join();
        // ctx's stream continues after the children's work
        sabr_timing sum{};
        for (int64_t w = 0; w < W; ++w) {
            sabr_ctx* c = ctx->children[w];
            check_cuda(cudaEventRecord(c->ev1, c->stream), "event record");
            check_cuda(cudaStreamWaitEvent(ctx->stream, c->ev1, 0), "stream wait");
        }
        for (const sabr_timing& t : tm) {
            sum.units += t.units;
            sum.kernel_ms += t.kernel_ms;
            sum.kernel_launches += t.kernel_launches;
            sum.total_launches += t.total_launches;
        }
        sum.total_ms = 1e3 * seconds_since(t0);
        ctx->timing = sum;
    });
    if (s0 != SABR_OK) return s0;
    for (size_t i = 0; i < st.size(); ++i)
        if (st[i] != SABR_OK) {
            g_last_error = msg[i];
            return st[i];
        }
    return SABR_OK;
}

// calibrate_dynamic_case1_T1, proj/src/calibration.cpp:325-365
SABR_API sabr_status sabr_calibrate_dynamic_case1_T1(sabr_ctx* ctx, const sabr_surface* surface_in,
                                                     const sabr_bounds* bounds,
                                                     const sabr_schedule* schedule,
                                                     const sabr_fixed* fixed, sabr_report* report) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.calibrate_dynamic_case1_T1");
        if (!schedule) fail(SABR_E_INVALID, "schedule is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        surface.validate();
        if (surface.n() < 2)
            fail(SABR_E_DOMAIN, "calibrate_dynamic_case1_T1: need at least two slices");
        const auto t0 = std::chrono::steady_clock::now();
        const ParamSpace ps(case1_defs(), bounds_from_abi(bounds), fixed_from_abi(fixed),
                            atm_vol_guess(surface, 0));
        const SurfaceView sv = make_view(ctx, "view_case1", surface, nullptr);
        std::vector<double> best_full;
        double best_value;
        int64_t evals;
        std::vector<double> tt, tf;
        if (ps.free_ix.empty()) {
            best_full = ps.full({});
            validate_case1(best_full.data());
            best_value = device_costs(ctx, OBJ_CASE1, sv, best_full, 6)[0];
            evals = 1;
        } else {
            const auto start = ps.full(ps.start_point());
            validate_case1(start.data());
            check_box(SABR_MODEL_CASE1, ps);
            std::vector<double> lo(6), hi(6);
            for (int i = 0; i < 6; ++i) {
                lo[i] = ps.defs[i].lo;
                hi[i] = ps.defs[i].hi;
            }
            const T1Out r = run_sa_t1(ctx, OBJ_CASE1, sv, 6, ps.free_mask(), lo, hi, start, *schedule,
                                      0, SABR_PRED_NONE);
            best_full = r.best_full;
            best_value = r.best_value;
            evals = r.evals;
            tt = r.trace_t;
            tf = r.trace_f;
        }
        Report rep = evaluate_case1_impl(ctx, surface, best_full.data());
        rep.params = ps.named(best_full);
        rep.final_cost = best_value;
        rep.evals = evals;
        rep.seed = schedule->seed;
        rep.trace_t = tt;
        rep.trace_f = tf;
        rep.wall_seconds = seconds_since(t0);
        rep.write(report);
    });
}

// calibrate_case2_T2, proj/src/calibration.cpp:450-481
SABR_API sabr_status sabr_calibrate_case2_T2(sabr_ctx* ctx, const sabr_surface* surface_in,
                                             const sabr_bounds* bounds,
                                             const sabr_schedule* schedule, const sabr_plan* plan,
                                             const sabr_fixed* fixed, const sabr_plan* report_plan,
                                             const double* start_override, int64_t start_len,
                                             sabr_report* report) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.calibrate_case2_T2");
        if (!schedule || !plan) fail(SABR_E_INVALID, "schedule/plan is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        surface.validate();
        validate_plan(*plan);
        const auto t0 = std::chrono::steady_clock::now();
        const double horizon = surface.T.back();
        const ParamSpace ps(case2_defs(), bounds_from_abi(bounds), fixed_from_abi(fixed),
                            atm_vol_guess(surface, 0));
        const auto market = market_prices(surface);
        std::vector<double> best_full;
        double best_value;
        int64_t evals;
        std::vector<double> tt, tf;
        auto with_h = [&](std::vector<double> v) {
            v.push_back(horizon);
            return v;
        };
        if (ps.free_ix.empty()) {
            best_full = ps.full({});
            const auto p = with_h(best_full);
            validate_case2(p.data());
            std::vector<double> value, se;
            mc_price_single(ctx, SABR_MODEL_CASE2, p.data(), surface.spot, surface.T, surface.r,
                            surface.y, surface.off, surface.K, *plan, value, se);
            best_value = 0.0;
            for (size_t i = 0; i < surface.n(); ++i)
                for (int64_t j = surface.off[i]; j < surface.off[i + 1]; ++j) {
                    const double rel = (market[j] - value[j]) / market[j];
                    best_value += rel * rel;
                }
            evals = 1;
        } else {
            validate_schedule(*schedule);
            std::vector<double> start;
            if (start_override) start.assign(start_override, start_override + start_len);
            else start = ps.start_point();
            bool ok = start.size() == ps.free_ix.size();
            for (size_t k = 0; ok && k < start.size(); ++k) {
                const auto& d = ps.defs[ps.free_ix[k]];
                if (start[k] < d.lo || start[k] > d.hi) ok = false;
            }
            if (ok) ok = case2_feasible_host(with_h(ps.full(start)).data());
            if (!ok) fail(SABR_E_DOMAIN, "annealer: start point is infeasible");
            const AnnealOut r = run_sa_case2(ctx, surface, market, ps, ps.full(start), horizon,
                                             *schedule, *plan);
            best_full = r.best_full;
            best_value = r.best_value;
            evals = r.evals;
            tt = r.trace_t;
            tf = r.trace_f;
        }
        const auto bp = with_h(best_full);
        const sabr_timing sa_timing = ctx->timing;  // the report's MC run must not replace it
        Report rep = evaluate_case2_impl(ctx, surface, bp.data(), report_plan ? *report_plan : *plan);
        ctx->timing = sa_timing;
        rep.params = ps.named(best_full);
        rep.final_cost = best_value;
        rep.evals = evals;
        rep.seed = schedule->seed;
        rep.trace_t = tt;
        rep.trace_f = tf;
        rep.wall_seconds = seconds_since(t0);
        rep.write(report);
    });
}

// calibrate_case2_formula, proj/src/calibration.cpp:483-534
SABR_API sabr_status sabr_calibrate_case2_formula(sabr_ctx* ctx, const sabr_surface* surface_in,
                                                  const sabr_bounds* bounds,
                                                  const sabr_schedule* schedule,
                                                  const sabr_fixed* fixed, sabr_report* report) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.calibrate_case2_formula");
        if (!schedule) fail(SABR_E_INVALID, "schedule is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        surface.validate();
        const auto t0 = std::chrono::steady_clock::now();
        const double horizon = surface.T.back();
        const ParamSpace ps(case2_defs(), bounds_from_abi(bounds), fixed_from_abi(fixed),
                            atm_vol_guess(surface, 0));
        const auto market = market_prices(surface);
        const C2fView v = make_c2f_view(ctx, surface, market, horizon);
        auto with_h = [&](std::vector<double> x) {
            x.push_back(horizon);
            return x;
        };
        Report rep{"case2", "T_I", "price"};
        std::vector<double> best_full;
        if (ps.free_ix.empty()) {  // run_or_evaluate: one objective call (dyn_coeffs_case2 validates)
            best_full = ps.full({});
            validate_case2(with_h(best_full).data());
            double c = c2f_costs(ctx, v, with_h(best_full))[0];
            rep.final_cost = c;
            rep.evals = 1;
        } else {
            validate_schedule(*schedule);
            const auto start = ps.full(ps.start_point());
            const bool start_ok = case2_feasible_host(with_h(start).data());
            double v0 = 0.0;
            if (start_ok) {
                v0 = c2f_costs(ctx, v, with_h(start))[0];
                if (std::isnan(v0)) v0 = INFINITY;  // safe_eval, annealer.cpp:84-87
            }
            std::vector<double> lo(10), hi(10);
            for (int i = 0; i < 10; ++i) {
                lo[i] = ps.defs[i].lo;
                hi[i] = ps.defs[i].hi;
            }
            const int64_t n_chains = static_cast<int64_t>(schedule->workers) * schedule->groups;
            const int64_t n_local =
                (ctx->rank + 1) * n_chains / ctx->nranks - ctx->rank * n_chains / ctx->nranks;
            cudaStream_t s = ctx->stream;
            const T1Out r = run_sa_generic(
                ctx, 10, ps.free_mask(), lo, hi, start, *schedule, start_ok, n_local,
                [&](const SaLevelArgs& a) {
                    cudaError_t e = cudaMemcpyAsync(&a.state->incumbent_value, &v0, sizeof(double),
                                                    cudaMemcpyHostToDevice, s);
                    if (e != cudaSuccess) return e;
                    e = cudaMemcpyAsync(&a.state->best_value, &v0, sizeof(double), cudaMemcpyHostToDevice, s);
                    if (e != cudaSuccess) return e;
                    return cudaStreamSynchronize(s);  // v0 lives on this stack frame
                },
                [&](const SaLevelArgs& a, int64_t level, double temp) {
                    return launch_c2f_level(v, a, level, temp, s);
                },
                0, SABR_PRED_NONE, /*use_peer=*/false, nullptr,
                /*skips_infeasible=*/true);  // case2_feasible inside the level kernel
            best_full = r.best_full;
            rep.final_cost = r.best_value;
            rep.evals = r.evals;
            rep.trace_t = r.trace_t;
            rep.trace_f = r.trace_f;
        }
        rep.params = ps.named(best_full);
        rep.seed = schedule->seed;
        rep.wall_seconds = seconds_since(t0);
        rep.write(report);
    });
}

SABR_API sabr_status sabr_evaluate_case1(sabr_ctx* ctx, const sabr_surface* surface_in,
                                         const double* p, sabr_report* report) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.evaluate_case1");
        if (!p) fail(SABR_E_INVALID, "params is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        evaluate_case1_impl(ctx, surface, p).write(report);
    });
}

SABR_API sabr_status sabr_evaluate_case2_prices(sabr_ctx* ctx, const sabr_surface* surface_in,
                                                const double* p, const sabr_plan* plan,
                                                sabr_report* report) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.evaluate_case2_prices");
        if (!p || !plan) fail(SABR_E_INVALID, "params/plan is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        evaluate_case2_impl(ctx, surface, p, *plan).write(report);
    });
}

SABR_API sabr_status sabr_cost_batch(sabr_ctx* ctx, int32_t model, const sabr_surface* surface_in,
                                     int64_t slice, const double* params, int64_t n,
                                     const sabr_plan* plan, double* cost) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.cost_batch");
        if (n < 0 || (n > 0 && (!params || !cost))) fail(SABR_E_INVALID, "params/cost is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        if (model == SABR_MODEL_STATIC) {
            if (slice < 0) surface.at(static_cast<size_t>(-1));
            surface.at(static_cast<size_t>(slice));
            for (int64_t i = 0; i < n; ++i) validate_static(params + 4 * i);
            const HostSurface one = surface.slice_only(static_cast<size_t>(slice));
            one.forward(0);
            const SurfaceView sv = make_view(ctx, "view_static", one, nullptr);
            const auto c = device_costs(ctx, OBJ_STATIC, sv, std::vector<double>(params, params + 4 * n), 4);
            std::copy(c.begin(), c.end(), cost);
        } else if (model == SABR_MODEL_CASE1) {
            if (slice != -1) fail(SABR_E_DOMAIN, "case1 objective is joint: slice must be -1");
            for (int64_t i = 0; i < n; ++i) validate_case1(params + 6 * i);
            const SurfaceView sv = make_view(ctx, "view_case1", surface, nullptr);
            const auto c = device_costs(ctx, OBJ_CASE1, sv, std::vector<double>(params, params + 6 * n), 6);
            std::copy(c.begin(), c.end(), cost);
        } else if (model == SABR_OBJECTIVE_CASE2_FORMULA) {
            if (slice != -1) fail(SABR_E_DOMAIN, "case2 objective is joint: slice must be -1");
            surface.validate();
            const auto market = market_prices(surface);
            for (int64_t i = 0; i < n; ++i) validate_case2(params + 11 * i);  // dyn_coeffs_case2 validates
            const C2fView v = make_c2f_view(ctx, surface, market, surface.T.back());
            const auto c = c2f_costs(ctx, v, std::vector<double>(params, params + 11 * n));
            std::copy(c.begin(), c.end(), cost);
        } else if (model == SABR_MODEL_CASE2) {
            if (!plan) fail(SABR_E_INVALID, "case2 objective needs a plan");
            if (slice != -1) fail(SABR_E_DOMAIN, "case2 objective is joint: slice must be -1");
            surface.validate();
            const auto market = market_prices(surface);
            for (int64_t i = 0; i < n; ++i) {
                const double* p = params + 11 * i;
                validate_case2(p);
                std::vector<double> value, se;
                mc_price_single(ctx, SABR_MODEL_CASE2, p, surface.spot, surface.T, surface.r, surface.y,
                                surface.off, surface.K, *plan, value, se);
                double sum = 0.0;
                for (size_t q = 0; q < value.size(); ++q) {
                    const double rel = (market[q] - value[q]) / market[q];
                    sum += rel * rel;
                }
                cost[i] = sum;
            }
        } else {
            fail(SABR_E_DOMAIN, "unknown model");
        }
    });
}

SABR_API sabr_status sabr_implied_vol_batch(sabr_ctx* ctx, int32_t model,
                                            const sabr_surface* surface_in, int64_t slice,
                                            const double* params, int64_t n, double* vols) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.implied_vol_batch");
        if (n < 0 || (n > 0 && (!params || !vols))) fail(SABR_E_INVALID, "params/vols is null");
        const HostSurface surface = HostSurface::from_abi(surface_in);
        if (model == SABR_MODEL_STATIC) {
            if (slice < 0) surface.at(static_cast<size_t>(-1));
            surface.at(static_cast<size_t>(slice));
            for (int64_t i = 0; i < n; ++i) validate_static(params + 4 * i);
            const HostSurface one = surface.slice_only(static_cast<size_t>(slice));
            const SurfaceView sv = make_view(ctx, "view_static", one, nullptr);
            const auto v = device_vols(ctx, OBJ_STATIC, sv, std::vector<double>(params, params + 4 * n), 4,
                                       static_cast<int64_t>(one.total_quotes()));
            std::copy(v.begin(), v.end(), vols);
        } else if (model == SABR_MODEL_CASE1) {
            for (int64_t i = 0; i < n; ++i) validate_case1(params + 6 * i);
            const SurfaceView sv = make_view(ctx, "view_case1", surface, nullptr);
            const auto v = device_vols(ctx, OBJ_CASE1, sv, std::vector<double>(params, params + 6 * n), 6,
                                       static_cast<int64_t>(surface.total_quotes()));
            std::copy(v.begin(), v.end(), vols);
        } else if (model == SABR_MODEL_CASE2) {
            // dynamic_implied_vol(dyn_coeffs_case2(p, T, 64), ...): the smile of
            // sabr_cli.cpp:234-243; p = n x 11 (horizon last), validated first
            for (int64_t i = 0; i < n; ++i) validate_case2(params + 11 * i);
            const C2fView v = make_c2f_view(ctx, surface, std::vector<double>(surface.total_quotes(), 1.0),
                                            n > 0 ? params[10] : 1.0, 64);
            auto* dp = upload(ctx, "c2v_params", std::vector<double>(params, params + 11 * n));
            const int64_t nq = static_cast<int64_t>(surface.total_quotes());
            auto* dv = static_cast<double*>(dev_buf(ctx, "c2v_vols", sizeof(double) * std::max<int64_t>(1, n * nq)));
            check_cuda(launch_c2f_vols(v, dp, n, dv, ctx->stream), "c2f_vols");
            check_cuda(cudaMemcpyAsync(vols, dv, sizeof(double) * n * nq, cudaMemcpyDeviceToHost, ctx->stream),
                       "D2H vols");
            sync(ctx);
        } else {
            fail(SABR_E_DOMAIN, "unknown model");
        }
    });
}

SABR_API sabr_status sabr_case2_feasible_batch(sabr_ctx* ctx, const double* params, int64_t n,
                                               uint8_t* feasible) {
    return guarded([&] {
        CtxLock l(ctx);
        if (n <= 0) return;
        if (!params || !feasible) fail(SABR_E_INVALID, "params/feasible is null");
        double* dp = upload(ctx, "feas_params", std::vector<double>(params, params + 11 * n));
        auto* df = static_cast<uint8_t*>(dev_buf(ctx, "feas_out", static_cast<size_t>(n)));
        check_cuda(launch_case2_feasible(dp, n, df, ctx->stream), "case2_feasible");
        check_cuda(cudaMemcpyAsync(feasible, df, static_cast<size_t>(n), cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H feasible");
        sync(ctx);
    });
}

// mc::simulate_terminals, proj/src/mc.cpp:231-240
SABR_API sabr_status sabr_mc_simulate_terminals(sabr_ctx* ctx, int32_t model, const double* params,
                                                double forward0, double alpha0, double maturity,
                                                const sabr_plan* plan, double* terminals) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.mc_simulate_terminals");
        if (!plan || !terminals) fail(SABR_E_INVALID, "plan/terminals is null");
        validate_model(model, params);
        validate_plan(*plan);
        const HostGrid g = build_grid(maturity, plan->dt);
        if (forward0 <= 0 || alpha0 < 0)
            fail(SABR_E_DOMAIN, "mc: forward0 must be positive and alpha0 nonnegative");
        const int ppt = choose_ppt(*plan);
        McJob job;
        job.slices.resize(1);
        const auto jump = mc_layout(ctx, *plan, ppt, {g}, job);
        std::vector<StepCoef> coef;
        for (size_t i = 0; i < g.dt.size(); ++i) {
            const double nu = model_nu_at(model, params, g.t_end[i]);
            const double rho = model_rho_at(model, params, g.t_end[i]);
            const double srho = std::sqrt(std::max(0.0, 1.0 - rho * rho));
            coef.push_back({nu * g.sdt[i], 0.5 * nu * nu * g.dt[i], rho * g.sdt[i], srho * g.sdt[i]});
        }
        McSlice& sl = job.slices[0];
        sl.q_begin = sl.q_end = 0;
        sl.forward0 = forward0;
        sl.lnf0 = std::log(forward0);
        sl.discount = 1.0;
        McParams P{};
        P.n_slices = 1;
        P.n_cand = 1;
        P.ppt = ppt;
        P.n_tiles = static_cast<int32_t>((plan->num_paths + static_cast<uint64_t>(kMcThreads) * ppt - 1) /
                                         (static_cast<uint64_t>(kMcThreads) * ppt));
        P.rng = plan->rng;
        P.total_steps = job.total_steps;
        P.num_paths = plan->num_paths;
        P.block_size = plan->block_size;
        P.seed = plan->seed;
        P.slices = upload(ctx, "mc_slices", job.slices);
        P.alpha0 = upload(ctx, "mc_alpha0", std::vector<double>{alpha0});
        P.beta = upload(ctx, "mc_beta", std::vector<double>{params[1]});
        set_coefficients(ctx, P, coef, plan->precision);
        P.cand_stride = 1;
        P.hdt = upload(ctx, "mc_hdt", job.hdt);
        P.strikes = upload(ctx, "mc_strikes", std::vector<double>{0.0});
        P.jump = upload(ctx, "mc_jump", jump);
        P.exptab = exp_table_device(ctx);
    P.logtab = log_table_device(ctx);
    P.sctab = sincos_table_device(ctx);
        P.partials = nullptr;
        P.terminals = static_cast<double*>(dev_buf(ctx, "mc_terminals", sizeof(double) * plan->num_paths));
        P.bad = static_cast<int*>(dev_buf(ctx, "mc_bad", sizeof(int)));
        check_cuda(cudaMemsetAsync(P.bad, 0, sizeof(int), ctx->stream), "memset bad");
        Timer timer(ctx);
        timer.start();
        check_cuda(launch_mc_tiles(P, 1, ctx->stream), "mc_tiles");
        int bad = 0;
        check_cuda(cudaMemcpyAsync(&bad, P.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        check_cuda(cudaMemcpyAsync(terminals, P.terminals, sizeof(double) * plan->num_paths,
                                   cudaMemcpyDeviceToHost, ctx->stream), "D2H terminals");
        sync(ctx);
        timer.stop(static_cast<double>(plan->num_paths) * job.total_steps,
                   static_cast<double>(plan->num_paths) * job.total_steps, 1, 1);
        if (bad) fail(SABR_E_RUNTIME, "mc: non-finite path value (scheme unstable for these inputs)");
    });
}

// mc::price_european_batch, proj/src/mc.cpp:249-273
SABR_API sabr_status sabr_mc_price_european_batch(sabr_ctx* ctx, int32_t model, const double* params,
                                                  double spot, const double* strikes, int64_t m,
                                                  double rate, double dividend, double maturity,
                                                  const sabr_plan* plan, double* value,
                                                  double* std_error) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.mc_price_european_batch");
        if (!plan || m < 0 || (m > 0 && (!strikes || !value || !std_error)))
            fail(SABR_E_INVALID, "null argument");
        validate_model(model, params);
        if (spot <= 0) fail(SABR_E_DOMAIN, "price_european_batch: spot must be positive");
        for (int64_t j = 0; j < m; ++j)
            if (strikes[j] <= 0) fail(SABR_E_DOMAIN, "price_european_batch: strikes must be positive");
        std::vector<double> v, s;
        mc_price_single(ctx, model, params, spot, {maturity}, {rate}, {dividend}, {0, m},
                        std::vector<double>(strikes, strikes + m), *plan, v, s);
        std::copy(v.begin(), v.end(), value);
        std::copy(s.begin(), s.end(), std_error);
    });
}

// mc::price_cliquet, proj/src/mc.cpp:275-320
SABR_API sabr_status sabr_mc_price_cliquet(sabr_ctx* ctx, int32_t model, const double* params,
                                           double spot, double rate, double dividend,
                                           double local_floor, double local_cap, double global_floor,
                                           double global_cap, const double* reset_dates,
                                           int64_t n_resets, const sabr_plan* plan, double* value,
                                           double* std_error) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.mc_price_cliquet");
        if (!plan || !value || !std_error || (n_resets > 0 && !reset_dates))
            fail(SABR_E_INVALID, "null argument");
        validate_model(model, params);
        // CliquetSpec::validate, mc.cpp:168-181
        if (local_floor > local_cap) fail(SABR_E_DOMAIN, "CliquetSpec: local floor above local cap");
        if (global_floor > global_cap) fail(SABR_E_DOMAIN, "CliquetSpec: global floor above global cap");
        if (n_resets < 2) fail(SABR_E_DOMAIN, "CliquetSpec: need at least two reset dates");
        for (int64_t i = 0; i < n_resets; ++i) {
            if (reset_dates[i] <= 0) fail(SABR_E_DOMAIN, "CliquetSpec: reset dates must be positive");
            if (i > 0 && reset_dates[i] <= reset_dates[i - 1])
                fail(SABR_E_DOMAIN, "CliquetSpec: reset dates must be strictly increasing");
        }
        validate_plan(*plan);
        if (spot <= 0) fail(SABR_E_DOMAIN, "price_cliquet: spot must be positive");
        if (n_resets > kMaxCliquetObs) fail(SABR_E_DOMAIN, "price_cliquet: at most 128 reset dates");
        const double maturity = reset_dates[n_resets - 1];
        const double forward0 = spot * std::exp((rate - dividend) * maturity);
        const HostGrid g = build_grid(maturity, plan->dt);
        // snap each reset date to the nearest grid node (mc.cpp:285-300)
        std::vector<double> node_time{0.0};
        node_time.insert(node_time.end(), g.t_end.begin(), g.t_end.end());
        CliquetSpecDev spec{};
        spec.n_obs = static_cast<int32_t>(n_resets);
        spec.local_floor = local_floor;
        spec.local_cap = local_cap;
        spec.global_floor = global_floor;
        spec.global_cap = global_cap;
        for (int64_t k = 0; k < n_resets; ++k) {
            const double d = reset_dates[k];
            size_t best = 0;
            for (size_t j = 1; j < node_time.size(); ++j)
                if (std::abs(node_time[j] - d) < std::abs(node_time[best] - d)) best = j;
            if (std::abs(node_time[best] - d) > 0.5 * plan->dt + 1e-12)
                fail(SABR_E_DOMAIN, "price_cliquet: reset date not within dt/2 of a grid node");
            if (k > 0 && static_cast<int32_t>(best) <= spec.obs_node[k - 1])
                fail(SABR_E_DOMAIN, "price_cliquet: reset dates collapse onto one grid node");
            spec.obs_node[k] = static_cast<int32_t>(best);
            spec.obs_discount[k] = std::exp(-(rate - dividend) * (maturity - node_time[best]));
        }
        const double alpha0 = params[0];
        if (forward0 <= 0 || alpha0 < 0)
            fail(SABR_E_DOMAIN, "mc: forward0 must be positive and alpha0 nonnegative");
        const int ppt = choose_ppt(*plan);
        McJob job;
        job.slices.resize(1);
        const auto jump = mc_layout(ctx, *plan, ppt, {g}, job);
        std::vector<StepCoef> coef;
        for (size_t i = 0; i < g.dt.size(); ++i) {
            const double nu = model_nu_at(model, params, g.t_end[i]);
            const double rho = model_rho_at(model, params, g.t_end[i]);
            const double srho = std::sqrt(std::max(0.0, 1.0 - rho * rho));
            coef.push_back({nu * g.sdt[i], 0.5 * nu * nu * g.dt[i], rho * g.sdt[i], srho * g.sdt[i]});
        }
        McSlice& sl = job.slices[0];
        sl.q_begin = 0;
        sl.q_end = 1;
        sl.forward0 = forward0;
        sl.lnf0 = std::log(forward0);
        sl.discount = std::exp(-rate * maturity);
        McParams P{};
        P.n_slices = 1;
        P.n_cand = 1;
        P.n_quotes = 1;
        P.max_q = 1;
        P.ppt = ppt;
        P.n_tiles = static_cast<int32_t>((plan->num_paths + static_cast<uint64_t>(kMcThreads) * ppt - 1) /
                                         (static_cast<uint64_t>(kMcThreads) * ppt));
        P.rng = plan->rng;
        P.total_steps = job.total_steps;
        P.num_paths = plan->num_paths;
        P.block_size = plan->block_size;
        P.seed = plan->seed;
        P.slices = upload(ctx, "mc_slices", job.slices);
        P.alpha0 = upload(ctx, "mc_alpha0", std::vector<double>{alpha0});
        P.beta = upload(ctx, "mc_beta", std::vector<double>{params[1]});
        set_coefficients(ctx, P, coef, SABR_FP64);
        P.cand_stride = 1;
        P.hdt = upload(ctx, "mc_hdt", job.hdt);
        P.strikes = upload(ctx, "mc_strikes", std::vector<double>{0.0});
        P.jump = upload(ctx, "mc_jump", jump);
        P.exptab = exp_table_device(ctx);
    P.logtab = log_table_device(ctx);
    P.sctab = sincos_table_device(ctx);
        P.partials = static_cast<double*>(dev_buf(ctx, "mc_partials", sizeof(double) * 2 * P.n_tiles));
        P.bad = static_cast<int*>(dev_buf(ctx, "mc_bad", sizeof(int)));
        check_cuda(cudaMemsetAsync(P.bad, 0, sizeof(int), ctx->stream), "memset bad");
        double* dv = static_cast<double*>(dev_buf(ctx, "mc_value", sizeof(double)));
        double* ds = static_cast<double*>(dev_buf(ctx, "mc_se", sizeof(double)));
        Timer timer(ctx);
        timer.start();
        timer.before();
        check_cuda(launch_mc_cliquet(P, spec, ctx->stream), "mc_cliquet");
        timer.after();
        check_cuda(launch_mc_reduce(P, dv, ds, nullptr, nullptr, ctx->stream), "mc_reduce");
        int bad = 0;
        check_cuda(cudaMemcpyAsync(value, dv, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        check_cuda(cudaMemcpyAsync(std_error, ds, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        check_cuda(cudaMemcpyAsync(&bad, P.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        sync(ctx);
        timer.stop(static_cast<double>(plan->num_paths) * job.total_steps,
                   static_cast<double>(plan->num_paths) * job.total_steps, 1, 2);
        if (bad) fail(SABR_E_RUNTIME, "mc: non-finite path value (scheme unstable for these inputs)");
    });
}

// minimize (annealer.cpp:76-167) on the closed-form objectives of test_annealer.cpp
SABR_API sabr_status sabr_minimize_builtin(sabr_ctx* ctx, int32_t objective, int32_t predicate,
                                           const double* lower, const double* upper, int64_t dim,
                                           const sabr_schedule* schedule, const double* start,
                                           sabr_anneal_result* result) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.minimize_builtin");
        if (!schedule || !result || !result->best_point) fail(SABR_E_INVALID, "null argument");
        validate_schedule(*schedule);
        if (dim < 1 || dim > 4) fail(SABR_E_DOMAIN, "SearchSpace: bounds must be nonempty and equal-sized");
        std::vector<double> lo(lower, lower + dim), hi(upper, upper + dim), st(start, start + dim);
        SurfaceView sv{};
        sv.exptab = exp_table_device(ctx);
        const T1Out r = run_sa_t1(ctx, OBJ_BUILTIN, sv, static_cast<int>(dim), (1u << dim) - 1u, lo, hi, st,
                                  *schedule, objective, predicate);
        for (int64_t i = 0; i < dim; ++i) result->best_point[i] = r.best_full[i];
        result->best_value = r.best_value;
        result->evals = r.evals;
        result->trace_len = static_cast<int64_t>(r.trace_f.size());
        if (result->trace_t && result->trace_f) {
            const size_t n = std::min(r.trace_f.size(), static_cast<size_t>(std::max<int64_t>(0, result->trace_capacity)));
            for (size_t i = 0; i < n; ++i) {
                result->trace_t[i] = r.trace_t[i];
                result->trace_f[i] = r.trace_f[i];
            }
        }
    });
}

SABR_API sabr_status sabr_merge_level_records(sabr_sa_state* state, const sabr_level_record* records,
                                              int64_t nranks, int64_t n_chains, int64_t max_evals,
                                              int64_t levels_total, double* trace_f) {
    return guarded([&] {
        if (!state || !records || nranks < 1) fail(SABR_E_INVALID, "null argument");
        sabr_dev::merge_level(state, records, nranks, n_chains, max_evals, levels_total, SABR_MAX_DIM,
                              trace_f);
    });
}

SABR_API sabr_status sabr_surface_csv_dims(const char* path, int64_t* n_slices, int64_t* n_quotes) {
    return guarded([&] {
        if (!path || !n_slices || !n_quotes) fail(SABR_E_INVALID, "null argument");
        const HostSurface s = parse_surface(path);
        *n_slices = static_cast<int64_t>(s.n());
        *n_quotes = static_cast<int64_t>(s.total_quotes());
    });
}

SABR_API sabr_status sabr_surface_csv_read(const char* path, double* spot, double* maturity,
                                           double* rate, double* dividend, int64_t* quote_offset,
                                           double* strike, double* vol) {
    return guarded([&] {
        if (!path || !spot || !maturity || !rate || !dividend || !quote_offset || !strike || !vol)
            fail(SABR_E_INVALID, "null argument");
        const HostSurface s = parse_surface(path);
        *spot = s.spot;
        std::copy(s.T.begin(), s.T.end(), maturity);
        std::copy(s.r.begin(), s.r.end(), rate);
        std::copy(s.y.begin(), s.y.end(), dividend);
        std::copy(s.off.begin(), s.off.end(), quote_offset);
        std::copy(s.K.begin(), s.K.end(), strike);
        std::copy(s.vol.begin(), s.vol.end(), vol);
    });
}

SABR_API sabr_status sabr_black_scholes_call(double spot, double strike, double rate, double dividend,
                                             double maturity, double vol, double* price) {
    return guarded([&] {
        if (!price) fail(SABR_E_INVALID, "price is null");
        *price = black_scholes_call(spot, strike, rate, dividend, maturity, vol);
    });
}

}

namespace {
// Upload the SoA inputs, run one batched Black-Scholes kernel, map the first
// rejected element (index order) to the reference's domain_error message.
template <class Launch>
void bs_batch(sabr_ctx* ctx, int64_t n, std::initializer_list<const double*> in, double* out, Launch&& launch) {
    std::vector<const double*> dev;
    int k = 0;
    for (const double* p : in) {
        if (!p) fail(SABR_E_INVALID, "input array is null");
        dev.push_back(upload(ctx, "bs_in" + std::to_string(k++), std::vector<double>(p, p + n)));
    }
    if (!out) fail(SABR_E_INVALID, "output array is null");
    auto* dout = static_cast<double*>(dev_buf(ctx, "bs_out", sizeof(double) * n));
    auto* dst = static_cast<int32_t*>(dev_buf(ctx, "bs_status", sizeof(int32_t) * n));
    check_cuda(launch(dev, dout, dst), "black_scholes batch");
    std::vector<int32_t> st(n);
    check_cuda(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    check_cuda(cudaMemcpyAsync(st.data(), dst, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync(ctx);
    for (int64_t i = 0; i < n; ++i) {
        if (st[i] == BS_E_INPUTS) fail(SABR_E_DOMAIN, "black_scholes_call: spot, strike, maturity must be positive");
        if (st[i] == BS_E_VOL) fail(SABR_E_DOMAIN, "black_scholes_call: vol must be nonnegative");
        if (st[i] == BS_E_BOUNDS) fail(SABR_E_DOMAIN, "implied_vol_from_price: price outside no-arbitrage bounds");
    }
}
}  // namespace

extern "C" {

SABR_API sabr_status sabr_black_scholes_call_batch(sabr_ctx* ctx, int64_t n, const double* spot,
                                                   const double* strike, const double* rate,
                                                   const double* dividend, const double* maturity,
                                                   const double* vol, double* price) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.black_scholes_call_batch");
        if (n <= 0) return;
        bs_batch(ctx, n, {spot, strike, rate, dividend, maturity, vol}, price,
                 [&](const std::vector<const double*>& d, double* o, int32_t* st) {
                     return launch_bs_call(n, d[0], d[1], d[2], d[3], d[4], d[5], o, st, ctx->stream);
                 });
    });
}

SABR_API sabr_status sabr_implied_vol_from_price_batch(sabr_ctx* ctx, int64_t n, const double* price,
                                                       const double* spot, const double* strike,
                                                       const double* rate, const double* dividend,
                                                       const double* maturity, double* vol) {
    return guarded([&] {
        CtxLock l(ctx);
        NvtxRange nvtx("sabr.implied_vol_from_price_batch");
        if (n <= 0) return;
        bs_batch(ctx, n, {price, spot, strike, rate, dividend, maturity}, vol,
                 [&](const std::vector<const double*>& d, double* o, int32_t* st) {
                     return launch_implied_vol(n, d[0], d[1], d[2], d[3], d[4], d[5], o, st, ctx->stream);
                 });
    });
}

}  // extern "C"
