// t2_driver.cu — the annealer of calibrate_case2_T2 (proj/src/calibration.cpp:450-481)
// with its Monte Carlo objective (case2_mc_cost, :399-416) on the device.
//
// The reference runs the chains of a level in an OpenMP loop and, inside each
// chain step, prices every slice with a fresh MC run (nested, serialized).
// Here the chains step in lockstep: one step of ALL chains is
//   propose+feasibility (1 thread/chain) -> grid coefficients (1 thread per
//   candidate-step) -> one batched MC launch over (candidate group x slice x
//   path tile), sharing the normals of a path-step across the candidates of a
//   group -> fixed-order tile reduction and cost -> Metropolis (1 thread/chain),
// and the level ends with the same in-kernel arg-min merge as the T_I driver.
// Nothing returns to the host inside a level.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "engine.hpp"

namespace sabr_gpu {

AnnealOut run_sa_case2(sabr_ctx* ctx, const HostSurface& surface, const std::vector<double>& market,
                       const ParamSpace& ps, const std::vector<double>& start_full, double horizon,
                       const sabr_schedule& sch, const sabr_plan& plan) {
    const std::vector<double> temps = temperatures(sch);
    const int64_t L = static_cast<int64_t>(temps.size());
    const int64_t n_chains = static_cast<int64_t>(sch.workers) * sch.groups;
    // Multi-rank decomposition.  Chains are split over the ranks
    // (one record all-gather per level) unless there are fewer chains than
    // ranks: then every rank runs every chain on its own slab of path tiles,
    // and the tile partials of every MC step are all-gathered and reduced in
    // the single-rank tile order, so costs, decisions and reports are the
    // same on every rank and for any rank count.  SABR_T2_SHARD=paths forces
    // the path split (tests).
    const bool path_mode = ctx->nranks > 1 && (n_chains < ctx->nranks || [] {
        const char* e = std::getenv("SABR_T2_SHARD");
        return e != nullptr && std::string(e) == "paths";
    }());
    const int64_t begin = path_mode ? 0 : ctx->rank * n_chains / ctx->nranks;
    const int64_t end = path_mode ? n_chains : (ctx->rank + 1) * n_chains / ctx->nranks;
    const int32_t n_local = static_cast<int32_t>(end - begin);
    const size_t ns = surface.n();
    const int nq = static_cast<int>(surface.total_quotes());

    // ---- start value: safe_eval(start), annealer.cpp:90 ----
    std::vector<double> p0 = start_full;
    p0.push_back(horizon);
    double start_value;
    {
        std::vector<double> value, se;
        mc_price_single(ctx, SABR_MODEL_CASE2, p0.data(), surface.spot, surface.T, surface.r, surface.y,
                        surface.off, surface.K, plan, value, se);
        double sum = 0.0;
        for (int q = 0; q < nq; ++q) {
            const double rel = (market[q] - value[q]) / market[q];
            sum += rel * rel;
        }
        start_value = std::isnan(sum) ? INFINITY : sum;
    }

    // ---- MC layout shared by every step ----
    std::vector<HostGrid> grids;
    for (size_t s = 0; s < ns; ++s) grids.push_back(build_grid(surface.T[s], plan.dt));
    const int ppt = choose_ppt(plan);
    McJob job;
    job.slices.resize(ns);
    const auto jump = mc_layout(ctx, plan, ppt, grids, job);
    // time-invariant dynamics for every chain: q_rho, q_nu, a, b (CaseIIParams
    // indices 3, 6, 8, 9) fixed at 0, so rho(t) = rho0 + d_rho, nu(t) = nu0 + d_nu
    // (analytics.cpp:138-143) and a uniform grid gives identical step rows
    bool invariant = true;
    for (int i : {3, 6, 8, 9}) invariant = invariant && !ps.is_free[i] && start_full[i] == 0.0;
    std::vector<double> t_end, dt, sdt;
    for (size_t s = 0; s < ns; ++s) {
        McSlice& sl = job.slices[s];
        sl.const_coef = invariant && uniform_grid(grids[s]);
        sl.q_begin = static_cast<int32_t>(surface.off[s]);
        sl.q_end = static_cast<int32_t>(surface.off[s + 1]);
        job.max_q = std::max(job.max_q, sl.q_end - sl.q_begin);
        sl.forward0 = surface.spot * std::exp((surface.r[s] - surface.y[s]) * surface.T[s]);  // mc.cpp:258
        sl.lnf0 = std::log(sl.forward0);
        sl.discount = std::exp(-surface.r[s] * surface.T[s]);
        t_end.insert(t_end.end(), grids[s].t_end.begin(), grids[s].t_end.end());
        dt.insert(dt.end(), grids[s].dt.begin(), grids[s].dt.end());
        sdt.insert(sdt.end(), grids[s].sdt.begin(), grids[s].sdt.end());
    }
    const int64_t S = job.total_steps;
    const int32_t n_tiles = static_cast<int32_t>(
        (plan.num_paths + static_cast<uint64_t>(kMcThreads) * ppt - 1) / (static_cast<uint64_t>(kMcThreads) * ppt));
    // path mode: rank r simulates tiles [r*tpr, min((r+1)*tpr, n_tiles)); the
    // partial buffer holds nranks*tpr tiles (rank slabs in rank order)
    const int32_t tpr = path_mode ? (n_tiles + ctx->nranks - 1) / ctx->nranks : n_tiles;
    const int32_t tile_begin = path_mode ? ctx->rank * tpr : 0;
    const int32_t tile_count = path_mode ? std::max(0, std::min(tpr, n_tiles - tile_begin)) : n_tiles;
    const int64_t tiles_alloc = path_mode ? static_cast<int64_t>(tpr) * ctx->nranks : n_tiles;
    // candidates per MC launch: bound the coefficient and partial buffers
    const int64_t per_cand = S * 32 + static_cast<int64_t>(nq) * tiles_alloc * 16;
    const int32_t chunk = static_cast<int32_t>(
        std::max<int64_t>(1, std::min<int64_t>(std::max(n_local, 1), (int64_t(1) << 31) / std::max<int64_t>(per_cand, 1))));
    const bool fp32 = plan.precision == SABR_FP32;
    // candidates per thread: 8 (register bound in FP64; in FP32 the
    // coefficient prefetch buffer takes the room a 16-wide group would need)
    int cb = chunk >= 8 ? 8 : (chunk >= 4 ? 4 : (chunk >= 2 ? 2 : 1));
    // FP32: 16 candidates per thread, the shared RNG and Box-Muller amortised
    // over twice the candidates, the coefficient rows read from shared memory
    // (kernels_mc.cu SMQ / WQ) (r02: C4 FP32 1.24e12 -> 1.54e12, C5 FP32
    // 1.33e12 -> 1.63e12 path-steps/s; FP64 spills at 16, 2x slower,
    // tools/ab_mc.py with SABR_MC_CB)
    if (fp32 && chunk >= 16) cb = 16;
    if (const char* e = std::getenv("SABR_MC_CB")) {  // tuning override (1, 2, 4, 8, 16)
        const int v = std::atoi(e);
        if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) cb = v;
    }
    // the payoff accumulators of a tile CTA grow with CB x quotes per slice
    const int cb_fit = mc_max_cand_block(job.max_q, fp32);
    if (cb_fit == 0) fail(SABR_E_RUNTIME, "case2_mc_cost: too many quotes in one slice for the MC tile kernel");
    while (cb > cb_fit) cb /= 2;
    const int32_t stride = (chunk + cb - 1) / cb * cb;  // coefficient row width

    McParams P{};
    P.n_slices = static_cast<int32_t>(ns);
    P.n_quotes = nq;
    P.max_q = job.max_q;
    P.n_tiles = n_tiles;
    P.ppt = ppt;
    P.rng = plan.rng;
    P.total_steps = S;
    P.num_paths = plan.num_paths;
    P.block_size = plan.block_size;
    P.seed = plan.seed;
    P.slices = upload(ctx, "t2_slices", job.slices);
    P.host_slices = job.slices.data();
    P.hdt = upload(ctx, "t2_hdt", job.hdt);
    P.strikes = upload(ctx, "t2_strikes", surface.K);
    P.jump = upload(ctx, "t2_jump", jump);
    {  // MC blocks of the longest slices first (C5: 62..1250 steps per slice)
        std::vector<int32_t> order(ns);
        for (size_t i = 0; i < ns; ++i) order[i] = static_cast<int32_t>(i);
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t x, int32_t y) { return job.slices[x].n_steps > job.slices[y].n_steps; });
        P.slice_order = upload(ctx, "t2_slice_order", order);
    }
    P.exptab = exp_table_device(ctx);
    P.logtab = log_table_device(ctx);
    P.sctab = sincos_table_device(ctx);
    const double* d_market = upload(ctx, "t2_market", market);
    const double* d_tend = upload(ctx, "t2_tend", t_end);
    const double* d_dt = upload(ctx, "t2_dt", dt);
    const double* d_sdt = upload(ctx, "t2_sdt", sdt);
    const size_t nl = static_cast<size_t>(std::max(n_local, 1));
    auto* chains = static_cast<T2Chain*>(dev_buf(ctx, "t2_chains", sizeof(T2Chain) * nl));
    auto* alpha0 = static_cast<double*>(dev_buf(ctx, "t2_alpha0", sizeof(double) * nl));
    auto* beta = static_cast<double*>(dev_buf(ctx, "t2_beta", sizeof(double) * nl));
    auto* active = static_cast<uint8_t*>(dev_buf(ctx, "t2_active", nl));
    auto* cost = static_cast<double*>(dev_buf(ctx, "t2_cost", sizeof(double) * nl));
    auto* bad = static_cast<int*>(dev_buf(ctx, "t2_bad", sizeof(int) * nl));
    // the step's feasible candidates, compacted (t2_compact_kernel)
    auto* cidx = static_cast<int32_t*>(dev_buf(ctx, "t2_cidx", sizeof(int32_t) * nl));
    auto* n_live = static_cast<int32_t*>(dev_buf(ctx, "t2_n_live", sizeof(int32_t)));
    auto* alpha0_c = static_cast<double*>(dev_buf(ctx, "t2_alpha0_c", sizeof(double) * nl));
    auto* beta_c = static_cast<double*>(dev_buf(ctx, "t2_beta_c", sizeof(double) * nl));
    auto* active_c = static_cast<uint8_t*>(dev_buf(ctx, "t2_active_c", nl));
    auto* cost_c = static_cast<double*>(dev_buf(ctx, "t2_cost_c", sizeof(double) * nl));
    auto* bad_c = static_cast<int*>(dev_buf(ctx, "t2_bad_c", sizeof(int) * nl));
    auto* nonfinite = static_cast<int*>(dev_buf(ctx, "t2_nonfinite", sizeof(int)));
    void* coef = dev_buf(ctx, "t2_coef", (fp32 ? sizeof(float4) : sizeof(StepCoef)) * S * stride);
    auto* partials = static_cast<double*>(
        dev_buf(ctx, "t2_partials", sizeof(double) * 2 * static_cast<size_t>(nq) * tiles_alloc * chunk));
    auto* values = static_cast<double*>(dev_buf(ctx, "t2_values", sizeof(double) * static_cast<size_t>(nq) * chunk));
    check_cuda(cudaMemsetAsync(nonfinite, 0, sizeof(int), ctx->stream), "memset");
    check_cuda(cudaMemsetAsync(bad, 0, sizeof(int) * nl, ctx->stream), "memset");

    // ---- annealer state (device resident) ----
    sabr_sa_state st{};
    for (size_t i = 0; i < start_full.size(); ++i) st.incumbent[i] = st.best[i] = start_full[i];
    st.incumbent_value = st.best_value = start_value;
    st.evals = 1;
    st.done = (L == 0 || st.evals >= sch.max_evals) ? 1 : 0;
    st.eval_cap = st.done ? 0 : (sch.max_evals - st.evals + n_chains - 1) / n_chains;

    SaLevelArgs a{};
    a.dim_full = 10;
    a.nranks = path_mode ? 1 : ctx->nranks;  // path mode: every rank holds every chain
    a.chain_begin = begin;
    a.n_local = n_local;
    a.n_chains = n_chains;
    a.max_evals = sch.max_evals;
    a.levels_total = L;
    const int64_t grid = std::max<int64_t>(1, (n_local + t2_block_threads() - 1) / t2_block_threads());
    a.state = static_cast<sabr_sa_state*>(dev_buf(ctx, "sa_state", sizeof(sabr_sa_state)));
    a.block_recs = static_cast<sabr_level_record*>(dev_buf(ctx, "sa_block_recs", sizeof(sabr_level_record) * grid));
    a.block_sum = static_cast<BlockSummary*>(dev_buf(ctx, "sa_block_sum", sizeof(BlockSummary) * grid));
    a.rank_rec = static_cast<sabr_level_record*>(dev_buf(ctx, "sa_rank_rec", sizeof(sabr_level_record)));
    auto* recv = static_cast<sabr_level_record*>(dev_buf(ctx, "sa_recv_recs", sizeof(sabr_level_record) * ctx->nranks));
    a.ticket = static_cast<unsigned int*>(dev_buf(ctx, "sa_ticket", sizeof(unsigned int)));
    a.trace_f = static_cast<double*>(dev_buf(ctx, "sa_trace", sizeof(double) * std::max<int64_t>(1, L)));
    check_cuda(cudaMemcpyAsync(a.state, &st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream), "H2D state");
    check_cuda(cudaMemsetAsync(a.ticket, 0, sizeof(unsigned int), ctx->stream), "memset ticket");

    T2StepArgs ta{};
    for (int i = 0; i < 10; ++i) {
        ta.lo[i] = ps.defs[i].lo;
        ta.hi[i] = ps.defs[i].hi;
        ta.range[i] = ps.defs[i].hi - ps.defs[i].lo;
    }
    ta.free_mask = ps.free_mask();
    ta.n_local = n_local;
    ta.t0 = sch.t0;
    ta.horizon = horizon;
    ta.seed = sch.seed;
    ta.chain_begin = begin;

    const bool one_chunk = n_local <= chunk;
    const int coef_layout = fp32 ? (cb >= 2 ? 2 : 1) : 0;
    Timer timer(ctx);
    timer.start();
    int64_t mc_launches = 0, launches = 0;
    auto* pinned = static_cast<int64_t*>(ctx->pinned);
    for (int64_t level = 0; level < L; ++level) {
        ta.level = level;
        ta.temp = temps[level];
        check_cuda(launch_t2_level_init(chains, a.state, ta, ctx->stream), "t2_level_init");
        for (int step = 0; step < sch.chain_length; ++step) {
            NvtxRange nvtx_step("sabr.t2_step");
            // the step's kernels form one PDL chain (pdl.cuh): each may be
            // scheduled while its predecessor runs, and waits for it in-kernel
            check_cuda(launch_t2_propose(chains, a.state, ta, alpha0, beta, active, ctx->stream), "t2_propose");
            // the MC launches run over the compacted feasible candidates: a
            // chunk past the live count exits in every kernel
            check_cuda(launch_t2_compact(active, alpha0, beta, n_local, cidx, alpha0_c, beta_c, active_c, n_live,
                                         bad_c, ctx->stream), "t2_compact");
            launches += 2;
            for (int32_t c0 = 0; c0 < n_local; c0 += chunk) {
                const int32_t nc = std::min(chunk, n_local - c0);
                const int32_t nc_pad = (nc + cb - 1) / cb * cb;
                check_cuda(launch_t2_coef(chains, cidx, n_live, c0, nc, nc_pad, d_tend, d_dt, d_sdt, S, coef,
                                          coef_layout, ctx->stream), "t2_coef");
                McParams Q = P;
                Q.n_cand = nc;
                Q.alpha0 = alpha0_c + c0;
                Q.beta = beta_c + c0;
                Q.active = active_c + c0;
                Q.fp32 = fp32 ? 1 : 0;
                Q.coef = fp32 ? nullptr : static_cast<const StepCoef*>(coef);
                Q.coef32 = fp32 ? static_cast<const float4*>(coef) : nullptr;
                Q.cand_stride = nc_pad;
                Q.partials = partials;
                Q.terminals = nullptr;
                Q.bad = bad_c + c0;
                Q.tile_begin = tile_begin;
                Q.tile_count = tile_count;
                timer.before();
                if (tile_count > 0) check_cuda(launch_mc_tiles(Q, cb, ctx->stream), "mc_tiles");
                timer.after();
                if (path_mode) {  // in-place all-gather of the rank slabs [tpr tiles][nc][nq][2]
                    const size_t slab = sizeof(double) * 2 * static_cast<size_t>(tpr) * nc * nq;
                    allgather(ctx, reinterpret_cast<unsigned char*>(partials) + ctx->rank * slab, partials, slab);
                }
                // one chunk (the step's candidates in one MC launch): the cost, the
                // scatter and the Metropolis test are one kernel (t2_finish)
                check_cuda(launch_mc_reduce(Q, values, nullptr, d_market, one_chunk ? nullptr : cost_c + c0,
                                            ctx->stream), "mc_reduce");
                mc_launches += 1;
                launches += one_chunk ? 3 : 4;
            }
            if (one_chunk) {
                check_cuda(launch_t2_finish(chains, ta, cidx, n_live, values, nq, d_market, bad_c, nonfinite,
                                            ctx->stream), "t2_finish");
                launches += 1;
            } else {
                check_cuda(launch_t2_scatter(cidx, n_live, n_local, cost_c, bad_c, cost, bad, ctx->stream),
                           "t2_scatter");
                check_cuda(launch_t2_accept(chains, ta, cost, bad, nonfinite, ctx->stream), "t2_accept");
                launches += 2;
            }
        }
        check_cuda(launch_t2_level_end(chains, a, level, ctx->stream), "t2_level_end");
        if (a.nranks > 1) {
            allgather(ctx, a.rank_rec, recv, sizeof(sabr_level_record));
            check_cuda(launch_sa_merge(a, recv, level, ctx->stream), "sa_merge");
        }
        check_cuda(cudaMemcpyAsync(pinned, &a.state->done, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                   ctx->stream), "D2H done");
        check_cuda(cudaStreamSynchronize(ctx->stream), "sync");
        if (*pinned) break;
    }
    sabr_sa_state out{};
    int nf = 0;
    check_cuda(cudaMemcpyAsync(&out, a.state, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream), "D2H state");
    if (path_mode) {  // a non-finite path may sit in any rank's tiles: OR the flags
        auto* flags = static_cast<int*>(dev_buf(ctx, "t2_nonfinite_all", sizeof(int) * ctx->nranks));
        allgather(ctx, nonfinite, flags, sizeof(int));
        std::vector<int> h(ctx->nranks);
        check_cuda(cudaMemcpyAsync(h.data(), flags, sizeof(int) * ctx->nranks, cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H");
        check_cuda(cudaStreamSynchronize(ctx->stream), "sync");
        for (int v : h) nf |= v;
    }
    int nf_local = 0;
    check_cuda(cudaMemcpyAsync(&nf_local, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    check_cuda(cudaStreamSynchronize(ctx->stream), "sync");
    nf |= nf_local;
    const double evals_run = static_cast<double>(out.evals - 1);
    timer.stop(evals_run, evals_run * static_cast<double>(plan.num_paths) * static_cast<double>(S),
               mc_launches, launches);
    if (nf) fail(SABR_E_RUNTIME, "mc: non-finite path value (scheme unstable for these inputs)");

    AnnealOut r;
    r.best_full.assign(out.best, out.best + 10);
    r.best_value = out.best_value;
    r.evals = out.evals;
    r.trace_f.resize(out.levels_run);
    if (out.levels_run > 0)
        check_cuda(cudaMemcpy(r.trace_f.data(), a.trace_f, sizeof(double) * out.levels_run,
                              cudaMemcpyDeviceToHost), "D2H trace");
    r.trace_t.assign(temps.begin(), temps.begin() + out.levels_run);
    return r;
}

}  // namespace sabr_gpu
