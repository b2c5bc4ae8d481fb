// engine.hpp — the context and the host drivers (internal).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "host_common.hpp"
#include "kernels.hpp"
#include "kernels_mc.hpp"

struct sabr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool profiling = false;
    sabr_timing timing{};
    std::mutex mu;
    // NCCL (one communicator per context; chains are split over ranks)
    void* comm = nullptr;
    int rank = 0, nranks = 1;
    // host-side record exchange instead of NCCL (sabr_ctx_init_host_exchange)
    sabr_allgather_fn exchange = nullptr;
    void* exchange_user = nullptr;
    // fused peer-memory exchange of the T_I level records (sabr_ctx_enable_peer_exchange)
    bool peer = false;
    sabr_gpu::PeerMailbox* peer_box = nullptr;          // this rank's mailbox (IPC-exported)
    std::vector<void*> peer_opened;           // peers' mailboxes mapped into this process
    sabr_gpu::PeerMailbox* const* peer_boxes = nullptr;  // device array [nranks]
    int* peer_error = nullptr;
    unsigned long long peer_epoch = 0;
    // grow-only device scratch, keyed by purpose
    std::map<std::string, std::pair<void*, size_t>> bufs;
    // host cache of xoshiro jump tables keyed by (draws per entry, count)
    std::map<std::pair<uint64_t, uint64_t>, std::vector<uint64_t>> jump_cache;
    void* pinned = nullptr;  // 4 KB pinned host scratch
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // per-launch event pairs of the dominant kernel when profiling
    std::vector<cudaEvent_t> kev;
    size_t kev_used = 0;
    // child contexts (own streams) of sabr_calibrate_static_T1_slices; a
    // child of a multi-rank context borrows its transport and has its own
    // peer mailboxes
    std::vector<sabr_ctx*> children;
    bool child = false;
};

namespace sabr_gpu {

// NVTX range (nsys / ncu timelines): the C-ABI entry points, each temperature
// level and each T_II step.  Header-only NVTX v3: no cost without a tool.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

void* dev_buf(sabr_ctx* ctx, const std::string& key, size_t bytes);
void check_cuda(cudaError_t e, const char* what);

template <class T>
T* upload(sabr_ctx* ctx, const std::string& key, const std::vector<T>& v) {
    T* d = static_cast<T*>(dev_buf(ctx, key, sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty())
        check_cuda(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice,
                                   ctx->stream),
                   "cudaMemcpyAsync H2D");
    return d;
}

// The exp_tab table (kernels_mc.cu) uploaded once per context.
const double2* exp_table_device(sabr_ctx* ctx);
// The log_tab table (Box-Muller's log in the MC kernels), uploaded once per context.
const double4* log_table_device(sabr_ctx* ctx);
const double2* sincos_table_device(sabr_ctx* ctx);
// Upload one candidate's step coefficients (FP64, + FP32 copy for SABR_FP32).
void set_coefficients(sabr_ctx* ctx, McParams& P, const std::vector<StepCoef>& coef, int precision);

// Device view of (part of) a surface; market = per-quote market values
// (null -> the quoted vols).
SurfaceView make_view(sabr_ctx* ctx, const std::string& key, const HostSurface& s,
                      const std::vector<double>* market);

// Time grid of build_grid (proj/src/mc.cpp:50-84): step lengths and the
// node time at each step END (where nu, rho are sampled).
struct HostGrid {
    std::vector<double> dt, sdt, t_end;
};
HostGrid build_grid(double maturity, double dt);
// every step of the grid has the same dt (no short last step)
bool uniform_grid(const HostGrid& g);

// Host-side CaseIIParams::validate with the reference message (input
// validation before a device run; the SA hot loop uses the device predicate).
void validate_case2(const double* p);
bool case2_feasible_host(const double* p);
void validate_model(int model, const double* p);
double model_nu_at(int model, const double* p, double t);
double model_rho_at(int model, const double* p, double t);

// MC launch description assembled on the host.
struct McJob {
    std::vector<McSlice> slices;
    std::vector<double> strikes;
    std::vector<double> hdt;
    int64_t total_steps = 0;
    int32_t max_q = 0;
};
int choose_ppt(const sabr_plan& plan);
// Fill slices/steps/jump offsets for maturities; returns the jump table
// (concatenated, 4 words per entry) for xoshiro mode.
std::vector<uint64_t> mc_layout(sabr_ctx* ctx, const sabr_plan& plan, int ppt,
                                const std::vector<HostGrid>& grids, McJob& job);

// Price `strikes` of every slice for ONE candidate (host-built coefficients):
// value/se per quote.  Used by price_european_batch, evaluate_case2_prices
// and the all-fixed T_II objective.
void mc_price_single(sabr_ctx* ctx, int model, const double* params, double spot,
                     const std::vector<double>& maturity, const std::vector<double>& rate,
                     const std::vector<double>& dividend, const std::vector<int64_t>& qoff,
                     const std::vector<double>& strikes, const sabr_plan& plan,
                     std::vector<double>& value, std::vector<double>& se);

// T_II annealer (calibrate_case2_T2's minimize): returns best full vector etc.
struct AnnealOut {
    std::vector<double> best_full;
    double best_value = 0.0;
    int64_t evals = 0;
    std::vector<double> trace_t, trace_f;
};
AnnealOut run_sa_case2(sabr_ctx* ctx, const HostSurface& surface, const std::vector<double>& market,
                       const ParamSpace& ps, const std::vector<double>& start_full, double horizon,
                       const sabr_schedule& sch, const sabr_plan& plan);

// NCCL all-gather of `bytes` per rank on the context stream (no-op for 1 rank).
void allgather(sabr_ctx* ctx, const void* send, void* recv, size_t bytes);

// Whole-call device time (events on the context stream) plus, when
// profiling, the summed duration of each dominant-kernel launch bracketed by
// its own event pair (before()/after()).
// Per-launch CUDA events (profiling mode) around one in kSample launches of
// the dominant kernel: events between kernels serialise them, so sampling
// keeps programmatic dependent launch (kernels_sa.cu) effective for the rest;
// kernel_ms is the sampled mean duration times the launch count.
struct Timer {
    static constexpr int64_t kSample = 8;
    sabr_ctx* ctx;
    std::chrono::steady_clock::time_point t0;
    int64_t calls = 0;
    bool sampling = false;
    explicit Timer(sabr_ctx* c);
    void start();
    void before();
    void after();
    void stop(double units, double path_steps, int64_t kernel_launches, int64_t total_launches);
};

}  // namespace sabr_gpu
