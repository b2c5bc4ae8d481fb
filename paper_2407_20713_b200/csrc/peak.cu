// peak.cu — FP64 pipe peak microbenchmark (the roofline denominator of the
// FP64-bound SA/MC kernels; MEASURED_PEAKS.json only carries HBM and bf16).
// Each thread runs 8 independent DFMA chains; FLOPs = 2 per DFMA.
#include "engine.hpp"

namespace sabr_gpu {
namespace {
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
           x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace
}  // namespace sabr_gpu

using namespace sabr_gpu;

extern "C" SABR_API sabr_status sabr_bench_fp64_peak(sabr_ctx* ctx, double* tflops) {
    try {
        if (!ctx || !tflops) fail(SABR_E_INVALID, "null argument");
        std::lock_guard<std::mutex> lock(ctx->mu);
        check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
        int sms = 0;
        check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device), "attr");
        double* out = static_cast<double*>(dev_buf(ctx, "peak_out", sizeof(double)));
        const int blocks = sms * 8, threads = 256, iters = 4096;
        dfma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, 64, 0.999999, 1e-7);  // warm-up
        check_cuda(cudaEventRecord(ctx->ev0, ctx->stream), "event");
        dfma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters, 0.999999, 1e-7);
        check_cuda(cudaEventRecord(ctx->ev1, ctx->stream), "event");
        check_cuda(cudaEventSynchronize(ctx->ev1), "event sync");
        float ms = 0.f;
        check_cuda(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "elapsed");
        const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
        *tflops = flops / (ms * 1e-3) / 1e12;
        return SABR_OK;
    } catch (const Error& e) {
        return e.status;
    }
}
