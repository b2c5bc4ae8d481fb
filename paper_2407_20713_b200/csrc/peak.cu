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
// MUFU (XU pipe) throughput: 8 independent ex2.approx.f32 chains per thread,
// the transcendental of the FP32 MC path (one ex2 per candidate-step).
__global__ void __launch_bounds__(256) mufu_peak_kernel(float* out, int iters, float a) {
    float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f, x4 = x0 + 0.4f,
          x5 = x0 + 0.5f, x6 = x0 + 0.6f, x7 = x0 + 0.7f;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            // ex2(-|x|) stays in (0, 1]: no overflow, no denormals
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x4));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x5));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x6));
            asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x7));
        }
    }
    const float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == a) out[0] = s;  // keep the chains alive
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

// Measured MUFU (XU) ex2 throughput of the context's GPU, in 1e12 ops/s.
extern "C" SABR_API sabr_status sabr_bench_mufu_peak(sabr_ctx* ctx, double* tops) {
    try {
        if (!ctx || !tops) fail(SABR_E_INVALID, "null argument");
        std::lock_guard<std::mutex> lock(ctx->mu);
        check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
        int sms = 0;
        check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device), "attr");
        float* out = static_cast<float*>(dev_buf(ctx, "peak_out", sizeof(double)));
        const int blocks = sms * 8, threads = 256, iters = 2048;
        mufu_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, 64, 12345.f);  // warm-up
        check_cuda(cudaEventRecord(ctx->ev0, ctx->stream), "event");
        mufu_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters, 12345.f);
        check_cuda(cudaEventRecord(ctx->ev1, ctx->stream), "event");
        check_cuda(cudaEventSynchronize(ctx->ev1), "event sync");
        float ms = 0.f;
        check_cuda(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "elapsed");
        const double ops = 8.0 * 16 * static_cast<double>(iters) * blocks * threads;
        *tops = ops / (ms * 1e-3) / 1e12;
        return SABR_OK;
    } catch (const Error& e) {
        return e.status;
    }
}
