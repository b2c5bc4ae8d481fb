// dispatch_probe.cu — does a DFMA block the warp scheduler's dispatch for the
// two cycles its 16-lane FP64 pipe needs, or can integer instructions issue
// in the second cycle?  Per iteration each thread issues 4 independent DFMAs
// and K independent 32-bit LOP3s mixing in the loop counter (nothing can be
// folded or hoisted); 32
// warps per SM.  If integer work fills the FP64 pipe's second cycle, the time
// per iteration stays 8 cycles per warp-quad up to K = 4; if not, it grows as
// 8 + K.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dispatch_probe tools/dispatch_probe.cu
#include <cstdio>

constexpr int N = 4096;

template <int K>
__global__ void __launch_bounds__(1024, 1) probe(double* out, long long* cyc, double a, double b) {
    double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    unsigned i0 = threadIdx.x, i1 = i0 + 1, i2 = i0 + 2, i3 = i0 + 3, i4 = i0 + 4, i5 = i0 + 5, i6 = i0 + 6,
             i7 = i0 + 7;
    const unsigned c = 0x9E3779B9u;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < N; ++it) {
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x0) : "d"(b), "d"(a));
        if (K > 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i0) : "r"(c), "r"(it));
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x1) : "d"(b), "d"(a));
        if (K > 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i1) : "r"(c), "r"(it));
        if (K > 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i4) : "r"(c), "r"(it));
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x2) : "d"(b), "d"(a));
        if (K > 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i2) : "r"(c), "r"(it));
        if (K > 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i5) : "r"(c), "r"(it));
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x3) : "d"(b), "d"(a));
        if (K > 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i3) : "r"(c), "r"(it));
        if (K > 6) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i6) : "r"(c), "r"(it));
        if (K > 7) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(i7) : "r"(c), "r"(it));
    }
    __syncthreads();
    const long long t1 = clock64();
    out[blockIdx.x * 1024 + threadIdx.x] = x0 + x1 + x2 + x3 + i0 + i1 + i2 + i3 + i4 + i5 + i6 + i7;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(double* out, long long* cyc, int sms) {
    probe<K><<<sms, 1024>>>(out, cyc, 1.0000001, 0.9999999);
    probe<K><<<sms, 1024>>>(out, cyc, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
    // 8 warps per SMSP, each iteration = 4 DFMA + K IADD per warp
    const double per_iter = static_cast<double>(cyc[0]) / N / 8;  // cycles per warp-iteration on one SMSP
    printf("4 DFMA + %d LOP3 per warp-iteration: %.2f SMSP cycles (pipe bound 8.0, issue bound %d)\n", K, per_iter,
           4 + K);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * 1024 * sms);
    cudaMallocManaged(&cyc, sizeof(long long) * sms);
    run<0>(out, cyc, sms);
    run<2>(out, cyc, sms);
    run<4>(out, cyc, sms);
    run<6>(out, cyc, sms);
    run<8>(out, cyc, sms);
    return 0;
}
