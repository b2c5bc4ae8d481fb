// throughput_probe.cu — per-SM issue throughput (thread-ops per cycle per SM)
// of the instruction kinds in the SA / MC hot loops, 8 independent chains per
// thread, 1024 threads per CTA, one CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o throughput_probe tools/throughput_probe.cu
#include <cstdint>
#include <cstdio>

constexpr int N = 2048;

template <int OP>
__global__ void __launch_bounds__(1024, 1) tp(double* out, long long* cyc, double a, double b) {
    double x[8];
    uint64_t u[8];
    for (int c = 0; c < 8; ++c) {
        x[c] = a + c * 1e-3 + threadIdx.x * 1e-9;
        u[c] = 0x9E3779B97F4A7C15ull * (threadIdx.x + 1 + c);
    }
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (OP == 0) x[c] = fma(x[c], b, a);                 // DFMA
            if (OP == 1) x[c] = x[c] + b;                        // DADD
            if (OP == 2) x[c] = x[c] * b;                        // DMUL
            if (OP == 3) x[c] = (x[c] > a) ? x[c] * 0.5 : x[c];  // DSETP + DMUL + 2 FSEL
            if (OP == 4) u[c] = (u[c] ^ (u[c] << 17)) + 0x5bd1e995ull;  // 64-bit xor-shift-add (INT)
            if (OP == 5) x[c] = static_cast<double>(u[c] >> (11 + (i & 1))) * b;  // I2F.F64.U64 + DMUL
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < 8; ++c) s += x[c] + static_cast<double>(u[c] & 1);
    out[blockIdx.x * 1024 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, double* out, long long* cyc, int sms) {
    tp<OP><<<sms, 1024>>>(out, cyc, 1.0000001, 0.9999999);
    tp<OP><<<sms, 1024>>>(out, cyc, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
    double ops = 1024.0 * 8 * N;
    printf("%-28s %7.2f thread-ops / cycle / SM\n", name, ops / static_cast<double>(cyc[0]));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * 1024 * sms);
    cudaMallocManaged(&cyc, sizeof(long long) * sms);
    run<0>("DFMA", out, cyc, sms);
    run<1>("DADD", out, cyc, sms);
    run<2>("DMUL", out, cyc, sms);
    run<3>("DSETP+DMUL+2 FSEL (per op)", out, cyc, sms);
    run<4>("u64 xor-shift-add (per op)", out, cyc, sms);
    run<5>("I2F.F64.U64+DMUL (per op)", out, cyc, sms);
    return 0;
}
