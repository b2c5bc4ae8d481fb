// latency_probe.cu — dependent-chain latency (cycles) of the instructions on
// the SA level kernel's critical path, measured with clock64 on one warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe tools/latency_probe.cu
#include <cstdio>
#include <cstdint>

constexpr int N = 4096;

__global__ void probe(double* out, long long* cyc, double a, double b, uint64_t s) {
    __shared__ double sm[64];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) sm[i] = i * 0.0;
    __syncthreads();
    double x = a;
    long long t0, t1;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(x, b, a);
    t1 = clock64();
    cyc[0] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = x + b;
    t1 = clock64();
    cyc[1] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = x * b;
    t1 = clock64();
    cyc[2] = t1 - t0;

    // DSETP + FSEL chain (compare then select)
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = (x > a) ? b : x;
    t1 = clock64();
    cyc[3] = t1 - t0;

    // LDS dependent chain (address from the loaded value)
    int idx = static_cast<int>(x) & 0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N / 8; ++i) idx = static_cast<int>(sm[idx]) & 63;
    t1 = clock64();
    cyc[4] = (t1 - t0) * 8;

    // 64-bit xor-shift chain (LOP3 + SHF)
    uint64_t u = s;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) u ^= u << 17;
    t1 = clock64();
    cyc[5] = t1 - t0;

    // u64 -> f64 convert chain (I2F.F64.U64 + F2I back)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N / 8; ++i) u = static_cast<uint64_t>(static_cast<double>(u >> 11));
    t1 = clock64();
    cyc[6] = (t1 - t0) * 8;

    // MUFU.RCP64H chain
    double r = b;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N / 8; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r));
    t1 = clock64();
    cyc[7] = (t1 - t0) * 8;

    out[threadIdx.x] = x + static_cast<double>(u) + r + idx;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMallocManaged(&cyc, 16 * sizeof(long long));
    for (int rep = 0; rep < 2; ++rep) probe<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, 0x1234567ull);
    cudaDeviceSynchronize();
    const char* names[] = {"DFMA", "DADD", "DMUL", "DSETP+FSEL", "LDS(+F2I)", "u64 xor-shift", "I2F.F64+F2I", "MUFU.RCP64H"};
    for (int i = 0; i < 8; ++i) printf("%-16s %6.2f cycles/op\n", names[i], cyc[i] / double(N));
    return 0;
}
