// Host build of the device log_tab / sqrt_pos (device_common.cuh) against
// x86 long double: max error in ulps over Box-Muller's inputs u1 = 1 - k 2^-53
// (all binades down to 2^-53) and random positive doubles.
//   nvcc -x cu -O2 -std=c++17 -I include -I paper_2407_20713_b200/csrc tools/mathtab_check.cpp -o /tmp/mathtab_check
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "device_common.cuh"

using namespace sabr_dev;

static double4 g_tab[kLogTableSize];
static double2 g_sc[kSinCosTableSize];

static double ulp_err(double got, long double want) {
    const double w = static_cast<double>(want);
    const double ulp = std::nextafter(std::fabs(w), INFINITY) - std::fabs(w);
    return w == 0 ? std::fabs(got) : static_cast<double>(std::fabs(static_cast<long double>(got) - want) / ulp);
}

int main(int argc, char** argv) {
    const long iters = argc > 1 ? std::atol(argv[1]) : 20000000;
    for (int i = 0; i < kLogTableSize; ++i) {
        const double c = bitsd(0x3fe6000000000000ull + (static_cast<uint64_t>(i) << 45) + (1ull << 44));
        // the two intervals around 1 use invc = 1 exactly: r = z - 1 is then
        // exact and nothing cancels as log x -> 0
        const double invc = (i == kLogOne - 1 || i == kLogOne) ? 1.0
                                                                : static_cast<double>(1.0L / static_cast<long double>(c));
        const long double nl = -logl(static_cast<long double>(invc));
        // hi on a 2^-42 grid: k*ln2_hi + hi is then exact for every |k| < 2^10
        const double hi = static_cast<double>(roundl(nl * 0x1.0p42L) * 0x1.0p-42L);
        g_tab[i] = double4{invc, hi, static_cast<double>(nl - static_cast<long double>(hi)), 0.0};
    }
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < kSinCosTableSize; ++k)
        g_sc[k] = double2{static_cast<double>(sinl(pi * k / 64)), static_cast<double>(cosl(pi * k / 64))};
    std::mt19937_64 gen(1);
    double worst_sc = 0;  // absolute error in units of 2^-53 (the ulp at 1)
    double worst_log = 0, worst_sqrt = 0, worst_glibc = 0;
    for (long n = 0; n < iters; ++n) {
        // u1 = 1 - k 2^-53 with k spread over every binade
        const int b = static_cast<int>(gen() % 54);
        const uint64_t k = b == 0 ? 0 : ((gen() >> 11) >> (53 - b));
        const double u1 = 1.0 - static_cast<double>(k) * 0x1.0p-53;
        if (!(u1 > 0)) continue;
        const long double want = logl(static_cast<long double>(u1));
        worst_log = std::max(worst_log, ulp_err(log_tab(u1, g_tab), want));
        worst_glibc = std::max(worst_glibc, ulp_err(std::log(u1), want));
        const double a = -2.0 * std::log(u1);
        worst_sqrt = std::max(worst_sqrt, ulp_err(sqrt_pos(a), sqrtl(static_cast<long double>(a))));
        // Box-Muller's angle: u2 = (n >> 11) 2^-53
        const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
        double sn, cs;
        sincos_2pi(u2, g_sc, sn, cs);
        const long double th = 2 * pi * static_cast<long double>(u2);
        worst_sc = std::max(worst_sc, static_cast<double>(fabsl(sn - sinl(th)) * 0x1.0p53L));
        worst_sc = std::max(worst_sc, static_cast<double>(fabsl(cs - cosl(th)) * 0x1.0p53L));
    }
    std::printf("log_tab max err %.3f ulp (glibc log %.3f ulp); sqrt_pos max err %.3f ulp; sqrt_pos(0) = %g; "
                "sincos_2pi max abs err %.3f x 2^-53\n",
                worst_log, worst_glibc, worst_sqrt, sqrt_pos(0.0), worst_sc);
    return worst_log < 1.0 && worst_sqrt < 1.0 && sqrt_pos(0.0) == 0.0 && worst_sc < 1.0 ? 0 : 1;
}
