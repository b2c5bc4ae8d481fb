// slice_qr_check.cpp — host check of the factored slice cost (slice_qr.hpp):
// for random market grids of n = 1 .. 600 quotes (and grids of repeated
// strikes, whose factor is rank-deficient) and random coefficient
// vectors (C0, A1, A2), ||R (C0, A1, A2, -1)||^2 evaluated as the kernels do
// (nine FMAs) against the per-quote sum in x86 long double, next to the
// per-quote sum in double (the reference's arithmetic).  Mixed error
// (relative above a cost of 1e-8).  Exits 1 unless the factored form is
// within twice the double per-quote sum's error.
//   g++ -O2 -std=c++17 -I paper_2407_20713_b200/csrc tools/slice_qr_check.cpp \
//       paper_2407_20713_b200/csrc/slice_qr.cpp -o slice_qr_check
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "slice_qr.hpp"

int main() {
    std::mt19937_64 gen(20260);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    double worst = 0.0, worst_near = 0.0, base = 0.0, base_near = 0.0;
    for (int n : {1, 2, 3, 4, 5, 7, 19, 21, 30, 84, 600}) {
        for (int rep = 0; rep < 20; ++rep) {
            std::vector<double> l(n), m(n);
            for (int j = 0; j < n; ++j) {
                l[j] = -0.4 + 0.8 * U(gen);
                m[j] = 0.05 + 0.6 * U(gen);
            }
            if (rep == 19)  // repeated strikes: collinear columns, a rank-deficient factor
                for (int j = 1; j < n; ++j) l[j] = l[j % 2];
            double R[sabr_gpu::kQrStride];
            sabr_gpu::slice_qr_factor(l.data(), m.data(), n, R);
            for (int t = 0; t < 2000; ++t) {
                // generic vectors, and vectors near the least-squares fit (small residuals)
                const bool near = t % 2;
                double x0 = 0.05 + 0.6 * U(gen), x1 = -0.5 + U(gen), x2 = -2 + 4 * U(gen);
                if (near) {  // exact fit through three quotes' markets, perturbed
                    x1 *= 1e-3;
                    x2 *= 1e-3;
                    x0 = m[0] - x1 * l[0] - x2 * l[0] * l[0];
                }
                long double s = 0;
                double sd = 0;  // the per-quote sum in double (the reference's arithmetic)
                for (int j = 0; j < n; ++j) {
                    const double rd = (m[j] - (x0 + x1 * l[j] + x2 * l[j] * l[j])) / m[j];
                    sd += rd * rd;
                    const long double r = 1.0L - ((long double)x0 + (long double)x1 * l[j] +
                                                  (long double)x2 * l[j] * l[j]) / (long double)m[j];
                    s += r * r;
                }
                const double u0 = std::fma(R[2], x2, std::fma(R[1], x1, std::fma(R[0], x0, -R[3])));
                const double u1 = std::fma(R[5], x2, std::fma(R[4], x1, -R[6]));
                const double u2 = std::fma(R[7], x2, -R[8]);
                const double c = std::fma(u0, u0, std::fma(u1, u1, std::fma(u2, u2, R[9])));
                // mixed error: relative above 1e-8, absolute below (a perfect fit has cost -> 0)
                const long double den = s > 1e-8L ? s : 1e-8L;
                const double e = (double)(fabsl((long double)c - s) / den);
                const double eb = (double)(fabsl((long double)sd - s) / den);
                (near ? worst_near : worst) = std::fmax(near ? worst_near : worst, e);
                (near ? base_near : base) = std::fmax(near ? base_near : base, eb);
            }
        }
    }
    std::printf("vs the long-double per-quote sum, worst mixed error: factored %.3e (generic) %.3e (near fit); "
                "per-quote sum in double %.3e / %.3e\n", worst, worst_near, base, base_near);
    // the factored form must be as accurate as the reference's own double arithmetic
    return (worst <= std::fmax(2 * base, 1e-14) && worst_near <= std::fmax(2 * base_near, 1e-14)) ? 0 : 1;
}
