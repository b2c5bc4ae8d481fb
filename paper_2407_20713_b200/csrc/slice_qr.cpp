// slice_qr.cpp — the least-squares factor of one slice's market grid (host,
// binary128).  See slice_qr.hpp.
#include "slice_qr.hpp"

#include <cmath>
#include <vector>

namespace sabr_gpu {
namespace {

using quad = __float128;

quad qsqrt(quad a) {  // Newton from the double root; a >= 0
    if (a <= 0) return 0;
    quad x = std::sqrt(static_cast<double>(a));
    for (int i = 0; i < 3; ++i) x = quad(0.5) * (x + a / x);
    return x;
}

quad qabs(quad a) { return a < 0 ? -a : a; }

}  // namespace

void slice_qr_factor(const double* lm, const double* market, int64_t n, double out[kQrStride]) {
    // W = [1/m, l/m, l^2/m, 1] (n x 4, column-major), exact in binary128
    // (a double's square and reciprocal carry ~2^-113 relative error).
    std::vector<quad> w(4 * static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) {
        const quad inv = quad(1.0) / static_cast<quad>(market[j]);
        const quad l = lm[j];
        w[j] = inv;
        w[n + j] = inv * l;
        w[2 * n + j] = inv * l * l;
        w[3 * n + j] = quad(1.0);
    }
    // Householder QR: after min(n, 4) reflections the first rows hold R.
    const int64_t kmax = n < 4 ? n : 4;
    for (int64_t k = 0; k < kmax; ++k) {
        quad* col = &w[k * n];
        quad norm2 = 0;
        for (int64_t i = k; i < n; ++i) norm2 += col[i] * col[i];
        const quad norm = qsqrt(norm2);
        if (norm == 0) continue;
        const quad alpha = col[k] > 0 ? -norm : norm;  // no cancellation in v_k
        // v = x - alpha e_k, H = I - 2 v v^T / (v^T v); v^T v = 2 norm (norm + |x_k|)
        col[k] -= alpha;
        const quad vtv = quad(2.0) * norm * (norm + qabs(col[k] + alpha));
        for (int64_t c = k + 1; c < 4; ++c) {
            quad* y = &w[c * n];
            quad dot = 0;
            for (int64_t i = k; i < n; ++i) dot += col[i] * y[i];
            const quad f = quad(2.0) * dot / vtv;
            for (int64_t i = k; i < n; ++i) y[i] -= f * col[i];
        }
        col[k] = alpha;
        for (int64_t i = k + 1; i < n; ++i) col[i] = 0;
    }
    auto R = [&](int i, int c) -> quad { return i < n ? w[c * n + i] : quad(0.0); };
    out[0] = static_cast<double>(R(0, 0));
    out[1] = static_cast<double>(R(0, 1));
    out[2] = static_cast<double>(R(0, 2));
    out[3] = static_cast<double>(R(0, 3));
    out[4] = static_cast<double>(R(1, 1));
    out[5] = static_cast<double>(R(1, 2));
    out[6] = static_cast<double>(R(1, 3));
    out[7] = static_cast<double>(R(2, 2));
    out[8] = static_cast<double>(R(2, 3));
    out[9] = static_cast<double>(R(3, 3) * R(3, 3));
    out[10] = out[11] = 0.0;
}

}  // namespace sabr_gpu
