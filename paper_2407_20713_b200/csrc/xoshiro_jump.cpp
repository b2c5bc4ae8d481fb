// xoshiro_jump.cpp — F2-linear jump-ahead for the reference's xoshiro256++
// block streams.
//
// The reference consumes one xoshiro256++ substream per block of
// `block_size` paths sequentially (proj/src/mc.cpp:126-135): path p of a block
// starts 2*n_steps*p draws into the stream.  The state transition M of
// xoshiro256 is linear over GF(2)^256, so M^k = r(M) with
// r(x) = x^k mod P(x), P the characteristic polynomial of M.  The host finds
// P once (Berlekamp-Massey on one state bit), builds r for the offsets a GPU
// thread needs, and the device applies r(M) to the block's seed state with
// 256 masked accumulate steps (Xoshiro::jump in device_common.cuh).
#include "xoshiro_jump.hpp"

#include <array>
#include <mutex>
#include <stdexcept>

#include "device_common.cuh"

namespace sabr_gpu {

namespace {

using Poly = std::array<uint64_t, 4>;  // bits 0..255

struct CharPoly {
    Poly low;  // P(x) = x^256 + low(x)
};

// Berlekamp-Massey over GF(2) on a bit sequence.
std::vector<uint8_t> berlekamp_massey(const std::vector<uint8_t>& s, int& L_out) {
    const int n = static_cast<int>(s.size());
    std::vector<uint8_t> C(n + 1, 0), B(n + 1, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int k = 0; k < n; ++k) {
        uint8_t d = s[k];
        for (int i = 1; i <= L; ++i) d ^= C[i] & s[k - i];
        if (d == 0) {
            ++m;
        } else if (2 * L <= k) {
            T = C;
            for (int i = 0; i + m <= n; ++i) C[i + m] ^= B[i];
            L = k + 1 - L;
            B = T;
            m = 1;
        } else {
            for (int i = 0; i + m <= n; ++i) C[i + m] ^= B[i];
            ++m;
        }
    }
    L_out = L;
    return C;
}

const CharPoly& char_poly() {
    static CharPoly cp;
    static std::once_flag once;
    std::call_once(once, [] {
        sabr_dev::Xoshiro g;
        g.init(0x1234567ull, 99);
        std::vector<uint8_t> bits(1024);
        for (auto& b : bits) {
            b = static_cast<uint8_t>(g.s0 & 1ull);
            g.advance();
        }
        int L = 0;
        const auto C = berlekamp_massey(bits, L);
        if (L != 256) throw std::logic_error("xoshiro jump: characteristic polynomial degree != 256");
        // s_{k+256} = sum_{i<256} c_{256-i} s_{k+i}  =>  P(x) = x^256 + sum_i c_{256-i} x^i
        cp.low = {0, 0, 0, 0};
        for (int i = 0; i < 256; ++i)
            if (C[256 - i]) cp.low[i >> 6] |= 1ull << (i & 63);
    });
    return cp;
}

// r <- r * x mod P
inline void mulx(Poly& r, const Poly& low) {
    const uint64_t carry = r[3] >> 63;
    r[3] = (r[3] << 1) | (r[2] >> 63);
    r[2] = (r[2] << 1) | (r[1] >> 63);
    r[1] = (r[1] << 1) | (r[0] >> 63);
    r[0] <<= 1;
    if (carry) {
        r[0] ^= low[0];
        r[1] ^= low[1];
        r[2] ^= low[2];
        r[3] ^= low[3];
    }
}

Poly mulmod(const Poly& a, const Poly& b, const Poly& low) {
    Poly r{0, 0, 0, 0};
    for (int i = 255; i >= 0; --i) {
        mulx(r, low);
        if ((b[i >> 6] >> (i & 63)) & 1ull) {
            r[0] ^= a[0];
            r[1] ^= a[1];
            r[2] ^= a[2];
            r[3] ^= a[3];
        }
    }
    return r;
}

Poly xpow(uint64_t e, const Poly& low) {
    Poly result{1, 0, 0, 0};
    Poly base{2, 0, 0, 0};  // x
    while (e) {
        if (e & 1ull) result = mulmod(result, base, low);
        base = mulmod(base, base, low);
        e >>= 1;
    }
    return result;
}

}  // namespace

std::vector<uint64_t> xoshiro_jump_table(uint64_t draws_per_entry, uint64_t count) {
    const Poly& low = char_poly().low;
    const Poly step = xpow(draws_per_entry, low);
    std::vector<uint64_t> out(4 * count);
    Poly cur{1, 0, 0, 0};
    for (uint64_t k = 0; k < count; ++k) {
        for (int w = 0; w < 4; ++w) out[4 * k + w] = cur[w];
        cur = mulmod(cur, step, low);
    }
    return out;
}

bool xoshiro_jump_selftest() {
    for (uint64_t k : {0ull, 1ull, 2ull, 7ull, 255ull, 256ull, 1000ull, 4097ull}) {
        sabr_dev::Xoshiro a, b;
        a.init(42, 3);
        b = a;
        for (uint64_t i = 0; i < k; ++i) a.advance();
        const auto t = xoshiro_jump_table(k, 2);
        b.jump(t.data() + 4);
        if (a.s0 != b.s0 || a.s1 != b.s1 || a.s2 != b.s2 || a.s3 != b.s3) return false;
    }
    return true;
}

}  // namespace sabr_gpu
