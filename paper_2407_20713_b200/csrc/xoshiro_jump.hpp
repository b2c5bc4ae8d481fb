#pragma once

#include <cstdint>
#include <vector>

namespace sabr_gpu {

// count polynomials r_k(x) = x^(k*draws_per_entry) mod P(x), 4 words each:
// applying r_k(M) to a xoshiro256 state advances it by k*draws_per_entry
// draws (see xoshiro_jump.cpp).
std::vector<uint64_t> xoshiro_jump_table(uint64_t draws_per_entry, uint64_t count);

// jump(k) == k x advance() for a handful of k.
bool xoshiro_jump_selftest();

}  // namespace sabr_gpu
