// Common definitions of the libgmg host layer (C++17).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gmg.h"

namespace gmg {

// Internal error carrying a gmg_status; converted to a status code at the C ABI.
struct Error : std::runtime_error {
  gmg_status code;
  Error(gmg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(gmg_status c, const std::string& m) { throw Error(c, m); }

#define GMG_REQUIRE(cond, code, msg)                                   \
  do {                                                                 \
    if (!(cond)) ::gmg::fail(code, std::string(msg));                  \
  } while (0)

using i64 = int64_t;
using u64 = uint64_t;
using i32 = int32_t;
using u32 = uint32_t;
using Vec3 = std::array<int64_t, 3>;

// ---------------------------------------------------------------- Morton
// Bit interleaving with x as the least significant bit of every group.
inline u64 spread2(u64 v) {  // 32 -> 64 bits, one gap
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
inline u64 spread3(u64 v) {  // 21 -> 63 bits, two gaps
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
inline u64 compact2(u64 v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v >> 4)) & 0x00ff00ff00ff00ffull;
  v = (v | (v >> 8)) & 0x0000ffff0000ffffull;
  v = (v | (v >> 16)) & 0x00000000ffffffffull;
  return v;
}
inline u64 compact3(u64 v) {
  v &= 0x1249249249249249ull;
  v = (v | (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v | (v >> 4)) & 0x100f00f00f00f00full;
  v = (v | (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v | (v >> 16)) & 0x1f00000000ffffull;
  v = (v | (v >> 32)) & 0x1fffffull;
  return v;
}
inline u64 morton(int dim, const Vec3& c) {
  if (dim == 2) return spread2((u64)c[0]) | (spread2((u64)c[1]) << 1);
  return spread3((u64)c[0]) | (spread3((u64)c[1]) << 1) | (spread3((u64)c[2]) << 2);
}
inline Vec3 unmorton(int dim, u64 k) {
  if (dim == 2) return {(i64)compact2(k), (i64)compact2(k >> 1), 0};
  return {(i64)compact3(k), (i64)compact3(k >> 1), (i64)compact3(k >> 2)};
}

// ---------------------------------------------------------------- flat hash set
// Open addressing, linear probing, keys < 2^64 - 1.
struct FlatSet {
  std::vector<u64> slot;
  size_t count = 0;
  static constexpr u64 EMPTY = ~0ull;
  explicit FlatSet(size_t cap = 16) { rehash(cap); }
  static u64 mix(u64 z) {
    z ^= z >> 33; z *= 0xff51afd7ed558ccdull; z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ull; z ^= z >> 33;
    return z;
  }
  void rehash(size_t cap) {
    size_t n = 16;
    while (n < cap * 2) n <<= 1;
    std::vector<u64> old;
    old.swap(slot);
    slot.assign(n, EMPTY);
    count = 0;
    for (u64 k : old)
      if (k != EMPTY) insert(k);
  }
  bool insert(u64 k) {
    if ((count + 1) * 2 > slot.size()) rehash(slot.size());
    size_t m = slot.size() - 1, i = mix(k) & m;
    while (slot[i] != EMPTY) {
      if (slot[i] == k) return false;
      i = (i + 1) & m;
    }
    slot[i] = k;
    ++count;
    return true;
  }
  bool contains(u64 k) const {
    size_t m = slot.size() - 1, i = mix(k) & m;
    while (slot[i] != EMPTY) {
      if (slot[i] == k) return true;
      i = (i + 1) & m;
    }
    return false;
  }
  std::vector<u64> sorted_keys() const;
};

// LSD radix sort of (key, value) pairs by key; stable.
void radix_sort_pairs(std::vector<u64>& key, std::vector<u64>& val, int key_bits);
void radix_sort_keys(std::vector<u64>& key, int key_bits);

inline int bits_for(u64 v) {
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b < 1 ? 1 : b;
}

}  // namespace gmg
