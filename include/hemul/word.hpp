// hemul drop-in API (B200 build) — machine-word arithmetic.
//
// The scalar layer of the reference (proj/core/include/hemul/word.hpp:19-159):
// word size beta = 2^32 or 2^64, Shoup pairs {y, floor(y beta / p)} and the
// exact / lazy / approximate Shoup products, reduce_4p, add_mod, sub_mod and
// the runtime word dispatch. Host code (table builders, tests, user code)
// uses these; the GPU kernels carry their own sm_100a forms of the same
// operations (csrc/modarith.cuh, csrc/fields.cuh). Like the reference this is
// not constant-time code.
#pragma once

#include <cstdint>
#include <type_traits>

namespace hemul {

enum class WordSize : int { w32 = 32, w64 = 64 };

constexpr int log_beta(WordSize w) { return static_cast<int>(w); }

// A fixed multiplicand y < p and its scaled reciprocal floor(y * beta / p).
struct ShoupPair {
  uint64_t value = 0;
  uint64_t quotient = 0;
};

// Word primitives for beta = 2^LogBeta; every operand is < beta.
template <int LogBeta>
struct WordOps {
  static_assert(LogBeta == 32 || LogBeta == 64, "beta is 2^32 or 2^64");
  static constexpr int kLogBeta = LogBeta;
  static constexpr uint64_t kMask = LogBeta == 64 ? ~uint64_t{0} : 0xffffffffull;
  static constexpr int kHalf = LogBeta / 2;

  static uint64_t mulhi(uint64_t x, uint64_t y) {
    if constexpr (LogBeta == 64)
      return static_cast<uint64_t>((static_cast<unsigned __int128>(x) * y) >> 64);
    else
      return (x * y) >> 32;
  }
  static uint64_t mullo(uint64_t x, uint64_t y) { return (x * y) & kMask; }

  // High word from the three upper half-word partial products (lo * lo is
  // dropped): at most 2 below the exact high word.
  static uint64_t approx_mulhi(uint64_t x, uint64_t y) {
    constexpr uint64_t hm = (uint64_t{1} << kHalf) - 1;
    const uint64_t xl = x & hm, xh = x >> kHalf, yl = y & hm, yh = y >> kHalf;
    const uint64_t cross = xl * yh;
    const uint64_t mid = xh * yl + (cross & hm);
    return xh * yh + (cross >> kHalf) + (mid >> kHalf);
  }

  // floor((hi * beta + lo) / d), the quotient fitting one word
  static uint64_t div_word(uint64_t hi, uint64_t lo, uint64_t d) {
    if constexpr (LogBeta == 64)
      return static_cast<uint64_t>(((static_cast<unsigned __int128>(hi) << 64) | lo) / d);
    else
      return ((hi << 32) | lo) / d;
  }
};

template <int LB>
ShoupPair shoup_precompute_t(uint64_t y, uint64_t p) {
  ShoupPair s;
  s.value = y;
  s.quotient = WordOps<LB>::div_word(y, 0, p);
  return s;
}

// x * y - q * p for the Shoup quotient estimate q, wrapped to one word
template <int LB>
uint64_t shoup_remainder_t(uint64_t x, ShoupPair sp, uint64_t p, uint64_t q) {
  return (WordOps<LB>::mullo(x, sp.value) - WordOps<LB>::mullo(q, p)) & WordOps<LB>::kMask;
}

// x * y mod p in [0, p)
template <int LB>
uint64_t shoup_modmul_t(uint64_t x, ShoupPair sp, uint64_t p) {
  const uint64_t r = shoup_remainder_t<LB>(x, sp, p, WordOps<LB>::mulhi(x, sp.quotient));
  return r < p ? r : r - p;
}

// x * y mod p in [0, 2p): the caller does the final subtraction
template <int LB>
uint64_t shoup_modmul_lazy_t(uint64_t x, ShoupPair sp, uint64_t p) {
  return shoup_remainder_t<LB>(x, sp, p, WordOps<LB>::mulhi(x, sp.quotient));
}

// truncated quotient: x * y mod p in [0, 4p) (needs p < beta / 4)
template <int LB>
uint64_t shoup_modmul_approx_t(uint64_t x, ShoupPair sp, uint64_t p) {
  return shoup_remainder_t<LB>(x, sp, p, WordOps<LB>::approx_mulhi(x, sp.quotient));
}

// [0, 4p) -> [0, p)
inline uint64_t reduce_4p(uint64_t r, uint64_t p) {
  r = r >= 2 * p ? r - 2 * p : r;
  return r >= p ? r - p : r;
}

inline uint64_t add_mod(uint64_t a, uint64_t b, uint64_t p) {
  const uint64_t s = a + b;
  return s < p ? s : s - p;
}

inline uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t p) { return a < b ? a + (p - b) : a - b; }

// Calls f(std::integral_constant<int, log beta>) for the runtime word size.
template <typename F>
decltype(auto) dispatch_word(WordSize w, F&& f) {
  if (w == WordSize::w64) return f(std::integral_constant<int, 64>{});
  return f(std::integral_constant<int, 32>{});
}

inline uint64_t word_mulhi(WordSize w, uint64_t x, uint64_t y) {
  return dispatch_word(w, [&](auto lb) { return WordOps<decltype(lb)::value>::mulhi(x, y); });
}

inline ShoupPair shoup_precompute(uint64_t y, uint64_t p, WordSize w) {
  return dispatch_word(w, [&](auto lb) { return shoup_precompute_t<decltype(lb)::value>(y, p); });
}

inline uint64_t shoup_modmul(uint64_t x, ShoupPair sp, uint64_t p, WordSize w) {
  return dispatch_word(w, [&](auto lb) { return shoup_modmul_t<decltype(lb)::value>(x, sp, p); });
}

inline uint64_t shoup_modmul_approx(uint64_t x, ShoupPair sp, uint64_t p, WordSize w) {
  return dispatch_word(w,
                       [&](auto lb) { return shoup_modmul_approx_t<decltype(lb)::value>(x, sp, p); });
}

}  // namespace hemul
