// hemul drop-in API (B200 build) — word size.
//
// Mirrors proj/core/include/hemul/word.hpp:19-23 of the reference. The B200
// HE Mul path is built for 64-bit limbs (the reference default and the
// paper-scale configuration); 32-bit word mode is accepted by the host-side
// containers but Scheme::he_mul rejects it with std::invalid_argument.
#pragma once

namespace hemul {

enum class WordSize : int { w32 = 32, w64 = 64 };

constexpr int log_beta(WordSize w) { return static_cast<int>(w); }

}  // namespace hemul
