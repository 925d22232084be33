// Host big integers of the drop-in API (include/hemul/bigint.hpp); only the
// scheme's host-side setup (keys, encryption, encoding) uses them — the GPU
// path works on fixed-width limb arrays. Semantics follow
// proj/core/src/bigint.cpp (little-endian limbs below 2^log_beta).
#include "hemul/bigint.hpp"

#include <algorithm>
#include <stdexcept>

namespace hemul {

namespace {

using u128 = unsigned __int128;

struct Word {
  int bits;
  uint64_t mask;
  explicit Word(WordSize w)
      : bits(log_beta(w)), mask(bits == 64 ? ~uint64_t{0} : (uint64_t{1} << bits) - 1) {}
};

size_t used(const BigInt& a) {
  size_t n = a.size();
  while (n && a[n - 1] == 0) --n;
  return n;
}

}  // namespace

int bigint_cmp(const BigInt& a, const BigInt& b) {
  const size_t na = used(a), nb = used(b);
  if (na != nb) return na < nb ? -1 : 1;
  for (size_t k = na; k-- > 0;)
    if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
  return 0;
}

bool bigint_is_zero(const BigInt& a) { return used(a) == 0; }

void bigint_trim(BigInt& a) { a.resize(used(a)); }

int bigint_bit_length(const BigInt& a, WordSize w) {
  const size_t n = used(a);
  if (!n) return 0;
  int top = 0;
  for (uint64_t x = a[n - 1]; x; x >>= 1) ++top;
  return static_cast<int>(n - 1) * log_beta(w) + top;
}

uint64_t bigint_add(BigInt& r, const BigInt& a, const BigInt& b, WordSize w) {
  const Word wd(w);
  const size_t n = std::max(a.size(), b.size());
  BigInt out(n);
  u128 carry = 0;
  for (size_t k = 0; k < n; ++k) {
    const u128 s = u128(k < a.size() ? a[k] : 0) + (k < b.size() ? b[k] : 0) + carry;
    out[k] = static_cast<uint64_t>(s) & wd.mask;
    carry = s >> wd.bits;
  }
  r = std::move(out);
  return static_cast<uint64_t>(carry);
}

void bigint_sub(BigInt& r, const BigInt& a, const BigInt& b, WordSize w) {
  if (bigint_cmp(a, b) < 0) throw std::invalid_argument("bigint_sub: a < b");
  const Word wd(w);
  BigInt out(a.size());
  uint64_t borrow = 0;
  for (size_t k = 0; k < a.size(); ++k) {
    const uint64_t x = a[k], y = (k < b.size() ? b[k] : 0);
    const u128 sub = u128(y) + borrow;
    out[k] = static_cast<uint64_t>(u128(x) + (u128(1) << wd.bits) - sub) & wd.mask;
    borrow = u128(x) < sub ? 1 : 0;
  }
  r = std::move(out);
}

BigInt bigint_mul(const BigInt& a, const BigInt& b, WordSize w) {
  const Word wd(w);
  const size_t na = used(a), nb = used(b);
  if (!na || !nb) return {};
  BigInt r(na + nb, 0);
  for (size_t i = 0; i < na; ++i) {
    u128 carry = 0;
    for (size_t j = 0; j < nb; ++j) {
      const u128 t = u128(a[i]) * b[j] + r[i + j] + carry;
      r[i + j] = static_cast<uint64_t>(t) & wd.mask;
      carry = t >> wd.bits;
    }
    r[i + nb] = static_cast<uint64_t>(carry);
  }
  bigint_trim(r);
  return r;
}

BigInt bigint_mul_word(const BigInt& a, uint64_t b, WordSize w) {
  return bigint_mul(a, bigint_from_u64(b, w), w);
}

void bigint_add_word(BigInt& a, uint64_t b, WordSize w) {
  const uint64_t c = bigint_add(a, a, bigint_from_u64(b, w), w);
  if (c) a.push_back(c);
}

BigInt bigint_shl(const BigInt& a, int bits, WordSize w) {
  const Word wd(w);
  if (bits < 0) return bigint_shr(a, -bits, w);
  const int ws = bits / wd.bits, bs = bits % wd.bits;
  BigInt r(a.size() + ws + 1, 0);
  for (size_t k = 0; k < a.size(); ++k) {
    const u128 v = u128(a[k]) << bs;
    r[k + ws] |= static_cast<uint64_t>(v) & wd.mask;
    r[k + ws + 1] |= static_cast<uint64_t>(v >> wd.bits) & wd.mask;
  }
  bigint_trim(r);
  return r;
}

BigInt bigint_shr(const BigInt& a, int bits, WordSize w) {
  const Word wd(w);
  const int ws = bits / wd.bits, bs = bits % wd.bits;
  if (static_cast<size_t>(ws) >= a.size()) return {};
  BigInt r(a.size() - ws, 0);
  for (size_t k = 0; k < r.size(); ++k) {
    const uint64_t lo = a[k + ws] >> bs;
    const uint64_t hi = (bs && k + ws + 1 < a.size()) ? (a[k + ws + 1] << (wd.bits - bs)) : 0;
    r[k] = (lo | hi) & wd.mask;
  }
  bigint_trim(r);
  return r;
}

int bigint_bit(const BigInt& a, int i, WordSize w) {
  const int lb = log_beta(w);
  const size_t k = static_cast<size_t>(i / lb);
  return k < a.size() ? static_cast<int>((a[k] >> (i % lb)) & 1) : 0;
}

BigInt bigint_mod(const BigInt& a, const BigInt& m, WordSize w) {
  if (bigint_is_zero(m)) throw std::invalid_argument("bigint_mod: zero modulus");
  BigInt r = a;
  bigint_trim(r);
  if (bigint_cmp(r, m) < 0) return r;
  // binary long division: subtract m << s for s from high to low
  const int shift = bigint_bit_length(r, w) - bigint_bit_length(m, w);
  for (int s = shift; s >= 0; --s) {
    const BigInt ms = bigint_shl(m, s, w);
    if (bigint_cmp(r, ms) >= 0) bigint_sub(r, r, ms, w);
  }
  bigint_trim(r);
  return r;
}

uint64_t bigint_mod_word(const BigInt& a, uint64_t m, WordSize w) {
  uint64_t rem = 0;
  bigint_div_word(a, m, &rem, w);
  return rem;
}

BigInt bigint_div_word(const BigInt& a, uint64_t m, uint64_t* rem, WordSize w) {
  if (m == 0) throw std::invalid_argument("bigint_div_word: zero divisor");
  const int lb = log_beta(w);
  BigInt q(a.size(), 0);
  u128 r = 0;
  for (size_t k = a.size(); k-- > 0;) {
    const u128 cur = (r << lb) | a[k];
    q[k] = static_cast<uint64_t>(cur / m);
    r = cur % m;
  }
  if (rem) *rem = static_cast<uint64_t>(r);
  bigint_trim(q);
  return q;
}

BigInt bigint_from_u64(uint64_t v, WordSize w) {
  const Word wd(w);
  BigInt r;
  while (v) {
    r.push_back(v & wd.mask);
    v = wd.bits == 64 ? 0 : v >> wd.bits;
  }
  return r;
}

BigInt bigint_pow2(int bits, WordSize w) {
  const int lb = log_beta(w);
  BigInt r(static_cast<size_t>(bits / lb + 1), 0);
  r.back() = uint64_t{1} << (bits % lb);
  return r;
}

uint64_t bigint_to_u64(const BigInt& a, WordSize w) {
  const int lb = log_beta(w);
  uint64_t v = 0;
  for (size_t k = 0; k < a.size() && static_cast<int>(k) * lb < 64; ++k) v |= a[k] << (k * lb);
  return v;
}

std::string bigint_to_hex(const BigInt& a, WordSize w) {
  static const char* digits = "0123456789abcdef";
  const int bits = bigint_bit_length(a, w);
  if (!bits) return "0";
  std::string s;
  for (int nib = (bits + 3) / 4 - 1; nib >= 0; --nib) {
    int v = 0;
    for (int b = 3; b >= 0; --b) v = (v << 1) | bigint_bit(a, 4 * nib + b, w);
    s.push_back(digits[v]);
  }
  return s;
}

BigInt bigint_from_hex(const std::string& s, WordSize w) {
  BigInt r;
  for (char ch : s) {
    int v;
    if (ch >= '0' && ch <= '9') v = ch - '0';
    else if (ch >= 'a' && ch <= 'f') v = ch - 'a' + 10;
    else if (ch >= 'A' && ch <= 'F') v = ch - 'A' + 10;
    else throw std::invalid_argument("bigint_from_hex: bad digit");
    r = bigint_shl(r, 4, w);
    if (v) bigint_add_word(r, static_cast<uint64_t>(v), w);
  }
  bigint_trim(r);
  return r;
}

}  // namespace hemul
