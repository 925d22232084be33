// Host-side level tables: deterministic primes, twiddles, CRT weights and the
// exact-iCRT table, built by the same rules as the reference so that every
// intermediate residue matches (params.cpp:76-240, heaan.cpp:132-147).
#include "level_tables.hpp"

#include <algorithm>
#include <stdexcept>
#include <thread>

namespace hemul_gpu {

namespace {

using u128 = unsigned __int128;

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return uint64_t(u128(a) * b % m); }

uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  a %= m;
  for (; e; e >>= 1) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
  }
  return r;
}

// Miller-Rabin with the twelve prime bases below 40 (deterministic < 2^64),
// as params.cpp:22-47 does.
bool is_prime(uint64_t n) {
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (uint64_t b : bases)
    if (n % b == 0) return n == b;
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) d >>= 1, ++s;
  for (uint64_t b : bases) {
    uint64_t x = powmod(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool witness = true;
    for (int r = 1; r < s && witness; ++r) {
      x = mulmod(x, x, n);
      witness = x != n - 1;
    }
    if (witness) return false;
  }
  return true;
}

uint64_t shoup_q(uint64_t w, uint64_t p) { return uint64_t((u128(w) << 64) / p); }
uint32_t shoup_q32(uint64_t w, uint64_t p) { return uint32_t((w << 32) / p); }

// smallest generator power of exact order 2n (params.cpp:49-54)
uint64_t min_root(uint64_t p, uint64_t two_n) {
  for (uint64_t g = 2;; ++g) {
    const uint64_t psi = powmod(g, (p - 1) / two_n, p);
    if (powmod(psi, two_n / 2, p) == p - 1) return psi;
  }
}

// little-endian natural number
using Nat = std::vector<uint64_t>;

void nat_mul_word(Nat& a, uint64_t w) {
  uint64_t carry = 0;
  for (auto& x : a) {
    const u128 t = u128(x) * w + carry;
    x = uint64_t(t);
    carry = uint64_t(t >> 64);
  }
  if (carry) a.push_back(carry);
}

Nat nat_div_word(const Nat& a, uint64_t d, uint64_t* rem) {
  Nat q(a.size());
  u128 r = 0;
  for (size_t k = a.size(); k-- > 0;) {
    const u128 cur = (r << 64) | a[k];
    q[k] = uint64_t(cur / d);
    r = cur % d;
  }
  if (rem) *rem = uint64_t(r);
  return q;
}

int nat_bits(const Nat& a) {
  for (size_t k = a.size(); k-- > 0;)
    if (a[k]) return int(k * 64 + 64 - __builtin_clzll(a[k]));
  return 0;
}

// low `bits` bits of a as `limbs` words
Nat nat_low(const Nat& a, int bits) {
  const int limbs = (bits + 63) / 64;
  Nat r(limbs, 0);
  for (int k = 0; k < limbs && k < int(a.size()); ++k) r[k] = a[k];
  if (bits % 64) r[limbs - 1] &= (uint64_t(1) << (bits % 64)) - 1;
  return r;
}

// 2^bits - a  for 0 < a < 2^bits (two's complement in `bits` bits)
Nat nat_neg_mod_pow2(const Nat& a, int bits) {
  Nat r = nat_low(a, bits);
  uint64_t borrow = 0;
  for (auto& x : r) {  // 0 - r
    const uint64_t v = 0 - x - borrow;
    borrow = (x != 0) || borrow;
    x = v;
  }
  if (bits % 64) r.back() &= (uint64_t(1) << (bits % 64)) - 1;
  return r;
}

// (a << s) mod 2^bits
Nat nat_shl_low(const Nat& a, int s, int bits) {
  const int limbs = (bits + 63) / 64;
  Nat r(limbs, 0);
  const int ws = s / 64, bs = s % 64;
  for (int k = 0; k < limbs; ++k) {
    const int src = k - ws;
    uint64_t v = 0;
    if (src >= 0 && src < int(a.size())) v = a[src] << bs;
    if (bs && src - 1 >= 0 && src - 1 < int(a.size())) v |= a[src - 1] >> (64 - bs);
    r[k] = v;
  }
  if (bits % 64) r[limbs - 1] &= (uint64_t(1) << (bits % 64)) - 1;
  return r;
}

// bits [bit, bit + width) of a, width <= 32
uint32_t bits_at(const Nat& a, int bit, int width) {
  const int k = bit / 64, off = bit % 64;
  uint64_t v = k < int(a.size()) ? a[k] >> off : 0;
  if (off + width > 64 && k + 1 < int(a.size())) v |= a[k + 1] << (64 - off);
  return uint32_t(v & ((uint64_t(1) << width) - 1));
}

uint32_t bit_reverse(uint32_t i, int bits) {
  uint32_t r = 0;
  for (int b = 0; b < bits; ++b, i >>= 1) r = (r << 1) | (i & 1);
  return r;
}

template <typename F>
void parallel_for(int count, int threads, F&& f) {
  threads = std::max(1, std::min(threads, count));
  if (threads == 1) {
    for (int i = 0; i < count; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (int i = t; i < count; i += threads) f(i);
    });
  for (auto& th : pool) th.join();
}

}  // namespace

int prime_count(int bound_bits, int log_n) {
  // ceil((bound + log_n) / 58): every w64 prime exceeds 2^57 (params.cpp:76-79)
  return (bound_bits + log_n + 57) / 58;
}

void generate_primes(int count, int log_n, std::vector<uint64_t>& primes,
                     std::vector<uint64_t>& roots) {
  const uint64_t two_n = uint64_t(1) << (log_n + 1);
  const uint64_t top = uint64_t(1) << 60, floor_ = uint64_t(1) << 57;
  primes.clear();
  roots.clear();
  // the largest candidate = 1 (mod 2n) not above 2^60, then downward in 2n steps
  for (uint64_t c = top - (top - 1) % two_n; int(primes.size()) < count; c -= two_n) {
    if (c <= floor_) throw std::runtime_error("prime range exhausted for this ring degree");
    if (!is_prime(c)) continue;
    primes.push_back(c);
    roots.push_back(min_root(c, two_n));
  }
}

void generate_primes30(int count, int log_n, std::vector<uint64_t>& primes,
                       std::vector<uint64_t>& roots) {
  const uint64_t two_n = uint64_t(1) << (log_n + 1);
  const uint64_t top = (uint64_t(1) << kPrime30Bits) - 1, floor_ = uint64_t(1) << 20;
  primes.clear();
  roots.clear();
  for (uint64_t c = top - (top - 1) % two_n; int(primes.size()) < count; c -= two_n) {
    if (c <= floor_ || c < two_n)
      throw BasisUnavailable("30-bit prime range exhausted for this ring degree");
    if (!is_prime(c)) continue;
    primes.push_back(c);
    roots.push_back(min_root(c, two_n));
  }
}

std::vector<uint64_t> reference_primes(int region, int log_q, int log_q_max, int log_n,
                                       int* p_limbs) {
  const int bound = region == 1 ? 2 * log_q + log_n + 1 : log_q + 2 * log_q_max + log_n + 1;
  int count = region == 1 ? prime_count(2 * log_q, log_n) : prime_count(log_q + 2 * log_q_max, log_n);
  std::vector<uint64_t> primes, roots;
  Nat P;
  for (;; ++count) {
    generate_primes(count, log_n, primes, roots);
    P.assign(1, 1);
    for (uint64_t p : primes) nat_mul_word(P, p);
    if (nat_bits(P) > bound) break;
  }
  if (p_limbs) *p_limbs = (nat_bits(P) + 63) / 64;
  return primes;
}

namespace {
void build_tables(RegionHost& r, const Nat& P, const std::vector<int>& crt_bits, int threads,
                  int log_q);
}  // namespace

RegionHost build_region(int region, int log_q, int log_q_max, int log_n,
                        const std::vector<int>& crt_bits, int threads, int word, int split_h) {
  RegionHost r;
  r.region = region;
  r.log_n = log_n;
  r.word = word;
  const int h = region == 1 ? split_h : 0;
  r.split_h = h;
  // Largest |v| the iCRT must recover: region 1 carries d1 = A1 B2 + A2 B1,
  // |v| < 2 n q^2 (split: the high product sums four h-bit x h-bit
  // products, |v| < 4 n 2^(2h)); region 2 carries d2 * evk, |v| < n q Q^2
  // with the reference's full 2 log Q-bit key (w64 basis, heaan.cpp:139-143).
  // The 30-bit basis reduces the key mod 2^(log q + log Q) before its CRT
  // (the product is only needed mod qQ, a power of two), so |v| < n q^2 Q
  // and region 2 shrinks with the level.
  const int vbits = region == 2 ? (word == 64 ? log_q + 2 * log_q_max + log_n
                                              : 2 * log_q + log_q_max + log_n)
                                : (h ? 2 * h + log_n + 2 : 2 * log_q + log_n + 1);
  Nat P;
  int count;
  if (word == 64) {
    // prime count with the grow-until-bound loop of heaan.cpp:132-135 / 139-143
    const int bound = region == 1 ? 2 * log_q + log_n + 1 : log_q + 2 * log_q_max + log_n + 1;
    count = region == 1 ? prime_count(2 * log_q, log_n) : prime_count(log_q + 2 * log_q_max, log_n);
    for (;; ++count) {
      generate_primes(count, log_n, r.primes, r.roots);
      P.assign(1, 1);
      for (uint64_t p : r.primes) nat_mul_word(P, p);
      if (nat_bits(P) > bound) break;  // P >= 2^bound
    }
  } else {
    // the B200 basis: the fewest 30-bit primes that leave the iCRT headroom
    count = (vbits + 2 + kMinSlackBits) / kPrime30Bits;
    for (;; ++count) {
      generate_primes30(count, log_n, r.primes, r.roots);
      P.assign(1, 1);
      for (uint64_t p : r.primes) nat_mul_word(P, p);
      if ((nat_bits(P) - 1) - 1 - vbits >= kMinSlackBits) break;
    }
  }
  r.np = count;
  r.target_bits = region == 1 ? log_q : log_q + log_q_max;
  r.slack_bits = (nat_bits(P) - 1) - 1 - vbits;
  if (r.slack_bits < kMinSlackBits)
    throw std::runtime_error("prime set leaves less than 4 bits of iCRT headroom");
  build_tables(r, P, crt_bits, threads, log_q);
  return r;
}

RegionHost build_explicit_region(const std::vector<uint64_t>& primes,
                                 const std::vector<uint64_t>& roots, int log_n, int target_bits,
                                 const std::vector<int>& crt_bits, int threads) {
  // roots empty: a CRT / pointwise / iCRT-only set (no NTT of this degree;
  // the twiddle slots are filled with 1)
  if (primes.empty() || (!roots.empty() && primes.size() != roots.size()))
    throw std::invalid_argument("prime set and roots differ in size");
  const uint64_t two_n = uint64_t(2) << log_n;
  for (size_t j = 0; j < primes.size(); ++j) {
    const uint64_t p = primes[j];
    if (p < 3 || p >= (uint64_t(1) << 62) || (p & 1) == 0)
      throw std::invalid_argument("primes must be odd and below 2^62");
    if (roots.empty()) continue;
    if ((p - 1) % two_n != 0) throw std::invalid_argument("primes must be 1 mod 2n");
    if (powmod(roots[j], two_n / 2, p) != p - 1)
      throw std::invalid_argument("root is not a primitive 2n-th root of unity");
  }
  RegionHost r;
  r.region = 0;
  r.log_n = log_n;
  r.word = 64;
  r.split_h = 0;
  r.primes = primes;
  r.roots = roots.empty() ? std::vector<uint64_t>(primes.size(), 1) : roots;
  r.np = static_cast<int>(primes.size());
  r.target_bits = target_bits;
  Nat P(1, 1);
  for (uint64_t p : primes) nat_mul_word(P, p);
  r.slack_bits = 0;  // arbitrary residues: the iCRT runs with the exact fix-up
  build_tables(r, P, crt_bits, threads, 0);
  return r;
}

namespace {

void build_tables(RegionHost& r, const Nat& P, const std::vector<int>& crt_bits, int threads,
                  int log_q) {
  const int count = r.np, log_n = r.log_n, n = 1 << log_n, word = r.word, h = r.split_h,
            region = r.region;
  // per-prime constants
  std::vector<Nat> hat(count);
  std::vector<uint64_t> inv(count), ninv(count);
  for (int j = 0; j < count; ++j) {
    const uint64_t p = r.primes[j];
    uint64_t hat_mod = 0;
    hat[j] = nat_div_word(P, p, nullptr);
    nat_div_word(hat[j], p, &hat_mod);
    inv[j] = powmod(hat_mod, p - 2, p);
    ninv[j] = powmod(uint64_t(n) % p, p - 2, p);
  }
  if (word == 64) {
    r.dev.resize(count);
    for (int j = 0; j < count; ++j) {
      const uint64_t p = r.primes[j];
      DevPrime& d = r.dev[j];
      d = DevPrime{};
      d.p = p;
      d.one_q = shoup_q(1, p);
      d.beta = uint64_t((u128(1) << 64) % p);
      d.beta_q = shoup_q(d.beta, p);
      d.inv = inv[j];
      d.inv_q = shoup_q(d.inv, p);
      d.ninv = ninv[j];
      d.ninv_q = shoup_q(d.ninv, p);
      d.inv_p_dbl = 1.0 / double(p);
    }
    r.tw.resize(size_t(count) * n);
    r.itw.resize(size_t(count) * n);
  } else {
    r.dev32.resize(count);
    for (int j = 0; j < count; ++j) {
      const uint64_t p = r.primes[j];
      DevPrime32& d = r.dev32[j];
      d = DevPrime32{};
      d.p = uint32_t(p);
      d.one_q = shoup_q32(1, p);
      d.beta = uint32_t((uint64_t(1) << 32) % p);
      d.beta_q = shoup_q32(d.beta, p);
      d.inv = uint32_t(inv[j]);
      d.inv_q = shoup_q32(inv[j], p);
      d.ninv = uint32_t(ninv[j]);
      d.ninv_q = shoup_q32(ninv[j], p);
      d.inv_p_dbl = 1.0 / double(p);
      d.pad[0] = uint32_t((u128(1) << 55) / p);  // bigint_tc.cu: fixed-point k quotient
      uint32_t pinv = uint32_t(p);                // p^-1 mod 2^32 (Newton, p odd)
      for (int it = 0; it < 5; ++it) pinv *= 2u - uint32_t(p) * pinv;
      d.pad[1] = pinv;                            // ntt_blk.cu: Montgomery products
    }
    // the twiddle tables of the 30-bit basis are built on the device
    // (tables.cu build_twiddles32, from primes and roots); only the
    // per-prime constant w1n = itw[1] n^-1 is needed here
    r.roots_inv.resize(count);
    for (int j = 0; j < count; ++j) {
      const uint64_t p = r.primes[j];
      r.roots_inv[j] = powmod(r.roots[j], p - 2, p);
      const uint64_t itw1 = n > 1 ? powmod(r.roots_inv[j], uint64_t(n) / 2, p) : 1;
      const uint64_t w1n = n > 1 ? mulmod(itw1, ninv[j], p) : ninv[j];
      r.dev32[j].w1n = uint32_t(w1n);
      r.dev32[j].w1n_q = shoup_q32(w1n, p);
    }
  }

  // twiddles: tw[j*n + i] = psi^rev(i), itw = psi^-rev(i) (params.cpp:151-180)
  if (word == 64) parallel_for(count, threads, [&](int j) {
    const uint64_t p = r.primes[j], psi = r.roots[j];
    const uint64_t psi_inv = powmod(psi, p - 2, p);
    uint64_t pw = 1, ipw = 1, itw1 = 1;
    for (int i = 0; i < n; ++i) {
      const uint32_t k = bit_reverse(uint32_t(i), log_n);
      if (k == 1) itw1 = ipw;
      r.tw[size_t(j) * n + k] = Twiddle{pw, shoup_q(pw, p)};
      r.itw[size_t(j) * n + k] = Twiddle{ipw, shoup_q(ipw, p)};
      pw = mulmod(pw, psi, p);
      ipw = mulmod(ipw, psi_inv, p);
    }
    const uint64_t w1n = n > 1 ? mulmod(itw1, ninv[j], p) : ninv[j];
    r.dev[j].w1n = w1n;
    r.dev[j].w1n_q = shoup_q(w1n, p);
  });

  if (word == 32) {
    r.dev32_t = r.dev32;
    for (int j = 0; j < count; ++j) {
      const uint64_t p = r.primes[j];
      DevPrime32& d = r.dev32_t[j];
      const uint64_t nt = mulmod(d.ninv, inv[j], p), wt = mulmod(d.w1n, inv[j], p);
      d.ninv = uint32_t(nt);
      d.ninv_q = shoup_q32(nt, p);
      d.w1n = uint32_t(wt);
      d.w1n_q = shoup_q32(wt, p);
    }
    // Montgomery-compensated copies: ninv, w1n times 2^32 mod p
    auto mont = [&](const std::vector<DevPrime32>& src, std::vector<DevPrime32>& dst) {
      dst = src;
      for (int j = 0; j < count; ++j) {
        const uint64_t p = r.primes[j], r32 = (uint64_t(1) << 32) % p;
        DevPrime32& d = dst[j];
        const uint64_t nm = mulmod(d.ninv, r32, p), wm = mulmod(d.w1n, r32, p);
        d.ninv = uint32_t(nm);
        d.ninv_q = shoup_q32(nm, p);
        d.w1n = uint32_t(wm);
        d.w1n_q = shoup_q32(wm, p);
      }
    };
    mont(r.dev32, r.dev32_m);
    mont(r.dev32_t, r.dev32_tm);
  }

  // CRT weights of 2^(25 m) mod p_j (kernels.hpp CrtWeights): w64 as two
  // 30-bit halves, the 30-bit basis as one column
  const int wcols = word == 64 ? 2 : 1;
  std::vector<int> in_bits = crt_bits;
  if (h) in_bits = {h};  // both halves of a split input use the low half's table
  for (int bits : in_bits) {
    RegionHost::Crt c;
    c.in_bits = bits;
    c.chunks = (bits + kChunkBits - 1) / kChunkBits;
    c.ld = crt_cols_pad(wcols * count);
    c.wtab.assign(size_t(c.chunks) * c.ld, 0);
    for (int j = 0; j < count; ++j) {
      const uint64_t p = r.primes[j];
      const uint64_t step = powmod(2, kChunkBits, p);
      uint64_t u = 1 % p;
      for (int m = 0; m < c.chunks; ++m) {
        if (wcols == 2) {
          c.wtab[size_t(m) * c.ld + 2 * j] = uint32_t(u & 0x3fffffffu);
          c.wtab[size_t(m) * c.ld + 2 * j + 1] = uint32_t(u >> 30);
        } else {
          c.wtab[size_t(m) * c.ld + j] = uint32_t(u);
        }
        u = mulmod(u, step, p);
      }
    }
    r.crt.push_back(std::move(c));
  }
  if (word == 32) {
    // tensor-core CRT fields: region 1 the two halves, region 2 the ModUp input
    std::vector<std::pair<int, int>> fields;
    if (h && h % 8 == 0)
      fields = {{0, h}, {h, log_q - h}};
    else if (region == 2)
      fields = {{0, log_q}};
    // the split halves run in one launch (crt_forward_tc), which needs one
    // K padding and column tiling for both: build with the larger kpad
    int kpad = 0;
    for (auto [b0, nb] : fields) kpad = std::max(kpad, build_crt_tc_kpad(b0, nb));
    for (auto [b0, nb] : fields) r.crt_tc.push_back(build_crt_tc(r.primes, b0, nb, kpad));
  }

  // iCRT operands mod 2^T in A-row order: w64 H_j, H_j 2^30 (the two 30-bit
  // halves of t_j), the 30-bit basis H_j; then (-P). Then the 25-bit-chunk
  // table rows of the same order.
  const int T = r.target_bits;
  const int R = word == 64 ? 2 : 1;
  const int seg = R * count + 1;  // A rows of one RNS operand
  r.hat_t.resize(h ? 2 * seg : seg);
  for (int j = 0; j < count; ++j) {
    r.hat_t[R * j] = nat_low(hat[j], T);
    if (R == 2) r.hat_t[2 * j + 1] = nat_shl_low(hat[j], 30, T);
  }
  r.hat_t[R * count] = nat_neg_mod_pow2(P, T);
  // split: the high product c1 enters as 2^h c1 (a b = c0 + 2^h c1 mod 2^T)
  for (int row = 0; h && row < seg; ++row) r.hat_t[seg + row] = nat_shl_low(r.hat_t[row], h, T);
  r.m_out = (T + kChunkBits - 1) / kChunkBits;
  r.m_pad = (r.m_out + 15) / 16 * 16;
  const int K = static_cast<int>(r.hat_t.size());
  r.btab.assign(size_t(K) * r.m_pad, 0);
  for (int row = 0; row < K; ++row)
    for (int m = 0; m < r.m_out; ++m)
      r.btab[size_t(row) * r.m_pad + m] = bits_at(r.hat_t[row], kChunkBits * m, kChunkBits);
  r.p_limbs = (nat_bits(P) + 63) / 64;
  r.hat_full.assign(size_t(count) * r.p_limbs, 0);
  for (int j = 0; j < count; ++j)
    for (int k = 0; k < r.p_limbs && k < int(hat[j].size()); ++k)
      r.hat_full[size_t(j) * r.p_limbs + k] = hat[j][k];
  r.big_p.assign(r.p_limbs, 0);
  r.half_p.assign(r.p_limbs, 0);
  for (int k = 0; k < r.p_limbs && k < int(P.size()); ++k) r.big_p[k] = P[k];
  for (int k = 0; k < r.p_limbs; ++k)
    r.half_p[k] = (r.big_p[k] >> 1) | (k + 1 < r.p_limbs ? r.big_p[k + 1] << 63 : 0);
}

}  // namespace

int build_crt_tc_kpad(int bit0, int bits) {
  const int byte0 = bit0 / 8, nbytes = (bits + 7) / 8;
  const int d = byte0 - 8 * (byte0 / 8);
  return (d + nbytes + 31) / 32 * 32;
}

RegionHost::CrtTc build_crt_tc(const std::vector<uint64_t>& primes, int bit0, int bits,
                               int kpad_min) {
  RegionHost::CrtTc t;
  const int np = static_cast<int>(primes.size());
  t.bit0 = bit0;
  t.bits = bits;
  const int byte0 = bit0 / 8, nbytes = (bits + 7) / 8;
  t.limb0 = byte0 / 8;
  const int d = byte0 - 8 * t.limb0;
  t.kpad = std::max(build_crt_tc_kpad(bit0, bits), kpad_min);
  t.end_bit = bit0 + bits;
  // shared memory of crt_tc.cu: col_tile x K + 2 stages x 128 x K (K rounded
  // to 128-byte atom columns) + 1 KB alignment, within kMaxDynSmem (224 KB)
  const int kc = (t.kpad + 127) / 128 * 128;
  for (t.ncol_tiles = (4 * np + 255) / 256;; ++t.ncol_tiles) {
    t.primes_per_tile = (np + t.ncol_tiles - 1) / t.ncol_tiles;
    t.col_tile = (4 * t.primes_per_tile + 15) / 16 * 16;
    if (t.col_tile * kc + 2 * 128 * kc + 1024 <= 224 * 1024 || t.col_tile <= 16) break;
  }
  t.btab.assign(size_t(t.ncol_tiles) * t.col_tile * t.kpad, 0);
  for (int j = 0; j < np; ++j) {
    const int ct = j / t.primes_per_tile, jj = j - ct * t.primes_per_tile;
    const uint64_t p = primes[j];
    const uint64_t step = powmod(2, 8, p);
    uint64_t u = powmod(2, 32, p);  // Montgomery factor: crt_tc.cu planes_mont
    for (int k = d; k < d + nbytes; ++k) {
      for (int b = 0; b < 4; ++b)
        t.btab[(size_t(ct) * t.col_tile + 4 * jj + b) * t.kpad + k] = uint8_t(u >> (8 * b));
      u = mulmod(u, step, p);
    }
  }
  return t;
}

namespace {

uint8_t nat_byte(const Nat& v, long e) {
  if (e < 0 || size_t(e / 8) >= v.size()) return 0;
  return uint8_t(v[e / 8] >> (8 * (e % 8)));
}

// segs[s] = {rows V_j..., k row V_k}; values < 2^T. The A operand carries a
// constant 1 at K byte 4 k_slot + 6: its row adds `round` (< 2^T) to every
// coefficient (the finisher's rounding halves).
BigTcHost build_bigint(const std::vector<std::vector<Nat>>& segs, int T, int base8,
                       const Nat& round) {
  BigTcHost t;
  t.nseg = static_cast<int>(segs.size());
  t.base8 = base8;
  // every segment starts on a 16-row (64-byte) chunk: a chunk's rows belong to
  // one segment (padding rows have zero B rows)
  int slot = 0;
  for (int s = 0; s < t.nseg; ++s) {
    t.slot0[s] = slot;
    t.np[s] = static_cast<int>(segs[s].size()) - 1;
    slot += (t.np[s] + 15) / 16 * 16;
  }
  t.k_slot = slot;
  t.k_bytes = 4 * t.k_slot + 64;
  t.n_cols = ((T - base8 + 7) / 8 + 31) / 32 * 32;
  const long m0 = base8 / 8;
  t.btab.assign(size_t(t.n_cols) * t.k_bytes, 0);
  for (int s = 0; s < t.nseg; ++s) {
    for (int j = 0; j <= t.np[s]; ++j) {
      const Nat& v = segs[s][j];
      const bool krow = j == t.np[s];
      const int kb0 = krow ? 4 * t.k_slot + 2 * s : 4 * (t.slot0[s] + j);
      const int nb = krow ? 2 : 4;  // k < 2^16, t < 2^32
      for (int m = 0; m < t.n_cols; ++m)
        for (int b = 0; b < nb; ++b)
          t.btab[size_t(m) * t.k_bytes + kb0 + b] = nat_byte(v, m + m0 - b);
    }
  }
  for (int m = 0; m < t.n_cols; ++m) t.btab[size_t(m) * t.k_bytes + 4 * t.k_slot + 6] = nat_byte(round, m + m0);
  // device layout: chunk-major blocks of n_cols x 64 K-bytes, each already in
  // the 64-byte-swizzled K-major order the UMMA descriptor reads (16-byte
  // piece q of row m at piece q ^ ((m >> 1) & 3)), so one linear bulk copy per
  // chunk fills a pipeline stage (bigint_tc.cu)
  std::vector<uint8_t> dev(t.btab.size());
  const int nchunks = t.k_bytes / 64;
  for (int c = 0; c < nchunks; ++c)
    for (int m = 0; m < t.n_cols; ++m)
      for (int kb = 0; kb < 64; ++kb)
        dev[(size_t(c) * t.n_cols + m) * 64 + ((((kb >> 4) ^ ((m >> 1) & 3)) << 4) | (kb & 15))] =
            t.btab[size_t(m) * t.k_bytes + 64 * c + kb];
  t.btab.swap(dev);
  return t;
}

}  // namespace

BigTcHost build_icrt_tc(const RegionHost& r1) {
  const int np = r1.np, T = r1.target_bits;
  std::vector<std::vector<Nat>> segs(2);
  for (int h = 0; h < 2; ++h)
    for (int j = 0; j <= np; ++j) segs[h].push_back(r1.hat_t[size_t(h) * (np + 1) + j]);
  BigTcHost t = build_bigint(segs, T, 0, Nat{});
  t.out_bit = 0;
  t.out_bits = T;
  return t;
}

BigTcHost build_finisher_tc(const RegionHost& r1, const RegionHost& r2, int log_q, int log_q_max,
                            int log_p) {
  const int T2 = log_q + log_q_max;
  const int base8 = std::max(0, log_q_max - kFinisherGuardBits) / 8 * 8;
  std::vector<std::vector<Nat>> segs(3);
  for (int j = 0; j <= r2.np; ++j) segs[0].push_back(r2.hat_t[j]);
  for (int h = 0; h < 2; ++h)
    for (int j = 0; j <= r1.np; ++j)
      segs[1 + h].push_back(nat_shl_low(r1.hat_t[size_t(h) * (r1.np + 1) + j], log_q_max, T2));
  // rounding halves of R_logQ and R_logp: 2^(logQ-1) + 2^(logQ+logp-1)
  Nat round(size_t((T2 + 63) / 64), 0);
  round[(log_q_max - 1) / 64] |= uint64_t(1) << ((log_q_max - 1) % 64);
  round[(log_q_max + log_p - 1) / 64] |= uint64_t(1) << ((log_q_max + log_p - 1) % 64);
  BigTcHost t = build_bigint(segs, T2, base8, round);
  t.out_bit = log_q_max + log_p - base8;
  t.out_bits = log_q - log_p;
  return t;
}

FinisherHost build_finisher(const RegionHost& r1, const RegionHost& r2, int log_q,
                            int log_q_max, int log_p) {
  // V = X2 + 2^logQ X1 (+ both rounding halves), evaluated from bit `base`
  // up: region-2 rows are H_j-type values mod 2^(logq+logQ) truncated below
  // base, region-1 rows are exact values mod 2^logq placed at bit logQ.
  FinisherHost f;
  const int T2 = log_q + log_q_max;
  f.base = std::max(0, log_q_max - kFinisherGuardBits);
  f.width = T2 - f.base;
  f.cols = (f.width + kChunkBits - 1) / kChunkBits;
  f.cols_pad = (f.cols + 15) / 16 * 16;
  f.k2 = static_cast<int>(r2.hat_t.size());
  f.k1 = static_cast<int>(r1.hat_t.size());
  const int K = f.k2 + f.k1;
  f.btab.assign(size_t(K) * f.cols_pad, 0);
  for (int row = 0; row < f.k2; ++row)
    for (int m = 0; m < f.cols; ++m)
      f.btab[size_t(row) * f.cols_pad + m] =
          bits_at(r2.hat_t[row], f.base + kChunkBits * m, kChunkBits);
  const int shift = log_q_max - f.base;  // region-1 values sit at bit logQ
  for (int row = 0; row < f.k1; ++row) {
    const Nat v = nat_shl_low(r1.hat_t[row], shift, f.width);
    for (int m = 0; m < f.cols; ++m)
      f.btab[size_t(f.k2 + row) * f.cols_pad + m] = bits_at(v, kChunkBits * m, kChunkBits);
  }
  f.half_q_bit = log_q_max - 1 - f.base;
  f.half_p_bit = log_q_max + log_p - 1 - f.base;
  f.out_bit = log_q_max + log_p - f.base;
  f.out_bits = log_q - log_p;
  return f;
}

}  // namespace hemul_gpu
