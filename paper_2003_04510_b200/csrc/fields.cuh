// Residue "fields" the RNS kernels are templated on.
//
//   F64: the reference's own prime basis (w64 primes in (2^57, 2^60),
//        params.cpp:76-115), 64-bit residues built from 32-bit IMAD.WIDE
//        (modarith.cuh). Used by the stage entry points, whose outputs are
//        compared residue-for-residue with the reference.
//   F32: a B200 basis of primes p = 1 (mod 2n) below 2^30, 32-bit residues.
//        HE Mul is an exact big-integer product (the CRT is lossless), so its
//        result does not depend on the basis: the same ciphertext comes out
//        with ~2x as many 30-bit primes, and each butterfly costs one
//        IMAD.HI + two IMAD instead of five IMAD.WIDE + four IMAD.
//
// Every field exposes the same lazy-reduction contract to the kernels:
//   ct()   Cooley-Tukey butterfly, closed on the forward domain
//          (F64: [0, 8p), F32: [0, 4p))
//   gs()   Gentleman-Sande butterfly, closed on the inverse domain
//          (F64: [0, 4p), F32: [0, 2p))
//   fwd_canon()  forward-domain value -> [0, p)
//   inv_level0() last inverse level with n^-1 folded in, outputs in [0, p)
//   mul(), mul_add2()  products of forward-domain values -> inverse domain
//   hat_inv()    t_j = x (P/p_j)^-1 mod p_j in [0, p) (the iCRT A rows)
#pragma once
#include <cstdint>

#include "device_tables.cuh"
#include "modarith.cuh"

namespace hemul_gpu {

// ---- 32-bit arithmetic (p < 2^30: lazy values < 4p fit 32 bits) -----------

__device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// x in [0, 2m) -> [0, m) for m < 2^31: x - m wraps above x when x < m.
__device__ __forceinline__ uint32_t csub32(uint32_t x, uint32_t m) { return umin32(x, x - m); }

// Shoup product x w mod p in [0, 2p) for any x < 2^32 (wq = floor(w 2^32 / p)).
__device__ __forceinline__ uint32_t shoup32(uint32_t x, uint32_t w, uint32_t wq, uint32_t negp) {
  const uint32_t q = __umulhi(x, wq);
  return x * w + q * negp;
}

// z mod p in [0, 2p) for any z < 2^64:  z = zh 2^32 + zl,
// zh 2^32 = zh beta (beta = 2^32 mod p), zl = zl * 1 — two Shoup products.
__device__ __forceinline__ uint32_t reduce64_32(uint64_t z, uint32_t p, uint32_t negp,
                                                uint32_t one_q, uint32_t beta, uint32_t beta_q) {
  const uint32_t zh = static_cast<uint32_t>(z >> 32), zl = static_cast<uint32_t>(z);
  const uint32_t r = shoup32(zh, beta, beta_q, negp) + (zl + __umulhi(zl, one_q) * negp);
  return csub32(r, 2 * p);  // [0, 4p) -> [0, 2p)
}

// Montgomery: z < p 2^32 -> z 2^-32 mod p in (0, 2p), pinv = p^-1 mod 2^32.
// z - m p with m = zl pinv has a zero low word, so (z - m p) / 2^32 =
// zh - mulhi(m, p), in (-p, p) because zh < p and m p < p 2^32.
__device__ __forceinline__ uint32_t mont32(uint64_t z, uint32_t p, uint32_t pinv) {
  const uint32_t zh = static_cast<uint32_t>(z >> 32), m = static_cast<uint32_t>(z) * pinv;
  return zh + p - __umulhi(m, p);
}

struct F64 {
  using W = uint64_t;
  using Prime = DevPrime;
  using Tw = Twiddle;
  static constexpr int kRowsPerPrime = 2;    // iCRT A rows per residue (30-bit halves)
  static constexpr int kCrtColsPerPrime = 2; // CRT weight columns per prime (30-bit halves)
  struct Mod {
    uint64_t p, p4, negp;
    __device__ __forceinline__ explicit Mod(const Prime& pr) : p(pr.p), p4(4 * pr.p), negp(0 - pr.p) {}
  };
  // a, b in [0, 8p) -> [0, 8p)
  static __device__ __forceinline__ void ct(W& a, W& b, W w, W wq, const Mod& m) {
    const W u = csub(a, m.p4);
    const W v = shoup_mul_4p(b, w, wq, m.negp);
    a = u + v;
    b = u + m.p4 - v;
  }
  // a, b in [0, 4p) -> [0, 4p)
  static __device__ __forceinline__ void gs(W& a, W& b, W w, W wq, const Mod& m) {
    const W u = a, v = b;
    a = csub(u + v, m.p4);
    b = shoup_mul_4p(u + m.p4 - v, w, wq, m.negp);
  }
  static __device__ __forceinline__ W fwd_canon(W x, const Mod& m) {
    return reduce_4p(csub(x, m.p4), m.p);
  }
  static __device__ __forceinline__ void inv_level0(W& a, W& b, const Prime& pr, const Mod& m) {
    const W u = a, v = b;
    a = shoup_mul(u + v, pr.ninv, pr.ninv_q, m.p);
    b = shoup_mul(u + m.p4 - v, pr.w1n, pr.w1n_q, m.p);
  }
  static __device__ __forceinline__ W mul(W x, W y, const Prime& pr) {
    return mulmod(x, y, pr.p, pr.one_q, pr.beta, pr.beta_q);
  }
  static __device__ __forceinline__ W mul_add2(W x1, W y1, W x2, W y2, const Prime& pr) {
    return add_mod(mul(x1, y1, pr), mul(x2, y2, pr), pr.p);
  }
  // canonical t = x (P/p_j)^-1 mod p_j for a canonical or lazy residue x
  static __device__ __forceinline__ W hat_inv(W x, const Prime& pr) {
    return shoup_mul(x, pr.inv, pr.inv_q, pr.p);
  }
};

struct F32 {
  using W = uint32_t;
  using Prime = DevPrime32;
  using Tw = Twiddle32;
  static constexpr int kRowsPerPrime = 1;     // t_j < 2^30 is one A row
  static constexpr int kCrtColsPerPrime = 1;  // weights < 2^30 are one column
  struct Mod {
    uint32_t p, p2, negp;
    __device__ __forceinline__ explicit Mod(const Prime& pr) : p(pr.p), p2(2 * pr.p), negp(0u - pr.p) {}
  };
  // Harvey: a, b in [0, 4p) -> [0, 4p)
  static __device__ __forceinline__ void ct(W& a, W& b, W w, W wq, const Mod& m) {
    const W u = csub32(a, m.p2);
    const W v = shoup32(b, w, wq, m.negp);
    a = u + v;
    b = u + m.p2 - v;
  }
  // a, b in [0, 2p) -> [0, 2p)
  static __device__ __forceinline__ void gs(W& a, W& b, W w, W wq, const Mod& m) {
    const W u = a, v = b;
    a = csub32(u + v, m.p2);
    b = shoup32(u + m.p2 - v, w, wq, m.negp);
  }
  static __device__ __forceinline__ W fwd_canon(W x, const Mod& m) {
    return csub32(csub32(x, m.p2), m.p);
  }
  static __device__ __forceinline__ void inv_level0(W& a, W& b, const Prime& pr, const Mod& m) {
    const W u = a, v = b;
    a = csub32(shoup32(u + v, pr.ninv, pr.ninv_q, m.negp), m.p);
    b = csub32(shoup32(u + m.p2 - v, pr.w1n, pr.w1n_q, m.negp), m.p);
  }
  // x, y in [0, 4p): x y < 16 p^2 < 2^64
  static __device__ __forceinline__ W mul(W x, W y, const Prime& pr) {
    return reduce64_32(static_cast<uint64_t>(x) * y, pr.p, 0u - pr.p, pr.one_q, pr.beta,
                       pr.beta_q);
  }
  // x1 y1 + x2 y2 with lazy inputs: reduce the inputs to [0, p) so that the
  // sum of the two products stays below 2 p^2 < 2^61, then reduce once
  static __device__ __forceinline__ W mul_add2(W x1, W y1, W x2, W y2, const Prime& pr) {
    const Mod m(pr);
    x1 = fwd_canon(x1, m);
    y1 = fwd_canon(y1, m);
    x2 = fwd_canon(x2, m);
    y2 = fwd_canon(y2, m);
    const uint64_t z = static_cast<uint64_t>(x1) * y1 + static_cast<uint64_t>(x2) * y2;
    return reduce64_32(z, pr.p, m.negp, pr.one_q, pr.beta, pr.beta_q);
  }
  static __device__ __forceinline__ W hat_inv(W x, const Prime& pr) {
    return csub32(shoup32(x, pr.inv, pr.inv_q, 0u - pr.p), pr.p);
  }
  // Split tensor product (context.cu, level_tables.hpp split_h): v = the
  // halves x1 X1 y1 Y1 x2 X2 y2 Y2 of ax1 bx1 ax2 bx2 (forward domain, lazy)
  // -> d2 = (x1x2, x1X2 + X1x2), d0 = (y1y2, y1Y2 + Y1y2),
  //    d1 = (x1y2 + x2y1, x1Y2 + X1y2 + x2Y1 + X2y1) in v[0..5].
  // Inputs are reduced to [0, p) first: a sum of four products < 4 p^2 < 2^62.
  static __device__ __forceinline__ void tensor_split(W (&v)[8], const Prime& pr) {
    const Mod m(pr);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fwd_canon(v[i], m);
    auto P = [](W a, W b) { return static_cast<uint64_t>(a) * b; };
    auto R = [&](uint64_t z) { return reduce64_32(z, pr.p, m.negp, pr.one_q, pr.beta, pr.beta_q); };
    const W x1 = v[0], X1 = v[1], y1 = v[2], Y1 = v[3], x2 = v[4], X2 = v[5], y2 = v[6], Y2 = v[7];
    v[0] = R(P(x1, x2));
    v[1] = R(P(x1, X2) + P(X1, x2));
    v[2] = R(P(y1, y2));
    v[3] = R(P(y1, Y2) + P(Y1, y2));
    v[4] = R(P(x1, y2) + P(x2, y1));
    v[5] = R(P(x1, Y2) + P(X1, y2) + P(x2, Y1) + P(X2, y1));
  }
  // The same six sums Montgomery-reduced: v = (sum) 2^-32 mod p in [0, 2p)
  // (every sum < 4 p^2 < p 2^32); the inverse pass multiplies 2^32 back in
  // (level_tables.hpp dev32_m / dev32_tm).
  static __device__ __forceinline__ void tensor_split_mont(W (&v)[8], const Prime& pr) {
    const Mod m(pr);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fwd_canon(v[i], m);
    auto P = [](W a, W b) { return static_cast<uint64_t>(a) * b; };
    const uint32_t pinv = pr.pad[1];
    auto R = [&](uint64_t z) { return mont32(z, pr.p, pinv); };
    const W x1 = v[0], X1 = v[1], y1 = v[2], Y1 = v[3], x2 = v[4], X2 = v[5], y2 = v[6], Y2 = v[7];
    v[0] = R(P(x1, x2));
    v[1] = R(P(x1, X2) + P(X1, x2));
    v[2] = R(P(y1, y2));
    v[3] = R(P(y1, Y2) + P(Y1, y2));
    v[4] = R(P(x1, y2) + P(x2, y1));
    v[5] = R(P(x1, Y2) + P(X1, y2) + P(x2, Y1) + P(X2, y1));
  }
  // x y 2^-32 mod p in [0, 2p) for x y < 4 p^2 (one factor canonical, the other < 4p)
  static __device__ __forceinline__ W mul_mont(W x, W y, const Prime& pr) {
    return mont32(static_cast<uint64_t>(x) * y, pr.p, pr.pad[1]);
  }
};

}  // namespace hemul_gpu
