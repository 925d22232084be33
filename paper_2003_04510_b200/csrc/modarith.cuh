// 64-bit modular arithmetic for sm_100a, built from 32-bit IMAD.WIDE.U32
// (measured on B200: 64 IMAD.WIDE / clk / SM, the same rate as a 32-bit
// IMAD, while mul.hi.u64 costs ~9 slots; see profiles/r01_imad_probe.txt).
//
// Residues live below primes p < 2^60 (params.cpp:93-96 picks them from
// (2^57, 2^60)), so lazy values in [0, 4p) still fit 62 bits.
//
// Reference counterparts: ShoupPair / shoup_modmul_t / _lazy_t / _approx_t,
// add_mod, sub_mod (proj/core/include/hemul/word.hpp:25-127). All results
// that leave a kernel are canonical, so they are bit-identical to the
// reference whatever reduction variant is used inside.
#pragma once
#include <cstdint>

namespace hemul_gpu {

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return static_cast<uint32_t>(x >> 32); }

__device__ __forceinline__ uint64_t wide(uint32_t a, uint32_t b) {
  return static_cast<uint64_t>(a) * b;
}

// floor(x*y / 2^64) minus e, e in {0,1,2}: the x0*y0 partial product and the
// carries of the two cross terms' low halves are dropped (cf. word.hpp:45-51
// approx_mulhi, which drops lo*lo the same way). 3 IMAD.WIDE + 1 add.
__device__ __forceinline__ uint64_t mulhi_approx(uint64_t x, uint64_t y) {
  // x1 y1 + hi(x1 y0) + hi(x0 y1): the 33-bit sum of the two high halves is
  // formed with one add/addc pair and fed as the 64-bit addend of the last
  // IMAD.WIDE (written in PTX so no {hi, 0} register pairs get materialised
  // with moves on the FMA pipe)
  uint64_t q;
  asm("{\n\t"
      ".reg .u32 x0, x1, y0, y1, al, ah, bl, bh, sl, sh;\n\t"
      ".reg .u64 a, b, s;\n\t"
      "mov.b64 {x0, x1}, %1;\n\t"
      "mov.b64 {y0, y1}, %2;\n\t"
      "mul.wide.u32 a, x1, y0;\n\t"
      "mul.wide.u32 b, x0, y1;\n\t"
      "mov.b64 {al, ah}, a;\n\t"
      "mov.b64 {bl, bh}, b;\n\t"
      "add.cc.u32 sl, ah, bh;\n\t"
      "addc.u32 sh, 0, 0;\n\t"
      "mov.b64 s, {sl, sh};\n\t"
      "mad.wide.u32 %0, x1, y1, s;\n\t"
      "}"
      : "=l"(q)
      : "l"(x), "l"(y));
  return q;
}

// Exact floor(x*y / 2^64).
__device__ __forceinline__ uint64_t mulhi(uint64_t x, uint64_t y) { return __umul64hi(x, y); }

// x*y + q*(2^64 - p) mod 2^64 == x*y - q*p mod 2^64, in 2 IMAD.WIDE + 4 IMAD.
__device__ __forceinline__ uint64_t mul_sub_lo(uint64_t x, uint64_t y, uint64_t q, uint64_t negp) {
  // lo64(x0 y0 + q0 n0) then the four cross terms on the high word only
  uint64_t r;
  asm("{\n\t"
      ".reg .u32 x0, x1, y0, y1, q0, q1, n0, n1, rl, rh;\n\t"
      ".reg .u64 t;\n\t"
      "mov.b64 {x0, x1}, %1;\n\t"
      "mov.b64 {y0, y1}, %2;\n\t"
      "mov.b64 {q0, q1}, %3;\n\t"
      "mov.b64 {n0, n1}, %4;\n\t"
      "mul.wide.u32 t, x0, y0;\n\t"
      "mad.wide.u32 t, q0, n0, t;\n\t"
      "mov.b64 {rl, rh}, t;\n\t"
      "mad.lo.u32 rh, x0, y1, rh;\n\t"
      "mad.lo.u32 rh, x1, y0, rh;\n\t"
      "mad.lo.u32 rh, q0, n1, rh;\n\t"
      "mad.lo.u32 rh, q1, n0, rh;\n\t"
      "mov.b64 %0, {rl, rh};\n\t"
      "}"
      : "=l"(r)
      : "l"(x), "l"(y), "l"(q), "l"(negp));
  return r;
}

// Shoup multiplication by a fixed operand w with wq = floor(w 2^64 / p).
// Approximate quotient: result in [0, 4p) for any x < 2^64 (word.hpp:102-111).
__device__ __forceinline__ uint64_t shoup_mul_4p(uint64_t x, uint64_t w, uint64_t wq, uint64_t negp) {
  const uint64_t q = mulhi_approx(x, wq);
  return mul_sub_lo(x, w, q, negp);
}

// Conditional subtraction: x in [0, 2m) -> [0, m). Works for m < 2^63.
__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) {
  const uint64_t t = x - m;
  return static_cast<int64_t>(t) < 0 ? x : t;
}

// [0, 4p) -> [0, p)  (word.hpp:114-118 reduce_4p)
__device__ __forceinline__ uint64_t reduce_4p(uint64_t x, uint64_t p) {
  return csub(csub(x, 2 * p), p);
}

// Exact x*w mod p in [0, p) for x < 2^62.
__device__ __forceinline__ uint64_t shoup_mul(uint64_t x, uint64_t w, uint64_t wq, uint64_t p) {
  return reduce_4p(shoup_mul_4p(x, w, wq, 0 - p), p);
}

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t p) { return csub(a + b, p); }
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t p) { return csub(a + p - b, p); }

// Exact a*b mod p for a, b < 2^62 via the 128-bit product and two Shoup
// reductions (the reference's reduce2, rns.cpp:14-19):
//   a*b = hi*2^64 + lo ;  r = lo*1 + hi*(2^64 mod p)  (mod p)
// one_q = floor(2^64 / p), beta = 2^64 mod p, beta_q = floor(beta 2^64 / p).
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p, uint64_t one_q,
                                           uint64_t beta, uint64_t beta_q) {
  const uint64_t lo = a * b;
  const uint64_t hi = __umul64hi(a, b);
  const uint64_t negp = 0 - p;
  const uint64_t r0 = shoup_mul_4p(lo, 1, one_q, negp);
  const uint64_t r1 = shoup_mul_4p(hi, beta, beta_q, negp);
  return reduce_4p(csub(r0 + r1, 4 * p), p);
}

}  // namespace hemul_gpu
