// Device-resident per-region constants shared by all kernels.
#pragma once
#include <cstdint>

namespace hemul_gpu {

// One RNS prime of a region and every per-prime constant a kernel needs.
// Source of each field in the reference:
//   p                         PrimeSet::primes            params.cpp:89-115
//   one_q, beta, beta_q       pair_one / pair_beta         params.cpp:106-111
//   inv, inv_q                IcrtTables::inv_p            params.cpp:196-197
//   ninv, ninv_q              NttTables::n_inv             params.cpp:176-177
//   w1n, w1n_q                itw[1] * n^-1 (the last GS stage with the n^-1
//                             scaling of ntt.cpp:127-136 folded in)
//   inv_p_dbl                 1/p_j for the exact iCRT quotient
struct DevPrime {
  uint64_t p;
  uint64_t one_q;   // floor(2^64 / p)
  uint64_t beta;    // 2^64 mod p
  uint64_t beta_q;  // floor(beta * 2^64 / p)
  uint64_t inv, inv_q;
  uint64_t ninv, ninv_q;
  uint64_t w1n, w1n_q;
  double inv_p_dbl;
  uint64_t pad;
};
static_assert(sizeof(DevPrime) == 96, "DevPrime layout");

// Twiddle with its Shoup quotient (ShoupPair, word.hpp:25-28).
struct Twiddle {
  uint64_t w, wq;
};

// One prime of the B200 30-bit basis (fields.cuh F32); Shoup quotients are
// floor(w 2^32 / p). No reference counterpart: the HE Mul result does not
// depend on the basis (see fields.cuh).
struct DevPrime32 {
  uint32_t p;
  uint32_t one_q;   // floor(2^32 / p)
  uint32_t beta;    // 2^32 mod p
  uint32_t beta_q;  // floor(beta 2^32 / p)
  uint32_t inv, inv_q;    // (P / p)^-1 mod p
  uint32_t ninv, ninv_q;  // n^-1 mod p
  uint32_t w1n, w1n_q;    // itw[1] n^-1
  uint32_t pad[2];         // [0] floor(2^55 / p) (bigint_tc.cu), [1] p^-1 mod 2^32
  double inv_p_dbl;       // 1 / p
  double pad2;
};
static_assert(sizeof(DevPrime32) == 64, "DevPrime32 layout");

struct Twiddle32 {
  uint32_t w, wq;
};

}  // namespace hemul_gpu
