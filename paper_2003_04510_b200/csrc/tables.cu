// Level tables built on the device (sm_100a): the 30-bit basis' twiddle
// tables, the bulk of a level's setup (np x n Shoup pairs per direction,
// 2 x 328 x 2^17 x 8 bytes at X) that the host used to compute and upload.
//
// Reference: make_ntt_tables (proj/core/src/params.cpp:151-180): tw[j][rev(i)]
// = psi_j^i, itw[j][rev(i)] = psi_j^-i with Shoup quotients floor(w 2^w / p)
// (here w = 32 bits: Twiddle32, fields.cuh F32). Same entries as the host
// builder in level_tables.cpp (build_tables), checked by
// tests/test_gpu_basis32.py::test_device_twiddles_match_rule.
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace hemul_gpu {

namespace {

// a b mod p for a, b < p < 2^31: the fp64 quotient of a b < 2^62 is off by
// at most one, corrected on the exact 64-bit remainder
__device__ __forceinline__ uint32_t mulmod30(uint32_t a, uint32_t b, uint32_t p, double inv_p) {
  const uint64_t z = uint64_t(a) * b;
  const uint64_t q = static_cast<uint64_t>(__dmul_rz(static_cast<double>(z), inv_p));
  int64_t r = static_cast<int64_t>(z - q * p);
  if (r < 0) r += p;
  if (r >= int64_t(p)) r -= p;
  return static_cast<uint32_t>(r);
}

__device__ __forceinline__ uint32_t powmod30(uint32_t b, uint32_t e, uint32_t p, double inv_p) {
  uint32_t r = 1;
  while (e) {
    if (e & 1) r = mulmod30(r, b, p, inv_p);
    b = mulmod30(b, b, p, inv_p);
    e >>= 1;
  }
  return r;
}

// floor(w 2^32 / p) for w < p
__device__ __forceinline__ uint32_t shoup_q30(uint32_t w, uint32_t p, double inv_p) {
  const uint64_t z = uint64_t(w) << 32;
  uint64_t q = static_cast<uint64_t>(__dmul_rz(static_cast<double>(z), inv_p));
  int64_t r = static_cast<int64_t>(z - q * p);
  while (r < 0) r += p, --q;
  while (r >= int64_t(p)) r -= p, ++q;
  return static_cast<uint32_t>(q);
}

constexpr int kChunk = 2048, kThreads = 256;

// CTA (x, j): exponents i in [x kChunk, (x+1) kChunk) of prime j; thread t
// starts from psi^(i0 + t) and steps by psi^kThreads
__global__ void __launch_bounds__(kThreads) twiddles32_kernel(const uint32_t* __restrict__ primes,
                                                              const uint32_t* __restrict__ roots,
                                                              const uint32_t* __restrict__ roots_inv,
                                                              int log_n, Twiddle32* tw,
                                                              Twiddle32* itw) {
  const int j = blockIdx.y;
  const uint32_t p = primes[j], psi = roots[j], psi_inv = roots_inv[j];
  const double inv_p = 1.0 / static_cast<double>(p);
  const size_t n = size_t(1) << log_n;
  const uint32_t i0 = blockIdx.x * kChunk + threadIdx.x;
  if (i0 >= n) return;
  uint32_t x = powmod30(psi, i0, p, inv_p), y = powmod30(psi_inv, i0, p, inv_p);
  const uint32_t sx = powmod30(psi, kThreads, p, inv_p), sy = powmod30(psi_inv, kThreads, p, inv_p);
  Twiddle32* tj = tw + size_t(j) * n;
  Twiddle32* ij = itw + size_t(j) * n;
  for (uint32_t i = i0; i < n && i < (blockIdx.x + 1u) * kChunk; i += kThreads) {
    const uint32_t k = __brev(i) >> (32 - log_n);
    tj[k] = Twiddle32{x, shoup_q30(x, p, inv_p)};
    ij[k] = Twiddle32{y, shoup_q30(y, p, inv_p)};
    x = mulmod30(x, sx, p, inv_p);
    y = mulmod30(y, sy, p, inv_p);
  }
}

}  // namespace

cudaError_t build_twiddles32(const uint32_t* primes, const uint32_t* roots,
                             const uint32_t* roots_inv, int np, int log_n, Twiddle32* tw,
                             Twiddle32* itw, cudaStream_t st) {
  if (np <= 0 || log_n < 1 || log_n > 17) return cudaErrorInvalidValue;
  const size_t n = size_t(1) << log_n;
  dim3 grid(static_cast<unsigned>((n + kChunk - 1) / kChunk), static_cast<unsigned>(np));
  twiddles32_kernel<<<grid, kThreads, 0, st>>>(primes, roots, roots_inv, log_n, tw, itw);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
