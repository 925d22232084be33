// Element-wise RNS products and big-integer polynomial epilogues (sm_100a).
//
// pointwise / tensor_product / evk_product:  rns_pointwise_mul
//   (proj/core/src/rns.cpp:108-130, 360-371), one exact 64x64 -> 128 product
//   reduced with two Shoup steps (the reference's reduce2, rns.cpp:14-19).
// keyswitch_epilogue: poly_shift_right by log_Q (ModDown), poly_add with the
//   region-1 term, poly_shift_right by log_p (rescale) — heaan.cpp:401-409,
//   poly.cpp:46-70, 98-115 — fused into one pass per coefficient.
// These kernels are HBM-bound; each coefficient's limbs are read once.
#include <cuda_runtime.h>

#include "fields.cuh"
#include "kernels.hpp"

namespace hemul_gpu {

namespace {

__device__ __forceinline__ uint64_t mm(uint64_t a, uint64_t b, const DevPrime& pr) {
  return mulmod(a, b, pr.p, pr.one_q, pr.beta, pr.beta_q);
}

__global__ void pointwise_kernel(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                 uint64_t* __restrict__ out, size_t total, int np, int log_n,
                                 const DevPrime* __restrict__ primes) {
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
       idx += size_t(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>((idx >> log_n) % np);
    out[idx] = mm(a[idx], b[idx], primes[j]);
  }
}

// The products of the unfused path (logN < 12): forward-domain inputs,
// inverse-domain outputs (F64 canonical, F32 in [0, 2p), fields.cuh).
template <class F>
__global__ void tensor_kernel(const typename F::W* a1, const typename F::W* b1,
                              const typename F::W* a2, const typename F::W* b2,
                              typename F::W* d0, typename F::W* d1, typename F::W* d2,
                              size_t total, int np, int log_n,
                              const typename F::Prime* __restrict__ primes) {
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
       idx += size_t(gridDim.x) * blockDim.x) {
    const typename F::Prime pr = primes[(idx >> log_n) % np];
    const typename F::W x1 = a1[idx], y1 = b1[idx], x2 = a2[idx], y2 = b2[idx];
    d0[idx] = F::mul(y1, y2, pr);
    d2[idx] = F::mul(x1, x2, pr);
    d1[idx] = F::mul_add2(x1, y2, x2, y1, pr);
  }
}

// split region 1 (F32::tensor_split): 8 operand slots -> slots 0..5
__global__ void tensor_split_kernel(uint32_t* __restrict__ r1, size_t slot, int np, int log_n,
                                    const DevPrime32* __restrict__ primes) {
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < slot;
       idx += size_t(gridDim.x) * blockDim.x) {
    const DevPrime32 pr = primes[(idx >> log_n) % np];
    uint32_t v[8];
#pragma unroll
    for (int op = 0; op < 8; ++op) v[op] = r1[op * slot + idx];
    F32::tensor_split(v, pr);
#pragma unroll
    for (int op = 0; op < 6; ++op) r1[op * slot + idx] = v[op];
  }
}

template <class F>
__global__ void evk_kernel(const typename F::W* f, const typename F::W* __restrict__ ea,
                           const typename F::W* __restrict__ eb, typename F::W* ka,
                           typename F::W* __restrict__ kb, size_t total, int np, int log_n,
                           const typename F::Prime* __restrict__ primes) {
  const size_t per = size_t(np) << log_n;  // evk forms are shared by the batch
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
       idx += size_t(gridDim.x) * blockDim.x) {
    const size_t e = idx % per;
    const typename F::Prime pr = primes[e >> log_n];
    const typename F::W x = f[idx];
    ka[idx] = F::mul(x, ea[e], pr);
    kb[idx] = F::mul(x, eb[e], pr);
  }
}

constexpr int kMaxLimbs = 96;  // supports log_q + log_Q up to 6144 bits

__device__ __forceinline__ uint64_t mask_of(int bits) {
  return bits % 64 ? (uint64_t(1) << (bits % 64)) - 1 : ~uint64_t(0);
}

// s (len limbs) += 2^bit, then reduce mod 2^mod_bits (mod_bits <= 64 len).
__device__ __forceinline__ void add_pow2_mod(uint64_t* s, int len, int bit, int mod_bits) {
  uint64_t carry = uint64_t(1) << (bit % 64);
  for (int k = bit / 64; k < len && carry; ++k) {
    const uint64_t v = s[k] + carry;
    carry = v < carry;
    s[k] = v;
  }
  const int top = (mod_bits + 63) / 64;
  if (top <= len) s[top - 1] &= mask_of(mod_bits);
}

// out[0..olen) = (s >> bits), s has len limbs.
__device__ __forceinline__ void shr_limbs(const uint64_t* s, int len, int bits, uint64_t* out,
                                          int olen) {
  const int w = bits / 64, sh = bits % 64;
  for (int k = 0; k < olen; ++k) {
    const uint64_t lo = w + k < len ? s[w + k] : 0;
    const uint64_t hi = w + k + 1 < len ? s[w + k + 1] : 0;
    out[k] = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
  }
}

__global__ void keyswitch_epilogue_kernel(const uint64_t* __restrict__ ks,
                                          const uint64_t* __restrict__ d,
                                          uint64_t* __restrict__ out, size_t total, int log_q,
                                          int log_Q, int log_p) {
  const int L2 = (log_q + log_Q + 63) / 64, L = (log_q + 63) / 64;
  const int Lo = (log_q - log_p + 63) / 64;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    uint64_t s[kMaxLimbs], t[kMaxLimbs];
    const uint64_t* src = ks + i * L2;
    for (int k = 0; k < L2; ++k) s[k] = src[k];
    // R_logQ: (v + 2^(Q-1)) mod 2^(q+Q), >> Q   (poly.cpp:98-115)
    add_pow2_mod(s, L2, log_Q - 1, log_q + log_Q);
    shr_limbs(s, L2, log_Q, t, L);
    t[L - 1] &= mask_of(log_q);
    // + d mod 2^q   (poly.cpp:46-70)
    const uint64_t* dd = d + i * L;
    uint64_t carry = 0;
    for (int k = 0; k < L; ++k) {
      const uint64_t x = t[k] + carry;
      const uint64_t c1 = x < carry;
      const uint64_t y = x + dd[k];
      carry = c1 + (y < x);
      t[k] = y;
    }
    t[L - 1] &= mask_of(log_q);
    // rescale R_logp   (heaan.cpp:328-337)
    add_pow2_mod(t, L, log_p - 1, log_q);
    uint64_t* o = out + i * Lo;
    shr_limbs(t, L, log_p, s, Lo);
    s[Lo - 1] &= mask_of(log_q - log_p);
    for (int k = 0; k < Lo; ++k) o[k] = s[k];
  }
}

__global__ void shift_right_kernel(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                                   size_t total, int log_q, int bits) {
  const int L = (log_q + 63) / 64, Lo = (log_q - bits + 63) / 64;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    uint64_t s[kMaxLimbs], t[kMaxLimbs];
    for (int k = 0; k < L; ++k) s[k] = a[i * L + k];
    add_pow2_mod(s, L, bits - 1, log_q);
    shr_limbs(s, L, bits, t, Lo);
    t[Lo - 1] &= mask_of(log_q - bits);
    for (int k = 0; k < Lo; ++k) out[i * Lo + k] = t[k];
  }
}

// poly_mod_down (poly.cpp:117-127): the low ceil(new_log_q / 64) limbs of
// each coefficient, top limb masked; one thread per output word.
__global__ void mod_down_kernel(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                                size_t words, int L, int Lo, uint64_t top_mask) {
  for (size_t o = blockIdx.x * size_t(blockDim.x) + threadIdx.x; o < words;
       o += size_t(gridDim.x) * blockDim.x) {
    const size_t i = o / Lo;
    const int k = static_cast<int>(o - i * Lo);
    const uint64_t v = a[i * L + k];
    out[o] = k == Lo - 1 ? v & top_mask : v;
  }
}

// BigPoly (rows x cols words, row-major) -> cols x rows, 32 x 32 tiles
// through shared memory (both sides coalesced).
__global__ void word_transpose_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                      int rows, int cols) {
  __shared__ uint64_t tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[y][threadIdx.x] = in[size_t(r) * cols + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[size_t(c) * rows + r] = tile[threadIdx.x][y];
  }
}

// Scheme::mul_by_ternary (heaan.cpp:234-256) on limb-major operands: out =
// sum_j s_j X^(i_j) a mod (X^n + 1, 2^log_q) for a sparse ternary s given
// as nz[j] = 2 i_j + (s_j < 0). One thread per output coefficient d walks
// the limbs low to high; per limb the positive and negative terms
// a[(d - i_j) mod n] (negated once more on the X^n = -1 wrap) are summed in
// 128 bits and the signed difference plus the incoming carry gives the limb
// and the next carry — exact for any nonzero count below 2^62.
__global__ void ternary_mul_kernel(const uint64_t* __restrict__ aT, const int* __restrict__ nz,
                                   int nnz, uint64_t* __restrict__ rT, int n, int L,
                                   uint64_t top_mask) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  __int128 carry = 0;
  for (int k = 0; k < L; ++k) {
    const uint64_t* col = aT + size_t(k) * n;
    unsigned __int128 pos = 0, neg = 0;
    for (int j = 0; j < nnz; ++j) {
      const int e = __ldg(nz + j);
      int src = d - (e >> 1);
      const int wrap = src < 0;
      src += wrap ? n : 0;
      const uint64_t v = col[src];
      const uint64_t m = 0 - uint64_t((e & 1) ^ wrap);  // all ones: a negative term
      pos += v & ~m;
      neg += v & m;
    }
    const __int128 val = static_cast<__int128>(pos) - static_cast<__int128>(neg) + carry;
    uint64_t w = static_cast<uint64_t>(val);
    if (k == L - 1) w &= top_mask;
    rT[size_t(k) * n + d] = w;
    carry = val >> 64;
  }
}

unsigned grid_for(size_t total, int threads) {
  size_t blocks = (total + threads - 1) / threads;
  const size_t cap = 148 * 64;
  return static_cast<unsigned>(blocks < cap ? blocks : cap);
}

}  // namespace

cudaError_t pointwise(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t batch, int np,
                      int log_n, const DevPrime* primes, cudaStream_t st) {
  const size_t total = (batch * np) << log_n;
  pointwise_kernel<<<grid_for(total, 256), 256, 0, st>>>(a, b, out, total, np, log_n, primes);
  return cudaGetLastError();
}

template <class F>
cudaError_t tensor_product(const typename F::W* a1, const typename F::W* b1,
                           const typename F::W* a2, const typename F::W* b2, typename F::W* d0,
                           typename F::W* d1, typename F::W* d2, size_t batch, int np,
                           int log_n, const typename F::Prime* primes, cudaStream_t st) {
  const size_t total = (batch * np) << log_n;
  tensor_kernel<F><<<grid_for(total, 256), 256, 0, st>>>(a1, b1, a2, b2, d0, d1, d2, total, np,
                                                         log_n, primes);
  return cudaGetLastError();
}

cudaError_t tensor_split_product(uint32_t* r1, size_t batch, int np, int log_n,
                                 const DevPrime32* primes, cudaStream_t st) {
  const size_t slot = (batch * np) << log_n;
  tensor_split_kernel<<<grid_for(slot, 256), 256, 0, st>>>(r1, slot, np, log_n, primes);
  return cudaGetLastError();
}

template <class F>
cudaError_t evk_product(const typename F::W* f, const typename F::W* ea, const typename F::W* eb,
                        typename F::W* ka, typename F::W* kb, size_t batch, int np, int log_n,
                        const typename F::Prime* primes, cudaStream_t st) {
  const size_t total = (batch * np) << log_n;
  evk_kernel<F><<<grid_for(total, 256), 256, 0, st>>>(f, ea, eb, ka, kb, total, np, log_n,
                                                      primes);
  return cudaGetLastError();
}

#define HEMUL_POLY_INSTANTIATE(F)                                                             \
  template cudaError_t tensor_product<F>(const F::W*, const F::W*, const F::W*, const F::W*,  \
                                         F::W*, F::W*, F::W*, size_t, int, int,               \
                                         const F::Prime*, cudaStream_t);                      \
  template cudaError_t evk_product<F>(const F::W*, const F::W*, const F::W*, F::W*, F::W*,    \
                                      size_t, int, int, const F::Prime*, cudaStream_t);
HEMUL_POLY_INSTANTIATE(F64)
HEMUL_POLY_INSTANTIATE(F32)
#undef HEMUL_POLY_INSTANTIATE

cudaError_t keyswitch_epilogue(const uint64_t* ks, const uint64_t* d, uint64_t* out, size_t batch,
                               int log_n, int log_q, int log_Q, int log_p, cudaStream_t st) {
  if ((log_q + log_Q + 63) / 64 > kMaxLimbs) return cudaErrorInvalidValue;
  const size_t total = batch << log_n;
  keyswitch_epilogue_kernel<<<grid_for(total, 128), 128, 0, st>>>(ks, d, out, total, log_q,
                                                                   log_Q, log_p);
  return cudaGetLastError();
}

cudaError_t mod_down(const uint64_t* a, uint64_t* out, size_t batch, int log_n, int log_q,
                     int new_log_q, cudaStream_t st) {
  if (new_log_q <= 0 || new_log_q > log_q) return cudaErrorInvalidValue;
  const int L = (log_q + 63) / 64, Lo = (new_log_q + 63) / 64;
  const size_t words = (batch << log_n) * size_t(Lo);
  const int rest = new_log_q - 64 * (Lo - 1);
  const uint64_t top = rest == 64 ? ~uint64_t(0) : (uint64_t(1) << rest) - 1;
  mod_down_kernel<<<grid_for(words, 256), 256, 0, st>>>(a, out, words, L, Lo, top);
  return cudaGetLastError();
}

cudaError_t shift_right(const uint64_t* a, uint64_t* out, size_t batch, int log_n, int log_q,
                        int bits, cudaStream_t st) {
  if ((log_q + 63) / 64 > kMaxLimbs) return cudaErrorInvalidValue;
  const size_t total = batch << log_n;
  shift_right_kernel<<<grid_for(total, 128), 128, 0, st>>>(a, out, total, log_q, bits);
  return cudaGetLastError();
}

cudaError_t word_transpose(const uint64_t* in, uint64_t* out, int rows, int cols,
                           cudaStream_t st) {
  const dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  word_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
  return cudaGetLastError();
}

cudaError_t mul_by_ternary(const uint64_t* aT, const int* nz, int nnz, uint64_t* rT, int log_n,
                           int log_q, cudaStream_t st) {
  const int n = 1 << log_n, L = (log_q + 63) / 64;
  const int rest = log_q - 64 * (L - 1);
  const uint64_t top = rest == 64 ? ~uint64_t(0) : (uint64_t(1) << rest) - 1;
  ternary_mul_kernel<<<(n + 127) / 128, 128, 0, st>>>(aT, nz, nnz, rT, n, L, top);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
