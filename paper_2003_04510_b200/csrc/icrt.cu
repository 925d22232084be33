// Exact inverse CRT: prime-major residues -> coefficients mod 2^T (sm_100a).
//
// Reference: icrt_reordered (proj/core/src/rns.cpp:132-190, 235-290, 395-415):
//   t_j = x_j (P/p_j)^-1 mod p_j ; acc = sum_j t_j (P/p_j) ; fold below P ;
//   centered lift (acc > floor(P/2) -> acc - P) ; reduce mod the target 2^T.
//
// B200 form (bit-identical):
//   v = sum_j t_j H_j - k P with k = rint(sum_j t_j / p_j) computed in fp64.
// sum_j t_j / p_j = k + v/P and the centered v satisfies |v|/P < 1/2 - 2^-s
// (s = the level's slack, >= 4 bits is asserted at level setup), so fp64's
// ~2^-45 error can never move the rounding. Then
//   out = sum_j t_j (H_j mod 2^T) + k ((-P) mod 2^T)   mod 2^T,
// so the MAC width is ceil(T/30) chunks instead of the limbs of P (40->80
// chunks of 30 bits at region 1, N=2^16).
// The accumulation is a small-K integer GEMM S[i][m] = sum_k A[k][i] B[k][m]
// with A = {t_j low 30 bits, t_j high 30 bits, k} and B = {H_j chunks, H_j
// chunks shifted one chunk up, (-P) chunks}; every product is one
// IMAD.WIDE.U32 < 2^60, folded into 128 bits every 16 rows. A final carry
// pass turns the 30-bit column sums into 64-bit limbs.
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "modarith.cuh"

namespace hemul_gpu {

namespace {

constexpr int kCoefs = 32;   // coefficients per CTA
constexpr int kKt = 16;      // B rows per shared-memory tile

// A CTA: 32 coefficients x m_pad chunks; lane -> (coef group = lane % 8,
// chunk group = lane / 8 + 4 * warp); thread tile 4 coefs x 4 chunks.
__global__ void __launch_bounds__(512) icrt_kernel(const uint64_t* __restrict__ rns,
                                                  int log_n, const DevPrime* __restrict__ primes,
                                                  int np, const uint32_t* __restrict__ btab,
                                                  int m_out, int m_pad, int tbits,
                                                  uint64_t* __restrict__ out, IcrtFlags flags) {
  extern __shared__ __align__(16) unsigned char smem[];
  const size_t n = size_t(1) << log_n;
  const int b = blockIdx.y;
  const size_t c0 = size_t(blockIdx.x) * kCoefs;
  const int K = 2 * np + 1;
  uint32_t* A = reinterpret_cast<uint32_t*>(smem);    // [K][kCoefs]
  uint32_t* Bt = A + size_t(K) * kCoefs;              // [kKt][m_pad]
  // ---- t_j = x_j * inv_j mod p_j, split in 30-bit halves ------------------
  for (int idx = threadIdx.x; idx < np * kCoefs; idx += blockDim.x) {
    const int j = idx / kCoefs, c = idx % kCoefs;
    const DevPrime& pr = primes[j];
    const uint64_t x = rns[(size_t(b) * np + j) * n + c0 + c];
    const uint64_t t = shoup_mul(x, pr.inv, pr.inv_q, pr.p);
    A[(2 * j) * kCoefs + c] = static_cast<uint32_t>(t) & 0x3fffffffu;
    A[(2 * j + 1) * kCoefs + c] = static_cast<uint32_t>(t >> 30);
  }
  __syncthreads();
  // ---- k = rint(sum_j t_j / p_j) ------------------------------------------
  if (threadIdx.x < kCoefs) {
    const int c = threadIdx.x;
    double s = 0;
    for (int j = 0; j < np; ++j) {
      const uint64_t t = uint64_t(A[(2 * j) * kCoefs + c]) |
                         (uint64_t(A[(2 * j + 1) * kCoefs + c]) << 30);
      s += static_cast<double>(t) * primes[j].inv_p_dbl;
    }
    const double k = rint(s);
    A[(2 * np) * kCoefs + c] = static_cast<uint32_t>(k);
    if (flags.count && fabs(s - k) > 0.25) {
      const unsigned slot = atomicAdd(flags.count, 1u);
      if (slot < flags.capacity) flags.ids[slot] = unsigned(size_t(b) * n + c0 + c);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane & 7;                        // coefficient group (4 coefs)
  const int mg = (lane >> 3) + 4 * warp;          // chunk group (4 chunks)
  const bool active = 4 * mg < m_pad;
  uint64_t lo[4][4], hi[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) lo[i][q] = hi[i][q] = 0;
  for (int kb = 0; kb < K; kb += kKt) {
    const int ke = min(kb + kKt, K);
    __syncthreads();
    for (int idx = threadIdx.x; idx < (ke - kb) * m_pad; idx += blockDim.x)
      Bt[idx] = btab[size_t(kb) * m_pad + idx];
    __syncthreads();
    if (active) {
      uint64_t acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = 0;
      for (int k = kb; k < ke; ++k) {
        const uint4 a = *reinterpret_cast<const uint4*>(A + size_t(k) * kCoefs + 4 * cg);
        const uint4 w = *reinterpret_cast<const uint4*>(Bt + size_t(k - kb) * m_pad + 4 * mg);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w};
        const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] += wide(av[i], wv[q]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t s = lo[i][q] + acc[i][q];
          hi[i][q] += s < acc[i][q];
          lo[i][q] = s;
        }
    }
  }
  __syncthreads();
  // ---- column sums to shared memory, then a carry pass per coefficient ----
  uint64_t* Slo = reinterpret_cast<uint64_t*>(smem);            // [kCoefs][m_pad]
  uint32_t* Shi = reinterpret_cast<uint32_t*>(Slo + size_t(kCoefs) * m_pad);
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = 4 * cg + i, m = 4 * mg + q;
        Slo[size_t(c) * m_pad + m] = lo[i][q];
        Shi[size_t(c) * m_pad + m] = static_cast<uint32_t>(hi[i][q]);
      }
  }
  __syncthreads();
  const int tl = (tbits + 63) / 64;
  uint64_t* packed = reinterpret_cast<uint64_t*>(Shi + size_t(kCoefs) * m_pad);  // [kCoefs][tl]
  if (threadIdx.x < kCoefs) {
    const int c = threadIdx.x;
    // carry = (chi:clo), 30-bit digit emitted each step, packed into limbs
    uint64_t clo = 0, chi = 0, word = 0;
    int fill = 0, limb = 0;
    for (int m = 0; m < m_out; ++m) {
      const uint64_t slo = Slo[size_t(c) * m_pad + m];
      const uint64_t shi = Shi[size_t(c) * m_pad + m];
      const uint64_t vlo = slo + clo;
      const uint64_t vhi = shi + chi + (vlo < slo);
      const uint64_t digit = vlo & 0x3fffffffu;
      clo = (vlo >> 30) | (vhi << 34);
      chi = vhi >> 30;
      word |= digit << fill;
      fill += 30;
      if (fill >= 64) {
        if (limb < tl) packed[size_t(c) * tl + limb] = word;
        ++limb;
        fill -= 64;
        word = fill > 0 ? digit >> (30 - fill) : 0;
      }
    }
    if (fill > 0 && limb < tl) packed[size_t(c) * tl + limb++] = word;
    while (limb < tl) packed[size_t(c) * tl + limb++] = 0;
    if (tbits % 64) packed[size_t(c) * tl + tl - 1] &= (uint64_t(1) << (tbits % 64)) - 1;
  }
  __syncthreads();
  uint64_t* dst = out + (size_t(b) * n + c0) * tl;
  for (int idx = threadIdx.x; idx < kCoefs * tl; idx += blockDim.x) dst[idx] = packed[idx];
}

// Exact reconstruction of the flagged coefficients, the reference's own
// algorithm (rns.cpp:148-169, 192-233): acc = sum_j t_j H_j, fold below P,
// centered lift, mod 2^T. One thread per flagged coefficient.
constexpr int kFixMaxLimbs = 136;
__global__ void icrt_fixup_kernel(const uint64_t* __restrict__ rns, int log_n,
                                  const DevPrime* __restrict__ primes, int np,
                                  const uint64_t* __restrict__ hat, const uint64_t* __restrict__ P,
                                  const uint64_t* __restrict__ halfP, int pl, int tbits,
                                  uint64_t* __restrict__ out, IcrtFlags flags) {
  const unsigned cnt = min(*flags.count, flags.capacity);
  const size_t n = size_t(1) << log_n;
  const int tl = (tbits + 63) / 64;
  const int al = pl + 2;
  for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < cnt; f += gridDim.x * blockDim.x) {
    const size_t id = flags.ids[f];
    const size_t b = id / n, i = id % n;
    uint64_t acc[kFixMaxLimbs];
    for (int k = 0; k < al; ++k) acc[k] = 0;
    for (int j = 0; j < np; ++j) {
      const DevPrime& pr = primes[j];
      const uint64_t t = shoup_mul(rns[(b * np + j) * n + i], pr.inv, pr.inv_q, pr.p);
      const uint64_t* h = hat + size_t(j) * pl;
      uint64_t carry = 0;
      for (int k = 0; k < al; ++k) {
        const uint64_t hk = k < pl ? h[k] : 0;
        const uint64_t lo = t * hk, hi = __umul64hi(t, hk);
        const uint64_t s1 = acc[k] + lo;
        const uint64_t c1 = s1 < lo;
        const uint64_t s2 = s1 + carry;
        carry = hi + c1 + (s2 < s1);
        acc[k] = s2;
      }
    }
    auto geq = [&](const uint64_t* x) {  // acc >= x (x has pl limbs)
      for (int k = al - 1; k >= 0; --k) {
        const uint64_t xk = k < pl ? x[k] : 0;
        if (acc[k] != xk) return acc[k] > xk;
      }
      return true;
    };
    while (geq(P)) {
      uint64_t borrow = 0;
      for (int k = 0; k < al; ++k) {
        const uint64_t xk = (k < pl ? P[k] : 0) + borrow;
        const uint64_t nb = (xk < borrow) | (acc[k] < xk);
        acc[k] -= xk;
        borrow = nb;
      }
    }
    bool neg = geq(halfP);
    if (neg) {  // acc > floor(P/2)  <=>  acc >= floor(P/2) + 1; equality impossible for odd P
      bool eq = true;
      for (int k = 0; k < al && eq; ++k) eq = acc[k] == (k < pl ? halfP[k] : 0);
      neg = !eq;
    }
    uint64_t* o = out + (b * n + i) * tl;
    uint64_t borrow = 0;
    for (int k = 0; k < tl; ++k) {
      const uint64_t a = k < al ? acc[k] : 0;
      if (neg) {
        const uint64_t xk = (k < pl ? P[k] : 0) + borrow;
        const uint64_t nb = (xk < borrow) | (a < xk);
        o[k] = a - xk;
        borrow = nb;
      } else {
        o[k] = a;
      }
    }
    if (tbits % 64) o[tl - 1] &= (uint64_t(1) << (tbits % 64)) - 1;
  }
}

size_t icrt_smem(int np, int m_pad, int tbits) {
  const int K = 2 * np + 1;
  const size_t main = size_t(K) * kCoefs * 4 + size_t(kKt) * m_pad * 4;
  const int tl = (tbits + 63) / 64;
  const size_t epi = size_t(kCoefs) * m_pad * 12 + size_t(kCoefs) * tl * 8;
  return main > epi ? main : epi;
}

}  // namespace

cudaError_t icrt_setup_attributes() {
  return cudaFuncSetAttribute(icrt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024);
}

cudaError_t icrt(const uint64_t* rns, size_t batch, int log_n, const DevPrime* primes, int np,
                 const IcrtTable& t, uint64_t* out, cudaStream_t st, const IcrtFlags* flags) {
  const size_t n = size_t(1) << log_n;
  if (n < kCoefs) return cudaErrorInvalidValue;
  int threads = 8 * (t.m_pad / 4);  // one thread per (coef group, chunk group)
  threads = (threads + 31) / 32 * 32;
  if (threads > 512) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(n / kCoefs), static_cast<unsigned>(batch));
  IcrtFlags f;
  if (flags) {
    if (t.p_limbs + 2 > kFixMaxLimbs) return cudaErrorInvalidValue;
    f = *flags;
    cudaError_t e = cudaMemsetAsync(f.count, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
  }
  icrt_kernel<<<grid, threads, icrt_smem(np, t.m_pad, t.target_bits), st>>>(
      rns, log_n, primes, np, t.btab, t.m_out, t.m_pad, t.target_bits, out, f);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !flags) return e;
  icrt_fixup_kernel<<<64, 64, 0, st>>>(rns, log_n, primes, np, t.hat, t.big_p, t.half_p,
                                       t.p_limbs, t.target_bits, out, f);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
