// Batched negacyclic NTT / iNTT over prime-major RNS rows (sm_100a).
//
// Reference: ntt_forward / ntt_inverse (proj/core/src/ntt.cpp:59-137,
// 153-197). Forward = Cooley-Tukey, natural in -> bit-reversed out; level L
// (2^L groups, half-distance t = n / 2^(L+1)) uses tw[2^L + g] for group g.
// Inverse = Gentleman-Sande from the last level back to level 0 with itw,
// then x n^-1 (folded here into level 0's butterfly).
//
// B200 mapping. One transform of n = 2^logN 64-bit residues is split into
// two memory passes (2^s1 x 2^s2, s1 = ceil(logN/2)):
//   pass A: levels [0, s1) on 2^s1-point columns at stride 2^s2; a CTA owns
//           C adjacent columns (C x 8 B contiguous per global row);
//   pass B: levels [s1, logN) on contiguous 2^s2-point blocks.
// Inside a pass the CTA's 4096 residues sit in shared memory and each thread
// holds 8 of them in registers, running radix-8 butterfly units (3 levels)
// between barriers, so shared memory is touched once per 3 levels. The pass
// size S is a template parameter: every level group, unit and register index
// is resolved at compile time (no local memory). Values stay lazy in [0, 4p)
// (forward) / [0, 2p) (inverse) and are canonicalised at the end, so every
// output is bit-identical to the reference's canonical residues (ntt.hpp:
// 12-16, all variants bit-identical, test_ntt.cpp:120-165).
//
// Rows are visited prime-major (all batch rows of prime j back to back), so a
// prime's twiddle table is streamed from HBM once per launch and re-read from
// L2 by the other rows.
#include <cuda_runtime.h>

#include "device_tables.cuh"
#include "kernels.hpp"
#include "modarith.cuh"

namespace hemul_gpu {

namespace {

constexpr int kPassElems = 4096;  // residues per CTA (32 KB of shared memory)

// Lazy Cooley-Tukey butterfly: a, b in [0, 4p) -> [0, 4p) (Harvey).
__device__ __forceinline__ void ct_bfly(uint64_t& a, uint64_t& b, const Twiddle w, uint64_t p2,
                                        uint64_t negp) {
  const uint64_t u = csub(a, p2);
  const uint64_t v = csub(shoup_mul_4p(b, w.w, w.wq, negp), p2);
  a = u + v;
  b = u + p2 - v;
}

// Lazy Gentleman-Sande butterfly: a, b in [0, 2p) -> [0, 2p).
__device__ __forceinline__ void gs_bfly(uint64_t& a, uint64_t& b, const Twiddle w, uint64_t p2,
                                        uint64_t negp) {
  const uint64_t u = a, v = b;
  a = csub(u + v, p2);
  b = csub(shoup_mul_4p(u + p2 - v, w.w, w.wq, negp), p2);
}

struct PassArgs {
  uint64_t* data;
  const Twiddle* tw;
  const DevPrime* primes;
  int np;
  int log_n;
  int st0;        // first global level of the pass
  int log_c;      // log2 of sub-problems per CTA
  int rows_per_prime;
  int last;       // final pass: canonicalise (fwd) / fold n^-1 (inv)
};

// One pass of S levels. STRIDED: pass A layout (sub-problems are columns at
// stride tlast); else pass B (contiguous blocks of 2^S).
template <int S, bool STRIDED, bool INV>
__global__ void __launch_bounds__(512) ntt_pass_kernel(PassArgs a) {
  extern __shared__ uint64_t sbuf[];
  constexpr int NG = (S + 2) / 3;  // level groups
  // prime-major traversal: blockIdx.y = j * rows_per_prime + b (row-major
  // when the rows are not whole prime sets)
  int j, row;
  if (a.rows_per_prime) {
    j = blockIdx.y / a.rows_per_prime;
    row = (blockIdx.y - j * a.rows_per_prime) * a.np + j;
  } else {
    row = blockIdx.y;
    j = row % a.np;
  }
  const DevPrime& pr = a.primes[j];
  const uint64_t p = pr.p, p2 = 2 * p, negp = 0 - p;
  const size_t n = size_t(1) << a.log_n;
  uint64_t* rowp = a.data + size_t(row) * n;
  const Twiddle* twr = a.tw + size_t(j) * n;
  const int C = 1 << a.log_c;
  const int elems = C << S;
  const int tlast = 1 << (a.log_n - a.st0 - S);
  const int sp0 = blockIdx.x << a.log_c;  // first sub-problem of the CTA
  const int m0 = 1 << a.st0;
  const int T = blockDim.x;               // = elems / 8
  // ---- load ---------------------------------------------------------------
  if (STRIDED) {
    for (int idx = threadIdx.x; idx < elems; idx += T) {
      const int e = idx >> a.log_c, c = idx & (C - 1);
      sbuf[idx] = rowp[size_t(e) * tlast + sp0 + c];
    }
  } else {
    const uint64_t* src = rowp + (size_t(sp0) << S);
    for (int idx = threadIdx.x; idx < elems; idx += T) sbuf[idx] = src[idx];
  }
  __syncthreads();
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    const int grp = INV ? NG - 1 - gi : gi;
    const int l = 3 * grp;
    const int k = S - l < 3 ? S - l : 3;   // levels in this group
    const int ubits = S - l - k;           // log2 of units per group
    const int per = 8 >> k;                // units per thread
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q >= per) break;
      const int uid = threadIdx.x + q * T;
      int c, h, u;
      if (STRIDED) {
        c = uid & (C - 1);
        const int rest = uid >> a.log_c;
        u = rest & ((1 << ubits) - 1);
        h = rest >> ubits;
      } else {
        u = uid & ((1 << ubits) - 1);
        h = (uid >> ubits) & ((1 << l) - 1);
        c = uid >> (ubits + l);
      }
      const int gsub = STRIDED ? 0 : sp0 + c;
      const int e0 = (h << (S - l)) + u;
      const int stride = 1 << ubits;
      uint64_t x[8];
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) {
          const int e = e0 + v * stride;
          x[v] = sbuf[STRIDED ? (e << a.log_c) + c : (c << S) + e];
        }
      if (!INV) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          if (i < k) {
            const int half = 1 << (k - i - 1);
            const size_t tb = (size_t(m0 + gsub) << (l + i)) + (size_t(h) << i);
#pragma unroll
            for (int blk = 0; blk < 4; ++blk)
              if (blk < (1 << i)) {
                const Twiddle w = twr[tb + blk];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                  if (r < half)
                    ct_bfly(x[blk * 2 * half + r], x[blk * 2 * half + r + half], w, p2, negp);
              }
          }
        }
        if (a.last && grp == NG - 1) {
#pragma unroll
          for (int v = 0; v < 8; ++v)
            if (v < (1 << k)) x[v] = reduce_4p(x[v], p);
        }
      } else {
#pragma unroll
        for (int ii = 2; ii >= 0; --ii) {
          if (ii < k) {
            const int half = 1 << (k - ii - 1);
            const int L = a.st0 + l + ii;
            const size_t tb = (size_t(m0 + gsub) << (l + ii)) + (size_t(h) << ii);
#pragma unroll
            for (int blk = 0; blk < 4; ++blk)
              if (blk < (1 << ii)) {
                if (L == 0 && a.last) {
                  // level 0 with n^-1 folded in: a' = (u+v) n^-1,
                  // b' = (u-v) itw[1] n^-1, outputs canonical
#pragma unroll
                  for (int r = 0; r < 4; ++r)
                    if (r < half) {
                      const int i0 = blk * 2 * half + r;
                      const uint64_t uu = x[i0], vv = x[i0 + half];
                      x[i0] = shoup_mul(uu + vv, pr.ninv, pr.ninv_q, p);
                      x[i0 + half] = shoup_mul(uu + p2 - vv, pr.w1n, pr.w1n_q, p);
                    }
                } else {
                  const Twiddle w = twr[tb + blk];
#pragma unroll
                  for (int r = 0; r < 4; ++r)
                    if (r < half)
                      gs_bfly(x[blk * 2 * half + r], x[blk * 2 * half + r + half], w, p2, negp);
                }
              }
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) {
          const int e = e0 + v * stride;
          sbuf[STRIDED ? (e << a.log_c) + c : (c << S) + e] = x[v];
        }
    }
    __syncthreads();
  }
  // ---- store --------------------------------------------------------------
  if (STRIDED) {
    for (int idx = threadIdx.x; idx < elems; idx += T) {
      const int e = idx >> a.log_c, c = idx & (C - 1);
      rowp[size_t(e) * tlast + sp0 + c] = sbuf[idx];
    }
  } else {
    uint64_t* dst = rowp + (size_t(sp0) << S);
    for (int idx = threadIdx.x; idx < elems; idx += T) dst[idx] = sbuf[idx];
  }
}

void split_levels(int log_n, int& s1, int& s2) {
  if (log_n <= 11) {
    s1 = log_n;
    s2 = 0;
  } else {
    s1 = (log_n + 1) / 2;
    s2 = log_n - s1;
  }
}

template <int S, bool STRIDED, bool INV>
cudaError_t launch_s(const PassArgs& a, size_t rows, int C, cudaStream_t st) {
  const int subproblems = STRIDED ? (1 << (a.log_n - a.st0 - S)) : (1 << a.st0);
  dim3 grid(subproblems / C, static_cast<unsigned>(rows));
  const int threads = (C << S) / 8;
  ntt_pass_kernel<S, STRIDED, INV><<<grid, threads, sizeof(uint64_t) * (C << S), st>>>(a);
  return cudaGetLastError();
}

template <bool STRIDED, bool INV>
cudaError_t launch_any(int S, const PassArgs& a, size_t rows, int C, cudaStream_t st) {
  switch (S) {
    case 3: return launch_s<3, STRIDED, INV>(a, rows, C, st);
    case 4: return launch_s<4, STRIDED, INV>(a, rows, C, st);
    case 5: return launch_s<5, STRIDED, INV>(a, rows, C, st);
    case 6: return launch_s<6, STRIDED, INV>(a, rows, C, st);
    case 7: return launch_s<7, STRIDED, INV>(a, rows, C, st);
    case 8: return launch_s<8, STRIDED, INV>(a, rows, C, st);
    case 9: return launch_s<9, STRIDED, INV>(a, rows, C, st);
    case 10: return launch_s<10, STRIDED, INV>(a, rows, C, st);
    case 11: return launch_s<11, STRIDED, INV>(a, rows, C, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pass(bool inv, uint64_t* data, const Twiddle* tw, const DevPrime* primes, int np,
                        size_t rows, int log_n, int st0, int S, bool strided, bool last,
                        cudaStream_t st) {
  const int rpp = rows % np ? 0 : static_cast<int>(rows / np);
  PassArgs a{data, tw, primes, np, log_n, st0, 0, rpp, last ? 1 : 0};
  const int subproblems = strided ? (1 << (log_n - st0 - S)) : (1 << st0);
  int C = (1 << S) >= kPassElems ? 1 : kPassElems >> S;
  if (C > subproblems) C = subproblems;
  if ((C << S) / 8 > 512 || (C << S) < 8) return cudaErrorInvalidValue;
  while ((1 << a.log_c) < C) ++a.log_c;
  if (strided)
    return inv ? launch_any<true, true>(S, a, rows, C, st)
               : launch_any<true, false>(S, a, rows, C, st);
  return inv ? launch_any<false, true>(S, a, rows, C, st)
             : launch_any<false, false>(S, a, rows, C, st);
}

template <int S, bool STRIDED, bool INV>
cudaError_t attr_s() {
  return cudaFuncSetAttribute(ntt_pass_kernel<S, STRIDED, INV>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
}

template <bool STRIDED, bool INV>
cudaError_t attr_all() {
  cudaError_t e = cudaSuccess;
  if ((e = attr_s<3, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<4, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<5, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<6, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<7, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<8, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<9, STRIDED, INV>()) != cudaSuccess) return e;
  if ((e = attr_s<10, STRIDED, INV>()) != cudaSuccess) return e;
  return attr_s<11, STRIDED, INV>();
}

}  // namespace

cudaError_t ntt_setup_attributes() {
  cudaError_t e;
  if ((e = attr_all<true, false>()) != cudaSuccess) return e;
  if ((e = attr_all<true, true>()) != cudaSuccess) return e;
  if ((e = attr_all<false, false>()) != cudaSuccess) return e;
  return attr_all<false, true>();
}

int ntt_num_passes(int log_n) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  return s2 == 0 ? 1 : 2;
}

cudaError_t ntt_forward_pass(int pass, uint64_t* data, size_t rows, int np, int log_n,
                             const Twiddle* tw, const DevPrime* primes, cudaStream_t st) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  if (pass == 0)
    return launch_pass(false, data, tw, primes, np, rows, log_n, 0, s1, true, s2 == 0, st);
  return launch_pass(false, data, tw, primes, np, rows, log_n, s1, s2, false, true, st);
}

cudaError_t ntt_inverse_pass(int pass, uint64_t* data, size_t rows, int np, int log_n,
                             const Twiddle* itw, const DevPrime* primes, cudaStream_t st) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  if (pass == 0 && s2 > 0)
    return launch_pass(true, data, itw, primes, np, rows, log_n, s1, s2, false, false, st);
  return launch_pass(true, data, itw, primes, np, rows, log_n, 0, s1, true, true, st);
}

cudaError_t ntt_forward(uint64_t* data, size_t rows, int np, int log_n, const Twiddle* tw,
                        const DevPrime* primes, cudaStream_t st, int* launches) {
  for (int pass = 0; pass < ntt_num_passes(log_n); ++pass) {
    cudaError_t e = ntt_forward_pass(pass, data, rows, np, log_n, tw, primes, st);
    ++*launches;
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t ntt_inverse(uint64_t* data, size_t rows, int np, int log_n, const Twiddle* itw,
                        const DevPrime* primes, cudaStream_t st, int* launches) {
  for (int pass = 0; pass < ntt_num_passes(log_n); ++pass) {
    cudaError_t e = ntt_inverse_pass(pass, data, rows, np, log_n, itw, primes, st);
    ++*launches;
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace hemul_gpu
