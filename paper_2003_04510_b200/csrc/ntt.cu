// Batched negacyclic NTT / iNTT over prime-major RNS rows (sm_100a).
//
// Reference: ntt_forward / ntt_inverse (proj/core/src/ntt.cpp:59-137,
// 153-197). Forward = Cooley-Tukey, natural in -> bit-reversed out; level L
// (2^L groups, half-distance t = n / 2^(L+1)) uses tw[2^L + g] for group g.
// Inverse = Gentleman-Sande from the last level back to level 0 with itw,
// then x n^-1 (folded here into level 0's butterfly).
//
// B200 mapping. One transform of n = 2^logN 64-bit residues is split into
// two memory passes (2^s1 x 2^s2):
//   pass A: levels [0, s1) on 2^s1-point columns at stride 2^s2, a CTA owns
//           C adjacent columns (C x 8 B contiguous per global row);
//   pass B: levels [s1, logN) on contiguous 2^s2-point blocks.
// Inside a pass the block sits in shared memory and each thread runs radix-8
// butterfly units (3 levels on 8 registers) between barriers, so shared
// memory is touched once per 3 levels. Values stay lazy in [0, 4p) (forward)
// or [0, 2p) (inverse) and are canonicalised at the end, so every output is
// bit-identical to the reference's canonical residues (ntt.hpp:12-16, all
// variants bit-identical, test_ntt.cpp:120-165).
#include <cuda_runtime.h>

#include "device_tables.cuh"
#include "kernels.hpp"
#include "modarith.cuh"

namespace hemul_gpu {

namespace {

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

struct PassGeom {
  int S;        // levels in this pass
  int st0;      // first global level
  int log_n;
  int tlast;    // element stride inside a sub-problem = n >> (st0 + S)
  int C;        // sub-problems per CTA
  bool strided; // pass A layout (columns) vs pass B (contiguous blocks)
};

// Shared-memory slot of element e of the CTA's sub-problem c.
__device__ __forceinline__ int sidx(const PassGeom& g, int e, int c) {
  return g.strided ? e * g.C + c : (c << g.S) + e;
}

// Decomposes unit index `uid` of a level group (levels l..l+k-1) into
// (sub-problem c, group h, offset u).
__device__ __forceinline__ void unit_coords(const PassGeom& g, int l, int k, int uid, int& c,
                                            int& h, int& u) {
  const int ubits = g.S - l - k;  // log2 of units per group
  if (g.strided) {
    c = uid % g.C;
    const int rest = uid / g.C;
    u = rest & ((1 << ubits) - 1);
    h = rest >> ubits;
  } else {
    u = uid & ((1 << ubits) - 1);
    h = (uid >> ubits) & ((1 << l) - 1);
    c = uid >> (ubits + l);
  }
}

// One pass of a forward (INV=false) or inverse (INV=true) transform.
// grid.x = CTA index within the row, grid.y = row (batch x prime).
// LAST: this pass produces the final output (canonicalise / n^-1 fold).
template <bool INV>
__global__ void __launch_bounds__(512) ntt_pass_kernel(uint64_t* __restrict__ data,
                                                      const Twiddle* __restrict__ tw,
                                                      const DevPrime* __restrict__ primes, int np,
                                                      PassGeom g, int last) {
  extern __shared__ uint64_t sbuf[];
  const int row = blockIdx.y;
  const int j = row % np;
  const DevPrime pr = primes[j];
  const uint64_t p = pr.p, p2 = 2 * p, negp = 0 - p;
  const size_t n = size_t(1) << g.log_n;
  uint64_t* rowp = data + size_t(row) * n;
  const Twiddle* twr = tw + size_t(j) * n;
  const int elems = g.C << g.S;
  // global offset of the CTA's first sub-problem
  const int sp0 = blockIdx.x * g.C;
  const int m0 = 1 << g.st0;
  // ---- load ---------------------------------------------------------------
  if (g.strided) {
    // sub-problems sp0..sp0+C-1 are columns r (g = 0): element e at r + e*tlast
    for (int idx = threadIdx.x; idx < elems; idx += blockDim.x) {
      const int e = idx / g.C, c = idx % g.C;
      sbuf[idx] = rowp[size_t(e) * g.tlast + sp0 + c];
    }
  } else {
    const uint64_t* src = rowp + (size_t(sp0) << g.S);
    for (int idx = threadIdx.x; idx < elems; idx += blockDim.x) sbuf[idx] = src[idx];
  }
  __syncthreads();
  // ---- level groups -------------------------------------------------------
  // forward: l = 0, 3, 6, ... ; inverse walks the same groups in reverse order
  int ngroups = (g.S + 2) / 3;
  for (int gi = 0; gi < ngroups; ++gi) {
    const int grp = INV ? ngroups - 1 - gi : gi;
    const int l = grp * 3;
    const int k = min(3, g.S - l);
    const int units = elems >> k;
    for (int uid = threadIdx.x; uid < units; uid += blockDim.x) {
      int c, h, u;
      unit_coords(g, l, k, uid, c, h, u);
      // sub-problem global group index (pass A: gsub = 0)
      const int gsub = g.strided ? 0 : sp0 + c;
      const int e0 = (h << (g.S - l)) + u;
      const int stride = 1 << (g.S - l - k);
      uint64_t x[8];
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) x[v] = sbuf[sidx(g, e0 + v * stride, c)];
      if (!INV) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          if (i < k) {
            const int L = g.st0 + l + i;  // global level
            const int half = 1 << (k - i - 1);
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
              if (blk < (1 << i)) {
                const int hh = (h << i) + blk;  // group inside sub-problem at level l+i
                const Twiddle w = twr[(size_t(m0) << (l + i)) + (size_t(gsub) << (l + i)) + hh];
                (void)L;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (q < half) {
                    const int a = blk * 2 * half + q;
                    ct_bfly(x[a], x[a + half], w, p2, negp);
                  }
              }
            }
          }
        }
        if (last && grp == ngroups - 1) {
#pragma unroll
          for (int v = 0; v < 8; ++v)
            if (v < (1 << k)) x[v] = reduce_4p(x[v], p);
        }
      } else {
#pragma unroll
        for (int ii = 2; ii >= 0; --ii) {
          if (ii < k) {
            const int L = g.st0 + l + ii;
            const int half = 1 << (k - ii - 1);
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
              if (blk < (1 << ii)) {
                const int hh = (h << ii) + blk;
                if (L == 0 && last) {
                  // level 0 of the inverse with n^-1 folded in: a' = (u+v) n^-1,
                  // b' = (u-v) itw[1] n^-1, outputs canonical.
#pragma unroll
                  for (int q = 0; q < 4; ++q)
                    if (q < half) {
                      const int a = blk * 2 * half + q;
                      const uint64_t uu = x[a], vv = x[a + half];
                      x[a] = shoup_mul(uu + vv, pr.ninv, pr.ninv_q, p);
                      x[a + half] = shoup_mul(uu + p2 - vv, pr.w1n, pr.w1n_q, p);
                    }
                } else {
                  const Twiddle w = twr[(size_t(m0) << (l + ii)) + (size_t(gsub) << (l + ii)) + hh];
#pragma unroll
                  for (int q = 0; q < 4; ++q)
                    if (q < half) {
                      const int a = blk * 2 * half + q;
                      gs_bfly(x[a], x[a + half], w, p2, negp);
                    }
                }
              }
            }
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) sbuf[sidx(g, e0 + v * stride, c)] = x[v];
    }
    __syncthreads();
  }
  // ---- store --------------------------------------------------------------
  if (g.strided) {
    for (int idx = threadIdx.x; idx < elems; idx += blockDim.x) {
      const int e = idx / g.C, c = idx % g.C;
      rowp[size_t(e) * g.tlast + sp0 + c] = sbuf[idx];
    }
  } else {
    uint64_t* dst = rowp + (size_t(sp0) << g.S);
    for (int idx = threadIdx.x; idx < elems; idx += blockDim.x) dst[idx] = sbuf[idx];
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

cudaError_t launch_pass(bool inv, uint64_t* data, const Twiddle* tw, const DevPrime* primes, int np,
                        size_t rows, int log_n, int st0, int S, bool strided, bool last,
                        cudaStream_t st) {
  PassGeom g;
  g.S = S;
  g.st0 = st0;
  g.log_n = log_n;
  g.tlast = 1 << (log_n - st0 - S);
  g.strided = strided;
  // aim at ~4096 elements (32 KB) per CTA
  const int per = 1 << S;
  const int subproblems = strided ? g.tlast : (1 << st0);
  int C = per >= 4096 ? 1 : 4096 / per;
  if (C > subproblems) C = subproblems;
  g.C = C;
  const int elems = C * per;
  int threads = elems / 8;
  if (threads < 32) threads = 32;
  if (threads > 512) threads = 512;
  dim3 grid(subproblems / C, static_cast<unsigned>(rows));
  const size_t smem = sizeof(uint64_t) * elems;
  if (inv)
    ntt_pass_kernel<true><<<grid, threads, smem, st>>>(data, tw, primes, np, g, last);
  else
    ntt_pass_kernel<false><<<grid, threads, smem, st>>>(data, tw, primes, np, g, last);
  return cudaGetLastError();
}

}  // namespace

cudaError_t ntt_setup_attributes() {
  cudaError_t e = cudaFuncSetAttribute(ntt_pass_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(ntt_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              64 * 1024);
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
  if (pass == 0) return launch_pass(false, data, tw, primes, np, rows, log_n, 0, s1, true, s2 == 0, st);
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
