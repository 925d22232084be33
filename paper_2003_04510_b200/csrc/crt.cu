// Forward CRT: big-integer coefficients -> prime-major residues (sm_100a).
//
// Reference: crt_forward / crt_kernel<64> (proj/core/src/rns.cpp:43-106,
// 331-358): r_j(i) = sum_k a_{i,k} (2^64k mod p_j) mod p_j with a 3-word
// accumulator. The result is the canonical a_i mod p_j, so any exact method
// is bit-identical.
//
// B200 form: a small-K integer GEMM on the IMAD.WIDE pipe. A coefficient is
// re-cut into 30-bit chunks c_m (m < M = ceil(bits/30)) and every weight
// u_{j,m} = 2^(30m) mod p_j into two 30-bit halves, so each partial product
// c_m * half < 2^60 is ONE IMAD.WIDE.U32 and 16 of them accumulate in a u64
// without overflow; every 16 chunks the u64 is folded into a 128-bit sum.
//   C[i][2j+h] = sum_m c_m(i) * half_h(u_{j,m})
//   a_i mod p_j = (C[i][2j] + 2^30 C[i][2j+1]) mod p_j
// Tiling: a CTA owns 128 coefficients (their chunks staged once in shared
// memory) and walks the primes 16 at a time; a warp owns 2 primes (4 weight
// columns, broadcast loads) and a lane owns 4 coefficients (one LDS.128), so
// each lane issues 16 IMAD.WIDE per 2 shared loads. Output rows are written
// prime-major directly (no transpose; cf. rns_transpose, rns.cpp:303-311).
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "modarith.cuh"

namespace hemul_gpu {

namespace {

constexpr int kCoefs = 128;             // coefficients per CTA
constexpr int kWarps = 8;               // 8 warps x 2 primes = 16 primes per tile
constexpr int kCols = 2 * kCrtPrimesPerTile;  // 32 weight columns per tile

__device__ __forceinline__ uint32_t chunk30(const uint64_t* limbs, int nlimbs, int m) {
  const int bit = 30 * m;
  const int k = bit >> 6, off = bit & 63;
  uint64_t v = k < nlimbs ? limbs[k] >> off : 0;
  if (off > 34 && k + 1 < nlimbs) v |= limbs[k + 1] << (64 - off);
  return static_cast<uint32_t>(v) & 0x3fffffffu;
}

__global__ void __launch_bounds__(256) crt_kernel(const uint64_t* __restrict__ poly, int limbs,
                                                 int log_n, const uint32_t* __restrict__ wtab,
                                                 int M, int np_pad,
                                                 const DevPrime* __restrict__ primes, int np,
                                                 uint64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const size_t n = size_t(1) << log_n;
  const int b = blockIdx.y;
  const size_t c0 = size_t(blockIdx.x) * kCoefs;
  uint32_t* A = reinterpret_cast<uint32_t*>(smem);                 // [M][kCoefs]
  uint32_t* W = A + size_t(M) * kCoefs;                            // [M][kCols]
  uint64_t* raw = reinterpret_cast<uint64_t*>(W + size_t(M) * kCols);  // [kCoefs][limbs]
  // stage the CTA's limbs (contiguous in the BigPoly layout), then re-cut
  const uint64_t* src = poly + (size_t(b) * n + c0) * limbs;
  for (int idx = threadIdx.x; idx < kCoefs * limbs; idx += blockDim.x) raw[idx] = src[idx];
  __syncthreads();
  for (int idx = threadIdx.x; idx < kCoefs * M; idx += blockDim.x) {
    const int m = idx / kCoefs, c = idx % kCoefs;
    A[idx] = chunk30(raw + size_t(c) * limbs, limbs, m);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tiles = np_pad / kCrtPrimesPerTile;
  for (int tile = 0; tile < tiles; ++tile) {
    __syncthreads();
    // weight tile: rows m, columns [tile*kCols, +kCols)
    for (int idx = threadIdx.x; idx < M * kCols; idx += blockDim.x) {
      const int m = idx / kCols, col = idx % kCols;
      W[idx] = wtab[size_t(m) * 2 * np_pad + tile * kCols + col];
    }
    __syncthreads();
    uint64_t lo[4][4], hi[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) lo[i][q] = hi[i][q] = 0;
    for (int mb = 0; mb < M; mb += 16) {
      uint64_t acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = 0;
      const int me = min(mb + 16, M);
      for (int m = mb; m < me; ++m) {
        const uint4 a = *reinterpret_cast<const uint4*>(A + size_t(m) * kCoefs + 4 * lane);
        const uint4 w = *reinterpret_cast<const uint4*>(W + size_t(m) * kCols + 4 * warp);
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
    // epilogue: 2 primes x 4 coefficients
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int j = tile * kCrtPrimesPerTile + 2 * warp + pp;
      if (j >= np) continue;
      const DevPrime pr = primes[j];
      const uint64_t negp = 0 - pr.p;
      uint64_t r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // V = X + 2^30 Y, X = (hx:lx), Y = (hy:ly)
        const uint64_t lx = lo[i][2 * pp], hx = hi[i][2 * pp];
        const uint64_t ly = lo[i][2 * pp + 1], hy = hi[i][2 * pp + 1];
        const uint64_t vlo = lx + (ly << 30);
        const uint64_t vhi = hx + (ly >> 34) + (hy << 30) + (vlo < lx);
        const uint64_t r0 = shoup_mul_4p(vlo, 1, pr.one_q, negp);
        const uint64_t r1 = shoup_mul_4p(vhi, pr.beta, pr.beta_q, negp);
        r[i] = reduce_4p(csub(r0 + r1, 4 * pr.p), pr.p);
      }
      uint64_t* dst = out + (size_t(b) * np + j) * n + c0 + 4 * lane;
      reinterpret_cast<ulonglong2*>(dst)[0] = make_ulonglong2(r[0], r[1]);
      reinterpret_cast<ulonglong2*>(dst)[1] = make_ulonglong2(r[2], r[3]);
    }
  }
}

size_t crt_smem(int limbs, int M) {
  return size_t(M) * kCoefs * 4 + size_t(M) * kCols * 4 + size_t(kCoefs) * limbs * 8;
}

}  // namespace

cudaError_t crt_setup_attributes() {
  return cudaFuncSetAttribute(crt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kMaxDynSmem);
}

cudaError_t crt_forward(const uint64_t* poly, int limbs, size_t batch, int log_n,
                        const CrtWeights& w, const DevPrime* primes, int np, uint64_t* out,
                        cudaStream_t st) {
  const size_t n = size_t(1) << log_n;
  if (n < kCoefs) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(n / kCoefs), static_cast<unsigned>(batch));
  crt_kernel<<<grid, kWarps * 32, crt_smem(limbs, w.chunks), st>>>(
      poly, limbs, log_n, w.wtab, w.chunks, w.np_pad, primes, np, out);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
