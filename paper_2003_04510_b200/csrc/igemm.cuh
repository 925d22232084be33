// Small-K integer GEMM core on the IMAD.WIDE pipe (sm_100a), shared by the
// forward CRT, the exact iCRT and the fused key-switch finisher.
//
//   C[c][n] = sum_k A[k][c] * B[k][n]      A: <= 30-bit, B: <= 25-bit (u32)
//
// Every product is < 2^55, so one IMAD.WIDE.U32 per product accumulates into
// a u64 with no carry handling for K <= 480 (480 * 2^55 < 2^64): the CRT/iCRT
// big-integer inner products of the reference (rns.cpp:43-106, 235-290 — 64x64
// MACs into 3-word accumulators with ADC chains) become straight IMAD.WIDE
// streams.
//
// Tile: a CTA of NW warps owns 32 coefficients (columns of A, staged in shared
// memory for all K) x 16*NW output columns. Lane -> (coefficient group
// lane&7: 4 coefficients, column group lane>>3: 4 columns), so each lane does
// 16 IMAD.WIDE per k from one LDS.128 of A (8 distinct addresses per warp)
// and one LDS.128 of B (4 distinct addresses), i.e. 2 shared-memory
// wavefronts per 16 warp-IMADs: IMAD-bound. B streams from global/L2 through
// a STAGES-deep cp.async ring of KT rows.
#pragma once
#include <cstdint>

namespace hemul_gpu {

constexpr int kGemmCoefs = 32;   // A columns (coefficients) per CTA
constexpr int kMaxGemmK = 480;   // 480 * (2^30-1)(2^25-1) < 2^64

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// acc[i][q] += sum_{k<K} A[k][4cg+i] * B[k][col0 + 16w + 4ng + q]
// As: shared [K][32]; Bg: global [>=K][ldb] (ldb, col0 multiples of 4, 16-B
// aligned rows); Bs: shared ring of STAGES*KT*16*NW u32.
// All threads of the CTA must call it (it synchronises).
template <int NW, int KT, int STAGES>
__device__ __forceinline__ void igemm_32xN(const uint32_t* __restrict__ As, int K,
                                           const uint32_t* __restrict__ Bg, int ldb, int col0,
                                           uint32_t* __restrict__ Bs, uint64_t (&acc)[4][4]) {
  constexpr int NC = 16 * NW;       // columns in the tile
  constexpr int CH = NC / 4;        // 16-byte chunks per B row
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int cg = lane & 7, ng = lane >> 3;
  const int tiles = (K + KT - 1) / KT;
  auto load = [&](int t) {
    if (t < tiles) {
      const int k0 = t * KT;
      const int rows = min(KT, K - k0);
      uint32_t* dst = Bs + (t % STAGES) * KT * NC;
      for (int idx = tid; idx < rows * CH; idx += NW * 32) {
        const int r = idx / CH, c = idx - r * CH;
        cp_async16(dst + r * NC + 4 * c, Bg + size_t(k0 + r) * ldb + col0 + 4 * c);
      }
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) load(s);
  const uint32_t* a_ptr = As + 4 * cg;
  const int b_off = 16 * warp + 4 * ng;
  for (int t = 0; t < tiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    load(t + STAGES - 1);
    const int k0 = t * KT;
    const int rows = min(KT, K - k0);
    const uint32_t* bt = Bs + (t % STAGES) * KT * NC + b_off;
    const uint32_t* at = a_ptr + k0 * kGemmCoefs;
    if (rows == KT) {
#pragma unroll 8
      for (int r = 0; r < KT; ++r) {
        const uint4 a = *reinterpret_cast<const uint4*>(at + r * kGemmCoefs);
        const uint4 b = *reinterpret_cast<const uint4*>(bt + r * NC);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] += static_cast<uint64_t>(av[i]) * bv[q];
      }
    } else {
      for (int r = 0; r < rows; ++r) {
        const uint4 a = *reinterpret_cast<const uint4*>(at + r * kGemmCoefs);
        const uint4 b = *reinterpret_cast<const uint4*>(bt + r * NC);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] += static_cast<uint64_t>(av[i]) * bv[q];
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// The same product with no CTA-wide barrier in the K loop: a warp only ever
// reads its own 16 B columns, so each warp streams them through a private
// cp.async ring (STAGES x KT rows x 64 bytes at Bw) and synchronises with
// __syncwarp. Warps then run their IMAD.WIDE loops at their own pace instead
// of meeting at a __syncthreads every tile. A (all K rows) must be complete
// and visible (one __syncthreads) before the call; col0 is the CTA tile's
// first column (the warp uses col0 + 16 * warp).
template <int KT, int STAGES>
__device__ __forceinline__ void igemm_32x16_warp(const uint32_t* __restrict__ As, int K,
                                                 const uint32_t* __restrict__ Bg, int ldb,
                                                 int col0, uint32_t* __restrict__ Bw,
                                                 uint64_t (&acc)[4][4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane & 7, ng = lane >> 3;
  const int colw = col0 + 16 * warp;
  const int tiles = (K + KT - 1) / KT;
  auto load = [&](int t) {
    if (t < tiles) {
      const int k0 = t * KT;
      const int rows = min(KT, K - k0);
      uint32_t* dst = Bw + (t % STAGES) * KT * 16;
      for (int idx = lane; idx < rows * 4; idx += 32) {
        const int r = idx >> 2, c = idx & 3;
        cp_async16(dst + r * 16 + 4 * c, Bg + size_t(k0 + r) * ldb + colw + 4 * c);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) load(s);
  const uint32_t* a_ptr = As + 4 * cg;
  for (int t = 0; t < tiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncwarp();
    load(t + STAGES - 1);
    const int k0 = t * KT;
    const int rows = min(KT, K - k0);
    const uint32_t* bt = Bw + (t % STAGES) * KT * 16 + 4 * ng;
    const uint32_t* at = a_ptr + k0 * kGemmCoefs;
    auto step = [&](int r) {
      const uint4 a = *reinterpret_cast<const uint4*>(at + r * kGemmCoefs);
      const uint4 b = *reinterpret_cast<const uint4*>(bt + r * 16);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] += static_cast<uint64_t>(av[i]) * bv[q];
    };
    if (rows == KT) {
#pragma unroll 8
      for (int r = 0; r < KT; ++r) step(r);
    } else {
      for (int r = 0; r < rows; ++r) step(r);
    }
  }
  cp_async_wait<0>();
  __syncwarp();
}

}  // namespace hemul_gpu
