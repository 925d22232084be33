// Exact inverse CRT and the fused key-switch finisher on the int8 tensor
// cores (sm_100a tcgen05, 30-bit basis).
//
// Reference: icrt_reordered (proj/core/src/rns.cpp:132-190, 235-290,
// 395-415) and the ModDown / add / rescale tail of Scheme::he_mul
// (heaan.cpp:398-409, poly.cpp:98-115). As in icrt.cu (the IMAD.WIDE form),
// every RNS operand ("segment") of a coefficient is reconstructed as
//   v = sum_j t_j H_j + k (-P),  t_j = x_j (P/p_j)^-1 mod p_j,
//   k = round(sum_j t_j / p_j)   (exact: >= 4 bits of slack, level_tables.cpp)
// and the kernel evaluates, per coefficient, the big integer
//   V = sum_segments sum_rows a_row V_row     (mod 2^T, from bit base8 up)
// whose rows V_row are the segment's H_j / -P already shifted to their place
// in the output (region-1 rows at bit logQ for the finisher; the split high
// product at 2^h), so that one pass gives d2 (iCRT) or
// R_logp(d + R_logQ(ks)) (finisher).
//
// Tensor-core form: with a_row = sum_b a_{row,b} 2^(8b) (bytes) and
// V_row = sum_e v_{row,e} 2^(8e),
//   D[i][m] = sum_{row,b} a_{row,b}(i) * v_{row, m + m0 - b}      (u8 x u8 -> s32)
//   V = sum_m D[i][m] 2^(8 (m + m0))
// i.e. a GEMM of the coefficients' bytes (A, M = 128 coefficients, K = 4
// bytes per row) against a constant table B[m][K] of shifted row bytes
// (level_tables.cpp build_bigint). The A operand lives in TMEM (the .kind::i8
// "TS" form): TMEM lane = coefficient, column = 4 K-bytes, so a residue t_j
// stored as one 32-bit column IS its four K-bytes; no byte transposition and
// no shared-memory traffic for A. D < K 2^16 < 2^27 is exact in s32; the
// epilogue carries the columns into 32-bit digits and extracts the output
// window. Columns below m0 (the finisher's bits under logQ - 125) are
// dropped: the truncation error is < 2^(8 m0 + 19), far below the 64 guard
// bits the ambiguity check inspects, exactly as in the IMAD finisher
// (kernels.hpp Finisher).
//
// Persistent warp-specialised CTA (one per SM, 512 TMEM columns: 3 x N/2
// accumulator columns, 2 x 16 A columns):
//   warp 4      bulk copies of the B chunks (64 K-bytes x n_cols rows, stored
//               chunk-major and pre-swizzled for the 64-byte UMMA layout)
//   warp 5      MMA issue: 2 k-steps x 2 MMAs (N = n_cols / 2 each) per chunk,
//               A from TMEM
//   warp 14     TMA of the t_j rows (16 rows x 128 coefficients per chunk; the
//               inverse NTT already scaled x_j by (P/p_j)^-1, context.cu
//               ntt_inv to_t)
//   warps 6-13  producers, two quads of four warps (one per TMEM lane
//               quadrant): quad q mod 2 takes chunk q into TMEM A stage q mod 2
//               (16 LDS + one 16-column tcgen05.st per thread) and keeps the
//               fixed-point sum_j umulhi(t_j, 2^55 / p_j) of its coefficient;
//               the last chunk of a tile carries the k bytes, from both quads'
//               posted partial sums
//   warps 0-3   epilogue: TMEM columns -> 32-bit digits -> output limbs
// Shared-memory traffic per chunk: the B chunk (written once, read once) and
// the t rows (TMA write, one LDS pass): 56 KB instead of 80 KB with a
// byte-plane A operand in shared memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include "fields.cuh"
#include "igemm.cuh"
#include "kernels.hpp"
#include "tc.cuh"

namespace hemul_gpu {

namespace {

#ifndef HEMUL_BIG_ABL
#define HEMUL_BIG_ABL 0  // ablation experiments (tools/run_variants.sh); 0 in production
// (1: B chunks loaded once, 2: A stages never written,
// 4: epilogue without the carry pass and the stores, 5: carry pass without the limb stores,
// 6: the high block's TMEM reads without the carry pass)
// (1: B chunks loaded once, 2: A stages never written, 3: MMAs not waiting for the A hand-off)
#endif
constexpr int kRows = 128;           // coefficients per tile (TMEM lanes)
constexpr int kChunk = 64;           // K bytes per pipeline chunk (2 MMA k-steps)
constexpr int kSlots = kChunk / 4;   // row slots (4-byte residues) per chunk
constexpr int kEpiWarps = 4;
constexpr int kTmaWarp = 4, kRawWarp = 5, kProd0 = 6, kProdWarps = 8;
constexpr int kMmaWarp = kProd0 + kProdWarps;  // highest warp id: first in issue arbitration
constexpr int kThreads = 32 * (kMmaWarp + 1);
constexpr int kSR = 8;               // raw t stages
constexpr int kMaxSB = 4;            // B (table) stages, 2 .. 4 by shared memory
constexpr int kRawBytes = kSlots * kRows * 4;    // 8 KB
constexpr int kMaxSeg = 3;
constexpr int kMaxRows = 1024;       // A rows (residues) per coefficient
constexpr int kACol = 512 - 2 * kSlots;          // TMEM A stages: columns 480 .. 511
constexpr int kXWords = 2 * 2 * kMaxSeg * kRows; // posted k partial sums [tile&1][quad][seg][i]

struct Params {
  BigTcSeg seg[kMaxSeg];
  int nseg, B, entries, log_n;
  int n_cols, k_bytes, k_slot, rows_total;
  int nsb;    // B stages
  int lobuf;  // the epilogue copies each tile's low accumulator block to shared memory
  BigTcOut o;
  uint32_t s8, s16, s24;  // 2^8, 2^16, 2^24 (arguments: kept as IMAD.WIDE)
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tc::smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(tc::smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b)
               : "memory");
}

// row (in the segment's tensor map) of residue row j of entry e
__device__ __forceinline__ int seg_row(const BigTcSeg& s, int e, int B, int j) {
  const int b = e % B, hi = e / B;
  return s.row0 + b * s.erows + (hi ? s.half_rows : 0) + j;
}

__global__ void __launch_bounds__(kThreads, 1)
    bigint_tc_kernel(const uint8_t* __restrict__ btab, const __grid_constant__ CUtensorMap rmap0,
                     const __grid_constant__ CUtensorMap rmap1, Params P) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t a_full[2], a_empty[2], b_full[kMaxSB], b_empty[kMaxSB];
  __shared__ __align__(8) uint64_t t_full[2], blk_free[3], r_full[kSR], r_empty[kSR];
  __shared__ __align__(8) uint64_t f_done[2], f_free[2];
  __shared__ uint32_t tmem_base;
  // 1024-byte aligned by pointer arithmetic on the shared array (an integer
  // round trip would lose the state space: generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_addr(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t n = size_t(1) << P.log_n;
  const int N = P.n_cols, NH = N / 2;
  const int nsb = P.nsb;
  const uint32_t b_bytes = uint32_t(N) * kChunk;
  uint8_t* sB = smem;                                  // nsb x [N][64] (SW64 K-major)
  uint8_t* sR = sB + nsb * b_bytes;                    // kSR x [16 rows][128] u32
  uint32_t* xbuf = reinterpret_cast<uint32_t*>(sR + kSR * kRawBytes);
  uint32_t* mu_tab = xbuf + kXWords;                   // [k_slot]
  // epilogue copy of the low accumulator block: [128 coefficients][LB]
  // words, LB = NH + 4 (mod 32): 16-byte accesses of 8 lanes hit 32 banks
  const int LB = NH + (NH % 32 == 0 ? 4 : 20);
  uint32_t* lobuf = P.lobuf ? mu_tab + kMaxRows : nullptr;
  const int C = P.k_bytes / kChunk;                    // chunks per tile (last: k bytes)
  const int tiles_per_entry = static_cast<int>(n / kRows);
  const int tiles = P.entries * tiles_per_entry;
  const int my_tiles = tiles > int(blockIdx.x) ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int total = my_tiles * C;                      // this CTA's chunk sequence

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&a_full[s], kProdWarps / 2 * 32);
      tc::mbar_init(&a_empty[s], 1);
      tc::mbar_init(&t_full[s], 1);
      tc::mbar_init(&f_done[s], kProdWarps * 32);
      tc::mbar_init(&f_free[s], kProdWarps / 2 * 32);
    }
    for (int s = 0; s < nsb; ++s) {
      tc::mbar_init(&b_full[s], 1);
      tc::mbar_init(&b_empty[s], 1);
    }
    for (int s = 0; s < kSR; ++s) {
      tc::mbar_init(&r_full[s], 1);
      tc::mbar_init(&r_empty[s], kProdWarps / 2);
    }
    for (int b = 0; b < 3; ++b) tc::mbar_init(&blk_free[b], kEpiWarps * 32);
    tc::mbar_fence_init();
  }
  // floor(2^55 / p) of every A row slot (the fixed-point k quotient; 0 for
  // padding slots, whose t values are whatever the TMA box held)
  for (int g = threadIdx.x; g < P.k_slot; g += kThreads) {
    const int s = (g >= P.seg[1].slot0) + (g >= P.seg[2].slot0);
    const int j = g - P.seg[s].slot0;
    mu_tab[g] = j < P.seg[s].np ? P.seg[s].primes[j].pad[0] : 0u;
  }
  if (warp == kTmaWarp) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  // TMEM: the accumulator is two column blocks of NH (low / high columns).
  // With 3 NH <= 480 the blocks rotate through three slots, tile t using
  // slots (2t mod 3, 2t+1 mod 3): the MMAs of tile t+1 need only the low
  // block of tile t, which the epilogue releases half way through.
  const int nslots = 3 * NH <= kACol ? 3 : 2;
  auto slot_lo = [&](int t) { return nslots == 3 ? (2 * t) % 3 : 0; };
  auto slot_hi = [&](int t) { return nslots == 3 ? (2 * t + 1) % 3 : 1; };

  if (warp == kTmaWarp) {
    // ---- B chunks: one linear bulk copy each (the table is stored chunk-
    // major and pre-swizzled, level_tables.cpp build_bigint) ---------------
    if (lane == 0) {
      for (int q = 0, c = 0, s = 0, ph = 0; q < total; ++q) {
        tc::mbar_wait(&b_empty[s], ph ^ 1);
#if HEMUL_BIG_ABL == 1  // ablation: B stages loaded once, reused (wrong results)
        if (q >= nsb) {
          tc::mbar_arrive(&b_full[s]);
        } else
#endif
        {
          mbar_expect_tx(&b_full[s], b_bytes);
          bulk_load(tc::smem_addr(sB + s * b_bytes), btab + size_t(c) * b_bytes, b_bytes,
                    &b_full[s]);
        }
        if (++c == C) c = 0;
        if (++s == nsb) s = 0, ph ^= 1;
      }
    }
  } else if (warp == kRawWarp) {
    // ---- TMA: the t rows of each chunk (kSR stages ahead of the producers)
    if (lane == 0) {
      for (int tl = 0, qr = 0; tl < my_tiles; ++tl) {
        const int tile = blockIdx.x + tl * gridDim.x;
        const int e = tile / tiles_per_entry;
        const int i0 = (tile - e * tiles_per_entry) * kRows;
        for (int c = 0; c < C - 1; ++c, ++qr) {
          // rows 16 c .. 16 c + 15 of one segment (segments start on chunks;
          // rows past the segment read neighbours or zero-filled OOB, unused)
          const int g0 = kSlots * c;
          const int sg = (g0 >= P.seg[1].slot0) + (g0 >= P.seg[2].slot0);
          const BigTcSeg& S = P.seg[sg];
          const int r = qr % kSR;
          tc::mbar_wait(&r_empty[r], ((qr / kSR) & 1) ^ 1);
          mbar_expect_tx(&r_full[r], kRawBytes);
          tma_load_2d(tc::smem_addr(sR + r * kRawBytes), S.map ? &rmap1 : &rmap0, i0,
                      seg_row(S, e, P.B, g0 - S.slot0), &r_full[r]);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issue (A: TMEM stage q mod 2, B: shared memory) --------------
    // The whole warp walks the chunk sequence (its barrier waits are warp-
    // uniform) and one elected lane issues; the B descriptors are the stage-0
    // descriptor plus a 16-byte-unit offset (shared addresses < 256 KB keep
    // the 14-bit start field from carrying), so a chunk costs a handful of
    // uniform adds instead of four descriptor builds. (With a lane-0 branch
    // and per-MMA descriptors the MMA warp spent ~110 instructions per chunk,
    // as long as the four MMAs themselves take.)
    const uint32_t idesc = tc::idesc_u8(kRows, NH, 0, 0);
    const uint64_t bdesc0 = tc::smem_desc(tc::smem_addr(sB), 16, 512, tc::kSw64);
    const uint32_t b_step = b_bytes >> 4, hi_off = uint32_t(NH * kChunk) >> 4;
    const bool leader = tc::elect_one();
    {
      int uses[3] = {0, 0, 0};
      uint32_t dlo = 0, dhi = 0;
      for (int q = 0, c = 0, it = 0, sb = 0; q < total; ++q) {
        if (c == 0) {  // a new tile: its two TMEM blocks must be drained
          const int bl = slot_lo(it), bh = slot_hi(it);
#pragma unroll
          for (int b = 0; b < 3; ++b)
            if ((b == bl || b == bh) && uses[b]++ > 0)
              tc::mbar_wait(&blk_free[b], (uses[b] - 2) & 1);
          dlo = tmem + bl * NH;
          dhi = tmem + bh * NH;
        }
        const int sa = q & 1;
#if HEMUL_BIG_ABL == 3  // ablation: MMAs decoupled from the A hand-off (wrong results)
        tc::mbar_wait(&b_full[sb], (q / nsb) & 1);
#else
        tc::mbar_wait(&a_full[sa], (q >> 1) & 1);  // the producers saw b_full too
#endif
        tc::fence_after();
        const uint64_t bd = bdesc0 + uint64_t(uint32_t(sb) * b_step);
        const uint32_t a0 = tmem + kACol + sa * kSlots;
        if (leader) {
          const uint32_t acc0 = c > 0 ? 1u : 0u;
          tc::mma_u8_ts(dlo, a0, bd, idesc, acc0);
          tc::mma_u8_ts(dhi, a0, bd + hi_off, idesc, acc0);
          tc::mma_u8_ts(dlo, a0 + 8, bd + 2, idesc, 1u);
          tc::mma_u8_ts(dhi, a0 + 8, bd + hi_off + 2, idesc, 1u);
          tc::mma_commit(&b_empty[sb]);
          tc::mma_commit(&a_empty[sa]);
        }
        if (++sb == nsb) sb = 0;
        if (++c == C) {
          if (leader) tc::mma_commit(&t_full[it & 1]);
          c = 0;
          ++it;
        }
        __syncwarp();
      }
    }
  } else if (warp >= kProd0) {
    // ---- producers: quad (warp - kProd0) / 4 takes the chunks q with
    // q mod 2 == quad into TMEM A stage quad; the warp writes the lanes of its
    // quadrant (warp mod 4), one coefficient per thread. Barrier phases: a
    // stage belongs to one quad; a quad's raw chunks are at most 3 apart
    // (< kSR), and tile t's partial sums are posted only after tile t - 2's
    // k chunk has read the buffer, so no wait can alias two phases ahead.
    const int quad = (warp - kProd0) >> 2, lq = warp & 3;
    const int ci = 32 * lq + lane;
    const uint32_t a_st = tmem + kACol + quad * kSlots + (uint32_t(32 * lq) << 16);
    const int sl1 = P.seg[1].slot0, sl2 = P.seg[2].slot0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int q0 = tl * C;
      int c = (quad - q0) & 1;  // (q0 + c) mod 2 == quad
      uint32_t F0 = 0, F1 = 0, F2 = 0;
      for (; c < C - 1; c += 2) {
        const int q = q0 + c;
        const int qr = tl * (C - 1) + c;
        const int r = qr % kSR;
        tc::mbar_wait_sleep<32>(&r_full[r], (qr / kSR) & 1);
        const uint32_t* R = reinterpret_cast<const uint32_t*>(sR + r * kRawBytes) + ci;
        const int g0 = kSlots * c;
        uint32_t t[kSlots];
#pragma unroll
        for (int i = 0; i < kSlots; ++i) t[i] = R[i * kRows];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&r_empty[r]);
        uint32_t f = 0;
#pragma unroll
        for (int i = 0; i < kSlots; ++i) f += __umulhi(t[i], mu_tab[g0 + i]);
        const int sg = (g0 >= sl1) + (g0 >= sl2);  // one segment per chunk
        F0 += sg == 0 ? f : 0u;
        F1 += sg == 1 ? f : 0u;
        F2 += sg == 2 ? f : 0u;
#if HEMUL_BIG_ABL != 3
        tc::mbar_wait_sleep<32>(&a_empty[quad], ((q >> 1) & 1) ^ 1);
        tc::mbar_wait_sleep<32>(&b_full[q % nsb], (q / nsb) & 1);
#endif
        tc::fence_after();
#if HEMUL_BIG_ABL != 2  // ablation 2: A stages never written (wrong results)
        tc::tmem_st16(a_st, t);
        tc::tmem_wait_st();
#endif
        tc::fence_before();
        tc::mbar_arrive(&a_full[quad]);
      }
      // post this tile's partial k sums (buffer tl & 1 is free once the k
      // chunk of tile tl - 2 has read it)
      const int xb = tl & 1;
      uint32_t* X = xbuf + (xb * 2 + quad) * kMaxSeg * kRows + ci;
      if (tl >= 2) tc::mbar_wait_sleep<32>(&f_free[xb], ((tl >> 1) - 1) & 1);
      X[0] = F0;
      X[kRows] = F1;
      X[2 * kRows] = F2;
      tc::mbar_arrive(&f_done[xb]);
      if (c == C - 1) {
        // k chunk: k_s = round(sum_j t_j / p_j) from both quads' partial sums
        const int q = q0 + c;
        tc::mbar_wait(&f_done[xb], (tl >> 1) & 1);
        const uint32_t* Y = xbuf + xb * 2 * kMaxSeg * kRows + ci;
        uint32_t k[kMaxSeg];
#pragma unroll
        for (int sg = 0; sg < kMaxSeg; ++sg) {
          const uint32_t tot = Y[sg * kRows] + Y[(kMaxSeg + sg) * kRows];
          k[sg] = sg < P.nseg ? (tot + (1u << 22)) >> 23 : 0u;
        }
        tc::mbar_arrive(&f_free[xb]);
#if HEMUL_BIG_ABL != 3
        tc::mbar_wait_sleep<32>(&a_empty[quad], ((q >> 1) & 1) ^ 1);
        tc::mbar_wait_sleep<32>(&b_full[q % nsb], (q / nsb) & 1);
#endif
        tc::fence_after();
        // K bytes 2s, 2s+1 = k_s (< 2^16), byte 6 = 1 (the constant row)
        tmem_st2(a_st, k[0] | k[1] << 16, k[2] | 1u << 16);
        tc::tmem_wait_st();
        tc::fence_before();
        tc::mbar_arrive(&a_full[quad]);
      }
    }
  } else {
    // ---- epilogue: lane = coefficient i0 + 32 warp + lane -----------------------
    // Column sums -> 32-bit digits d_h = (sum_{c<4} D[4h+c] 2^(8c) + carry) mod
    // 2^32. Output limb j (j = 0 is the guard limb below out_bit when the
    // ambiguity check is on) = bits [B0 + 64 j, +64) = e_{q+2j} | e_{q+2j+1} << 32
    // with e_h = (d_{h+1}:d_h) >> S, B0 = 32 q + S. Digits 0..q only carry;
    // then every 4 digits (one 16-column TMEM load) complete two limbs.
    // (The rounding constants enter through a constant A row, build_bigint.)
    const BigTcOut& o = P.o;
    const int H = N / 4;
    const int kst = (o.check_amb || o.force_exact) ? -1 : 0;
    const int B0 = o.out_bit + 64 * kst;
    const int S = B0 & 31, q = B0 >> 5;
    const int L = o.out_limbs, nl = L - kst;
    const uint64_t top = o.out_bits % 64 ? (uint64_t(1) << (o.out_bits % 64)) - 1 : ~0ull;
    const uint32_t lane_base = tmem + (uint32_t(32 * warp) << 16);
    auto digit = [&](const uint32_t* v, int h, uint64_t& carry) -> uint32_t {
      // the column sum does not depend on the carry: only the last 64-bit
      // add is on the digit-to-digit chain (iCRT 0.432 -> 0.416 ms at X)
      uint64_t t = 0;
      if (h < H) {  // warp-uniform
        const uint64_t t01 = uint64_t(v[1]) * P.s8 + v[0];
        const uint64_t t23 = uint64_t(v[3]) * P.s24 + uint64_t(v[2]) * P.s16;
        t = t01 + t23;
      }
      const uint64_t z = t + carry;
      carry = z >> 32;
      return static_cast<uint32_t>(z);
    };
    for (int it = 0; it < my_tiles; ++it) {
      const int tile = blockIdx.x + it * gridDim.x;
      const int e = tile / tiles_per_entry;
      // position of this lane's residues in the t rows -> its coefficient
      const size_t ipos = size_t(tile - e * tiles_per_entry) * kRows + 32 * warp + lane;
      const size_t i = o.tS ? ((ipos & ((size_t(1) << o.tS) - 1)) << (P.log_n - o.tS)) |
                                  (ipos >> o.tS)
                            : ipos;
      const int eb = e % P.B;
      uint64_t* dst = (e < P.B ? o.out0 : o.out1) + (size_t(eb) * n + i) * L;
      tc::mbar_wait_sleep<128>(&t_full[it & 1], (it >> 1) & 1);
      tc::fence_after();
      const int bl = slot_lo(it), bh = slot_hi(it);
      const uint32_t alo = lane_base + bl * NH, ahi = lane_base + bh * NH - NH;
      bool lo_held = true;
      uint32_t* lb = lobuf + (32 * warp + lane) * LB;  // this coefficient's row of lobuf
      if (lobuf) {
        // the next tile's MMAs need the low block: copy it out and hand it
        // back before the (sequential) carry pass (each thread reads back
        // only its own coefficient: no synchronisation)
        for (int c0 = 0; c0 < NH; c0 += 16) {
          uint32_t v[16];
          tc::tmem_ld16(alo + c0, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int d = 0; d < 16; d += 4)
            *reinterpret_cast<uint4*>(lb + c0 + d) = make_uint4(v[d], v[d + 1], v[d + 2], v[d + 3]);
        }
        tc::fence_before();
        tc::mbar_arrive(&blk_free[bl]);
        lo_held = false;
      }
      // 16 columns from col (multiple of 4); without lobuf the low block is
      // handed back as soon as every column below NH has been read
      auto load16 = [&](int col, uint32_t (&v)[16]) {
        if (lobuf) {
          if (col + 16 <= NH) {
#pragma unroll
            for (int d = 0; d < 16; d += 4) {
              const uint4 x = *reinterpret_cast<const uint4*>(lb + col + d);
              v[d] = x.x, v[d + 1] = x.y, v[d + 2] = x.z, v[d + 3] = x.w;
            }
            return;
          }
          if (col < NH) {
#pragma unroll
            for (int d = 0; d < 4; ++d) {
              const int cc = col + 4 * d;
              if (cc < NH) {
                const uint4 x = *reinterpret_cast<const uint4*>(lb + cc);
                v[4 * d] = x.x, v[4 * d + 1] = x.y, v[4 * d + 2] = x.z, v[4 * d + 3] = x.w;
              } else {
                tc::tmem_ld4(ahi + cc, *reinterpret_cast<uint32_t(*)[4]>(v + 4 * d));
              }
            }
            tc::tmem_wait_ld();
            return;
          }
          tc::tmem_ld16(ahi + col, v);
          tc::tmem_wait_ld();
          return;
        }
        if (col + 16 <= NH) {
          tc::tmem_ld16(alo + col, v);
        } else if (col >= NH) {
          tc::tmem_ld16(ahi + col, v);
        } else {
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const int cc = col + 4 * d;
            tc::tmem_ld4((cc < NH ? alo : ahi) + cc, *reinterpret_cast<uint32_t(*)[4]>(v + 4 * d));
          }
        }
        tc::tmem_wait_ld();
        if (lo_held && col + 16 >= NH) {
          tc::fence_before();
          tc::mbar_arrive(&blk_free[bl]);
          lo_held = false;
        }
      };
#if HEMUL_BIG_ABL == 6  // ablation: the high block's TMEM reads only (wrong results)
      {
        uint32_t acc = 0;
        for (int col = NH; col < N; col += 16) {
          uint32_t v[16];
          tc::tmem_ld16(ahi + col, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int d = 0; d < 16; ++d) acc ^= v[d];
        }
        dst[0] = acc;
        tc::fence_before();
        if (lo_held) tc::mbar_arrive(&blk_free[bl]);
        tc::mbar_arrive(&blk_free[bh]);
        continue;
      }
#endif
#if HEMUL_BIG_ABL == 4  // ablation: no carry pass / output (wrong results)
      if (lo_held) {
        uint32_t v[16];
        load16(0, v);
      }
      tc::fence_before();
      if (lo_held) tc::mbar_arrive(&blk_free[bl]);
      tc::mbar_arrive(&blk_free[bh]);
      continue;
#endif
      uint64_t carry = 0;
      uint32_t dprev = 0;
      // digits 0 .. q: carry only
      for (int h0 = 0; h0 <= q; h0 += 4) {
        uint32_t v[16];
        load16(4 * h0, v);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (h0 + c <= q) dprev = digit(v + 4 * c, h0 + c, carry);
      }
      bool skip = false;
      uint64_t xacc = 0;  // (ablation 5)
      for (int j = 0; j < nl; j += 2) {
        const int h = q + 1 + 2 * j;  // digits h .. h + 3 -> limbs j, j + 1
        uint32_t v[16];
        if (4 * h < N) load16(4 * h, v);
        const uint32_t d0 = digit(v, h, carry), d1 = digit(v + 4, h + 1, carry);
        const uint32_t d2 = digit(v + 8, h + 2, carry), d3 = digit(v + 12, h + 3, carry);
        const uint64_t l0 = __funnelshift_r(dprev, d0, S) |
                            (uint64_t(__funnelshift_r(d0, d1, S)) << 32);
        const uint64_t l1 = __funnelshift_r(d1, d2, S) |
                            (uint64_t(__funnelshift_r(d2, d3, S)) << 32);
        dprev = d3;
        const int k0 = j + kst;
        if (k0 < 0) {
          // guard limb: exact unless its 64 bits are all ones (kernels.hpp Finisher)
          skip = (o.check_amb && l0 == ~0ull) || o.force_exact;
          if (skip) {
            const unsigned slot = atomicAdd(o.flags.count, 1u);
            if (slot < o.flags.capacity) o.flags.ids[slot] = static_cast<unsigned>(size_t(e) * n + i);
          }
        } else if (!skip) {
          if (HEMUL_BIG_ABL == 5) xacc ^= l0;
          else dst[k0] = k0 == L - 1 ? l0 & top : l0;
        }
        if (!skip && k0 + 1 < L) {
          if (HEMUL_BIG_ABL == 5) xacc ^= l1;
          else dst[k0 + 1] = k0 + 1 == L - 1 ? l1 & top : l1;
        }
      }
      if (HEMUL_BIG_ABL == 5) dst[0] = xacc;  // ablation: one store per coefficient
      tc::fence_before();
      if (lo_held) tc::mbar_arrive(&blk_free[bl]);
      tc::mbar_arrive(&blk_free[bh]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == kTmaWarp) tc::tmem_dealloc<512>(tmem);
}

}  // namespace


namespace {
size_t smem_for(int n_cols, int nsb, bool lobuf) {
  return size_t(nsb) * n_cols * kChunk + size_t(kSR) * kRawBytes + size_t(kXWords) * 4 +
         kMaxRows * 4 +
         (lobuf ? size_t(n_cols / 2 + (n_cols / 2 % 32 == 0 ? 4 : 20)) * kRows * 4 : 0) + 1024;
}
// the low-block copy when it fits next to >= 3 B stages; B stages: as many as fit
bool use_lobuf(int n_cols) { return smem_for(n_cols, 3, true) <= size_t(kMaxDynSmem); }
int b_stages(int n_cols) {
  const bool lb = use_lobuf(n_cols);
  int nsb = kMaxSB;
  while (nsb > 2 && smem_for(n_cols, nsb, lb) > size_t(kMaxDynSmem)) --nsb;
  return nsb;
}
}  // namespace

// Shapes the kernel runs: the low-block copy must fit (forcing the path
// without it failed the M ladder at log_q = 60, n_cols = 32 — not reachable
// while the copy fits, i.e. n_cols <= 352, every he_mul level with logQ up to
// ~2700; larger tables take the IMAD.WIDE finisher)
bool bigint_tc_supported(int n_cols) {
  return n_cols % 32 == 0 && n_cols <= 480 && use_lobuf(n_cols) &&
         bigint_tc_smem(n_cols) <= size_t(kMaxDynSmem);
}

size_t bigint_tc_smem(int n_cols) {
  return smem_for(n_cols, b_stages(n_cols), use_lobuf(n_cols));
}

cudaError_t bigint_tc_setup_attributes() {
  return cudaFuncSetAttribute(bigint_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kMaxDynSmem);
}

cudaError_t bigint_tc(const BigTcTable& t, const BigTcSeg* segs, int entries, int B, int log_n,
                      const BigTcOut& o, const void* const* rmaps, cudaStream_t st) {
  const size_t n = size_t(1) << log_n;
  if (!t.btab || !rmaps || !rmaps[0] || !rmaps[1] || t.nseg < 1 || t.nseg > kMaxSeg || n < size_t(kRows) || t.n_cols % 32 ||
      !bigint_tc_supported(t.n_cols) || t.k_bytes % kChunk)
    return cudaErrorInvalidValue;
  if ((o.check_amb || o.force_exact) && !o.flags.count) return cudaErrorInvalidValue;
  if (t.k_slot > kMaxRows) return cudaErrorInvalidValue;
  for (int s2 = 0; s2 < t.nseg; ++s2)
    if (t.np[s2] > 511) return cudaErrorInvalidValue;  // fixed-point k sum < 2^32
  Params P{};
  for (int s = 0; s < kMaxSeg; ++s) {
    if (s < t.nseg) {
      P.seg[s] = segs[s];
      P.seg[s].slot0 = t.slot0[s];
      P.seg[s].np = t.np[s];
    } else {
      P.seg[s].slot0 = 1 << 30;  // never selected
    }
  }
  P.nseg = t.nseg;
  P.B = B;
  P.entries = entries;
  P.log_n = log_n;
  P.n_cols = t.n_cols;
  P.nsb = b_stages(t.n_cols);
  P.lobuf = use_lobuf(t.n_cols) ? 1 : 0;
  P.k_bytes = t.k_bytes;
  P.k_slot = t.k_slot;
  P.rows_total = t.slot0[t.nseg - 1] + t.np[t.nseg - 1];  // real rows; padding up to k_slot
  P.o = o;
  P.s8 = 1u << 8;
  P.s16 = 1u << 16;
  P.s24 = 1u << 24;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = entries * static_cast<int>(n / kRows);
  const int grid = tiles < sms ? tiles : sms;
  if (o.check_amb || o.force_exact) {
    cudaError_t e = cudaMemsetAsync(o.flags.count, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
  }
  bigint_tc_kernel<<<grid, kThreads, bigint_tc_smem(t.n_cols), st>>>(
      t.btab, *static_cast<const CUtensorMap*>(rmaps[0]),
      *static_cast<const CUtensorMap*>(rmaps[1]), P);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
