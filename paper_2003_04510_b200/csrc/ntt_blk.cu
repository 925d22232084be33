// Fused NTT middle pass for the 30-bit basis, one warp per contiguous block
// (sm_100a): forward levels [s1, logN) of every operand, the evaluation-
// domain product, inverse levels [logN-1, s1) of every product.
//
// Reference: ntt_forward / ntt_inverse (proj/core/src/ntt.cpp:59-137,
// 153-197) and the pointwise products pm_pointwise / rns_pointwise_mul
// (polymul.cpp:22-27, rns.cpp:108-130); the same computation as ntt.cu's
// ntt_mid_kernel (OP_TENSOR2 / OP_EVK) with the same lazy ranges, so the
// results are identical.
//
// A warp owns one 2^S-point block (S = logN - s1) of one row for all
// operands: its loads and stores are coalesced 128-byte rows of the block,
// its twiddles ((2^s1 + block) 2^L + group, shared by every operand) sit in
// registers, and the three register / shuffle / register level groups of
// ntt_col.cu run between __syncwarp exchanges through the warp's own padded
// shared-memory slots. No CTA barrier at all: warps progress independently,
// so the HBM traffic of one warp overlaps the arithmetic of the others.
// The evaluation-domain products are Montgomery-reduced (3 instructions
// instead of 7 for the 64 -> 32-bit reduction): they come out as x y 2^-32,
// and the inverse pass A that follows uses n^-1 constants carrying 2^32
// (level_tables.hpp dev32_m / dev32_tm; context.cu blk_mont).
#include <cuda_runtime.h>

#include <type_traits>

#include "fields.cuh"
#include "igemm.cuh"
#include "kernels.hpp"

namespace hemul_gpu {

namespace {

#ifndef HEMUL_BLK_WARPS
#define HEMUL_BLK_WARPS 4
#endif
// blocks (warps) per CTA; 2 warps at 12 / 16 CTAs per SM and 8 warps at 3 / 4
// time the same or slower (mid r1 2.15-2.25 ms, r2 1.70-1.74 ms per step at X)
constexpr int kWarps = HEMUL_BLK_WARPS;
constexpr int kTensor2 = 0, kEvk = 1;

__device__ __forceinline__ int padf(int y) { return y + (y >> 5); }

struct BlkArgs {
  const uint32_t* in[8];   // operand rows (batch x np x n each)
  const uint32_t* evk[2];  // kEvk: evk NTT forms, np x n each
  uint32_t* out[6];        // product rows
  const Twiddle32* tw;
  const Twiddle32* itw;
  const DevPrime32* primes;
  int np, log_n, s1, rows_per_prime;
};

#pragma nv_diag_suppress 177
template <int S>
struct BlkGeo {
  static constexpr int EPT = (1 << S) / 32;
  static constexpr int R = S - 5;
  static constexpr int NSH = S - 2 * R;
  static constexpr int NH = EPT - 1;  // twiddles of R register levels
  // padded slot (words); S = 8 also holds the f1pad exchange (< 284)
  static constexpr int BS = S == 8 ? 288 : (1 << S) + (1 << (S - 5));
};
#pragma nv_diag_default 177

__device__ __forceinline__ Twiddle32 ldtw(const Twiddle32* p) {
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  return Twiddle32{v.x, v.y};
}

// The block's twiddles at levels s1 + L: index (gbase << L) + group
template <int S>
struct BlkTw {
  using G = BlkGeo<S>;
  uint32_t hw[G::NH], hq[G::NH];      // layout H levels 0 .. R-1 (uniform)
  uint32_t sw[G::NSH], sq[G::NSH];    // lane levels R .. S-R-1
  uint32_t lw[G::NH], lq[G::NH];      // layout L levels S-R .. S-1
  __device__ __forceinline__ void load(const Twiddle32* t, uint32_t gbase, int lane) {
    constexpr int R = G::R, NSH = G::NSH;
#pragma unroll
    for (int L = 0; L < R; ++L)
#pragma unroll
      for (int b = 0; b < (1 << L); ++b) {
        const Twiddle32 x = ldtw(t + (size_t(gbase) << L) + b);
        hw[(1 << L) - 1 + b] = x.w;
        hq[(1 << L) - 1 + b] = x.wq;
      }
#pragma unroll
    for (int k = 0; k < NSH; ++k) {
      const int L = R + k;
      const Twiddle32 x = ldtw(t + (size_t(gbase) << L) + (lane >> (S - L - R)));
      sw[k] = x.w;
      sq[k] = x.wq;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int L = S - R + i;
#pragma unroll
      for (int b = 0; b < (1 << i); ++b) {
        const Twiddle32 x = ldtw(t + (size_t(gbase) << L) + (size_t(lane) << i) + b);
        lw[(1 << i) - 1 + b] = x.w;
        lq[(1 << i) - 1 + b] = x.wq;
      }
    }
  }
};

__device__ __forceinline__ void ct(uint32_t& a, uint32_t& b, uint32_t w, uint32_t wq, uint32_t p2,
                                   uint32_t negp) {
  const uint32_t u = csub32(a, p2);
  const uint32_t v = shoup32(b, w, wq, negp);
  a = u + v;
  b = u + p2 - v;
}
__device__ __forceinline__ void gs(uint32_t& a, uint32_t& b, uint32_t w, uint32_t wq, uint32_t p2,
                                   uint32_t negp) {
  const uint32_t u = a, v = b;
  a = csub32(u + v, p2);
  b = shoup32(u + p2 - v, w, wq, negp);
}

// Forward levels of one operand: v in layout H (y = lane + 32 r) on entry,
// layout L (y = EPT lane + r) on exit; slot = the warp's scratch slot.
template <int S>
__device__ __forceinline__ void fwd(uint32_t (&v)[BlkGeo<S>::EPT], const BlkTw<S>& T,
                                    uint32_t* slot, int lane, uint32_t p2, uint32_t negp) {
  using G = BlkGeo<S>;
  constexpr int EPT = G::EPT, R = G::R, NSH = G::NSH;
#pragma unroll
  for (int L = 0; L < R; ++L) {
    const int half = EPT >> (L + 1);
#pragma unroll
    for (int b = 0; b < (1 << L); ++b)
#pragma unroll
      for (int rr = 0; rr < half; ++rr)
        ct(v[b * 2 * half + rr], v[b * 2 * half + rr + half], T.hw[(1 << L) - 1 + b],
           T.hq[(1 << L) - 1 + b], p2, negp);
  }
#pragma unroll
  for (int r = 0; r < EPT; ++r) slot[padf(lane + 32 * r)] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < EPT; ++r) v[r] = slot[padf(EPT * lane + r)];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < NSH; ++k) {
    const int lb = S - 1 - (R + k) - R;
    const bool upper = (lane >> lb) & 1;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], 1 << lb);
      const uint32_t top = upper ? o : v[r], bot = upper ? v[r] : o;
      const uint32_t u = csub32(top, p2);
      const uint32_t t = shoup32(bot, T.sw[k], T.sq[k], negp);
      v[r] = upper ? u + p2 - t : u + t;
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int half = EPT >> (i + 1);
#pragma unroll
    for (int b = 0; b < (1 << i); ++b)
#pragma unroll
      for (int rr = 0; rr < half; ++rr)
        ct(v[b * 2 * half + rr], v[b * 2 * half + rr + half], T.lw[(1 << i) - 1 + b],
           T.lq[(1 << i) - 1 + b], p2, negp);
  }
}

// Inverse levels (mirror of fwd): layout L on entry, layout H on exit.
template <int S>
__device__ __forceinline__ void inv(uint32_t (&v)[BlkGeo<S>::EPT], const BlkTw<S>& T,
                                    uint32_t* slot, int lane, uint32_t p2, uint32_t negp) {
  using G = BlkGeo<S>;
  constexpr int EPT = G::EPT, R = G::R, NSH = G::NSH;
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    const int half = EPT >> (i + 1);
#pragma unroll
    for (int b = 0; b < (1 << i); ++b)
#pragma unroll
      for (int rr = 0; rr < half; ++rr)
        gs(v[b * 2 * half + rr], v[b * 2 * half + rr + half], T.lw[(1 << i) - 1 + b],
           T.lq[(1 << i) - 1 + b], p2, negp);
  }
#pragma unroll
  for (int k = NSH - 1; k >= 0; --k) {
    const int lb = S - 1 - (R + k) - R;
    const bool upper = (lane >> lb) & 1;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], 1 << lb);
      const uint32_t top = upper ? o : v[r], bot = upper ? v[r] : o;
      v[r] = upper ? shoup32(top + p2 - bot, T.sw[k], T.sq[k], negp) : csub32(top + bot, p2);
    }
  }
#pragma unroll
  for (int r = 0; r < EPT; ++r) slot[padf(EPT * lane + r)] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < EPT; ++r) v[r] = slot[padf(lane + 32 * r)];
  __syncwarp();
#pragma unroll
  for (int L = R - 1; L >= 0; --L) {
    const int half = EPT >> (L + 1);
#pragma unroll
    for (int b = 0; b < (1 << L); ++b)
#pragma unroll
      for (int rr = 0; rr < half; ++rr)
        gs(v[b * 2 * half + rr], v[b * 2 * half + rr + half], T.hw[(1 << L) - 1 + b],
           T.hq[(1 << L) - 1 + b], p2, negp);
  }
}

// ---- S = 8 without shuffle levels ----------------------------------------
// The generic form above runs levels R .. S-R-1 (two of them at S = 8) as
// shuffle levels: every lane computes the whole butterfly (a duplicated
// Shoup product) plus a shuffle and three selects. At S = 8 the 8 levels are
// split instead into
//   layout H: y = lane + 32 r              levels 0-2 (r = y7 y6 y5)
//   -- shared exchange (pad f1(y) = y + 4 (y >> 5): H stores and M loads
//      are both bank-conflict free) --
//   layout M: y = (lane & 3) + 4 r + 32 (lane >> 2)   levels 3-5 (r = y4 y3 y2)
//   -- two register <-> lane bit swaps: lane bit 1 (y1) <-> r bit 2 (y4),
//      lane bit 0 (y0) <-> r bit 1 (y3); one shuffle per register pair --
//   layout L': lane = y >> 3, r = (y1, y0, y2)   levels 6-7
// and L' is the parked layout L (y = 8 lane + rL) with the registers renamed
// (rL = 4 b0 + 2 b2 + b1 for r = b2 b1 b0). Same butterflies, same lazy
// ranges, same outputs; the inverse runs the mirror image.
__device__ __forceinline__ int f1pad(int y) { return y + 4 * (y >> 5); }
__device__ __forceinline__ constexpr int rl_of(int r) {  // L' register -> L index
  return 4 * (r & 1) + 2 * ((r >> 2) & 1) + ((r >> 1) & 1);
}

struct BlkTw8 {
  uint32_t hw[7], hq[7];   // H levels 0-2: (gbase << L) + blk (uniform)
  uint32_t mw[7], mq[7];   // M levels 3-5: (gbase << L) + (lane >> 2) 2^(L-3) + blk
  uint32_t w6[2], q6[2];   // level 6: (gbase << 6) + 2 lane + b0
  uint32_t w7[4], q7[4];   // level 7: (gbase << 7) + 4 lane + 2 b0 + b2
  __device__ __forceinline__ void load(const Twiddle32* t, uint32_t gbase, int lane) {
#pragma unroll
    for (int L = 0; L < 3; ++L)
#pragma unroll
      for (int b = 0; b < (1 << L); ++b) {
        const Twiddle32 x = ldtw(t + (size_t(gbase) << L) + b);
        hw[(1 << L) - 1 + b] = x.w;
        hq[(1 << L) - 1 + b] = x.wq;
      }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int b = 0; b < (1 << k); ++b) {
        const int L = 3 + k;
        const Twiddle32 x = ldtw(t + (size_t(gbase) << L) + (size_t(lane >> 2) << k) + b);
        mw[(1 << k) - 1 + b] = x.w;
        mq[(1 << k) - 1 + b] = x.wq;
      }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const Twiddle32 x = ldtw(t + (size_t(gbase) << 6) + 2 * lane + b);
      w6[b] = x.w;
      q6[b] = x.wq;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {  // b = 2 b0 + b2
      const Twiddle32 x = ldtw(t + (size_t(gbase) << 7) + 4 * lane + b);
      w7[b] = x.w;
      q7[b] = x.wq;
    }
  }
};

// exchange register bit RB with lane bit LB (see the S = 8 notes)
template <int RB>
__device__ __forceinline__ void swap_bit(uint32_t (&v)[8], int lane, int lb) {
  const bool c = (lane >> lb) & 1;
#pragma unroll
  for (int r0 = 0; r0 < 8; ++r0) {
    if (r0 & (1 << RB)) continue;
    const int r1 = r0 | (1 << RB);
    const uint32_t send = c ? v[r0] : v[r1];
    const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 1 << lb);
    v[r0] = c ? recv : v[r0];
    v[r1] = c ? v[r1] : recv;
  }
}

// register level over pairs (r, r + 2^K) of an 8-array; TW(blk) = group twiddle
template <int K, bool INV, typename TwF>
__device__ __forceinline__ void reg_level8(uint32_t (&v)[8], const TwF& tw, uint32_t p2,
                                           uint32_t negp) {
  constexpr int half = 1 << K;
#pragma unroll
  for (int blk = 0; blk < 8 / (2 * half); ++blk) {
    uint32_t w, wq;
    tw(blk, w, wq);
#pragma unroll
    for (int rr = 0; rr < half; ++rr) {
      if constexpr (INV)
        gs(v[blk * 2 * half + rr], v[blk * 2 * half + rr + half], w, wq, p2, negp);
      else
        ct(v[blk * 2 * half + rr], v[blk * 2 * half + rr + half], w, wq, p2, negp);
    }
  }
}

// levels 6 / 7 in layout L': level 6 pairs bit 2 (twiddle by b0), level 7
// pairs bit 1 (twiddle by b0, b2)
template <bool INV>
__device__ __forceinline__ void level6(uint32_t (&v)[8], const BlkTw8& T, uint32_t p2,
                                       uint32_t negp) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if constexpr (INV)
      gs(v[r], v[r + 4], T.w6[r & 1], T.q6[r & 1], p2, negp);
    else
      ct(v[r], v[r + 4], T.w6[r & 1], T.q6[r & 1], p2, negp);
  }
}
template <bool INV>
__device__ __forceinline__ void level7(uint32_t (&v)[8], const BlkTw8& T, uint32_t p2,
                                       uint32_t negp) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (r & 2) continue;
    const int b = 2 * (r & 1) + (r >> 2);
    if constexpr (INV)
      gs(v[r], v[r + 2], T.w7[b], T.q7[b], p2, negp);
    else
      ct(v[r], v[r + 2], T.w7[b], T.q7[b], p2, negp);
  }
}

// forward levels: v in layout H on entry, L' on exit (slot = scratch)
__device__ __forceinline__ void fwd8(uint32_t (&v)[8], const BlkTw8& T, uint32_t* slot, int lane,
                                     uint32_t p2, uint32_t negp) {
  reg_level8<2, false>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.hw[0]; q = T.hq[0]; }, p2, negp);
  reg_level8<1, false>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.hw[1 + b]; q = T.hq[1 + b]; }, p2, negp);
  reg_level8<0, false>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.hw[3 + b]; q = T.hq[3 + b]; }, p2, negp);
#pragma unroll
  for (int r = 0; r < 8; ++r) slot[f1pad(lane + 32 * r)] = v[r];
  __syncwarp();
  const int mbase = f1pad((lane & 3) + 32 * (lane >> 2));
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = slot[mbase + 4 * r];
  __syncwarp();
  reg_level8<2, false>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.mw[0]; q = T.mq[0]; }, p2, negp);
  reg_level8<1, false>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.mw[1 + b]; q = T.mq[1 + b]; }, p2, negp);
  reg_level8<0, false>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.mw[3 + b]; q = T.mq[3 + b]; }, p2, negp);
  swap_bit<2>(v, lane, 1);
  swap_bit<1>(v, lane, 0);
  level6<false>(v, T, p2, negp);
  level7<false>(v, T, p2, negp);
}

// inverse levels: layout L' on entry, layout H on exit
__device__ __forceinline__ void inv8(uint32_t (&v)[8], const BlkTw8& T, uint32_t* slot, int lane,
                                     uint32_t p2, uint32_t negp) {
  level7<true>(v, T, p2, negp);
  level6<true>(v, T, p2, negp);
  swap_bit<1>(v, lane, 0);
  swap_bit<2>(v, lane, 1);
  reg_level8<0, true>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.mw[3 + b]; q = T.mq[3 + b]; }, p2, negp);
  reg_level8<1, true>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.mw[1 + b]; q = T.mq[1 + b]; }, p2, negp);
  reg_level8<2, true>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.mw[0]; q = T.mq[0]; }, p2, negp);
  const int mbase = f1pad((lane & 3) + 32 * (lane >> 2));
#pragma unroll
  for (int r = 0; r < 8; ++r) slot[mbase + 4 * r] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = slot[f1pad(lane + 32 * r)];
  __syncwarp();
  reg_level8<0, true>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.hw[3 + b]; q = T.hq[3 + b]; }, p2, negp);
  reg_level8<1, true>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.hw[1 + b]; q = T.hq[1 + b]; }, p2, negp);
  reg_level8<2, true>(v, [&](int b, uint32_t& w, uint32_t& q) { w = T.hw[0]; q = T.hq[0]; }, p2, negp);
}

// register caps that buy one or two more CTAs per SM without spills
// (measured at X: split tensor 2.25 -> 2.22 ms at 6 CTAs, evk 1.78 -> 1.72 at 7;
// with the Montgomery products the evk pass fits 8: 1.74 -> 1.71 ms; 9 or a
// 5-CTA split tensor pass are slower)
#ifndef HEMUL_BLK_MINB_R1
#define HEMUL_BLK_MINB_R1 6
#endif
#ifndef HEMUL_BLK_MINB_R2
#define HEMUL_BLK_MINB_R2 8
#endif
// S = 8 key-switch pass: the lane's evk words are copied to shared memory by
// cp.async when the warp starts, so their L2 latency hides behind the forward
// levels of F instead of stalling the products (the pass's top stall was
// long_scoreboard)
#ifndef HEMUL_BLK_EVK_PREFETCH
#define HEMUL_BLK_EVK_PREFETCH 1
#endif
constexpr int kEvkStage = HEMUL_BLK_EVK_PREFETCH ? 2 * 256 : 0;  // words per warp (S = 8)
template <int S, int OP>
__global__ void __launch_bounds__(32 * kWarps, OP == kTensor2 ? HEMUL_BLK_MINB_R1 : HEMUL_BLK_MINB_R2)
    ntt_blk_kernel(BlkArgs a) {
  using G = BlkGeo<S>;
  constexpr int EPT = G::EPT, BS = G::BS;
  constexpr int NIN = OP == kTensor2 ? 8 : 1, NOUT = OP == kTensor2 ? 6 : 2;
  constexpr int NSLOT = (S == 8 && OP == kEvk) ? 1 : (NIN > NOUT ? NIN : NOUT);
  extern __shared__ uint32_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int EVS = (S == 8 && OP == kEvk) ? kEvkStage : 0;
  uint32_t* slots = smem + warp * (NSLOT * BS + EVS);
  const int j = blockIdx.y / a.rows_per_prime;
  const int bt = blockIdx.y - j * a.rows_per_prime;
  const DevPrime32& pr = a.primes[j];
  const uint32_t p2 = 2 * pr.p, negp = 0u - pr.p;
  const size_t n = size_t(1) << a.log_n;
  const int block = blockIdx.x * kWarps + warp;
  const uint32_t gbase = (1u << a.s1) + block;
  const size_t off = (size_t(bt) * a.np + j) * n + (size_t(block) << S) + lane;
  // S = 8: no shuffle levels (fwd8 / inv8); registers are renamed (rl_of)
  constexpr bool k8 = S == 8;
  auto rl = [](int r) { return k8 ? rl_of(r) : r; };
  std::conditional_t<k8, BlkTw8, BlkTw<S>> T;
  T.load(a.tw + size_t(j) * n, gbase, lane);
  if constexpr (k8 && OP == kEvk) {
    // key-switch product at S = 8 entirely in registers: forward levels of
    // F (layout L' on exit), F evk_a and F evk_b at the lane's own positions
    // y = 8 lane + rl(r), then the inverse levels of each product from L';
    // one scratch slot per warp (the H <-> M exchange)
    uint32_t v[EPT], pb[EPT];
    const size_t eb0 = size_t(j) * n + (size_t(block) << S) + EPT * lane;
    uint32_t* ev = slots + NSLOT * BS + EPT * lane;  // [2][256] (HEMUL_BLK_EVK_PREFETCH)
    if constexpr (EVS > 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        cp_async16(ev + 256 * h, a.evk[h] + eb0);
        cp_async16(ev + 256 * h + 4, a.evk[h] + eb0 + 4);
      }
      cp_async_commit();
    }
#pragma unroll
    for (int r = 0; r < EPT; ++r) v[r] = a.in[0][off + 32 * r];
    fwd8(v, T, slots, lane, p2, negp);
    if constexpr (EVS > 0) cp_async_wait<0>();  // this lane's own words: no barrier
    // f in [0, 4p); the evk forms are full forward transforms, canonical
    // (kernels.hpp), so f evk < 4 p^2 < p 2^32
    if constexpr (EVS > 0) {
      // the lane's 8 words of each key row as two 16-byte loads (2-way bank
      // conflicts instead of 8-way scalar ones), evk_b first so that F is
      // overwritten last
      uint32_t e[EPT];
      auto ld8 = [&](const uint32_t* src) {
        const uint4 x0 = *reinterpret_cast<const uint4*>(src);
        const uint4 x1 = *reinterpret_cast<const uint4*>(src + 4);
        e[0] = x0.x, e[1] = x0.y, e[2] = x0.z, e[3] = x0.w;
        e[4] = x1.x, e[5] = x1.y, e[6] = x1.z, e[7] = x1.w;
      };
      static_assert(EPT == 8, "S = 8");
      ld8(ev + 256);
#pragma unroll
      for (int r = 0; r < EPT; ++r) pb[r] = F32::mul_mont(v[r], e[rl(r)], pr);
      ld8(ev);
#pragma unroll
      for (int r = 0; r < EPT; ++r) v[r] = F32::mul_mont(v[r], e[rl(r)], pr);
    } else {
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const uint32_t f = v[r];
        v[r] = F32::mul_mont(f, __ldg(a.evk[0] + eb0 + rl(r)), pr);
        pb[r] = F32::mul_mont(f, __ldg(a.evk[1] + eb0 + rl(r)), pr);
      }
    }
    T.load(a.itw + size_t(j) * n, gbase, lane);
    inv8(v, T, slots, lane, p2, negp);
#pragma unroll
    for (int r = 0; r < EPT; ++r) a.out[0][off + 32 * r] = v[r];
    inv8(pb, T, slots, lane, p2, negp);
#pragma unroll
    for (int r = 0; r < EPT; ++r) a.out[1][off + 32 * r] = pb[r];
  } else {
  // ---- forward levels of every operand; results parked in layout L. The
  // next operand's rows are loaded while this one is transformed. ----------
  uint32_t nx[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) nx[r] = a.in[0][off + 32 * r];
#pragma unroll 1
  for (int o = 0; o < NIN; ++o) {
    uint32_t v[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) v[r] = nx[r];
    if (o + 1 < NIN) {
#pragma unroll
      for (int r = 0; r < EPT; ++r) nx[r] = a.in[o + 1][off + 32 * r];
    }
    if constexpr (k8)
      fwd8(v, T, slots + o * BS, lane, p2, negp);
    else
      fwd<S>(v, T, slots + o * BS, lane, p2, negp);
#pragma unroll
    for (int r = 0; r < EPT; ++r) slots[o * BS + padf(EPT * lane + rl(r))] = v[r];
  }
  // ---- products at this lane's own positions (no exchange needed) -------
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int e = padf(EPT * lane + r);
    if constexpr (OP == kTensor2) {
      uint32_t x[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) x[o] = slots[o * BS + e];
      F32::tensor_split_mont(x, pr);
#pragma unroll
      for (int o = 0; o < 6; ++o) slots[o * BS + e] = x[o];
    } else {
      const size_t ei = size_t(j) * n + (size_t(block) << S) + EPT * lane + r;
      // f in [0, 4p); the evk forms are full forward transforms, canonical
      // (kernels.hpp), so f evk < 4 p^2 < p 2^32
      const uint32_t f = slots[e];
      slots[e] = F32::mul_mont(f, __ldg(a.evk[0] + ei), pr);
      slots[BS + e] = F32::mul_mont(f, __ldg(a.evk[1] + ei), pr);
    }
  }
  // ---- inverse levels of every product ------------------------------------
  T.load(a.itw + size_t(j) * n, gbase, lane);
#pragma unroll 1
  for (int o = 0; o < NOUT; ++o) {
    uint32_t v[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) v[r] = slots[o * BS + padf(EPT * lane + rl(r))];
    if constexpr (k8)
      inv8(v, T, slots + o * BS, lane, p2, negp);
    else
      inv<S>(v, T, slots + o * BS, lane, p2, negp);
#pragma unroll
    for (int r = 0; r < EPT; ++r) a.out[o][off + 32 * r] = v[r];
  }
  }  // generic path
}

template <int S, int OP>
cudaError_t launch_blk(const BlkArgs& a, size_t rows, cudaStream_t st) {
  constexpr int NSLOT = OP == kTensor2 ? 8 : (S == 8 ? 1 : 2);
  constexpr int EVS = (S == 8 && OP == kEvk) ? kEvkStage : 0;
  const size_t smem = size_t(kWarps) * (NSLOT * BlkGeo<S>::BS + EVS) * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ntt_blk_kernel<S, OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(static_cast<unsigned>((1 << a.s1) / kWarps), static_cast<unsigned>(rows));
  ntt_blk_kernel<S, OP><<<grid, 32 * kWarps, smem, st>>>(a);
  return cudaGetLastError();
}

template <int OP>
cudaError_t launch_blk_any(const BlkArgs& a, int S, size_t rows, cudaStream_t st) {
  switch (S) {
    case 6: return launch_blk<6, OP>(a, rows, st);
    case 7: return launch_blk<7, OP>(a, rows, st);
    default: return launch_blk<8, OP>(a, rows, st);
  }
}

}  // namespace

bool ntt_blk_supported(int log_n) {
  if (log_n < 12 || log_n > 17) return false;
  const int s1 = (log_n + 1) / 2, s2 = log_n - s1;
  return s2 >= 6 && s2 <= 8 && (1 << s1) % kWarps == 0;
}

cudaError_t ntt_blk_tensor_split(uint32_t* R1, size_t batch, int np, int log_n,
                                 const Twiddle32* tw, const Twiddle32* itw,
                                 const DevPrime32* primes, cudaStream_t st) {
  if (!ntt_blk_supported(log_n)) return cudaErrorInvalidValue;
  const int s1 = (log_n + 1) / 2;
  BlkArgs a{};
  const size_t slot = batch * size_t(np) << log_n;
  for (int o = 0; o < 8; ++o) a.in[o] = R1 + o * slot;
  for (int o = 0; o < 6; ++o) a.out[o] = R1 + o * slot;
  a.tw = tw;
  a.itw = itw;
  a.primes = primes;
  a.np = np;
  a.log_n = log_n;
  a.s1 = s1;
  a.rows_per_prime = static_cast<int>(batch);
  return launch_blk_any<kTensor2>(a, log_n - s1, batch * np, st);
}

cudaError_t ntt_blk_evk(uint32_t* Fin, const uint32_t* ea, const uint32_t* eb, uint32_t* KA,
                        uint32_t* KB, size_t batch, int np, int log_n, const Twiddle32* tw,
                        const Twiddle32* itw, const DevPrime32* primes, cudaStream_t st) {
  if (!ntt_blk_supported(log_n)) return cudaErrorInvalidValue;
  const int s1 = (log_n + 1) / 2;
  BlkArgs a{};
  a.in[0] = Fin;
  a.evk[0] = ea;
  a.evk[1] = eb;
  a.out[0] = KA;
  a.out[1] = KB;
  a.tw = tw;
  a.itw = itw;
  a.primes = primes;
  a.np = np;
  a.log_n = log_n;
  a.s1 = s1;
  a.rows_per_prime = static_cast<int>(batch);
  return launch_blk_any<kEvk>(a, log_n - s1, batch * np, st);
}

}  // namespace hemul_gpu
