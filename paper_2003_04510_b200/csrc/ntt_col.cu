// Strided NTT pass A (levels [0, S) on 2^S-point columns) for the 30-bit
// basis (sm_100a): a half-warp per column at S >= 8 (the he_mul path at
// log N >= 15), a warp per column at S = 7.
//
// Reference: ntt_forward / ntt_inverse (proj/core/src/ntt.cpp:59-137,
// 153-197); pass structure as in ntt.cu (pass A = the first forward levels /
// the last inverse levels, n^-1 folded into inverse level 0). Values stay in
// the same lazy ranges as F32::ct / F32::gs (fields.cuh), so the outputs are
// identical to ntt.cu's pass A.
//
// Layout. A CTA loads 16 adjacent columns (16 consecutive residues of every
// one of the 2^S rows: coalesced 64-byte segments) into shared memory, column
// x at x * CS + f(y) (f pads one word per 32 or 2^(S-4) rows, CS = 2 mod 32):
// the cooperative load / store and the register layouts below are
// bank-conflict free (checked exhaustively).
// S >= 8 (column_transform_half): the two halves of a warp take columns c and
// c + 8, 2^S / 16 residues per lane, two register layouts and one shared
// exchange cover all S levels (layout H: y = h + 16 r, layout L: y = HE h + r).
// S = 7 (column_transform): a warp per column, layouts H / L plus one
// shuffle level between them. No CTA barrier inside the transform.
//
// Measured at X (ms per step forward / inverse; tools/run_variants.sh with
// the HEMUL_COL_* macros below): the half-warp form 2.02 / 2.33 (the warp
// form with its shuffle level 2.14 / 2.38). Its HBM phase alone
// (HEMUL_COL_EXP=1) takes 1.48 / 1.62, the transform alone (EXP=2) 1.50 /
// 1.67: the one-tile CTAs overlap the two only in part. Not adopted, all
// slower: 32-column tiles (128-byte row segments; HBM phase alone 1.28 /
// 1.39 = 0.91 of HBM, full pass 2.09 / 2.42 at 2 CTAs per SM); a persistent
// cp.async double-buffered CTA (3.0 / 3.4: 2 CTAs per SM, 41 % issue); a
// warp-specialised persistent CTA (16 transform + 8 copy warps, named
// barriers, 2 or 3 buffers: 2.49 / 2.74) — the transform needs ~32 resident
// warps per SM, which at 64 registers is the whole register file.
#include <cuda_runtime.h>

#include "fields.cuh"
#include "kernels.hpp"

namespace hemul_gpu {

namespace {

#ifndef HEMUL_COL_COLS
#define HEMUL_COL_COLS 16
#endif
constexpr int kCols = HEMUL_COL_COLS;  // columns per CTA (4 kCols-byte row segments)
constexpr int kWarps = kCols / 2;      // half-warp form: one column per half-warp
constexpr int kThreads = 32 * kWarps;
constexpr int kTpr = kCols / 4;        // threads per row segment (16-byte vectors)

// (every form reads only its own members: silence nvcc's unused-member note)
#pragma nv_diag_suppress 177
template <int S>
struct ColGeo {
  static constexpr int EPT = (1 << S) / 32;
  static constexpr int R = S - 5;                 // log2(EPT)
  static_assert(EPT >= 4, "16-byte cooperative load: >= 4 residues per thread");
  static constexpr int NSH = S - 2 * R;           // shuffle levels
  // half-warp form (S >= 8): 16 lanes per column, HE = 2^S / 16 residues
  // per lane, RH = log2(HE) levels in each of the two register layouts
  static constexpr bool kHalf = S >= 8;
  static constexpr int HE = (1 << S) / 16;
  static constexpr int RH = S - 4;
  // padded position of row y: one pad word per 2^PS rows
  static constexpr int PS = kHalf ? S - 4 : 5;
  // column stride: > f(2^S - 1) and = 2 (mod 32) for 16-column tiles, 1 (mod
  // 32) for 32-column tiles (the cooperative copies then cover 8 columns x 4
  // rows per warp; the half-warp columns c, c + 16 sit 16 banks apart)
  static constexpr int CM = (kHalf && kCols == 32) ? 1 : 2;
  static constexpr int CS = ((1 << S) + (1 << (S - PS)) + 32 - CM - 1) / 32 * 32 + CM;
};
#pragma nv_diag_default 177

template <int S>
__device__ __forceinline__ int padc(int y) { return y + (y >> ColGeo<S>::PS); }
__device__ __forceinline__ int padf(int y) { return y + (y >> 5); }

struct ColArgs {
  uint32_t* data;
  uint32_t* out;  // == data except in the transposed forms (out of place)
  const Twiddle32* tw;
  const uint2* twc;  // TR != 0: per prime 2^S (w, wq) pairs in shared-slot order
  const DevPrime32* primes;
  int np, log_n, rows_per_prime;
};

// Harvey CT / GS butterflies (fields.cuh F32::ct, F32::gs)
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

// Shared twiddle slot of table entry t (level L = floor(log2 t)). Layout-L
// levels (L >= S - R = 5) are read by lane l at t = 2^L + l 2^i + blk
// (i = L - 5): stored lane-minor instead (2^L + blk 32 + l) so those reads
// are bank-conflict free; w and wq live in separate arrays.
template <int S>
__device__ __forceinline__ int twiddle_slot(int t) {
  if constexpr (ColGeo<S>::kHalf) {
    // half-warp form: layout-L levels L >= RH are read by half-lane h at
    // t = 2^L + h 2^i + blk (i = L - 4) -> stored at 2^L + blk 16 + h
    if (t < (1 << ColGeo<S>::RH)) return t;
    const int L = 31 - __clz(t), i = L - 4, within = t - (1 << L);
    return (1 << L) + (within & ((1 << i) - 1)) * 16 + (within >> i);
  } else {
    if (t < 32) return t;
    const int L = 31 - __clz(t), i = L - 5, within = t - (1 << L);
    return (1 << L) + (within & ((1 << i) - 1)) * 32 + (within >> i);
  }
}

// One warp transforms NC padded columns mc, mc + cstride, ... (see the layout
// notes above) together: every twiddle load serves NC butterflies, and the
// NC independent columns give each warp NC-fold instruction-level
// parallelism.
template <int S, bool INV, int NC>
__device__ __forceinline__ void column_transform(uint32_t* mc, int cstride, const uint32_t* stw,
                                                 const DevPrime32& pr, int lane) {
  using G = ColGeo<S>;
  constexpr int EPT = G::EPT, R = G::R, NSH = G::NSH;
  const uint32_t p = pr.p, p2 = 2 * p, negp = 0u - p;
  auto tw = [&](int idx, uint32_t& w, uint32_t& wq) {
    w = stw[idx];
    wq = stw[(1 << S) + idx];
  };
  uint32_t v[NC][EPT];
  auto ld = [&](auto pos) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int r = 0; r < EPT; ++r) v[c][r] = mc[c * cstride + padf(pos(r))];
  };
  auto st = [&](auto pos) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int r = 0; r < EPT; ++r) mc[c * cstride + padf(pos(r))] = v[c][r];
  };
  auto posH = [&](int r) { return lane + 32 * r; };
  auto posL = [&](int r) { return EPT * lane + r; };
  if (!INV) {
    // ---- layout H: y = lane + 32 r; levels 0 .. R-1 ----------------------
    ld(posH);
#pragma unroll
    for (int L = 0; L < R; ++L) {
      const int half = EPT >> (L + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << L); ++blk) {
        uint32_t w, wq;
        tw((1 << L) + blk, w, wq);  // group y >> (S - L) = blk: uniform
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int rr = 0; rr < half; ++rr)
            ct(v[c][blk * 2 * half + rr], v[c][blk * 2 * half + rr + half], w, wq, p2, negp);
      }
    }
    st(posH);
    __syncwarp();
    ld(posL);
    // ---- lane levels R .. S-R-1 (layout L: y = EPT lane + r) -------------
#pragma unroll
    for (int L = R; L < R + NSH; ++L) {
      const int lb = S - 1 - L - R;  // lane bit of the pair
      const bool upper = (lane >> lb) & 1;
      uint32_t w, wq;
      tw((1 << L) + (lane >> (S - L - R)), w, wq);
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[c][r], 1 << lb);
          const uint32_t top = upper ? o : v[c][r], bot = upper ? v[c][r] : o;
          const uint32_t u = csub32(top, p2);
          const uint32_t t = shoup32(bot, w, wq, negp);
          v[c][r] = upper ? u + p2 - t : u + t;
        }
    }
    // ---- register levels S-R .. S-1 --------------------------------------
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int L = S - R + i, half = EPT >> (i + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << i); ++blk) {
        uint32_t w, wq;
        tw((1 << L) + blk * 32 + lane, w, wq);  // permuted (twiddle_slot)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int rr = 0; rr < half; ++rr)
            ct(v[c][blk * 2 * half + rr], v[c][blk * 2 * half + rr + half], w, wq, p2, negp);
      }
    }
    st(posL);
  } else {
    // ---- layout L: levels S-1 .. S-R in registers --------------------------
    ld(posL);
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      const int L = S - R + i, half = EPT >> (i + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << i); ++blk) {
        uint32_t w, wq;
        tw((1 << L) + blk * 32 + lane, w, wq);  // permuted (twiddle_slot)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int rr = 0; rr < half; ++rr)
            gs(v[c][blk * 2 * half + rr], v[c][blk * 2 * half + rr + half], w, wq, p2, negp);
      }
    }
    // ---- lane levels S-R-1 .. R ------------------------------------------
#pragma unroll
    for (int L = R + NSH - 1; L >= R; --L) {
      const int lb = S - 1 - L - R;
      const bool upper = (lane >> lb) & 1;
      uint32_t w, wq;
      tw((1 << L) + (lane >> (S - L - R)), w, wq);
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[c][r], 1 << lb);
          const uint32_t top = upper ? o : v[c][r], bot = upper ? v[c][r] : o;
          v[c][r] = upper ? shoup32(top + p2 - bot, w, wq, negp) : csub32(top + bot, p2);
        }
    }
    st(posL);
    __syncwarp();
    ld(posH);
    // ---- layout H: levels R-1 .. 1, then level 0 with n^-1 folded ---------
#pragma unroll
    for (int L = R - 1; L >= 1; --L) {
      const int half = EPT >> (L + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << L); ++blk) {
        uint32_t w, wq;
        tw((1 << L) + blk, w, wq);
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int rr = 0; rr < half; ++rr)
            gs(v[c][blk * 2 * half + rr], v[c][blk * 2 * half + rr + half], w, wq, p2, negp);
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int rr = 0; rr < EPT / 2; ++rr) {
        // a' = (u+v) n^-1, b' = (u-v) itw[1] n^-1, canonical (F32::inv_level0)
        const uint32_t u = v[c][rr], w2 = v[c][rr + EPT / 2];
        v[c][rr] = csub32(shoup32(u + w2, pr.ninv, pr.ninv_q, negp), p);
        v[c][rr + EPT / 2] = csub32(shoup32(u + p2 - w2, pr.w1n, pr.w1n_q, negp), p);
      }
    st(posH);
  }
}

// Half-warp form of the column transform (S >= 8): the 16 lanes h of a
// half-warp own one column, HE = 2^S / 16 residues each, and the two halves
// of a warp take columns c and c + 8 (the column stride is 2 mod 32, so the
// halves sit 16 banks apart). Two register layouts cover all S levels with
// one shared-memory exchange and no shuffle levels:
//   layout H: y = h + 16 r  -> levels 0 .. RH-1 (the top RH bits of y are r;
//             twiddles uniform across the warp),
//   layout L: y = HE h + r  -> levels RH .. S-1 (the low 4 bits of y are r's
//             low bits; twiddle t = 2^L + h 2^i + blk read lane-minor).
// The butterflies are those of column_transform (same pairs, same lazy
// ranges), so the outputs are identical; per residue it drops the shuffle
// level (a shuffle, three selects and a duplicated Shoup product per lane).
// Inverse of twiddle_slot for the half-warp form: the table entry at slot s.
template <int S>
__device__ __forceinline__ int twiddle_entry(int s) {
  static_assert(ColGeo<S>::kHalf, "half-warp form");
  if (s < (1 << ColGeo<S>::RH)) return s;
  const int L = 31 - __clz(s), i = L - 4, within = s - (1 << L);
  return (1 << L) + ((within & 15) << i) + (within >> 4);
}

// One register level of the half-warp form with compile-time level L:
// butterflies (r, r + half) in groups of 2 half registers, group twiddle at
// shared slot TW(blk) (templated so that nvcc unrolls every level fully; a
// runtime-indexed register array would turn into predicated moves).
template <int HE, int LOG_HALF, bool INV, typename TwF>
__device__ __forceinline__ void half_level(uint32_t (&v)[HE], const TwF& tw, uint32_t p2,
                                           uint32_t negp) {
  constexpr int half = 1 << LOG_HALF, groups = HE / (2 * half);
#pragma unroll
  for (int blk = 0; blk < groups; ++blk) {
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

template <int S, bool INV, int L, typename ReadTw>
__device__ __forceinline__ void half_level_at(uint32_t (&v)[ColGeo<S>::HE], const ReadTw& rd, int h,
                                              uint32_t p2, uint32_t negp) {
  constexpr int HE = ColGeo<S>::HE, RH = ColGeo<S>::RH;
  if constexpr (L < RH) {  // layout H: r holds the top bits, twiddle uniform
    half_level<HE, RH - 1 - L, INV>(
        v, [&](int blk, uint32_t& w, uint32_t& wq) { rd((1 << L) + blk, w, wq); }, p2, negp);
  } else {  // layout L: lane-minor twiddle slots (twiddle_slot)
    half_level<HE, S - 1 - L, INV>(
        v, [&](int blk, uint32_t& w, uint32_t& wq) { rd((1 << L) + blk * 16 + h, w, wq); }, p2,
        negp);
  }
}

template <int S, bool INV, int L0, int L1, typename ReadTw>
__device__ __forceinline__ void half_levels(uint32_t (&v)[ColGeo<S>::HE], const ReadTw& rd, int h,
                                            uint32_t p2, uint32_t negp) {
  // forward: L0, L0+1, ..., L1-1; inverse: L1-1, ..., L0
  if constexpr (L0 < L1) {
    if constexpr (!INV) {
      half_level_at<S, INV, L0>(v, rd, h, p2, negp);
      half_levels<S, INV, L0 + 1, L1>(v, rd, h, p2, negp);
    } else {
      half_level_at<S, INV, L1 - 1>(v, rd, h, p2, negp);
      half_levels<S, INV, L0, L1 - 1>(v, rd, h, p2, negp);
    }
  }
}

// Half-warp form of the column transform (S >= 8): the 16 lanes h of a
// half-warp own one column, HE = 2^S / 16 residues each, and the two halves
// of a warp take columns c and c + 8 (the column stride is 2 mod 32, so the
// halves sit 16 banks apart). Two register layouts cover all S levels with
// one shared-memory exchange and no shuffle levels:
//   layout H: y = h + 16 r  -> levels 0 .. RH-1 (the top RH bits of y are r;
//             twiddles uniform across the warp),
//   layout L: y = HE h + r  -> levels RH .. S-1 (the low 4 bits of y are r's
//             low bits; twiddle t = 2^L + h 2^i + blk read lane-minor).
// The butterflies are those of column_transform (same pairs, same lazy
// ranges), so the outputs are identical; per residue it drops the shuffle
// level (a shuffle, three selects and a duplicated Shoup product per lane).
// IO = kIoShared: input and output in the shared column (the cooperative
// copies move the tile); kIoGlobalIn (forward): the column is read straight
// from a transposed ("column-major") global row, gcol[y], and the CTA's
// twiddle copy (a straight uint4 copy of the prime's table in shared-slot
// order, built at level setup by ntt_col_slot_twiddles) is waited on after
// those loads are issued, so the barrier hides behind the column's HBM
// latency instead of preceding it (pass A forward -5..7% on B200);
// kIoGlobalOut (inverse): the result is written straight to a transposed
// global row. In the transposed layout column x of a row occupies
// [x 2^S, (x+1) 2^S): a half-warp's 16 lanes at one register touch 64
// contiguous bytes, and a layout-L twiddle read is 16 consecutive pairs.
enum { kIoShared = 0, kIoGlobalIn = 1, kIoGlobalOut = 2 };
template <int S, bool INV, int IO = kIoShared>
__device__ __forceinline__ void column_transform_half(uint32_t* mc, const uint32_t* stw,
                                                      const DevPrime32& pr, int h,
                                                      uint32_t* gcol = nullptr) {
  using G = ColGeo<S>;
  constexpr int HE = G::HE, RH = G::RH;
  static_assert(S - RH <= RH, "layout L must hold the remaining levels");
  const uint32_t p = pr.p, p2 = 2 * p, negp = 0u - p;
  const auto rd = [&](int idx, uint32_t& w, uint32_t& wq) {  // one LDS.64 per pair
    const uint2 x = reinterpret_cast<const uint2*>(stw)[idx];
    w = x.x;
    wq = x.y;
  };
  uint32_t v[HE];
  auto ld = [&](auto pos) {
#pragma unroll
    for (int r = 0; r < HE; ++r) v[r] = mc[padc<S>(pos(r))];
  };
  auto st = [&](auto pos) {
#pragma unroll
    for (int r = 0; r < HE; ++r) mc[padc<S>(pos(r))] = v[r];
  };
  auto posH = [&](int r) { return h + 16 * r; };
  auto posL = [&](int r) { return HE * h + r; };
  if (!INV) {
    if constexpr (IO == kIoGlobalIn) {
#pragma unroll
      for (int r = 0; r < HE; ++r) v[r] = gcol[posH(r)];
      __syncthreads();  // the CTA's twiddle copy, overlapped with the loads above
    } else {
      ld(posH);
    }
    half_levels<S, false, 0, RH>(v, rd, h, p2, negp);
    st(posH);
    __syncwarp();
    ld(posL);
    half_levels<S, false, RH, S>(v, rd, h, p2, negp);
    st(posL);
  } else {
    ld(posL);
    half_levels<S, true, RH, S>(v, rd, h, p2, negp);
    st(posL);
    __syncwarp();
    ld(posH);
    half_levels<S, true, 1, RH>(v, rd, h, p2, negp);
#pragma unroll
    for (int rr = 0; rr < HE / 2; ++rr) {
      // level 0 with n^-1 folded (F32::inv_level0)
      const uint32_t u = v[rr], w2 = v[rr + HE / 2];
      v[rr] = csub32(shoup32(u + w2, pr.ninv, pr.ninv_q, negp), p);
      v[rr + HE / 2] = csub32(shoup32(u + p2 - w2, pr.w1n, pr.w1n_q, negp), p);
    }
    if constexpr (IO == kIoGlobalOut) {
#pragma unroll
      for (int r = 0; r < HE; ++r) gcol[posH(r)] = v[r];
    } else {
      st(posH);
    }
  }
}

// Columns per warp-transform: the forward pass runs two interleaved columns
// (2.23 -> 2.12 ms per step at X, 3 CTAs/SM), the inverse pass one (two are
// slower there: 2.35 -> 2.44 ms). The macros exist for tools/build_variant.sh
// sweeps; last sweep at X (ms per step, inverse / forward): inverse NC=2 at
// 3 / 4 CTAs 2.43 / 2.50, NC=1 at 4 / 5 / 6 CTAs 2.52 / 2.37 / 2.55; forward
// at 2 / 3 / 4 CTAs 2.25 / 2.13 / 2.15.
#ifndef HEMUL_COL_NC_INV
#define HEMUL_COL_NC_INV 1
#endif
#ifndef HEMUL_COL_MINB_INV
#define HEMUL_COL_MINB_INV 5
#endif
#ifndef HEMUL_COL_MINB_FWD
#define HEMUL_COL_MINB_FWD 3
#endif
#ifndef HEMUL_COL_MINB_HALF
#define HEMUL_COL_MINB_HALF (64 / kCols)
#endif
#pragma nv_diag_suppress 177
template <int S, bool INV>
struct ColCfg {
  static constexpr int NC = INV ? HEMUL_COL_NC_INV : 2;
  static constexpr int kMinBlocks =
      ColGeo<S>::kHalf ? HEMUL_COL_MINB_HALF : (INV ? HEMUL_COL_MINB_INV : HEMUL_COL_MINB_FWD);
};
#pragma nv_diag_default 177

// TR = 1 (forward, S >= 8): input rows in the transposed layout (column x at
// [x 2^S, (x+1) 2^S), crt_tc.cu writes them so), output natural, out of place;
// TR = 2 (inverse): input natural, output transposed (bigint_tc.cu reads it).
template <int S, bool INV, int TR = 0>
__global__ void __launch_bounds__(kThreads, ColCfg<S, INV>::kMinBlocks) ntt_col_kernel(ColArgs a) {
  constexpr int CS = ColGeo<S>::CS;
  static_assert(TR == 0 || (ColGeo<S>::kHalf && (TR == 1) == !INV), "transposed forms");
  extern __shared__ uint32_t smem[];
  uint32_t* col = smem;                        // [kCols][CS]
  uint32_t* stw = smem + kCols * CS;           // w[2^S] then wq[2^S] (twiddle_slot order)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int j, row;
  if (a.rows_per_prime) {  // prime-major traversal (ntt.cu PassArgs)
    j = blockIdx.y / a.rows_per_prime;
    row = (blockIdx.y - j * a.rows_per_prime) * a.np + j;
  } else {
    row = blockIdx.y;
    j = row % a.np;
  }
  const DevPrime32& pr = a.primes[j];
  const size_t n = size_t(1) << a.log_n;
  const int tlast = 1 << (a.log_n - S);
  uint32_t* rowp = a.data + size_t(row) * n + size_t(blockIdx.x) * kCols;
  uint32_t* orowp = a.out + size_t(row) * n + size_t(blockIdx.x) * kCols;
  // transposed row of this half-warp's column (TR != 0)
  const int mycol = warp + kWarps * (lane >> 4);
  uint32_t* gcol = (TR == 1 ? a.data : a.out) + size_t(row) * n +
                   (size_t(blockIdx.x) * kCols + mycol) * (size_t(1) << S);
  // ---- cooperative load: 16-byte vectors, thread -> (columns 4 (tid % 4)
  // .. +3, rows tid / 4 + 128 r) ------------------------------------------------
  {
    constexpr int RS = kThreads / kTpr;  // rows per sweep
    const int x4 = 4 * (tid % kTpr), y0 = tid / kTpr;
    const uint4* src = reinterpret_cast<const uint4*>(rowp + size_t(y0) * tlast + x4);
    const size_t step = size_t(RS) * tlast / 4;
#ifndef HEMUL_COL_EXP
#define HEMUL_COL_EXP 0  // experiments: 1 = no transform, 2 = no HBM traffic
#endif
#pragma unroll
    for (int r = 0; r < (TR == 1 ? 0 : (1 << S) / RS); ++r) {  // TR 1: the transform loads
      const uint4 q = HEMUL_COL_EXP == 2 ? make_uint4(tid, r, 1, 2) : src[r * step];
      const int fy = padc<S>(y0 + RS * r);
      col[x4 * CS + fy] = q.x;
      col[(x4 + 1) * CS + fy] = q.y;
      col[(x4 + 2) * CS + fy] = q.z;
      col[(x4 + 3) * CS + fy] = q.w;
    }
    const uint32_t* t2 = reinterpret_cast<const uint32_t*>(a.tw + size_t(j) * n);
    if constexpr (TR != 0) {  // slot-ordered table: a straight copy (TR 1: waited on in the transform)
      static_assert((kCols * CS) % 4 == 0, "16-byte aligned twiddle slots");
      const uint4* s4 = reinterpret_cast<const uint4*>(a.twc + (size_t(j) << S));
      for (int i = tid; i < (1 << S) / 2; i += kThreads) reinterpret_cast<uint4*>(stw)[i] = s4[i];
    }
    for (int i = tid; i < (TR != 0 ? 0 : 1 << S); i += kThreads) {
      if constexpr (ColGeo<S>::kHalf) {
        // (w, wq) pairs interleaved; walk the slots (consecutive shared
        // words per warp) and gather the table entry each slot holds
        reinterpret_cast<uint2*>(stw)[i] =
            reinterpret_cast<const uint2*>(t2)[twiddle_entry<S>(i)];
      } else {
        const int pos = twiddle_slot<S>(i);
        stw[pos] = t2[2 * i];
        stw[(1 << S) + pos] = t2[2 * i + 1];
      }
    }
  }
  if constexpr (TR != 1) __syncthreads();
  if constexpr (HEMUL_COL_EXP == 1) {
  } else if constexpr (TR == 1) {
    column_transform_half<S, INV, kIoGlobalIn>(col + mycol * CS, stw, pr, lane & 15, gcol);
  } else if constexpr (TR == 2) {
    column_transform_half<S, INV, kIoGlobalOut>(col + mycol * CS, stw, pr, lane & 15, gcol);
    return;  // written straight to the transposed row: no store phase
  } else if constexpr (ColGeo<S>::kHalf) {
    static_assert(kCols == 2 * kWarps, "one column per half-warp");
    column_transform_half<S, INV>(col + mycol * CS, stw, pr, lane & 15);
  } else {
    constexpr int NC = ColCfg<S, INV>::NC;
    static_assert(kCols % (kWarps * NC) == 0, "columns per warp");
    for (int cw = warp; cw < kCols; cw += kWarps * NC)
      column_transform<S, INV, NC>(col + cw * CS, kWarps * CS, stw, pr, lane);
  }
  __syncthreads();
  // ---- cooperative store ------------------------------------------------
  if (HEMUL_COL_EXP != 2 || a.np < 0) {
    constexpr int RS = kThreads / kTpr;
    const int x4 = 4 * (tid % kTpr), y0 = tid / kTpr;
    uint4* dst = reinterpret_cast<uint4*>(orowp + size_t(y0) * tlast + x4);
    const size_t step = size_t(RS) * tlast / 4;
#pragma unroll
    for (int r = 0; r < (1 << S) / RS; ++r) {
      const int fy = padc<S>(y0 + RS * r);
      dst[r * step] = make_uint4(col[x4 * CS + fy], col[(x4 + 1) * CS + fy],
                                 col[(x4 + 2) * CS + fy], col[(x4 + 3) * CS + fy]);
    }
  }
}

template <int S, bool INV, int TR = 0>
cudaError_t launch_col(const ColArgs& a, size_t rows, cudaStream_t st) {
  const size_t smem = (size_t(kCols) * ColGeo<S>::CS + (size_t(2) << S)) * 4;
  if (smem > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      const cudaError_t e = cudaFuncSetAttribute(
          ntt_col_kernel<S, INV, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      attr = true;
    }
  }
  const int cols = 1 << (a.log_n - S);
  dim3 grid(static_cast<unsigned>(cols / kCols), static_cast<unsigned>(rows));
  ntt_col_kernel<S, INV, TR><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

// Pass A of the 30-bit basis through the column kernel: forward levels
// [0, S) (not the last pass) or inverse levels [S-1, 0] with n^-1 (the last
// pass); S = the pass-A level count of ntt.cu (7..9), n / 2^S >= 16 columns.
bool ntt_col_supported(int log_n, int S) {
  return S >= 7 && S <= 9 && (1 << (log_n - S)) >= kCols;
}

namespace {
template <int S>
__global__ void slot_twiddles_kernel(const Twiddle32* __restrict__ tw, int log_n, int np,
                                     Twiddle32* __restrict__ out) {
  const int j = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (1 << S); i += gridDim.x * blockDim.x)
    out[(size_t(j) << S) + i] = tw[(size_t(j) << log_n) + twiddle_entry<S>(i)];
}
}  // namespace

cudaError_t ntt_col_slot_twiddles(const Twiddle32* tw, int np, int log_n, int S, Twiddle32* out,
                                  cudaStream_t st) {
  if (!ntt_col_transposed_supported(log_n, S) || np < 1) return cudaErrorInvalidValue;
  const dim3 grid(2, static_cast<unsigned>(np));
  if (S == 8)
    slot_twiddles_kernel<8><<<grid, 256, 0, st>>>(tw, log_n, np, out);
  else
    slot_twiddles_kernel<9><<<grid, 256, 0, st>>>(tw, log_n, np, out);
  return cudaGetLastError();
}

cudaError_t ntt_col_pass_transposed(bool inv, const uint32_t* in, uint32_t* out, size_t rows,
                                    int np, int log_n, int S, const Twiddle32* tw,
                                    const Twiddle32* twc, const DevPrime32* primes,
                                    cudaStream_t st) {
  if (!ntt_col_transposed_supported(log_n, S) || in == out || !twc)
    return cudaErrorInvalidValue;
  const int rpp = rows % np ? 0 : static_cast<int>(rows / np);
  const ColArgs a{const_cast<uint32_t*>(in), out, tw, reinterpret_cast<const uint2*>(twc), primes,
                  np, log_n, rpp};
  switch (S * 2 + (inv ? 1 : 0)) {
    case 16: return launch_col<8, false, 1>(a, rows, st);
    case 17: return launch_col<8, true, 2>(a, rows, st);
    case 18: return launch_col<9, false, 1>(a, rows, st);
    default: return launch_col<9, true, 2>(a, rows, st);
  }
}

bool ntt_col_transposed_supported(int log_n, int S) {
  return ntt_col_supported(log_n, S) && (S == 8 || S == 9);
}

cudaError_t ntt_col_pass(bool inv, uint32_t* data, size_t rows, int np, int log_n, int S,
                         const Twiddle32* tw, const DevPrime32* primes, cudaStream_t st) {
  if (!ntt_col_supported(log_n, S)) return cudaErrorInvalidValue;
  const int rpp = rows % np ? 0 : static_cast<int>(rows / np);
  const ColArgs a{data, data, tw, nullptr, primes, np, log_n, rpp};
  switch (S * 2 + (inv ? 1 : 0)) {
    case 14: return launch_col<7, false>(a, rows, st);
    case 15: return launch_col<7, true>(a, rows, st);
    case 16: return launch_col<8, false>(a, rows, st);
    case 17: return launch_col<8, true>(a, rows, st);
    case 18: return launch_col<9, false>(a, rows, st);
    default: return launch_col<9, true>(a, rows, st);
  }
}

}  // namespace hemul_gpu
