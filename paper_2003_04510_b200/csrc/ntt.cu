// Batched negacyclic NTT / iNTT over prime-major RNS rows (sm_100a).
//
// Reference: ntt_forward / ntt_inverse (proj/core/src/ntt.cpp:59-137,
// 153-197). Forward = Cooley-Tukey, natural in -> bit-reversed out; level L
// (2^L groups, half-distance t = n / 2^(L+1)) uses tw[2^L + g] for group g.
// Inverse = Gentleman-Sande from the last level back to level 0 with itw,
// then x n^-1 (folded here into level 0's butterfly).
//
// B200 mapping. One transform of n = 2^logN residues is split into two
// memory passes (2^s1 x 2^s2, s1 = ceil(logN/2)):
//   pass A: levels [0, s1) on 2^s1-point columns at stride 2^s2; a CTA owns
//           C adjacent columns (C residues contiguous per global row);
//   pass B: levels [s1, logN) on contiguous 2^s2-point blocks.
// A CTA holds 2^LP residues in shared memory (F64: 4096 x 8 B, 8 per
// thread; F32: 8192 x 4 B, 16 per thread — the Geo table below) and runs
// radix-8 butterfly units (3 levels) in registers between barriers, so
// shared memory is touched once per 3 levels. The pass size S, the
// sub-problems per CTA C and the thread count are template parameters: all
// index arithmetic folds to shifts of threadIdx, and no register array is
// dynamically indexed. Pass A's 2^S twiddles are staged in shared memory
// (every column of a row uses the same ones); pass B's are read once each
// from global memory. Values stay lazy (fields.cuh) and are canonicalised at
// the end, so every output is bit-identical to the reference's canonical
// residues (ntt.hpp:12-16; all reference variants are bit-identical,
// test_ntt.cpp:120-165).
//
// Rows are visited prime-major (all batch rows of prime j back to back), so a
// prime's twiddle table is streamed from HBM once per launch and re-read from
// L2 by the other rows.
#include <cuda_runtime.h>

#include <type_traits>

#include "device_tables.cuh"
#include "fields.cuh"
#include "kernels.hpp"

namespace hemul_gpu {

namespace {


// Shared-memory slot of residue index i. In every radix-8 group a warp's 32
// lanes take the lowest five index bits that are not the group's butterfly
// (v) bits, so whenever the three v bits sit below bit 5 the lanes spill into
// bits 5..7 and, with 32-bit residues, land in the same banks. XOR-ing bits
// 5, 6, 7 into the bank bits with the masks 31, 21, 25 makes the lanes' banks
// distinct for every position of the v bits (any group of 1..3 levels, any
// pass layout). The map is linear, so swz(base + off) = swz(base) ^ swz(off)
// for disjoint bit fields and compile-time offsets fold into immediates.
// 64-bit residues keep the identity layout.
template <class W>
__host__ __device__ constexpr int swz(int i) {
  return sizeof(W) != 4 ? i
                        : i ^ (((i >> 5) & 1) * 31) ^ (((i >> 6) & 1) * 21) ^ (((i >> 7) & 1) * 25);
}

// 16-byte vector r of a contiguous block <-> swizzled shared slots
template <class W>
__device__ __forceinline__ void put_vec(W* sb, uint4* sv, int r, uint4 v) {
  if constexpr (sizeof(W) == 4) {
    const int e = swz<W>(4 * r);
    sb[e] = v.x;
    sb[e ^ 1] = v.y;
    sb[e ^ 2] = v.z;
    sb[e ^ 3] = v.w;
  } else {
    sv[r] = v;
  }
}
template <class W>
__device__ __forceinline__ uint4 get_vec(const W* sb, const uint4* sv, int r) {
  if constexpr (sizeof(W) == 4) {
    const int e = swz<W>(4 * r);
    return make_uint4(sb[e], sb[e ^ 1], sb[e ^ 2], sb[e ^ 3]);
  } else {
    return sv[r];
  }
}

template <class F>
struct PassArgs {
  typename F::W* data;
  const typename F::Tw* tw;
  const typename F::Prime* primes;
  int np;
  int log_n;
  int st0;             // first global level of the pass
  int rows_per_prime;  // 0: row-major traversal (ragged row counts)
  int last;            // final pass: canonicalise (fwd) / fold n^-1 (inv)
};

// One pass of S levels over C = 2^LOGC sub-problems. STRIDED: pass A layout
// (sub-problems are columns at stride tlast); else pass B (contiguous blocks).
template <class F, int S, int LOGC, int LOGT, int MINB, bool STRIDED, bool INV>
__global__ void __launch_bounds__(1 << LOGT, MINB) ntt_pass_kernel(PassArgs<F> a) {
  using W = typename F::W;
  using Tw = typename F::Tw;
  constexpr int C = 1 << LOGC;
  constexpr int ELEMS = C << S;
  constexpr int T = 1 << LOGT;
  constexpr int EPT = ELEMS / T;  // residues per thread (8 or 16)
  constexpr int NG = (S + 2) / 3;
  constexpr int VPT = ELEMS * int(sizeof(W)) / 16 / T;  // 16-byte vectors per thread
  extern __shared__ uint4 smem_raw[];
  W* sbuf = reinterpret_cast<W*>(smem_raw);  // [ELEMS] residues, then pass-A twiddles
  W* stw = sbuf + ELEMS;                     // [2^S] x {w, wq}
  int j, row;
  if (a.rows_per_prime) {  // prime-major: blockIdx.y = j * rows_per_prime + b
    j = blockIdx.y / a.rows_per_prime;
    row = (blockIdx.y - j * a.rows_per_prime) * a.np + j;
  } else {
    row = blockIdx.y;
    j = row % a.np;
  }
  const typename F::Prime& pr = a.primes[j];
  const typename F::Mod md(pr);
  const size_t n = size_t(1) << a.log_n;
  W* rowp = a.data + size_t(row) * n;
  const Tw* twr = a.tw + size_t(j) * n;
  const int tlast = 1 << (a.log_n - a.st0 - S);
  const int sp0 = blockIdx.x << LOGC;  // first sub-problem of the CTA
  const int tid = threadIdx.x;
  // ---- load (+ pass-A twiddles) ------------------------------------------
  if (STRIDED) {
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int idx = tid + r * T;
      sbuf[swz<W>(idx)] = rowp[size_t(idx >> LOGC) * tlast + sp0 + (idx & (C - 1))];
    }
    const W* t2 = reinterpret_cast<const W*>(twr);
    for (int i = tid; i < 2 << S; i += T) stw[i] = t2[i];
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(rowp + (size_t(sp0) << S));
#pragma unroll
    for (int r = 0; r < VPT; ++r) put_vec(sbuf, smem_raw, tid + r * T, src[tid + r * T]);
  }
  __syncthreads();
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    const int grp = INV ? NG - 1 - gi : gi;
    const int l = 3 * grp;
    const int k = S - l < 3 ? S - l : 3;  // levels in this group
    const int ubits = S - l - k;          // log2 of units per group
    const int per = EPT >> k;             // units per thread
#pragma unroll
    for (int q = 0; q < EPT / 2; ++q) {
      if (q >= per) break;
      const int uid = tid + q * T;
      int c, h, u;
      if (STRIDED) {
        c = uid & (C - 1);
        const int rest = uid >> LOGC;
        u = rest & ((1 << ubits) - 1);
        h = rest >> ubits;
      } else {
        u = uid & ((1 << ubits) - 1);
        h = (uid >> ubits) & ((1 << l) - 1);
        c = uid >> (ubits + l);
      }
      const int e0 = (h << (S - l)) + u;
      W x[8];
      const int sbase = swz<W>(STRIDED ? (e0 << LOGC) + c : (c << S) + e0);
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) x[v] = sbuf[sbase ^ swz<W>((v << ubits) << (STRIDED ? LOGC : 0))];
      // twiddle of group hh at local level l + i
      auto tw_at = [&](int i, int blk, W& w, W& wq) {
        if (STRIDED) {
          const int t = (1 << (l + i)) + (h << i) + blk;
          w = stw[2 * t];
          wq = stw[2 * t + 1];
        } else {
          const Tw tt =
              twr[(size_t((1 << a.st0) + sp0 + c) << (l + i)) + (size_t(h) << i) + blk];
          w = tt.w;
          wq = tt.wq;
        }
      };
      if (!INV) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          if (i < k) {
            const int half = 1 << (k - i - 1);
#pragma unroll
            for (int blk = 0; blk < 4; ++blk)
              if (blk < (1 << i)) {
                W w, wq;
                tw_at(i, blk, w, wq);
#pragma unroll
                for (int r = 0; r < 4; ++r)
                  if (r < half) F::ct(x[blk * 2 * half + r], x[blk * 2 * half + r + half], w, wq, md);
              }
          }
        }
        if (a.last && grp == NG - 1) {
#pragma unroll
          for (int v = 0; v < 8; ++v)
            if (v < (1 << k)) x[v] = F::fwd_canon(x[v], md);
        }
      } else {
#pragma unroll
        for (int ii = 2; ii >= 0; --ii) {
          if (ii < k) {
            const int half = 1 << (k - ii - 1);
            const bool level0 = STRIDED && l + ii == 0 && a.last;
#pragma unroll
            for (int blk = 0; blk < 4; ++blk)
              if (blk < (1 << ii)) {
                if (level0) {
                  // level 0 with n^-1 folded in: a' = (u+v) n^-1,
                  // b' = (u-v) itw[1] n^-1, outputs canonical
#pragma unroll
                  for (int r = 0; r < 4; ++r)
                    if (r < half) {
                      const int i0 = blk * 2 * half + r;
                      F::inv_level0(x[i0], x[i0 + half], pr, md);
                    }
                } else {
                  W w, wq;
                  tw_at(ii, blk, w, wq);
#pragma unroll
                  for (int r = 0; r < 4; ++r)
                    if (r < half) F::gs(x[blk * 2 * half + r], x[blk * 2 * half + r + half], w, wq, md);
                }
              }
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) sbuf[sbase ^ swz<W>((v << ubits) << (STRIDED ? LOGC : 0))] = x[v];
    }
    __syncthreads();
  }
  // ---- store --------------------------------------------------------------
  if (STRIDED) {
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int idx = tid + r * T;
      rowp[size_t(idx >> LOGC) * tlast + sp0 + (idx & (C - 1))] = sbuf[swz<W>(idx)];
    }
  } else {
    uint4* dst = reinterpret_cast<uint4*>(rowp + (size_t(sp0) << S));
#pragma unroll
    for (int r = 0; r < VPT; ++r) dst[tid + r * T] = get_vec(sbuf, smem_raw, tid + r * T);
  }
}

// ---- fused middle pass: forward levels [s1, logN) + product + inverse ------
//
// The evaluation-domain product of the reference (pm_pointwise,
// polymul.cpp:22-27 / rns_pointwise_mul rns.cpp:108-130, 360-371) sits
// between the last forward levels and the first inverse levels, and both
// act on the same contiguous 2^s2-point blocks. One CTA therefore loads a
// block of every operand once, finishes the forward transforms, multiplies,
// runs the first inverse levels and stores only the products' blocks:
//   OP_TENSOR (region 1): A1 B1 A2 B2 -> d2 = A1A2, d0 = B1B2,
//                         d1 = A1B2 + A2B1 (written over A1, B1, A2)
//   OP_EVK    (region 2): F, evk_a, evk_b -> F evk_a, F evk_b
//   OP_TENSOR2 (split region 1, F32): the eight halves x1 X1 y1 Y1 x2 X2 y2
//                         Y2 -> the six half products of F32::tensor_split
//                         (written over the first six)
// Each twiddle is loaded once per unit and reused for every operand.
enum { OP_TENSOR = 0, OP_EVK = 1, OP_TENSOR2 = 2 };

template <class F, int S, int LOGC, int LOGT, int NOPS, bool INV>
__device__ __forceinline__ void block_group(typename F::W* sb, int grp, int sp0, int m0,
                                            const typename F::Tw* twr,
                                            const typename F::Mod& md) {
  using W = typename F::W;
  constexpr int C = 1 << LOGC;
  constexpr int T = 1 << LOGT;
  constexpr int OPS = C << S;  // residues per operand in shared memory
  constexpr int EPT = OPS / T;
  const int l = 3 * grp;
  const int k = S - l < 3 ? S - l : 3;
  const int ubits = S - l - k;
  const int per = EPT >> k;
#pragma unroll
  for (int q = 0; q < EPT / 2; ++q) {
    if (q >= per) break;
    const int uid = threadIdx.x + q * T;
    const int u = uid & ((1 << ubits) - 1);
    const int h = (uid >> ubits) & ((1 << l) - 1);
    const int c = uid >> (ubits + l);
    const int e0 = (c << S) + (h << (S - l)) + u;
    W w[7], wq[7];
    const size_t g = size_t(m0 + sp0 + c);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (i < k)
#pragma unroll
        for (int blk = 0; blk < 4; ++blk)
          if (blk < (1 << i)) {
            const typename F::Tw t = twr[(g << (l + i)) + (size_t(h) << i) + blk];
            w[(1 << i) - 1 + blk] = t.w;
            wq[(1 << i) - 1 + blk] = t.wq;
          }
    const int sbase = swz<W>(e0);
#pragma unroll
    for (int op = 0; op < NOPS; ++op) {
      W x[8];
      W* base = sb + op * OPS;  // OPS is a multiple of 256: slots swizzle alike
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) x[v] = base[sbase ^ swz<W>(v << ubits)];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int i = INV ? 2 - s : s;
        if (i < k) {
          const int half = 1 << (k - i - 1);
#pragma unroll
          for (int blk = 0; blk < 4; ++blk)
            if (blk < (1 << i))
#pragma unroll
              for (int r = 0; r < 4; ++r)
                if (r < half) {
                  const int a = blk * 2 * half + r;
                  if (INV)
                    F::gs(x[a], x[a + half], w[(1 << i) - 1 + blk], wq[(1 << i) - 1 + blk], md);
                  else
                    F::ct(x[a], x[a + half], w[(1 << i) - 1 + blk], wq[(1 << i) - 1 + blk], md);
                }
        }
      }
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (1 << k)) base[sbase ^ swz<W>(v << ubits)] = x[v];
    }
  }
}

template <class F>
struct MidArgs {
  using W = typename F::W;
  W* in[8];          // operand rows (batch x np x n each)
  const W* evk[2];   // OP_EVK: evk forms, np x n each (shared by the batch)
  W* out[6];         // product rows (batch x np x n each)
  const typename F::Tw* tw;
  const typename F::Tw* itw;
  const typename F::Prime* primes;
  int np, log_n, s1, rows_per_prime;
};

template <class F, int S, int LOGC, int LOGT, int OP>
__global__ void __launch_bounds__(1 << LOGT) ntt_mid_kernel(MidArgs<F> a) {
  using W = typename F::W;
  constexpr int C = 1 << LOGC;
  constexpr int ELEMS = C << S;
  constexpr int T = 1 << LOGT;
  constexpr int EPT = ELEMS / T;
  constexpr int NG = (S + 2) / 3;
  constexpr int NIN = OP == OP_TENSOR ? 4 : OP == OP_TENSOR2 ? 8 : 1;
  constexpr int NOUT = OP == OP_TENSOR ? 3 : OP == OP_TENSOR2 ? 6 : 2;
  constexpr int VPT = ELEMS * int(sizeof(W)) / 16 / T;  // 16-byte vectors per thread
  constexpr int VOP = ELEMS * int(sizeof(W)) / 16;      // 16-byte vectors per operand
  extern __shared__ uint4 smem_raw[];
  W* sb = reinterpret_cast<W*>(smem_raw);  // NIN operands, products reuse the slots
  const int j = blockIdx.y / a.rows_per_prime;
  const int b = blockIdx.y - j * a.rows_per_prime;
  const typename F::Prime& pr = a.primes[j];
  const typename F::Mod md(pr);
  const size_t n = size_t(1) << a.log_n;
  const size_t row_off = (size_t(b) * a.np + j) * n;
  const int sp0 = blockIdx.x << LOGC;
  const size_t blk_off = size_t(sp0) << S;
  const int m0 = 1 << a.s1;
  const int tid = threadIdx.x;
#pragma unroll
  for (int op = 0; op < NIN; ++op) {
    const uint4* src = reinterpret_cast<const uint4*>(a.in[op] + row_off + blk_off);
#pragma unroll
    for (int r = 0; r < VPT; ++r)
      put_vec(sb + op * ELEMS, smem_raw + op * VOP, tid + r * T, src[tid + r * T]);
  }
  __syncthreads();
  const typename F::Tw* twr = a.tw + size_t(j) * n;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    block_group<F, S, LOGC, LOGT, NIN, false>(sb, gi, sp0, m0, twr, md);
    __syncthreads();
  }
  // evaluation-domain products of forward-domain (lazy) values
  const W* ea = OP == OP_EVK ? a.evk[0] + size_t(j) * n + blk_off : nullptr;
  const W* eb = OP == OP_EVK ? a.evk[1] + size_t(j) * n + blk_off : nullptr;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = tid + r * T, e = swz<W>(i);
    if constexpr (OP == OP_TENSOR2) {
      W v[8];
#pragma unroll
      for (int op = 0; op < 8; ++op) v[op] = sb[op * ELEMS + e];
      F::tensor_split(v, pr);
#pragma unroll
      for (int op = 0; op < 6; ++op) sb[op * ELEMS + e] = v[op];
    } else if (OP == OP_TENSOR) {
      const W x1 = sb[e], y1 = sb[ELEMS + e], x2 = sb[2 * ELEMS + e], y2 = sb[3 * ELEMS + e];
      sb[e] = F::mul(x1, x2, pr);                      // d2
      sb[ELEMS + e] = F::mul(y1, y2, pr);              // d0
      sb[2 * ELEMS + e] = F::mul_add2(x1, y2, x2, y1, pr);  // d1
    } else {
      const W f = sb[e];
      sb[e] = F::mul(f, ea[i], pr);
      sb[ELEMS + e] = F::mul(f, eb[i], pr);
    }
  }
  __syncthreads();
  const typename F::Tw* itwr = a.itw + size_t(j) * n;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    block_group<F, S, LOGC, LOGT, NOUT, true>(sb, NG - 1 - gi, sp0, m0, itwr, md);
    __syncthreads();
  }
#pragma unroll
  for (int op = 0; op < NOUT; ++op) {
    uint4* dst = reinterpret_cast<uint4*>(a.out[op] + row_off + blk_off);
#pragma unroll
    for (int r = 0; r < VPT; ++r)
      dst[tid + r * T] = get_vec(sb + op * ELEMS, smem_raw + op * VOP, tid + r * T);
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

template <class F, int S, int LOGC>
size_t smem_bytes(bool strided) {
  return sizeof(typename F::W) * ((size_t(1) << (S + LOGC)) + (strided ? (size_t(2) << S) : 0));
}

template <class F, int S, int LOGC, int LOGT, int MINB, bool STRIDED, bool INV>
cudaError_t launch_t(const PassArgs<F>& a, size_t rows, cudaStream_t st) {
  const int subproblems = STRIDED ? (1 << (a.log_n - a.st0 - S)) : (1 << a.st0);
  dim3 grid(subproblems >> LOGC, static_cast<unsigned>(rows));
  ntt_pass_kernel<F, S, LOGC, LOGT, MINB, STRIDED, INV>
      <<<grid, 1 << LOGT, smem_bytes<F, S, LOGC>(STRIDED), st>>>(a);
  return cudaGetLastError();
}

// Pass geometry of a field: two-pass sizes put 2^LP residues in a CTA,
// 2^LOGEPT per thread, with MINB resident CTAs per SM; single-pass
// transforms (logN <= 11) one row per CTA, 8 residues per thread.
template <int LP_, int LOGEPT_, int MINB_>
struct Geo {
  static constexpr int LP = LP_, LOGEPT = LOGEPT_, MINB = MINB_;
};

template <class F, class G, bool STRIDED, bool INV, typename Fn>
cudaError_t dispatch_geo(int S, int logc, Fn&& f) {
#define HEMUL_NTT_CASE2(s)                                                                   \
  if constexpr (G::LP - s >= 0)                                                             \
    if (S == s && logc == G::LP - s)                                                        \
      return f(ntt_pass_kernel<F, s, G::LP - s, G::LP - G::LOGEPT, G::MINB, STRIDED, INV>,  \
               launch_t<F, s, G::LP - s, G::LP - G::LOGEPT, G::MINB, STRIDED, INV>,         \
               smem_bytes<F, s, G::LP - s>(STRIDED));
#define HEMUL_NTT_CASE1(s)                                                              \
  if (S == s && logc == 0)                                                             \
    return f(ntt_pass_kernel<F, s, 0, s - 3, 2, STRIDED, INV>,                          \
             launch_t<F, s, 0, s - 3, 2, STRIDED, INV>, smem_bytes<F, s, 0>(STRIDED));
  HEMUL_NTT_CASE2(6) HEMUL_NTT_CASE2(7) HEMUL_NTT_CASE2(8) HEMUL_NTT_CASE2(9)
  HEMUL_NTT_CASE1(3) HEMUL_NTT_CASE1(4) HEMUL_NTT_CASE1(5) HEMUL_NTT_CASE1(6)
  HEMUL_NTT_CASE1(7) HEMUL_NTT_CASE1(8) HEMUL_NTT_CASE1(9) HEMUL_NTT_CASE1(10)
  HEMUL_NTT_CASE1(11)
#undef HEMUL_NTT_CASE1
#undef HEMUL_NTT_CASE2
  return cudaErrorInvalidValue;
}

// Measured on B200 at N=2^17 (30-bit basis): 8192 residues x 16 per thread
// beat 4096 x 8 (ntt_a 3.47 -> 2.85 ms, intt_a 3.90 -> 3.17 ms per step) and
// the 3-CTA / 1024-thread / 16384-residue variants.
using GeoF64 = Geo<12, 3, 2>;
using GeoF32 = Geo<13, 4, 2>;
template <class F>
using GeoOf = typename std::conditional<sizeof(typename F::W) == 8, GeoF64, GeoF32>::type;

// A CTA cannot hold more than a whole row: logN = 12 rows use 4096-residue
// CTAs whatever the field.
using GeoSmall = Geo<12, 3, 2>;
template <class F>
int pass_lp(int log_n) {
  return log_n < GeoOf<F>::LP ? GeoSmall::LP : GeoOf<F>::LP;
}

template <class F, bool STRIDED, bool INV, typename Fn>
cudaError_t dispatch(int S, int logc, int lp, Fn&& f) {
  if (lp == GeoOf<F>::LP) return dispatch_geo<F, GeoOf<F>, STRIDED, INV>(S, logc, f);
  return dispatch_geo<F, GeoSmall, STRIDED, INV>(S, logc, f);
}

template <class F>
cudaError_t launch_pass(bool inv, typename F::W* data, const typename F::Tw* tw,
                        const typename F::Prime* primes, int np, size_t rows, int log_n, int st0,
                        int S, bool strided, bool last, cudaStream_t st) {
  if constexpr (sizeof(typename F::W) == 4) {
    // 30-bit basis pass A (forward first pass / inverse last pass): the
    // warp-per-column kernel (ntt_col.cu)
    if (strided && st0 == 0 && log_n >= 12 && last == inv && ntt_col_supported(log_n, S))
      return ntt_col_pass(inv, data, rows, np, log_n, S, tw, primes, st);
  }
  const int rpp = rows % np ? 0 : static_cast<int>(rows / np);
  const PassArgs<F> a{data, tw, primes, np, log_n, st0, rpp, last ? 1 : 0};
  const int lp = pass_lp<F>(log_n);
  const int logc = log_n <= 11 ? 0 : lp - S;
  auto go = [&](auto kernel, auto launcher, size_t) { (void)kernel; return launcher(a, rows, st); };
  if (strided)
    return inv ? dispatch<F, true, true>(S, logc, lp, go)
               : dispatch<F, true, false>(S, logc, lp, go);
  return inv ? dispatch<F, false, true>(S, logc, lp, go)
             : dispatch<F, false, false>(S, logc, lp, go);
}

template <class F, bool STRIDED, bool INV>
cudaError_t set_attrs() {
  auto attr = [](auto kernel, auto, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes));
  };
  for (int lp : {GeoOf<F>::LP, GeoSmall::LP})
    for (int s = 6; s <= 9; ++s) {
      cudaError_t e = dispatch<F, STRIDED, INV>(s, lp - s, lp, attr);
      if (e != cudaSuccess) return e;
    }
  for (int s = 3; s <= 11; ++s) {
    cudaError_t e = dispatch<F, STRIDED, INV>(s, 0, GeoOf<F>::LP, attr);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <class F>
cudaError_t set_all_attrs() {
  cudaError_t e;
  if ((e = set_attrs<F, true, false>()) != cudaSuccess) return e;
  if ((e = set_attrs<F, true, true>()) != cudaSuccess) return e;
  if ((e = set_attrs<F, false, false>()) != cudaSuccess) return e;
  return set_attrs<F, false, true>();
}

}  // namespace

cudaError_t ntt_setup_attributes() {
  cudaError_t e = set_all_attrs<F64>();
  if (e != cudaSuccess) return e;
  return set_all_attrs<F32>();
}

namespace {

// Middle-pass geometry: 2^LM residues per operand per CTA, 2^LOGT threads.
template <int LM_, int LOGT_>
struct MidGeo {
  static constexpr int LM = LM_, LOGT = LOGT_;
};
template <class F, class G, int S, int OP>
cudaError_t launch_mid_g(const MidArgs<F>& a, size_t rows, cudaStream_t st) {
  constexpr int LOGC = G::LM - S;
  constexpr int NSLOT = OP == OP_TENSOR ? 4 : OP == OP_TENSOR2 ? 8 : 2;
  const size_t smem = sizeof(typename F::W) * NSLOT * (size_t(1) << G::LM);
  static bool attr = false;  // one-time opt-in above 48 KB
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ntt_mid_kernel<F, S, LOGC, G::LOGT, OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((1 << a.s1) >> LOGC, static_cast<unsigned>(rows));
  ntt_mid_kernel<F, S, LOGC, G::LOGT, OP><<<grid, 1 << G::LOGT, smem, st>>>(a);
  return cudaGetLastError();
}

template <class F, int S, int OP>
cudaError_t launch_mid(const MidArgs<F>& a, size_t rows, cudaStream_t st) {
  // 2048 residues per operand, 8 per thread: measured faster on B200 for
  // both fields than 4096 x 16 / 2048 x 16 / 4096 x 8
  return launch_mid_g<F, MidGeo<11, 8>, S, OP>(a, rows, st);
}

template <class F, int OP>
cudaError_t launch_mid_any(const MidArgs<F>& a, int s2, size_t rows, cudaStream_t st) {
  switch (s2) {
    case 6: return launch_mid<F, 6, OP>(a, rows, st);
    case 7: return launch_mid<F, 7, OP>(a, rows, st);
    case 8: return launch_mid<F, 8, OP>(a, rows, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool ntt_has_mid(int log_n) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  return s2 >= 6 && s2 <= 8;
}

template <class F>
cudaError_t ntt_mid_tensor(typename F::W* A1, typename F::W* B1, typename F::W* A2,
                           typename F::W* B2, size_t batch, int np, int log_n,
                           const typename F::Tw* tw, const typename F::Tw* itw,
                           const typename F::Prime* primes, cudaStream_t st) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  MidArgs<F> a{};
  a.in[0] = A1;
  a.in[1] = B1;
  a.in[2] = A2;
  a.in[3] = B2;
  a.out[0] = A1;  // d2
  a.out[1] = B1;  // d0
  a.out[2] = A2;  // d1
  a.tw = tw;
  a.itw = itw;
  a.primes = primes;
  a.np = np;
  a.log_n = log_n;
  a.s1 = s1;
  a.rows_per_prime = static_cast<int>(batch);
  return launch_mid_any<F, OP_TENSOR>(a, s2, batch * np, st);
}

cudaError_t ntt_mid_tensor_split(uint32_t* R1, size_t batch, int np, int log_n,
                                 const Twiddle32* tw, const Twiddle32* itw,
                                 const DevPrime32* primes, cudaStream_t st) {
  if (ntt_blk_supported(log_n))  // warp-per-block form (ntt_blk.cu)
    return ntt_blk_tensor_split(R1, batch, np, log_n, tw, itw, primes, st);
  int s1, s2;
  split_levels(log_n, s1, s2);
  MidArgs<F32> a{};
  const size_t slot = batch * size_t(np) << log_n;
  for (int op = 0; op < 8; ++op) a.in[op] = R1 + op * slot;
  for (int op = 0; op < 6; ++op) a.out[op] = R1 + op * slot;
  a.tw = tw;
  a.itw = itw;
  a.primes = primes;
  a.np = np;
  a.log_n = log_n;
  a.s1 = s1;
  a.rows_per_prime = static_cast<int>(batch);
  return launch_mid_any<F32, OP_TENSOR2>(a, s2, batch * np, st);
}

template <class F>
cudaError_t ntt_mid_evk(typename F::W* Fin, const typename F::W* ea, const typename F::W* eb,
                        typename F::W* KA, typename F::W* KB, size_t batch, int np, int log_n,
                        const typename F::Tw* tw, const typename F::Tw* itw,
                        const typename F::Prime* primes, cudaStream_t st) {
  if constexpr (sizeof(typename F::W) == 4) {
    if (ntt_blk_supported(log_n))  // warp-per-block form (ntt_blk.cu)
      return ntt_blk_evk(Fin, ea, eb, KA, KB, batch, np, log_n, tw, itw, primes, st);
  }
  int s1, s2;
  split_levels(log_n, s1, s2);
  MidArgs<F> a{};
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
  return launch_mid_any<F, OP_EVK>(a, s2, batch * np, st);
}

int ntt_pass_a_levels(int log_n) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  return s1;
}

int ntt_num_passes(int log_n) {
  int s1, s2;
  split_levels(log_n, s1, s2);
  return s2 == 0 ? 1 : 2;
}

// Rings below the tiled kernels' smallest pass (n < 8: the SPEC's N = 4
// known answer, test_ntt.cpp:59-93): one thread per row runs the reference's
// radix-2 loops (ntt.cpp:11-57) with canonical Shoup products.
template <class F>
__global__ void ntt_small_kernel(typename F::W* data, size_t rows, int np, int log_n,
                                 const typename F::Tw* tw, const typename F::Prime* primes,
                                 bool inv) {
  using W = typename F::W;
  const size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int n = 1 << log_n;
  const typename F::Prime& pr = primes[r % np];
  const W p = pr.p;
  const typename F::Tw* t = tw + size_t(r % np) * n;
  W* a = data + r * n;
  auto mulw = [&](W x, const typename F::Tw& w) { return shoup_mul(x, w.w, w.wq, p); };
  if (!inv) {
    for (int m = 1, h = n / 2; m < n; m *= 2, h /= 2)
      for (int i = 0; i < m; ++i)
        for (int j = 2 * i * h; j < 2 * i * h + h; ++j) {
          const W u = a[j], v = mulw(a[j + h], t[m + i]);
          a[j] = add_mod(u, v, p);
          a[j + h] = sub_mod(u, v, p);
        }
  } else {
    for (int m = n / 2, h = 1; m >= 1; m /= 2, h *= 2)
      for (int i = 0; i < m; ++i)
        for (int j = 2 * i * h; j < 2 * i * h + h; ++j) {
          const W u = a[j], v = a[j + h];
          a[j] = add_mod(u, v, p);
          a[j + h] = mulw(sub_mod(u, v, p), t[m + i]);
        }
    for (int i = 0; i < n; ++i) a[i] = shoup_mul(a[i], pr.ninv, pr.ninv_q, p);
  }
}

template <class F>
cudaError_t ntt_small(typename F::W* data, size_t rows, int np, int log_n,
                      const typename F::Tw* tw, const typename F::Prime* primes, bool inv,
                      cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  ntt_small_kernel<F><<<static_cast<unsigned>((rows + 127) / 128), 128, 0, st>>>(
      data, rows, np, log_n, tw, primes, inv);
  return cudaGetLastError();
}

template <class F>
cudaError_t ntt_forward_pass(int pass, typename F::W* data, size_t rows, int np, int log_n,
                             const typename F::Tw* tw, const typename F::Prime* primes,
                             cudaStream_t st) {
  if constexpr (sizeof(typename F::W) == 8)
    if (log_n < 3) return ntt_small<F>(data, rows, np, log_n, tw, primes, false, st);
  int s1, s2;
  split_levels(log_n, s1, s2);
  if (pass == 0)
    return launch_pass<F>(false, data, tw, primes, np, rows, log_n, 0, s1, true, s2 == 0, st);
  return launch_pass<F>(false, data, tw, primes, np, rows, log_n, s1, s2, false, true, st);
}

template <class F>
cudaError_t ntt_inverse_pass(int pass, typename F::W* data, size_t rows, int np, int log_n,
                             const typename F::Tw* itw, const typename F::Prime* primes,
                             cudaStream_t st) {
  if constexpr (sizeof(typename F::W) == 8)
    if (log_n < 3) return ntt_small<F>(data, rows, np, log_n, itw, primes, true, st);
  int s1, s2;
  split_levels(log_n, s1, s2);
  if (pass == 0 && s2 > 0)
    return launch_pass<F>(true, data, itw, primes, np, rows, log_n, s1, s2, false, false, st);
  return launch_pass<F>(true, data, itw, primes, np, rows, log_n, 0, s1, true, true, st);
}

#define HEMUL_NTT_INSTANTIATE(F)                                                              \
  template cudaError_t ntt_mid_tensor<F>(F::W*, F::W*, F::W*, F::W*, size_t, int, int,        \
                                         const F::Tw*, const F::Tw*, const F::Prime*,         \
                                         cudaStream_t);                                       \
  template cudaError_t ntt_mid_evk<F>(F::W*, const F::W*, const F::W*, F::W*, F::W*, size_t,  \
                                      int, int, const F::Tw*, const F::Tw*, const F::Prime*,  \
                                      cudaStream_t);                                          \
  template cudaError_t ntt_forward_pass<F>(int, F::W*, size_t, int, int, const F::Tw*,        \
                                           const F::Prime*, cudaStream_t);                    \
  template cudaError_t ntt_inverse_pass<F>(int, F::W*, size_t, int, int, const F::Tw*,        \
                                           const F::Prime*, cudaStream_t);
HEMUL_NTT_INSTANTIATE(F64)
HEMUL_NTT_INSTANTIATE(F32)
#undef HEMUL_NTT_INSTANTIATE

}  // namespace hemul_gpu
