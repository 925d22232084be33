// Forward CRT on the int8 tensor cores (sm_100a tcgen05, 30-bit basis).
//
// Reference: crt_forward / crt_kernel<64> (proj/core/src/rns.cpp:43-106,
// 331-358): r_j(i) = sum_k a_{i,k} (2^64k mod p_j) mod p_j. Any exact method
// gives the canonical a_i mod p_j, so the result is bit-identical.
//
// B200 form: the coefficient's own bytes are the GEMM's A operand (the
// BigPoly layout is coefficient-major: row i = limbs * 8 little-endian
// bytes), the weights u_{j,k} = 2^(8k) mod p_j (< 2^30) are cut into four
// byte planes, and one u8 x u8 -> s32 tensor-core GEMM gives
//   D[i][4j+b] = sum_k a_{i,k} byte_b(u_{j,k})        (< K 2^16: exact)
//   a_i mod p_j = (D0 + 2^8 D1 + 2^16 D2 + 2^24 D3) 2^-32 mod p_j  (epilogue;
//   the weights carry 2^32: one Montgomery step)
// with no carries anywhere. A coefficient costs K x 4 np MACs on a
// 4.1 POPS pipe instead of ceil(bits/25) x np IMAD.WIDE on a 8 T/s pipe.
//
// Persistent, warp-specialised CTA (one per SM): the column tile of the
// weight table (col_tile = 4 x primes-per-tile columns) stays resident in
// shared memory; 128-coefficient tiles stream through an S-stage A ring
// filled by 4 producer warps with zero-filling cp.async (128-byte-swizzled
// K-major); one thread issues the MMAs into one of two TMEM accumulators;
// 16 epilogue warps (four per TMEM lane quadrant) turn each coefficient's 4
// planes per prime into a residue and store the prime-major rows directly
// (no transpose, cf. rns_transpose rns.cpp:303-311).
//
// Inputs must be reduced (bits >= the field's end zero, the BigPoly
// invariant poly.cpp:12-18): the copies are byte-granular.
#include <cuda_runtime.h>

#include <algorithm>

#include "fields.cuh"
#include "igemm.cuh"
#include "kernels.hpp"
#include "tc.cuh"

namespace hemul_gpu {

namespace {

constexpr int kRows = 128;           // coefficients per tile (TMEM lanes)
#ifndef HEMUL_CRT_ABL
#define HEMUL_CRT_ABL 0  // ablations: 1 = no plane combination, 2 = no A loads (wrong results)
#endif
#ifndef HEMUL_CRT_EPI_WARPS
#define HEMUL_CRT_EPI_WARPS 16
#endif
constexpr int kEpiWarps = HEMUL_CRT_EPI_WARPS;  // four per TMEM lane quadrant (prime groups split); the
                                     // epilogue is latency bound: 8 -> 16 warps, 2.20 -> 1.93 ms
                                     // per step at X
constexpr int kMmaWarp = kEpiWarps;  // TMEM allocation + MMA issue
constexpr int kProdWarps = 4;
constexpr int kThreads = 32 * (kEpiWarps + 1 + kProdWarps);
constexpr int kMaxStages = 4;
constexpr int kMaxTilePrimes = 64;

struct TcInputs {
  const uint64_t* p[kMaxCrtInputs];
  const uint8_t* btab[2];       // the (at most two) distinct weight tables
  int slot[kMaxCrtInputs];      // input t's table
  int limb0[kMaxCrtInputs];
  int end_bit[kMaxCrtInputs];
  int aligned16[kMaxCrtInputs];  // rows and the field start 16-byte aligned
};

__host__ __device__ inline uint32_t round128(uint32_t k) { return (k + 127) & ~127u; }

// bytes of limb l (of `limbs`) below end_bit: the cp.async source size
__device__ __forceinline__ uint32_t limb_bytes(int l, int limbs, int end_bit) {
  if (l >= limbs) return 0;
  const int lim = end_bit - 64 * l;
  return lim <= 0 ? 0u : lim >= 64 ? 8u : uint32_t((lim + 7) >> 3);
}

// (d0 + 2^8 d1 + 2^16 d2 + 2^24 d3) 2^-32 mod p, lazy in [0, 2p) (inside the
// forward NTT's input domain [0, 4p), fields.cuh F32::ct), for plane sums
// d_b < 2^26. The table weights carry the factor 2^32 (build_crt_tc), so this
// is a mod p. z = d0 + ... < 2^51, then one Montgomery step: m = z (-p^-1)
// mod 2^32, (z + m p) / 2^32 < 2^19 + p < 2p (z + m p < 2^63: no overflow).
__device__ __forceinline__ uint32_t planes_mont(uint32_t d0, uint32_t d1, uint32_t d2,
                                                uint32_t d3, uint32_t p, uint32_t pinv) {
  // z = d0 + 2^8 d1 + 2^16 d2 + 2^24 d3 < 2^51: three IMAD.WIDE
  uint64_t z = static_cast<uint64_t>(d1) * 256u + d0;
  z += static_cast<uint64_t>(d2) * 65536u;
  z += static_cast<uint64_t>(d3) * 16777216u;
  // Montgomery: m = -z / p mod 2^32, (z + m p) / 2^32 exactly (one IMAD.WIDE)
  const uint32_t m = static_cast<uint32_t>(z) * pinv;
  return static_cast<uint32_t>((z + static_cast<uint64_t>(m) * p) >> 32);
}

#define LOGN_OR(x) (LOGN > 0 ? LOGN : (x))

// -p^-1 mod 2^32 (p odd): Newton, 5 steps from inv = p (correct to 3 bits)
__device__ __forceinline__ uint32_t neg_inv32(uint32_t p) {
  uint32_t inv = p;
#pragma unroll
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  return 0u - inv;
}

// LOGN > 0: the ring degree is a compile-time constant, so the epilogue's
// stores to the prime rows j, j+1, ... (n residues apart) take immediate
// offsets instead of a 64-bit address add each (LOGN = 0: any degree)
template <int LOGN>
__global__ void __launch_bounds__(kThreads, 1)
    crt_tc_kernel(TcInputs in, int count, int B, int limbs, int log_n, CrtTcTable tab,
                  const DevPrime32* __restrict__ primes, int np, uint32_t* __restrict__ out,
                  int stages, int nslots, int tS) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t a_full[kMaxStages], a_empty[kMaxStages], t_full[2], t_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ uint2 eprimes[kMaxTilePrimes];  // {p, -p^-1 mod 2^32} of the tile's primes
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_addr(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t n = size_t(1) << (LOGN > 0 ? LOGN : log_n);
  const int kpad = tab.kpad;                  // K bytes the MMAs read (multiple of 32)
  const uint32_t kcols = round128(kpad);      // K bytes per smem row (atom columns)
  const int ct = blockIdx.x % tab.ncol_tiles;  // this CTA's column tile
  const int cta_in_ct = blockIdx.x / tab.ncol_tiles;
  const int ctas_per_ct = gridDim.x / tab.ncol_tiles;
  const int col_tile = tab.col_tile;
  uint8_t* sB = smem;                                   // nslots x [col_tile][kcols]
  const uint32_t b_bytes = uint32_t(col_tile) * kcols;
  uint8_t* sA = smem + size_t(nslots) * b_bytes;        // stages x [128][kcols]
  const uint32_t a_bytes = kRows * kcols;
  const int tiles_per_poly = static_cast<int>(n / kRows);
  const int jbase = ct * tab.primes_per_tile;
  const int pcount = min(tab.primes_per_tile, np - jbase);

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&a_full[s], kProdWarps * 32);
      tc::mbar_init(&a_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&t_full[a], 1);
      tc::mbar_init(&t_empty[a], kEpiWarps * 32);
    }
    tc::mbar_fence_init();
  }
  for (int j = threadIdx.x; j < pcount; j += kThreads) {
    const DevPrime32& pr = primes[jbase + j];
    eprimes[j] = make_uint2(pr.p, neg_inv32(pr.p));
  }
  if (warp == kMmaWarp) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  // Both weight tables (the low and high halves' of split region 1, or the
  // one of region 2) stay resident. A CTA walks coefficient blocks (batch
  // entry b, 128 coefficients at ci) and converts every input's field of the
  // block in turn, so the halves of one poly read the same rows back to back.
  for (int sl = 0; sl < nslots; ++sl) {
    const uint8_t* g = in.btab[sl] + size_t(ct) * col_tile * kpad;
    const int chunks = kpad / 16;
    for (int idx = threadIdx.x; idx < col_tile * chunks; idx += kThreads) {
      const int r = idx / chunks, c = idx - r * chunks;
      tc::cp_async16z(tc::smem_addr(sB + sl * b_bytes + tc::kmaj_sw128(r, 16 * c, col_tile)),
                      g + size_t(r) * kpad + 16 * c, 16);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  tc::fence_async_smem();
  __syncthreads();
  int it = 0;  // local tile counter (ring / accumulator phases)
  const int poly_tiles = B * tiles_per_poly;
  int b = cta_in_ct / tiles_per_poly, ci = cta_in_ct - b * tiles_per_poly;
  const int step_b = ctas_per_ct / tiles_per_poly, step_c = ctas_per_ct - step_b * tiles_per_poly;
  for (int blk = cta_in_ct; blk < poly_tiles; blk += ctas_per_ct) {
  for (int t = 0; t < count; ++t) {
    const size_t i0 = size_t(ci) * kRows;
    const int s = it % stages;
    const int acc = it & 1;
    if (warp > kMmaWarp) {
      // ---- producers: 128 rows x kpad bytes of the input field -> sA[s] by
      // cp.async (zero-filled past the field); the stage's barrier completes
      // when every producer thread's copies have landed
      const int pt = threadIdx.x - 32 * (kMmaWarp + 1);
      tc::mbar_wait_sleep<32>(&a_empty[s], ((it / stages) & 1) ^ 1);
      uint8_t* dstA = sA + s * a_bytes;
      // output positions i0 .. i0+127; their coefficients: the same (natural
      // layout, tS = 0) or, in the column-major layout of NTT pass A (tS = S:
      // position x 2^S + y holds coefficient y n / 2^S + x), one column's
      // coefficients n / 2^S apart
      const size_t cb = tS ? ((i0 & ((size_t(1) << tS) - 1)) << (LOGN_OR(log_n) - tS)) | (i0 >> tS)
                           : i0;
      const size_t rs = tS ? size_t(1) << (LOGN_OR(log_n) - tS) : 1;
      const uint64_t* base = in.p[t] + (size_t(b) * n + cb) * limbs;
      const int chunks = kpad / 16;  // 16-byte chunks per row
      const int l0 = in.limb0[t], eb = in.end_bit[t];
      const bool al16 = in.aligned16[t] != 0;
      // thread -> rows 4 pw + lane / 8 + 16 i (i < 8), chunks lane % 8 + 8 m:
      // 8 lanes cover 128 contiguous bytes of a row; moving 16 rows down
      // moves 2048 bytes in the swizzled tile (no index division)
      const int pw = pt >> 5, r0 = 4 * pw + (lane >> 3);
      const uint64_t* rowp = base + size_t(r0) * rs * limbs;
      const size_t rstride = 16 * rs * limbs;  // 16 rows down
      const uint32_t sa0 = tc::smem_addr(dstA);
      for (int c = lane & 7; c < (HEMUL_CRT_ABL == 2 ? 0 : chunks); c += 8) {
        const int l = l0 + 2 * c;
        const uint32_t b0 = limb_bytes(l, limbs, eb), b1 = limb_bytes(l + 1, limbs, eb);
        const uint32_t dst = sa0 + tc::kmaj_sw128(r0, 16 * c, kRows);
        if (al16) {
          const uint32_t sz = b0 + (b0 == 8 ? b1 : 0);
          const uint64_t* g = sz ? rowp + l : rowp;
#pragma unroll
          for (int i = 0; i < kRows / 16; ++i)
            tc::cp_async16z(dst + 2048 * i, g + i * rstride, sz);
        } else {
          const uint64_t* g0 = b0 ? rowp + l : rowp;
          const uint64_t* g1 = b1 ? rowp + l + 1 : rowp;
#pragma unroll
          for (int i = 0; i < kRows / 16; ++i) {
            tc::cp_async8z(dst + 2048 * i, g0 + i * rstride, b0);
            tc::cp_async8z(dst + 2048 * i + 8, g1 + i * rstride, b1);
          }
        }
      }
      tc::cp_async_mbar_arrive(&a_full[s]);
    } else if (warp == kMmaWarp) {
      // ---- MMA issue (one thread)
      if (lane == 0) {
        tc::mbar_wait(&a_full[s], (it / stages) & 1);
        tc::fence_async_smem();  // cp.async (generic proxy) data -> tensor core
        tc::mbar_wait(&t_empty[acc], ((it >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t a0 = tc::smem_addr(sA + s * a_bytes);
        const uint32_t b0 = tc::smem_addr(sB + in.slot[t] * b_bytes);
        const uint32_t idesc = tc::idesc_u8(kRows, col_tile, 0, 0);
        const uint32_t d = tmem + acc * 256;
        for (int k = 0; k < kpad / 32; ++k)
          tc::mma_u8(d, tc::kmaj_sw128_desc(a0, k, kRows), tc::kmaj_sw128_desc(b0, k, col_tile),
                     idesc, k > 0);
        tc::mma_commit(&a_empty[s]);
        tc::mma_commit(&t_full[acc]);
      }
      __syncwarp();
    } else {
      // ---- epilogue: lane quadrant warp % 4 (coefficient i0 + 32 (warp % 4)
      // + lane), prime groups split between the two warps of a quadrant
      tc::mbar_wait_sleep<64>(&t_full[acc], (it >> 1) & 1);
      tc::fence_after();
      const int quad = warp & 3, part = warp >> 2;  // part < kEpiWarps / 4
      const uint32_t taddr = tmem + acc * 256 + (uint32_t(32 * quad) << 16);
      const int groups = (pcount + 3) / 4;  // 4 primes = 16 TMEM columns
      constexpr int kParts = kEpiWarps / 4;
      const int g0 = part * groups / kParts, g1 = (part + 1) * groups / kParts;
      uint32_t* o =
          out + (size_t(t) * B + b) * np * n + size_t(jbase) * n + i0 + 32 * quad + lane;
      for (int g = g0; g < g1; g += 2) {
        // two TMEM loads in flight per wait
        uint32_t v[32];
        tc::tmem_ld16(taddr + 16 * g, *reinterpret_cast<uint32_t(*)[16]>(v));
        if (g + 1 < g1) tc::tmem_ld16(taddr + 16 * g + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
        tc::tmem_wait_ld();
        uint32_t* op = o + size_t(4 * g) * n;
        const int jn = min((g + 1 < g1) ? 8 : 4, pcount - 4 * g);  // primes in this pair
        if (jn == 8) {  // full pair: no per-prime predicate
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint2 e = eprimes[4 * g + q];
            op[q * n] = HEMUL_CRT_ABL == 1 ? v[4 * q] ^ v[4 * q + 3]
                                           : planes_mont(v[4 * q], v[4 * q + 1], v[4 * q + 2],
                                                         v[4 * q + 3], e.x, e.y);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < jn) {
              const uint2 e = eprimes[4 * g + q];
              op[q * n] = planes_mont(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3], e.x, e.y);
            }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&t_empty[acc]);
    }
    ++it;
  }
    ci += step_c;
    b += step_b;
    if (ci >= tiles_per_poly) ci -= tiles_per_poly, ++b;
  }
  cp_async_wait<0>();
  tc::fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

size_t crt_tc_smem(const CrtTcTable& tab, int* stages, int nslots = 1) {
  const size_t kc = round128(tab.kpad);
  const size_t b = size_t(nslots) * tab.col_tile * kc, a = kRows * kc;
  const size_t cap = kMaxDynSmem - 1024;
  int s = kMaxStages;
  while (s > 2 && b + s * a > cap) --s;
  if (stages) *stages = s;
  return b + s * a + 1024;
}

bool crt_tc_supported(const CrtTcTable& tab) {
  int s = 0;
  const size_t need = crt_tc_smem(tab, &s);
  return tab.btab && tab.col_tile <= 256 && tab.col_tile % 16 == 0 && tab.kpad % 32 == 0 &&
         need <= size_t(kMaxDynSmem);
}

cudaError_t crt_tc_setup_attributes() {
  cudaError_t e = cudaFuncSetAttribute(crt_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kMaxDynSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(crt_tc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kMaxDynSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(crt_tc_kernel<17>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kMaxDynSmem);
  return e;
}

cudaError_t crt_forward_tc(const uint64_t* const* polys, const CrtTcTable* tabs, int count,
                           int limbs, size_t batch, int log_n, const DevPrime32* primes, int np,
                           uint32_t* out, cudaStream_t st, int transposed_S) {
  const size_t n = size_t(1) << log_n;
  if (count < 1 || count > kMaxCrtInputs || n < size_t(kRows)) return cudaErrorInvalidValue;
  if (transposed_S && (transposed_S < 7 || transposed_S >= log_n)) return cudaErrorInvalidValue;
  TcInputs in{};
  CrtTcTable tab = tabs[0];
  int nslots = 0;
  for (int t = 0; t < count; ++t) {
    if (tabs[t].kpad != tab.kpad || tabs[t].col_tile != tab.col_tile ||
        tabs[t].ncol_tiles != tab.ncol_tiles || !crt_tc_supported(tabs[t]))
      return cudaErrorInvalidValue;
    in.p[t] = polys[t];
    int sl = 0;
    while (sl < nslots && in.btab[sl] != tabs[t].btab) ++sl;
    if (sl == nslots) {
      if (nslots == 2) return cudaErrorInvalidValue;  // at most two distinct tables
      in.btab[nslots++] = tabs[t].btab;
    }
    in.slot[t] = sl;
    in.limb0[t] = tabs[t].limb0;
    in.end_bit[t] = tabs[t].end_bit;
    in.aligned16[t] = limbs % 2 == 0 && tabs[t].limb0 % 2 == 0 &&
                      reinterpret_cast<uintptr_t>(polys[t]) % 16 == 0;
  }
  if (tab.primes_per_tile > kMaxTilePrimes) return cudaErrorInvalidValue;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int stages = 0;
  const size_t smem = crt_tc_smem(tab, &stages, nslots);
  if (smem > size_t(kMaxDynSmem)) return cudaErrorInvalidValue;
  const int per_ct = std::max(1, sms / tab.ncol_tiles);
  const int grid = per_ct * tab.ncol_tiles;
  auto kern = log_n == 17 ? crt_tc_kernel<17> : log_n == 16 ? crt_tc_kernel<16> : crt_tc_kernel<0>;
  kern<<<grid, kThreads, smem, st>>>(in, count, static_cast<int>(batch), limbs, log_n, tab, primes,
                                     np, out, stages, nslots, transposed_S);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
