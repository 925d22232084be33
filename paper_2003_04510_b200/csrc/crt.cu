// Forward CRT: big-integer coefficients -> prime-major residues (sm_100a).
//
// Reference: crt_forward / crt_kernel<64> (proj/core/src/rns.cpp:43-106,
// 331-358): r_j(i) = sum_k a_{i,k} (2^64k mod p_j) mod p_j with a 3-word
// accumulator. The result is the canonical a_i mod p_j, so any exact method
// is bit-identical.
//
// B200 form: the small-K integer GEMM of igemm.cuh. A coefficient is re-cut
// into 25-bit chunks c_m (m < K = ceil(bits/25)), every weight
// u_{j,m} = 2^(25m) mod p_j into two 30-bit halves, and
//   C[i][2j+h] = sum_m c_m(i) * half_h(u_{j,m})          (< 2^64 for K <= 480)
//   a_i mod p_j = (C[i][2j] + 2^30 C[i][2j+1]) mod p_j   (two Shoup steps)
// A CTA owns 32 coefficients: their limbs are staged once (contiguous in the
// BigPoly layout) and re-cut in shared memory; the weight columns stream
// through the cp.async ring. Residues are written prime-major directly (no
// transpose; cf. rns_transpose, rns.cpp:303-311, polymul.cpp:13-16).
#include <cuda_runtime.h>

#include <type_traits>

#include "fields.cuh"
#include "igemm.cuh"
#include "kernels.hpp"

namespace hemul_gpu {

namespace {

constexpr int kKT = 32;  // B rows per cp.async stage
constexpr int kStages = 3;



// Input t: polys p[t], converting bits [bit0[t], bit0[t] + bits[t]) of each
// coefficient (the halves of a split operand, context.cu).
struct Inputs {
  const uint64_t* p[kMaxCrtInputs];
  int bit0[kMaxCrtInputs];
  int bits[kMaxCrtInputs];
};

// 25-bit chunk m of one coefficient's field (limbs l)
__device__ __forceinline__ uint32_t chunk_of(const uint64_t* l, int limbs, int bit0, int bits,
                                             int m) {
  const int lim = bits - 25 * m;
  if (lim <= 0) return 0;
  const int bit = bit0 + 25 * m, k = bit >> 6, off = bit & 63;
  uint64_t v = k < limbs ? l[k] >> off : 0;
  if (off > 39 && k + 1 < limbs) v |= l[k + 1] << (64 - off);
  return static_cast<uint32_t>(v) & (lim >= 25 ? 0x1ffffffu : (1u << lim) - 1);
}

// Residues of the thread's 4 coefficients x 4 accumulator columns. F64: the
// column pair (2j, 2j+1) holds the 30-bit halves of prime j's weights,
// V = X + 2^30 Y reduced with two Shoup steps. F32: column j is prime j,
// one 64 -> 32 reduction. obase points at coefficient 4 cg of prime 0.
template <class F>
__device__ __forceinline__ void crt_store(const uint64_t (&acc)[4][4], int col,
                                          const typename F::Prime* __restrict__ primes, int np,
                                          size_t n, typename F::W* obase) {
  if constexpr (F::kCrtColsPerPrime == 2) {
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int j = col / 2 + pp;
      if (j >= np) continue;
      const DevPrime& pr = primes[j];
      const uint64_t negp = 0 - pr.p;
      uint64_t r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t x = acc[i][2 * pp], y = acc[i][2 * pp + 1];
        const uint64_t vlo = x + (y << 30);
        const uint64_t vhi = (y >> 34) + (vlo < x);
        const uint64_t r0 = shoup_mul_4p(vlo, 1, pr.one_q, negp);
        const uint64_t r1 = shoup_mul_4p(vhi, pr.beta, pr.beta_q, negp);
        r[i] = reduce_4p(csub(r0 + r1, 4 * pr.p), pr.p);
      }
      uint64_t* dst = obase + size_t(j) * n;
      reinterpret_cast<ulonglong2*>(dst)[0] = make_ulonglong2(r[0], r[1]);
      reinterpret_cast<ulonglong2*>(dst)[1] = make_ulonglong2(r[2], r[3]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = col + q;
      if (j >= np) continue;
      const DevPrime32& pr = primes[j];
      const uint32_t negp = 0u - pr.p;
      uint32_t r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        r[i] = csub32(reduce64_32(acc[i][q], pr.p, negp, pr.one_q, pr.beta, pr.beta_q), pr.p);
      *reinterpret_cast<uint4*>(obase + size_t(j) * n) = make_uint4(r[0], r[1], r[2], r[3]);
    }
  }
}

template <class F, int NW>
__global__ void __launch_bounds__(NW * 32) crt_kernel(Inputs in, int B, int limbs, int log_n,
                                                      CrtWeights w,
                                                      const typename F::Prime* __restrict__ primes,
                                                      int np, typename F::W* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NC = 16 * NW;
  const size_t n = size_t(1) << log_n;
  const int bt = blockIdx.y;  // input t = bt / B, batch entry bt % B
  const int t = bt / B, b = bt - t * B;
  const size_t c0 = size_t(blockIdx.x) * kGemmCoefs;
  const int K = w.chunks;
  uint32_t* A = reinterpret_cast<uint32_t*>(smem);                          // [K][32]
  uint32_t* Bs = A + K * kGemmCoefs;                                        // ring
  uint64_t* raw = reinterpret_cast<uint64_t*>(Bs + kStages * kKT * NC);    // [32][limbs]
  const uint64_t* src = in.p[t] + (size_t(b) * n + c0) * limbs;
  // the CTA's limbs are one contiguous run: 16-byte cp.async copies
  for (int idx = threadIdx.x; idx < kGemmCoefs * limbs / 2; idx += blockDim.x)
    cp_async16(raw + 2 * idx, src + 2 * idx);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int idx = threadIdx.x; idx < kGemmCoefs * K; idx += blockDim.x) {
    const int m = idx >> 5, c = idx & 31;
    A[idx] = chunk_of(raw + c * limbs, limbs, in.bit0[t], in.bits[t], m);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane & 7, ng = lane >> 3;
  typename F::W* obase = out + size_t(t) * B * np * n + size_t(b) * np * n + c0 + 4 * cg;
  // (igemm_32xN synchronises before touching A; the CTA-wide ring measured
  // faster than per-warp rings here: 11 warps share each 704-byte B row)
  for (int col0 = 0; col0 < w.ld; col0 += NC) {
    uint64_t acc[4][4] = {};
    igemm_32xN<NW, kKT, kStages>(A, K, w.wtab, w.ld, col0, Bs, acc);
    crt_store<F>(acc, col0 + 16 * warp + 4 * ng, primes, np, n, obase);
  }
}

// ---- persistent variant: the CTA's weight columns stay in shared memory ---
//
// The weight table is the same for every coefficient, so a persistent CTA
// loads its column tile (K x 16 NW words) once and then walks coefficient
// tiles, double-buffering each tile's limbs with cp.async so the next tile's
// HBM reads overlap this tile's IMAD.WIDE loop. grid = (CTAs per column
// tile, column tiles).
template <class F, int NW>
__global__ void __launch_bounds__(NW * 32) crt_persistent_kernel(
    Inputs in, int count, int B, int limbs, int log_n, CrtWeights w,
    const typename F::Prime* __restrict__ primes, int np, typename F::W* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NC = 16 * NW;
  const size_t n = size_t(1) << log_n;
  const int K = w.chunks;
  const int col0 = blockIdx.y * NC;
  uint32_t* Bsm = reinterpret_cast<uint32_t*>(smem);       // [K][NC]
  uint32_t* A = Bsm + K * NC;                                // [K][32]
  uint64_t* raw = reinterpret_cast<uint64_t*>(A + K * kGemmCoefs);  // [2][32 * limbs]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cg = lane & 7, ng = lane >> 3;
  const int coef_tiles = static_cast<int>(n / kGemmCoefs);
  const int tiles = count * B * coef_tiles;
  const int rawsz = kGemmCoefs * limbs;
  // weight tile, once
  for (int idx = tid; idx < K * (NC / 4); idx += NW * 32) {
    const int k = idx / (NC / 4), c = idx - k * (NC / 4);
    cp_async16(Bsm + k * NC + 4 * c, w.wtab + size_t(k) * w.ld + col0 + 4 * c);
  }
  auto fetch = [&](int tile, uint64_t* dst) {
    const int ct = tile % coef_tiles, bt = tile / coef_tiles;  // bt = t * B + b
    const int t = bt / B, b = bt - t * B;
    const uint64_t* src = in.p[t] + (size_t(b) * n + size_t(ct) * kGemmCoefs) * limbs;
    for (int idx = tid; idx < rawsz / 2; idx += NW * 32) cp_async16(dst + 2 * idx, src + 2 * idx);
  };
  int tile = blockIdx.x;
  if (tile < tiles) fetch(tile, raw);
  cp_async_commit();
  for (int it = 0; tile < tiles; tile += gridDim.x, ++it) {
    uint64_t* cur = raw + (it & 1) * rawsz;
    cp_async_wait<0>();
    __syncthreads();  // limbs of this tile (and the weights) are in; A is free
    if (tile + gridDim.x < tiles) fetch(tile + gridDim.x, raw + ((it + 1) & 1) * rawsz);
    cp_async_commit();
    const int tin = tile / coef_tiles / B;  // input of this tile
    for (int idx = tid; idx < kGemmCoefs * K; idx += NW * 32) {
      const int m = idx >> 5, c = idx & 31;
      A[idx] = chunk_of(cur + c * limbs, limbs, in.bit0[tin], in.bits[tin], m);
    }
    __syncthreads();
    uint64_t acc[4][4] = {};
    const uint32_t* ap = A + 4 * cg;
    const uint32_t* bp = Bsm + 16 * warp + 4 * ng;
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
      const uint4 a = *reinterpret_cast<const uint4*>(ap + k * kGemmCoefs);
      const uint4 b = *reinterpret_cast<const uint4*>(bp + k * NC);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] += static_cast<uint64_t>(av[i]) * bv[q];
    }
    const int ct = tile % coef_tiles, bt = tile / coef_tiles;
    typename F::W* obase = out + size_t(bt) * np * n + size_t(ct) * kGemmCoefs + 4 * cg;
    crt_store<F>(acc, col0 + 16 * warp + 4 * ng, primes, np, n, obase);
  }
  cp_async_wait<0>();
}

template <int NW>
size_t crt_persistent_smem(int limbs, int K) {
  return size_t(K) * 16 * NW * 4 + size_t(K) * kGemmCoefs * 4 +
         2 * size_t(kGemmCoefs) * limbs * 8;
}

int nw_for(int ld) { return ld <= 192 ? ld / 16 : 8; }

template <int NW>
size_t crt_smem(int limbs, int K) {
  return size_t(K) * kGemmCoefs * 4 + size_t(kStages) * kKT * 16 * NW * 4 +
         size_t(kGemmCoefs) * limbs * 8;
}

template <class F, int NW>
cudaError_t launch(const Inputs& in, int count, int limbs, size_t batch, int log_n,
                   const CrtWeights& w, const typename F::Prime* primes, int np,
                   typename F::W* out, cudaStream_t st) {
  const size_t n = size_t(1) << log_n;
  dim3 grid(static_cast<unsigned>(n / kGemmCoefs), static_cast<unsigned>(count * batch));
  crt_kernel<F, NW><<<grid, NW * 32, crt_smem<NW>(limbs, w.chunks), st>>>(
      in, static_cast<int>(batch), limbs, log_n, w, primes, np, out);
  return cudaGetLastError();
}

template <typename F>
cudaError_t with_nw(int nw, F&& f) {
  switch (nw) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    case 7: return f(std::integral_constant<int, 7>{});
    case 8: return f(std::integral_constant<int, 8>{});
    case 9: return f(std::integral_constant<int, 9>{});
    case 10: return f(std::integral_constant<int, 10>{});
    case 11: return f(std::integral_constant<int, 11>{});
    case 12: return f(std::integral_constant<int, 12>{});
    default: return cudaErrorInvalidValue;
  }
}

template <class F>
cudaError_t crt_attrs() {
  for (int nw = 1; nw <= 12; ++nw) {
    cudaError_t e = with_nw(nw, [](auto v) {
      cudaError_t e2 = cudaFuncSetAttribute(crt_kernel<F, decltype(v)::value>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kMaxDynSmem);
      if (e2 != cudaSuccess) return e2;
      return cudaFuncSetAttribute(crt_persistent_kernel<F, decltype(v)::value>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    });
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t crt_setup_attributes() {
  cudaError_t e = crt_attrs<F64>();
  return e != cudaSuccess ? e : crt_attrs<F32>();
}

template <class F>
cudaError_t crt_forward_multi(const uint64_t* const* polys, int count, int limbs, size_t batch,
                              int log_n, const CrtWeights& w, const typename F::Prime* primes,
                              int np, typename F::W* out, cudaStream_t st, const int* bit0,
                              const int* bits) {
  const size_t n = size_t(1) << log_n;
  if (count < 1 || count > kMaxCrtInputs || n < kGemmCoefs || w.chunks > kMaxGemmK)
    return cudaErrorInvalidValue;
  Inputs in{};
  for (int t = 0; t < count; ++t) {
    in.p[t] = polys[t];
    in.bit0[t] = bit0 ? bit0[t] : 0;
    in.bits[t] = bits ? bits[t] : 25 * w.chunks;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return with_nw(nw_for(w.ld), [&](auto v) {
    constexpr int NW = decltype(v)::value;
    const size_t psmem = crt_persistent_smem<NW>(limbs, w.chunks);
    int resident = 0;  // persistent CTAs per SM at this shared-memory size
    if (psmem <= 110 * 1024 &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, crt_persistent_kernel<F, NW>,
                                                      NW * 32, psmem) != cudaSuccess)
      return cudaGetLastError();
    if (resident >= 2) {
      const int col_tiles = w.ld / (16 * NW);
      const int tiles = static_cast<int>(count * batch * (n / kGemmCoefs));
      const int per = std::max(1, std::min(tiles, resident * sms / col_tiles));
      crt_persistent_kernel<F, NW><<<dim3(per, col_tiles), NW * 32, psmem, st>>>(
          in, count, static_cast<int>(batch), limbs, log_n, w, primes, np, out);
      return cudaGetLastError();
    }
    return launch<F, NW>(in, count, limbs, batch, log_n, w, primes, np, out, st);
  });
}

template <class F>
cudaError_t crt_forward(const uint64_t* poly, int limbs, size_t batch, int log_n,
                        const CrtWeights& w, const typename F::Prime* primes, int np,
                        typename F::W* out, cudaStream_t st) {
  return crt_forward_multi<F>(&poly, 1, limbs, batch, log_n, w, primes, np, out, st, nullptr,
                              nullptr);
}

#define HEMUL_CRT_INSTANTIATE(F)                                                              \
  template cudaError_t crt_forward_multi<F>(const uint64_t* const*, int, int, size_t, int,    \
                                            const CrtWeights&, const F::Prime*, int, F::W*,   \
                                            cudaStream_t, const int*, const int*);            \
  template cudaError_t crt_forward<F>(const uint64_t*, int, size_t, int, const CrtWeights&,   \
                                      const F::Prime*, int, F::W*, cudaStream_t);
HEMUL_CRT_INSTANTIATE(F64)
HEMUL_CRT_INSTANTIATE(F32)
#undef HEMUL_CRT_INSTANTIATE

}  // namespace hemul_gpu
