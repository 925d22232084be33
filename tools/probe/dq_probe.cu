// Probe: throughput of the 30-bit Harvey CT butterfly with the Shoup quotient
// from IMAD.HI (fields.cuh shoup32) against a quotient from one DFMA on the
// FP64 pipe (q = floor(x w~), w~ = w / p rounded down to a multiple of 2^-53,
// computed as the low word of fma_rz(2^52 + x, w~, 2^52 (1 - w~))), which
// leaves the low products r = x w - q p to the integer pipe.
// Also checks the DFMA quotient gives a result in [0, 2p) congruent to x w.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dq_probe dq_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t csub32(uint32_t x, uint32_t m) { return min(x, x - m); }

__device__ __forceinline__ uint32_t shoup_hi(uint32_t x, uint32_t w, uint32_t wq, uint32_t negp) {
  return x * w + __umulhi(x, wq) * negp;
}
__device__ __forceinline__ uint32_t shoup_dp(uint32_t x, uint32_t w, double wd, double c,
                                             uint32_t negp) {
  const double xd = __hiloint2double(0x43300000, static_cast<int>(x));
  const uint32_t q = static_cast<uint32_t>(__double2loint(__fma_rz(xd, wd, c)));
  return x * w + q * negp;
}

template <int MODE>
__global__ void bench(uint32_t* out, uint32_t p, uint32_t w0, uint32_t wq0, double wd0, double c0,
                      int iters) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t p2 = 2 * p, negp = 0u - p;
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (tid * 2654435761u + i * 40503u) % p;
  const uint32_t w = w0, wq = wq0;
  const double wd = wd0, c = c0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t& a = v[i];
      uint32_t& b = v[i + 8];
      const uint32_t u = csub32(a, p2);
      const uint32_t t = MODE == 0 ? shoup_hi(b, w, wq, negp) : shoup_dp(b, w, wd, c, negp);
      a = u + t;
      b = u + p2 - t;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // second level: pairs (i, i + 4) within halves
      const int x = (i & 3) + (i >> 2) * 8;
      uint32_t& a = v[x];
      uint32_t& b = v[x + 4];
      const uint32_t u = csub32(a, p2);
      const uint32_t t = MODE == 0 ? shoup_hi(b, w, wq, negp) : shoup_dp(b, w, wd, c, negp);
      a = u + t;
      b = u + p2 - t;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= v[i];
  out[tid] = s;
}

__global__ void check(uint32_t* bad, uint32_t p, uint32_t w, double wd, double c, uint64_t seed) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint64_t s = seed ^ (tid * 0x9E3779B97F4A7C15ull);
  for (int k = 0; k < 64; ++k) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    uint32_t x = static_cast<uint32_t>(s);
    if (k == 0) x = 0xFFFFFFFFu - static_cast<uint32_t>(tid);  // near the top
    const uint32_t r = shoup_dp(x, w, wd, c, 0u - p);
    const uint64_t want = (uint64_t(x) * w) % p;
    if (r >= 2 * p || r % p != want) atomicAdd(bad, 1u);
  }
}

static double wtilde(uint32_t w, uint32_t p) {
  // floor(w 2^53 / p) 2^-53 (exact: w 2^53 / p < 2^53), minus one unit
  const unsigned __int128 num = (unsigned __int128)w << 53;
  const uint64_t k = static_cast<uint64_t>(num / p);
  return (double)(k ? k - 1 : 0) * 0x1p-53;
}

int main() {
  const uint32_t primes[3] = {1073479681u, 1068236801u, 998244353u};
  uint32_t *out, *bad;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaMalloc(&bad, 4);
  for (uint32_t p : primes) {
    for (uint32_t w : {1u, 2u, p - 1, p / 3, 123456789u % p, p - 2}) {
      const double wd = wtilde(w, p), c = 0x1p52 * (1.0 - wd);
      cudaMemset(bad, 0, 4);
      check<<<4096, 256>>>(bad, p, w, wd, c, 12345 + w);
      uint32_t nb = 0;
      cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost);
      printf("check p=%u w=%u: %u bad of %d\n", p, w, nb, 4096 * 256 * 64);
    }
  }
  const uint32_t p = primes[0], w = 987654321u % p;
  const uint32_t wq = static_cast<uint32_t>((uint64_t(w) << 32) / p);
  const double wd = wtilde(w, p), c = 0x1p52 * (1.0 - wd);
  const int iters = 4096;
  for (int blocks_per_sm : {4, 8}) {
    const int grid = 148 * blocks_per_sm;
    for (int mode = 0; mode < 2; ++mode) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) bench<0><<<grid, 256>>>(out, p, w, wq, wd, c, iters);
        else bench<1><<<grid, 256>>>(out, p, w, wq, wd, c, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bfly = double(grid) * 256 * iters * 16;
      printf("mode %s blocks/SM %d: %.3f ms, %.1f G butterflies/s (%s)\n",
             mode ? "dfma-quotient" : "imad.hi-quotient", blocks_per_sm, ms, bfly / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
