// tcgen05 kind::i8 with the A operand in TMEM ("TS" form): layout check and
// throughput against the shared-memory ("SS") form, alone and with other warps
// streaming shared-memory traffic beside the MMAs (the finisher's situation).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2003_04510_b200/csrc tools/tc_probe/tc_ts_test.cu -o tools/tc_probe/tc_ts_test
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace hemul_gpu;

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

// K-major 64-byte swizzle (the finisher's B layout)
__device__ uint32_t off_k_sw64(uint32_t r, uint32_t k, uint32_t rows) {
  const uint32_t kb = k & 63;
  return (k >> 6) * rows * 64 + (r >> 3) * 512 + (r & 7) * 64 + ((((kb >> 4) ^ (r >> 1)) & 3) << 4) + (kb & 15);
}

__global__ void ts_test(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
                        int32_t* __restrict__ D, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int Kp = (K + 63) / 64 * 64;
  uint8_t* sb = smem;
  for (int i = threadIdx.x; i < N * Kp; i += blockDim.x) smem[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) sb[off_k_sw64(i / K, i % K, N)] = B[i];
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = 32 * w + lane;
  // A row m -> TMEM lane m, columns 256 + c hold bytes 4c..4c+3
  for (int c0 = 0; c0 < Kp / 4; c0 += 8) {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) {
      uint32_t v = 0;
      for (int b = 0; b < 4; ++b) {
        const int k = 4 * (c0 + j) + b;
        if (k < K) v |= uint32_t(A[m * K + k]) << (8 * b);
      }
      r[j] = v;
    }
    tc::tmem_st8(tbase + ((32u * w) << 16) + 256 + c0, r);
  }
  tc::tmem_wait_st();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x == 0) {
    const uint32_t b0 = tc::smem_addr(sb);
    const uint32_t idesc = tc::idesc_u8(128, N, 0, 0);
    for (int s = 0; s < Kp / 32; ++s) {
      const uint64_t bd = tc::smem_desc(b0 + (s >> 1) * N * 64 + (s & 1) * 32, 16, 512, tc::kSw64);
      tc::mma_u8_ts(tbase, tbase + 256 + s * 8, bd, idesc, s > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tc::tmem_ld16(tbase + ((32u * w) << 16) + c, r);
    tc::tmem_wait_ld();
    for (int i = 0; i < 16; ++i)
      if (c + i < N) D[m * N + c + i] = static_cast<int32_t>(r[i]);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tbase);
}

// throughput: warp 0 issues iters x 2 k-steps x 2 MMAs (N each); ts selects A
// from TMEM; warps 4.. (if any) stream 16-byte shared stores + loads until done
__global__ void rate(int iters, int ts, int N, int32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = uint8_t(i * 7);
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
    done = 0;
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_addr(smem), b0 = a0 + 16384;
    const uint32_t idesc = tc::idesc_u8(128, N, ts ? 0 : 1, 0);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const uint64_t ad = tc::smem_desc(a0 + s * 4096, 8192, 1024, tc::kSw128);
        const uint64_t bd0 = tc::smem_desc(b0 + s * 32, 16, 512, tc::kSw64);
        const uint64_t bd1 = tc::smem_desc(b0 + N * 64 + s * 32, 16, 512, tc::kSw64);
        if (ts) {
          tc::mma_u8_ts(tbase, tbase + 480 + s * 8, bd0, idesc, 1);
          tc::mma_u8_ts(tbase + N, tbase + 480 + s * 8, bd1, idesc, 1);
        } else {
          tc::mma_u8(tbase, ad, bd0, idesc, 1);
          tc::mma_u8(tbase + N, ad, bd1, idesc, 1);
        }
      }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    done = 1;
  } else if (w >= 4) {
    // shared-memory traffic: 16-byte stores and loads over a 32 KB window
    uint4* p = reinterpret_cast<uint4*>(smem + 65536);
    const int t = threadIdx.x - 128;
    uint32_t acc = 0;
    while (!done) {
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        p[(t + i * 256) & 2047] = make_uint4(i, acc, 0, 0);
        acc += p[(t * 3 + i * 97) & 2047].x;
      }
    }
    if (acc == 12345) sink[0] = acc;
  }
  __syncwarp();
  if (w < 4) tc::mbar_wait(&bar, 0);
  tc::fence_after();
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t r[4];
    tc::tmem_ld4(tbase, r);
    tc::tmem_wait_ld();
    if (threadIdx.x == 0) sink[blockIdx.x] = r[0];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tbase);
}


// the finisher's operand walk: A (MN-major SW128, 8 KB per chunk) in a 3-stage
// ring, B (K-major SW64, 2N x 64 bytes per chunk) in a 6-stage ring, four MMAs
// and two commits per chunk; mode 1 adds warps streaming global -> shared
// bulk copies into an unused region, mode 2 also has 8 warps of STS/LDS
__global__ void ring_rate(int chunks, int N, int mode, const uint8_t* __restrict__ g, int32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar[2];
  __shared__ uint64_t cbar[4];
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t b_bytes = 2 * N * 64;
  uint8_t* sa = smem;                  // 3 x 8 KB
  uint8_t* sb = smem + 3 * 8192;       // 6 x b_bytes
  uint8_t* sx = sb + 6 * b_bytes;      // 4 x 8 KB scratch for the traffic warps
  for (int i = threadIdx.x; i < 3 * 8192 + 6 * b_bytes; i += blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    smem[i] = (mode & 4) ? uint8_t(h >> 8) : uint8_t(i * 7);
  }
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    for (int i = 0; i < 4; ++i) tc::mbar_init(&cbar[i], 1);
    tc::mbar_fence_init();
    tc::mbar_arrive(&cbar[0]);
    tc::mbar_arrive(&cbar[1]);
    done = 0;
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    const long long t_start = clock64();
    const uint32_t a0 = tc::smem_addr(sa), b0 = tc::smem_addr(sb);
    const uint32_t idesc = tc::idesc_u8(128, N, 1, 0);
    int sa_i = 0, sb_i = 0;
    for (int c = 0; c < chunks; ++c) {
      if (mode & 8) {  // the finisher's per-chunk barrier waits (already complete)
        tc::mbar_wait(&cbar[0], 0);
        tc::mbar_wait(&cbar[1], 0);
        tc::fence_after();
      }
      const uint32_t ab = a0 + sa_i * 8192, bb = b0 + sb_i * b_bytes;
      const uint32_t d = tbase + ((c / 29) & 1) * N;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const uint64_t ad = tc::smem_desc(ab + s * 4096, 8192, 1024, tc::kSw128);
        const uint64_t bd0 = tc::smem_desc(bb + s * 32, 16, 512, tc::kSw64);
        const uint64_t bd1 = tc::smem_desc(bb + N * 64 + s * 32, 16, 512, tc::kSw64);
        tc::mma_u8(d, ad, bd0, idesc, (c % 29) | s);
        tc::mma_u8(d + N, ad, bd1, idesc, (c % 29) | s);
      }
      tc::mma_commit(&cbar[2 + (c & 1)]);
      tc::mma_commit(&cbar[3 - (c & 1)]);
      sa_i = sa_i == 2 ? 0 : sa_i + 1;
      sb_i = sb_i == 5 ? 0 : sb_i + 1;
    }
    tc::mma_commit(&bar[0]);
    tc::mbar_wait(&bar[0], 0);
    done = 1;
    sink[gridDim.x + blockIdx.x] = int32_t((clock64() - t_start) >> 8);
  } else if (w >= 4 && w < 6 && (mode & 3) >= 1) {
    // bulk copies of 8 KB from global into the scratch region, 2 in flight per warp
    if (lane == 0) {
      const uint32_t dst = tc::smem_addr(sx) + (w - 4) * 16384;
      uint64_t* mb = &bar[1];
      if (w == 4) {
        uint32_t ph = 0;
        int it = 0;
        while (!done) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_addr(mb)), "r"(16384u) : "memory");
          for (int h = 0; h < 2; ++h)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst + h * 8192), "l"(g + ((size_t)(blockIdx.x * 977 + it * 2 + h) % 4096) * 8192), "r"(8192u), "r"(tc::smem_addr(mb)) : "memory");
          tc::mbar_wait(mb, ph);
          ph ^= 1;
          ++it;
        }
      }
    }
  } else if (w >= 6 && (mode & 3) >= 2) {
    uint4* p = reinterpret_cast<uint4*>(sx + 32768);
    const int t = threadIdx.x - 192;
    uint32_t acc = 0;
    while (!done) {
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        p[(t + i * 256) & 511] = make_uint4(i, acc, 0, 0);
        acc += p[(t * 3 + i * 97) & 511].x;
      }
    }
    if (acc == 12345) sink[0] = acc;
  }
  __syncwarp();
  if (w < 4) tc::mbar_wait(&bar[0], 0);
  tc::fence_after();
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t r[4];
    tc::tmem_ld4(tbase, r);
    tc::tmem_wait_ld();
    if (threadIdx.x == 0) sink[blockIdx.x] = r[0];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tbase);
}

// N sweep: 2 MMAs (N each) per k-step, A mode am (0 K-major SW128 smem, 1 MN-major
// SW128 smem, 2 TMEM), B K-major swizzle bs (64 or 128)
__global__ void sweep(int iters, int am, int bs, int N, int32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) smem[i] = uint8_t(i * 7);
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_addr(smem), b0 = a0 + 16384;
    const uint32_t idesc = tc::idesc_u8(128, N, am == 1 ? 1 : 0, 0);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const uint64_t ad = am == 1 ? tc::smem_desc(a0 + s * 4096, 8192, 1024, tc::kSw128)
                                    : tc::kmaj_sw128_desc(a0, s, 128);
        const uint64_t bd0 = bs == 64 ? tc::smem_desc(b0 + s * 32, 16, 512, tc::kSw64)
                                      : tc::kmaj_sw128_desc(b0, s, N);
        const uint64_t bd1 = bs == 64 ? tc::smem_desc(b0 + N * 64 + s * 32, 16, 512, tc::kSw64)
                                      : tc::kmaj_sw128_desc(b0 + N * 128, s, N);
        if (am == 2) {
          tc::mma_u8_ts(tbase, tbase + 480 + s * 8, bd0, idesc, 1);
          tc::mma_u8_ts(tbase + N, tbase + 480 + s * 8, bd1, idesc, 1);
        } else {
          tc::mma_u8(tbase, ad, bd0, idesc, 1);
          tc::mma_u8(tbase + N, ad, bd1, idesc, 1);
        }
      }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  if (threadIdx.x < 32) {
    uint32_t r[4];
    tc::tmem_ld4(tbase, r);
    tc::tmem_wait_ld();
    if (threadIdx.x == 0) sink[blockIdx.x] = r[0];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tbase);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int32_t* sink;
  CK(cudaMalloc(&sink, sms * 16));
  CK(cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  CK(cudaFuncSetAttribute(ts_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {128, 384})
    for (int ts : {0, 1})
      for (int N : {160, 128, 256}) {
        rate<<<sms, threads, 100 * 1024>>>(16, ts, N, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        rate<<<sms, threads, 100 * 1024>>>(iters, ts, N, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * sms * iters * 4 * 128.0 * N * 32;
        printf("%s A, N=%d x2, %s: %.1f TOPS\n", ts ? "TMEM" : "SMEM(MN)", N,
               threads > 128 ? "with 8 warps of smem traffic" : "alone", ops / (ms * 1e-3) / 1e12);
      }
  {
    uint8_t* g;
    CK(cudaMalloc(&g, 4096 * 8192));
    CK(cudaFuncSetAttribute(ring_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    for (int mode : {0, 8, 4, 12})
      for (int N : {160}) {
        const int chunks = 29 * 64;
        ring_rate<<<sms, 448, 220 * 1024>>>(58, N, mode, g, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        ring_rate<<<sms, 448, 220 * 1024>>>(chunks, N, mode, g, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * sms * chunks * 4 * 128.0 * N * 32;
        std::vector<int32_t> cyc(sms);
        CK(cudaMemcpy(cyc.data(), sink + sms, sms * 4, cudaMemcpyDeviceToHost));
        double cs = 0;
        for (int v : cyc) cs += double(v) * 256;
        printf("ring walk N=%d x2 mode %d: %.1f TOPS (%.0f ns per chunk, %.0f cycles per chunk, %.2f GHz)\n", N, mode,
               ops / (ms * 1e-3) / 1e12, ms * 1e6 / chunks, cs / sms / chunks, cs / sms / (ms * 1e6));
      }
  }
  CK(cudaFuncSetAttribute(sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  for (int am : {0, 1, 2})
    for (int bs : {64, 128}) {
      printf("A %s, B SW%d:", am == 0 ? "K-SW128" : am == 1 ? "MN-SW128" : "TMEM", bs);
      for (int N : {32, 64, 96, 128, 160, 192, 224, 256}) {
        if (am == 2 && N > 240) continue;
        sweep<<<sms, 128, 100 * 1024>>>(16, am, bs, N, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        sweep<<<sms, 128, 100 * 1024>>>(4096, am, bs, N, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  N=%d %.0f ns/MMA %.0fT", N, ms * 1e6 / (4096 * 4), 2.0 * sms * 4096 * 4 * 128.0 * N * 32 / (ms * 1e-3) / 1e12);
      }
      printf("\n");
    }
  srand(7);
  int fails = 0;
  for (int N : {160, 128, 96, 16})
    for (int K : {32, 64, 96, 128}) {
      std::vector<uint8_t> a(128 * K), b(N * K);
      for (auto& x : a) x = uint8_t(rand());
      for (auto& x : b) x = uint8_t(rand());
      std::vector<int32_t> ref(128 * N), got(128 * N);
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          int32_t s = 0;
          for (int k = 0; k < K; ++k) s += int32_t(a[m * K + k]) * int32_t(b[n * K + k]);
          ref[m * N + n] = s;
        }
      uint8_t *da, *db;
      int32_t* dd;
      CK(cudaMalloc(&da, a.size()));
      CK(cudaMalloc(&db, b.size()));
      CK(cudaMalloc(&dd, got.size() * 4));
      CK(cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
      ts_test<<<1, 128, 100 * 1024>>>(da, db, dd, N, K);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(got.data(), dd, got.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0, first = -1;
      for (size_t i = 0; i < ref.size(); ++i)
        if (ref[i] != got[i]) {
          if (first < 0) first = int(i);
          ++bad;
        }
      printf("TS N=%3d K=%3d : %s", N, K, bad ? "FAIL" : "ok");
      if (bad) printf(" (%d bad; first m=%d n=%d ref=%d got=%d)", bad, first / N, first % N, ref[first], got[first]);
      printf("\n");
      fails += bad != 0;
      cudaFree(da);
      cudaFree(db);
      cudaFree(dd);
    }
  printf("%s\n", fails ? "TS LAYOUT FAILED" : "ALL OK");
  return 0;
}
