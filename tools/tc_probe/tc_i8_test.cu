// tcgen05 kind::i8 layout / descriptor probe and throughput microbenchmark.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2003_04510_b200/csrc tools/tc_probe/tc_i8_test.cu -o tools/tc_probe/tc_i8_test
// Checks D = A . B^T (u8 x u8 -> s32, M = 128) against the CPU for each
// operand layout the GEMM kernels may use, then times back-to-back
// 128 x 256 x 32 MMAs on every SM (the dense int8 tensor peak).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
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

// layout variants
enum { V_KSW128 = 0, V_KNONE = 1, V_KNONE_SWAP = 2, V_AMN128 = 3, V_AMN128_SWAP = 4, V_KSW64 = 5, V_KSW32 = 6 };

__device__ uint32_t off_k_none(uint32_t r, uint32_t k, uint32_t rows) {
  return (k >> 4) * rows * 16 + (r >> 3) * 128 + (r & 7) * 16 + (k & 15);
}
// K-major 64-byte swizzle: rows of 64 K-bytes, 8-row atoms of 512 B, chunk ^= (r >> 1) & 3
__device__ uint32_t off_k_sw64(uint32_t r, uint32_t k, uint32_t rows) {
  const uint32_t kb = k & 63;
  return (k >> 6) * rows * 64 + (r >> 3) * 512 + (r & 7) * 64 + ((((kb >> 4) ^ (r >> 1)) & 3) << 4) + (kb & 15);
}
// K-major 32-byte swizzle: rows of 32 K-bytes, 8-row atoms of 256 B, chunk ^= (r >> 2) & 1
__device__ uint32_t off_k_sw32(uint32_t r, uint32_t k, uint32_t rows) {
  const uint32_t kb = k & 31;
  return (k >> 5) * rows * 32 + (r >> 3) * 256 + (r & 7) * 32 + ((((kb >> 4) ^ (r >> 2)) & 1) << 4) + (kb & 15);
}
__device__ uint32_t off_mn_sw128(uint32_t m, uint32_t k) {  // M = 128
  return (k >> 3) * 1024 + (k & 7) * 128 + ((((m >> 4) ^ k) & 7) << 4) + (m & 15);
}

__global__ void gemm_test(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
                          int32_t* __restrict__ D, int N, int K, int var) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int M = 128;
  const int Kp = (K + 127) / 128 * 128;
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * Kp;
  for (int i = threadIdx.x; i < M * Kp + N * Kp; i += blockDim.x) smem[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    uint32_t o;
    if (var == V_KSW128) o = tc::kmaj_sw128(r, k, M);
    else if (var == V_KSW64) o = off_k_sw64(r, k, M);
    else if (var == V_KSW32) o = off_k_sw32(r, k, M);
    else if (var == V_KNONE || var == V_KNONE_SWAP) o = off_k_none(r, k, M);
    else o = off_mn_sw128(r, k);
    sa[o] = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    uint32_t o;
    if (var == V_KNONE || var == V_KNONE_SWAP) o = off_k_none(r, k, N);
    else if (var == V_KSW64) o = off_k_sw64(r, k, N);
    else if (var == V_KSW32) o = off_k_sw32(r, k, N);
    else o = tc::kmaj_sw128(r, k, N);
    sb[o] = B[i];
  }
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  const int amn = (var == V_AMN128 || var == V_AMN128_SWAP);
  const uint32_t idesc = tc::idesc_u8(M, N, amn, 0);
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_addr(sa), b0 = tc::smem_addr(sb);
    for (int s = 0; s < K / 32; ++s) {
      uint64_t ad, bd;
      if (var == V_KSW128) {
        ad = tc::kmaj_sw128_desc(a0, s, M);
        bd = tc::kmaj_sw128_desc(b0, s, N);
      } else if (var == V_KSW64) {
        ad = tc::smem_desc(a0 + (s >> 1) * M * 64 + (s & 1) * 32, 16, 512, tc::kSw64);
        bd = tc::smem_desc(b0 + (s >> 1) * N * 64 + (s & 1) * 32, 16, 512, tc::kSw64);
      } else if (var == V_KSW32) {
        ad = tc::smem_desc(a0 + s * M * 32, 16, 256, tc::kSw32);
        bd = tc::smem_desc(b0 + s * N * 32, 16, 256, tc::kSw32);
      } else if (var == V_KNONE) {
        ad = tc::smem_desc(a0 + 2 * s * M * 16, M * 16, 128, tc::kSwNone);
        bd = tc::smem_desc(b0 + 2 * s * N * 16, N * 16, 128, tc::kSwNone);
      } else if (var == V_KNONE_SWAP) {
        ad = tc::smem_desc(a0 + 2 * s * M * 16, 128, M * 16, tc::kSwNone);
        bd = tc::smem_desc(b0 + 2 * s * N * 16, 128, N * 16, tc::kSwNone);
      } else if (var == V_AMN128) {
        ad = tc::smem_desc(a0 + s * 4096, Kp * 128, 1024, tc::kSw128);
        bd = tc::kmaj_sw128_desc(b0, s, N);
      } else {
        ad = tc::smem_desc(a0 + s * 4096, 1024, Kp * 128, tc::kSw128);
        bd = tc::kmaj_sw128_desc(b0, s, N);
      }
      tc::mma_u8(tbase, ad, bd, idesc, s > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < 4) {
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      tc::tmem_ld16(tbase + ((32u * w) << 16) + c, r);
      tc::tmem_wait_ld();
      for (int i = 0; i < 16; ++i)
        if (c + i < N) D[(32 * w + lane) * N + c + i] = static_cast<int32_t>(r[i]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tbase);
}

// throughput: every CTA issues `iters` x (128 x 256 x 32) MMAs on fixed tiles
__global__ void mma_rate(int iters, int32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 128 * 128 + 256 * 128; i += blockDim.x) smem[i] = uint8_t(i * 7);
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
    const uint32_t a0 = tc::smem_addr(smem), b0 = a0 + 128 * 128;
    const uint32_t idesc = tc::idesc_u8(128, 256, 0, 0);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int s = 0; s < 4; ++s)
        tc::mma_u8(tbase + (it & 1) * 256, tc::kmaj_sw128_desc(a0, s, 128),
                   tc::kmaj_sw128_desc(b0, s, 256), idesc, 1);
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

// throughput of one layout / shape: a_mn (A MN-major SW128, M=128), b_sw
// (B K-major swizzle 128 or 64), N per MMA, two MMAs per k-step (N each)
__global__ void mma_rate2(int iters, int a_mn, int b_sw, int N, int32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = uint8_t(i * 7);
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
    const uint32_t idesc = tc::idesc_u8(128, N, a_mn, 0);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const uint64_t ad = a_mn ? tc::smem_desc(a0 + s * 4096, 8192, 1024, tc::kSw128)
                                 : tc::kmaj_sw128_desc(a0, s, 128);
        const uint64_t bd0 = b_sw == 64 ? tc::smem_desc(b0 + s * 32, 16, 512, tc::kSw64)
                                        : tc::kmaj_sw128_desc(b0, s, N);
        const uint64_t bd1 = b_sw == 64 ? tc::smem_desc(b0 + N * 64 + s * 32, 16, 512, tc::kSw64)
                                        : tc::kmaj_sw128_desc(b0 + N * 128, s, N);
        tc::mma_u8(tbase, ad, bd0, idesc, 1);
        tc::mma_u8(tbase + N, ad, bd1, idesc, 1);
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

int main(int argc, char** argv) {
  const char* names[] = {"A,B K-major SW128", "A,B K-major interleave", "A,B K-major interleave (LBO/SBO swapped)",
                         "A MN-major SW128 / B K SW128", "A MN-major SW128 (LBO/SBO swapped) / B K SW128",
                         "A,B K-major SW64", "A,B K-major SW32"};
  CK(cudaFuncSetAttribute(gemm_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int32_t* sink;
  CK(cudaMalloc(&sink, sms * 4));
  const int iters = 4096;
  mma_rate<<<sms, 128, 64 * 1024>>>(64, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_rate<<<sms, 128, 64 * 1024>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * sms * iters * 4 * 128.0 * 256 * 32;
  printf("int8 MMA rate: %.1f TOPS dense (%d SMs, %.3f ms)\n", ops / (ms * 1e-3) / 1e12, sms, ms);
  CK(cudaFuncSetAttribute(mma_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  const int cfgs[][3] = {{0, 128, 256}, {1, 128, 256}, {0, 128, 160}, {1, 128, 160},
                         {0, 64, 160}, {1, 64, 160}, {1, 64, 128}, {1, 64, 240}};
  for (const auto& cf : cfgs) {
    mma_rate2<<<sms, 128, 100 * 1024>>>(16, cf[0], cf[1], cf[2], sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    mma_rate2<<<sms, 128, 100 * 1024>>>(4096, cf[0], cf[1], cf[2], sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms2 = 0;
    cudaEventElapsedTime(&ms2, e0, e1);
    const double ops2 = 2.0 * sms * 4096 * 4 * 128.0 * cf[2] * 32;
    printf("rate A %s, B K-major SW%d, N=%d x2: %.1f TOPS\n", cf[0] ? "MN-major" : "K-major", cf[1],
           cf[2], ops2 / (ms2 * 1e-3) / 1e12);
  }
  const int Ns[] = {256, 176, 80, 16};
  const int Ks[] = {32, 160, 320};
  srand(12345);
  int fails = 0;
  for (int ai = 1; ai < argc; ++ai) {
    const int var = atoi(argv[ai]);
    for (int N : Ns)
      for (int K : Ks) {
        if ((var == V_AMN128 || var == V_AMN128_SWAP) && K % 32) continue;
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
        CK(cudaMemset(dd, 0xff, got.size() * 4));
        const int Kp = (K + 127) / 128 * 128;
        gemm_test<<<1, 128, 1024 + (128 + N) * Kp>>>(da, db, dd, N, K, var);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(got.data(), dd, got.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0, first = -1;
        for (size_t i = 0; i < ref.size(); ++i)
          if (ref[i] != got[i]) {
            if (first < 0) first = int(i);
            ++bad;
          }
        printf("%-50s N=%3d K=%3d : %s", names[var], N, K, bad ? "FAIL" : "ok");
        if (bad)
          printf(" (%d bad; first m=%d n=%d ref=%d got=%d)", bad, first / N, first % N, ref[first],
                 got[first]);
        printf("\n");
        fails += bad != 0;
        cudaFree(da);
        cudaFree(db);
        cudaFree(dd);
      }
  }
  printf("%s\n", fails ? "SOME LAYOUTS FAILED" : "ALL OK");
  return 0;
}
