// Integer-pipe roofline denominator: IMAD.WIDE.U32 throughput measured on the
// device the context runs on (MEASURED_PEAKS.json records only HBM and bf16
// peaks). The multiplier changes every iteration so ptxas cannot hoist the
// products (a fixed multiplier gets strength-reduced into 64-bit adds); the
// accumulate is split by ptxas into product + IADD3 on the ALU pipe, which
// runs beside the FMA-heavy pipe. On B200 this measures ~27 IMAD.WIDE / clk
// / SM (profiles/r01_pipe_probe.txt), the same pipe the iGEMM kernels load
// (ncu sm__pipe_fmaheavy_cycles_active).
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "tc.cuh"

namespace hemul_gpu {

namespace {

constexpr int kIters = 2048;

__global__ void imad_probe_kernel(unsigned long long* out, unsigned seed) {
  unsigned a[8];
  unsigned long long acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed + i * 77 + threadIdx.x;
    acc[i] = i;
  }
  unsigned b = seed * 2654435761u + threadIdx.x;
  for (int it = 0; it < kIters; ++it) {
    b += 0x9e3779b9u;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
  }
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// int8 tensor-core roofline denominator: every CTA (one per SM) issues
// back-to-back 128 x 256 x 32 u8 MMAs on fixed shared-memory tiles into two
// TMEM accumulators (the shape the base-conversion GEMMs use).
__global__ void __launch_bounds__(128, 1) tc_probe_kernel(int iters, int* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_addr(smem_raw) & 1023u)) & 1023u);
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
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_addr(smem), b0 = a0 + 128 * 128;
    const uint32_t idesc = tc::idesc_u8(128, 256, 0, 0);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int s = 0; s < 4; ++s)
        tc::mma_u8(tmem + (it & 1) * 256, tc::kmaj_sw128_desc(a0, s, 128),
                   tc::kmaj_sw128_desc(b0, s, 256), idesc, 1);
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  if (threadIdx.x < 32) {
    uint32_t r[4];
    tc::tmem_ld4(tmem, r);
    tc::tmem_wait_ld();
    if (threadIdx.x == 0) sink[blockIdx.x] = static_cast<int>(r[0]);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

cudaError_t tc_peak(double* ops_per_s, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int kSmem = 64 * 1024, kIters = 4096;
  cudaError_t e = cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmem);
  if (e != cudaSuccess) return e;
  int* sink = nullptr;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&sink), sizeof(int) * sms, st)) != cudaSuccess)
    return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tc_probe_kernel<<<sms, 128, kSmem, st>>>(64, sink);  // warm-up
  cudaEventRecord(e0, st);
  tc_probe_kernel<<<sms, 128, kSmem, st>>>(kIters, sink);
  cudaEventRecord(e1, st);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, st);
  if (e != cudaSuccess) return e;
  *ops_per_s = 2.0 * sms * kIters * 4 * 128.0 * 256 * 32 / (ms * 1e-3);
  return cudaGetLastError();
}

cudaError_t imad_peak(double* ops_per_s, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256;
  unsigned long long* out = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&out),
                                  sizeof(unsigned long long) * blocks * threads, st);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  imad_probe_kernel<<<blocks, threads, 0, st>>>(out, 1);  // warm-up
  cudaEventRecord(e0, st);
  constexpr int kReps = 5;
  for (int r = 0; r < kReps; ++r) imad_probe_kernel<<<blocks, threads, 0, st>>>(out, 3 + r);
  cudaEventRecord(e1, st);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  if (e != cudaSuccess) return e;
  *ops_per_s = double(blocks) * threads * kIters * 8 * kReps / (ms * 1e-3);
  return cudaGetLastError();
}

}  // namespace hemul_gpu
