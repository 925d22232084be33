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

}  // namespace

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
