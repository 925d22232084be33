// Integer-pipe throughput probe for sm_100a (asm volatile so nothing folds).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
template <int KIND>
__global__ void probe(uint64_t* out, uint32_t seed) {
  uint32_t a[8], b = seed * 2654435761u + threadIdx.x;
  uint64_t acc[8];
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed + i * 77 + threadIdx.x; acc[i] = i; d[i] = a[i]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) {  // IMAD.WIDE.U32
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
      } else if (KIND == 1) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(i));
      } else if (KIND == 2) {
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(i));
      } else if (KIND == 3) {  // carry chain MAC: 3-word acc += a*b
        uint32_t lo = (uint32_t)acc[i], hi = (uint32_t)(acc[i] >> 32);
        asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;\n\taddc.u32 %4, %4, 0;"
                     : "+r"(lo), "+r"(hi) : "r"(a[i]), "r"(b), "r"(a[(i+1)&7]));
        acc[i] = ((uint64_t)hi << 32) | lo;
      } else if (KIND == 4) {  // mul.hi.u64
        asm volatile("mul.hi.u64 %0, %0, %1;" : "+l"(acc[i]) : "l"((uint64_t)b | 0x100000000ull));
      } else if (KIND == 5) {
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(1.0000001), "d"(0.5));
      } else if (KIND == 6) {  // mixed: 1 IMAD.WIDE + 1 DFMA
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(1.0000001), "d"(0.5));
      } else if (KIND == 7) {  // IADD3 64-bit add (alu)
        asm volatile("add.u64 %0, %0, %1;" : "+l"(acc[i]) : "l"((uint64_t)b));
      } else if (KIND == 8) {  // mul.lo.u64
        asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(acc[i]) : "l"((uint64_t)b | 0x100000000ull));
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i] + a[i] + (uint64_t)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
float run(uint64_t* out, int blocks, int threads) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<K><<<blocks, threads>>>(out, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) probe<K><<<blocks, threads>>>(out, 3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, clk);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  uint64_t* out; cudaMalloc(&out, sizeof(uint64_t) * blocks * threads);
  const char* names[] = {"mad.wide.u32", "mad.lo.u32", "mad.hi.u32", "mac3(lo.cc,hi.cc,addc)", "mul.hi.u64", "fma.f64", "wide+dfma pair", "add.u64", "mul.lo.u64"};
  float ms[9];
  ms[0] = run<0>(out, blocks, threads); ms[1] = run<1>(out, blocks, threads);
  ms[2] = run<2>(out, blocks, threads); ms[3] = run<3>(out, blocks, threads);
  ms[4] = run<4>(out, blocks, threads); ms[5] = run<5>(out, blocks, threads);
  ms[6] = run<6>(out, blocks, threads); ms[7] = run<7>(out, blocks, threads);
  ms[8] = run<8>(out, blocks, threads);
  for (int k = 0; k < 9; ++k) {
    double ops = (double)blocks * threads * ITERS * 8;
    double rate = ops / (ms[k] * 1e-3);
    printf("%-26s %.3f ms  %.2f Tops/s  %.1f ops/clk/SM(at max clk)\n", names[k], ms[k], rate / 1e12,
           rate / (p.multiProcessorCount * (clk * 1e3)));
  }
  return 0;
}
