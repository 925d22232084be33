// Integer / FP64 pipe throughput probe v2: the multiplier changes every
// iteration so ptxas cannot hoist the products (v1's mad.wide loop was
// strength-reduced into 64-bit adds).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
template <int KIND>
__global__ void probe(uint64_t* out, uint32_t seed) {
  uint32_t a[8];
  uint64_t acc[8];
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed + i * 77 + threadIdx.x; acc[i] = i; d[i] = a[i]; }
  uint32_t b = seed * 2654435761u + threadIdx.x;
  double db = (double)b;
  for (int it = 0; it < ITERS; ++it) {
    b += 0x9e3779b9u;  // one IADD per 8 (or 16) multiplies
    db += 1.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) {
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
      } else if (KIND == 1) {
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(a[(i + 1) & 7]));
      } else if (KIND == 2) {
        asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(a[(i + 1) & 7]));
      } else if (KIND == 3) {
        asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d[i]) : "d"((double)a[i]), "d"(db));
      } else if (KIND == 4) {  // one WIDE + one DFMA per slot: do the pipes overlap?
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
        asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d[i]) : "d"((double)a[i]), "d"(db));
      } else if (KIND == 5) {  // WIDE + 32-bit IMAD
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(a[(i + 1) & 7]));
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
  for (int r = 0; r < 5; ++r) probe<K><<<blocks, threads>>>(out, 3 + r);
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
  const char* names[] = {"mad.wide.u32", "mad.lo.u32", "mad.hi.u32", "fma.rn.f64", "wide+dfma (per pair)", "wide+imad (per pair)"};
  float ms[6];
  ms[0] = run<0>(out, blocks, threads); ms[1] = run<1>(out, blocks, threads);
  ms[2] = run<2>(out, blocks, threads); ms[3] = run<3>(out, blocks, threads);
  ms[4] = run<4>(out, blocks, threads); ms[5] = run<5>(out, blocks, threads);
  for (int k = 0; k < 6; ++k) {
    double ops = (double)blocks * threads * ITERS * 8;
    double rate = ops / (ms[k] * 1e-3);
    printf("%-24s %.3f ms  %.2f Tops/s  %.1f ops/clk/SM (at max clk)\n", names[k], ms[k], rate / 1e12,
           rate / (p.multiProcessorCount * (clk * 1e3)));
  }
  return 0;
}
