// Issue rate of FHFMA (fma.rn.f32.f16: fp16 x fp16 + fp32) against FFMA and
// FFMA2 on sm_100a: every thread runs 16 independent accumulator chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/fhfma_rate tools/fhfma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void rate_kernel(float* out, int iters, unsigned wbits, unsigned xbits) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = (float)(threadIdx.x + i);
  unsigned w = wbits + threadIdx.x, x = xbits;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {  // FHFMA
        unsigned short a, b, xx, x1;
        asm volatile("mov.b32 {%0, %1}, %2;" : "=h"(a), "=h"(b) : "r"(w));
        asm volatile("mov.b32 {%0, %1}, %2;" : "=h"(xx), "=h"(x1) : "r"(x));
        asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i]) : "h"(a), "h"(xx));
        asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i + 1]) : "h"(b), "h"(xx));
      } else if (MODE == 1) {  // FFMA
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[i]) : "f"(__uint_as_float(w)), "f"(__uint_as_float(x)));
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[i + 1]) : "f"(__uint_as_float(w)), "f"(__uint_as_float(x)));
      } else {  // FFMA2
        unsigned long long ab, xy, vv;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(ab) : "f"(__uint_as_float(w)), "f"(__uint_as_float(w)));
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(xy) : "f"(acc[i]), "f"(acc[i + 1]));
        asm volatile("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(__uint_as_float(x)));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(xy) : "l"(vv), "l"(ab));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(xy));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(const char* name, float* out, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = 148 * 8, block = 256;
  rate_kernel<MODE><<<grid, block>>>(out, 16, 0x3c003c00u, 0x3c00u);
  cudaEventRecord(a);
  rate_kernel<MODE><<<grid, block>>>(out, iters, 0x3c003c00u, 0x3c00u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double slots = (double)grid * block * iters * 16;
  printf("%-6s %8.3f ms  %7.2f G slot-updates/s  (%.1f per clk per SM at 1.965 GHz)\n", name, ms,
         slots / ms / 1e6, slots / (ms * 1e-3) / 148 / 1.965e9);
  return ms;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
  const int iters = 1 << 16;
  run<0>("FHFMA", out, iters);
  run<1>("FFMA", out, iters);
  run<2>("FFMA2", out, iters);
  return cudaDeviceSynchronize() != cudaSuccess;
}
