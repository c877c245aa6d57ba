// L2 -> SM read bandwidth on this GPU (the ceiling for the screen's posting
// reads, which hit L2: DESIGN.md §4).  Reads a buffer that fits in L2 with
// 16-B loads from a persistent grid, many passes, and reports GB/s for a few
// buffer sizes (and one much larger than L2 for the HBM figure).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_peak tools/l2_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void read_kernel(const uint4* __restrict__ buf, size_t n16, int passes,
                            unsigned* __restrict__ sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
      const uint4 v = __ldcg(buf + i);  // cache in L2 only: measures L2, not L1
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"results\": [", sms, l2);
  const size_t sizes_mb[] = {8, 16, 32, 48, 64, 2048};
  unsigned* sink;
  cudaMalloc(&sink, 4);
  bool first = true;
  for (size_t mb : sizes_mb) {
    const size_t bytes = mb << 20;
    uint4* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) continue;
    cudaMemset(buf, 1, bytes);
    const size_t n16 = bytes / 16;
    const int passes = mb >= 1024 ? 3 : (int)(4096 / mb);
    const int threads = 512, blocks = sms * 4;
    read_kernel<<<blocks, threads>>>(buf, n16, 1, sink);  // warm L2
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      read_kernel<<<blocks, threads>>>(buf, n16, passes, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double gbs = (double)bytes * passes / (best * 1e-3) / 1e9;
    printf("%s{\"buffer_mb\": %zu, \"passes\": %d, \"ms\": %.3f, \"GB_per_s\": %.1f}",
           first ? "" : ", ", mb, passes, best, gbs);
    first = false;
    cudaFree(buf);
  }
  printf("]}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
