// Build: nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/pcie_probe.cu -o tools/bin/pcie_probe
// PCIe probe: H2D / D2H bandwidth for pinned, write-combined and zero-copy
// (kernel reads mapped host memory) transfers of a few MB.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
__global__ void k_read(const double4* __restrict__ src, double4* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
int main() {
  const size_t bytes = 2880000;
  void *h_pin, *h_wc, *h_map, *d;
  cudaMallocHost(&h_pin, bytes);
  cudaHostAlloc(&h_wc, bytes, cudaHostAllocWriteCombined);
  cudaHostAlloc(&h_map, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto fn) {
    for (int i = 0; i < 5; ++i) fn();
    cudaStreamSynchronize(s);
    float best = 1e9, tot = 0;
    for (int i = 0; i < 30; ++i) {
      cudaEventRecord(a, s);
      fn();
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
      tot += ms;
    }
    printf("%-28s best %7.1f us  avg %7.1f us  (%.1f GB/s avg)\n", name, best * 1e3, tot / 30 * 1e3,
           bytes / (tot / 30 * 1e-3) / 1e9);
  };
  time("H2D pinned", [&] { cudaMemcpyAsync(d, h_pin, bytes, cudaMemcpyHostToDevice, s); });
  time("H2D write-combined", [&] { cudaMemcpyAsync(d, h_wc, bytes, cudaMemcpyHostToDevice, s); });
  time("D2H pinned", [&] { cudaMemcpyAsync(h_pin, d, bytes, cudaMemcpyDeviceToHost, s); });
  double4* dm;
  cudaHostGetDevicePointer((void**)&dm, h_map, 0);
  const long long n4 = bytes / 32;
  time("zero-copy kernel read", [&] { k_read<<<296, 256, 0, s>>>(dm, (double4*)d, n4); });
  time("zero-copy kernel write", [&] { k_read<<<296, 256, 0, s>>>((double4*)d, dm, n4); });
  // chunked H2D on 4 streams
  cudaStream_t ss[4];
  for (int i = 0; i < 4; ++i) cudaStreamCreate(&ss[i]);
  cudaEvent_t evs[4];
  for (int i = 0; i < 4; ++i) cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
  time("H2D pinned 4 streams", [&] {
    cudaEventRecord(a, s);
    for (int i = 0; i < 4; ++i) {
      cudaStreamWaitEvent(ss[i], a, 0);
      cudaMemcpyAsync((char*)d + i * bytes / 4, (char*)h_pin + i * bytes / 4, bytes / 4,
                      cudaMemcpyHostToDevice, ss[i]);
      cudaEventRecord(evs[i], ss[i]);
      cudaStreamWaitEvent(s, evs[i], 0);
    }
  });
  // effect of CPU writes to the source buffer
  memset(h_pin, 1, bytes);
  time("H2D pinned after memset", [&] { cudaMemcpyAsync(d, h_pin, bytes, cudaMemcpyHostToDevice, s); });
  void* h_def;
  cudaHostAlloc(&h_def, bytes, cudaHostAllocDefault);
  time("H2D hostalloc default", [&] { cudaMemcpyAsync(d, h_def, bytes, cudaMemcpyHostToDevice, s); });
  memset(h_def, 2, bytes);
  time("H2D hostalloc after memset", [&] { cudaMemcpyAsync(d, h_def, bytes, cudaMemcpyHostToDevice, s); });
  void* h_reg = aligned_alloc(4096, bytes + 4096);
  memset(h_reg, 3, bytes);
  cudaHostRegister(h_reg, bytes, cudaHostRegisterDefault);
  time("H2D registered", [&] { cudaMemcpyAsync(d, h_reg, bytes, cudaMemcpyHostToDevice, s); });
  printf("done\n");
  return 0;
}
