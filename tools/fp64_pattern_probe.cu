// DFMA issue-rate probe for the spread's operand pattern: 32 accumulators
// (4 rows x 8 planes) per thread, acc[r][s] += a[r] * wz[s], against the
// resident warps per SM.  Modes: 0 the spread's visit (weights from shared
// memory, a[r] = wx * wy[r]); 1 without the four products; 2 plane-major FMA
// order; 3 weights fixed in registers (no loads in the loop).  B200: 21.1 /
// 25.2 / 24.7 / 32.9 TFLOP/s at 32 warps per SM — a DFMA holds the issue
// port for two cycles and every other instruction adds one.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -o tools/bin/fp64_pattern_probe tools/fp64_pattern_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(64) k(double* out, int iters, const double* __restrict__ w) {
  __shared__ double sw[64 * 16];
  for (int i = threadIdx.x; i < 64 * 16; i += 64) sw[i] = w[i];
  __syncthreads();
  double acc[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int s = 0; s < 8; ++s) acc[r][s] = 0.0;
  double wfix[12];
#pragma unroll
  for (int t = 0; t < 12; ++t) wfix[t] = sw[threadIdx.x % 7 + t];
  for (int i = 0; i < iters; ++i) {
    const double* p = sw + (i & 63) * 16;
    double wz[8], a[4];
#pragma unroll
    for (int s = 0; s < 8; ++s) wz[s] = p[s];                 // broadcast loads
    if (MODE == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = p[8 + r] * p[12 + (threadIdx.x & 3)];
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = p[8 + r];
    }
    if (MODE == 2) {          // plane-major: consecutive FMAs share wz[s]
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r][s] = fma(a[r], wz[s], acc[r][s]);
    } else if (MODE == 3) {   // weights fixed in registers (no loads in the loop)
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[r][s] = fma(wfix[r], wfix[4 + s], acc[r][s]);
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[r][s] = fma(a[r], wz[s], acc[r][s]);
    }
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int s = 0; s < 8; ++s) t += acc[r][s];
  if (t == 1234.5) out[0] = t;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *d, *w;
  cudaMalloc(&d, 8);
  cudaMalloc(&w, 64 * 16 * 8);
  cudaMemset(w, 0, 64 * 16 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int mode = 0; mode < 4; ++mode)
    for (int cps : {2, 8, 16}) {   // CTAs (2 warps each) per SM
      // limit residency with dynamic shared memory
      const int smem = 220 * 1024 / cps - 9 * 1024;
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<nsm * cps, 64, smem>>>(d, 100, w);
      cudaEventRecord(e0);
      kern<<<nsm * cps, 64, smem>>>(d, iters, w);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * 32 * iters * (double)nsm * cps * 64;
      printf("mode %d warps/SM %2d: %.2f TFLOP/s (%.3f ms) %s\n", mode, 2 * cps, fl / ms / 1e9, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
