// Minimal TMA probe: rank-R tiled tensor map over a float64 / float32 array.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tma_probe2.cu -o tools/bin/tma_probe2
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k2(const __grid_constant__ CUtensorMap m, int rank, unsigned bytes, float* out, int variant) {
  __shared__ __align__(1024) float buf[4096];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
    const uint64_t mp = reinterpret_cast<uint64_t>(&m);
    if (rank == 1)
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(su(buf)), "l"(mp), "r"(0), "r"(su(&bar)) : "memory");
    else if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(buf)), "l"(mp), "r"(0), "r"(0), "r"(su(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred d;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n@!d bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int rank = argc > 1 ? atoi(argv[1]) : 1;
  const int link = argc > 2 ? atoi(argv[2]) : 0;
  float* d;
  cudaMalloc(&d, 1 << 20);
  std::vector<float> h(1 << 18);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  cudaMemcpy(d, h.data(), 4 * h.size(), cudaMemcpyHostToDevice);
  float* o;
  cudaMalloc(&o, 64 * 4);
  Enc enc = nullptr;
  if (link) {
    enc = &cuTensorMapEncodeTiled;
  } else {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    enc = (Enc)f;
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {256, 256};
  cuuint64_t str[1] = {256 * 4};
  cuuint32_t box[2] = {32, 8}, el[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = rank == 1 ? 32 * 4 : 32 * 8 * 4;
  printf("rank %d link %d encode %d\n", rank, link, (int)r);
  k2<<<1, 32>>>(m, rank, bytes, o, 0);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float g[64];
  cudaMemcpy(g, o, 256, cudaMemcpyDeviceToHost);
  printf("out %g %g %g %g\n", g[0], g[1], g[31], g[32]);
  return 0;
}
