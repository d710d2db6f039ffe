// TMA probe: float64, rank 2..4, static or dynamic smem, fence variant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tma_probe3.cu -o tools/bin/tma_probe3
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool DYN>
__global__ void k3(const __grid_constant__ CUtensorMap m, int rank, unsigned bytes, double* out, int fence, int c2, int x0, int y0, int z0) {
  __shared__ __align__(1024) double sbuf[DYN ? 1 : 16 * 16 * 4];
  __shared__ __align__(8) uint64_t sbar;
  extern __shared__ unsigned char dyn[];
  double* buf = sbuf;
  uint64_t* bar = &sbar;
  if (DYN) {
    unsigned char* b = reinterpret_cast<unsigned char*>(((uintptr_t)dyn + 1023) & ~uintptr_t(1023));
    buf = reinterpret_cast<double*>(b);
    bar = reinterpret_cast<uint64_t*>(b + 16 * 16 * 4 * 8);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(1));
    if (fence) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(bytes) : "memory");
    const uint64_t mp = reinterpret_cast<uint64_t>(&m);
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(buf)), "l"(mp), "r"(0), "r"(0), "r"(su(bar)) : "memory");
    else if (rank == 3)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(su(buf)), "l"(mp), "r"(0), "r"(0), "r"(0), "r"(su(bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(su(buf)), "l"(mp), "r"(x0), "r"(y0), "r"(z0), "r"(c2), "r"(su(bar)) : "memory");
  }
  asm volatile("{\n.reg .pred d;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n@!d bra W_%=;\n}\n" ::"r"(su(bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int rank = atoi(argv[1]), dyn = atoi(argv[2]), fence = atoi(argv[3]), sw = atoi(argv[4]);
  const int nthr = argc > 5 ? atoi(argv[5]) : 32;
  const int x0 = argc > 6 ? atoi(argv[6]) : 0, y0 = argc > 7 ? atoi(argv[7]) : 0, z0 = argc > 8 ? atoi(argv[8]) : 0;
  const int bz = argc > 9 ? atoi(argv[9]) : 4;
  double* d;
  const int E0 = 40, E1 = 36, E2 = 30;
  std::vector<double> h((size_t)E0 * E1 * E2 * 3);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  cudaMalloc(&d, 8 * h.size());
  cudaMemcpy(d, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
  double* o;
  cudaMalloc(&o, 64 * 8);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)E0, (cuuint64_t)E1, (cuuint64_t)E2, 3};
  cuuint64_t str[3] = {(cuuint64_t)E0 * 8, (cuuint64_t)E0 * E1 * 8, (cuuint64_t)E0 * E1 * E2 * 8};
  cuuint32_t box[4] = {16, 16, (cuuint32_t)bz, 1}, el[4] = {1, 1, 1, 1};
  CUresult r = ((Enc)f)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        (CUtensorMapSwizzle)sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = 16 * 16 * 8 * (rank >= 3 ? bz : 1);
  printf("rank %d dyn %d fence %d sw %d thr %d x%d y%d z%d bz%d encode %d: ", rank, dyn, fence, sw, nthr, x0, y0, z0, bz, (int)r);
  if (dyn) {
    cudaFuncSetAttribute(k3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k3<true><<<1, nthr, 64 * 1024>>>(m, rank, bytes, o, fence, 1, x0, y0, z0);
  } else {
    k3<false><<<1, nthr>>>(m, rank, bytes, o, fence, 1, x0, y0, z0);
  }
  printf("%s ", cudaGetErrorString(cudaDeviceSynchronize()));
  double g[64];
  cudaMemcpy(g, o, 512, cudaMemcpyDeviceToHost);
  printf("out %g %g %g\n", g[0], g[1], g[16]);
  return 0;
}
