// Standalone probe of the TMA gather's mechanics (tensor map over a padded
// fp64 array, 4D box {16,16,PZ,1}, 128B swizzle, mbarrier completion).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tma_probe.cu -o tools/bin/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// MODE 0: TMA 4D; 1: mbarrier arrive only (no TMA); 2: 1D cp.async.bulk; 3: TMA 4D without the
// init fence; 4: TMA 4D with try_wait without .shared::cta; 5: TMA 3D (c folded into z)
__global__ void k_probe(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap3,
                        int MODE, int PZ, int x0, int y0, int z0, int c, const double* src, double* out,
                        const CUtensorMap* gmap) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  double* buf = reinterpret_cast<double*>(base);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 16 * 16 * PZ);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    if (MODE != 3) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned bytes = 16 * 16 * PZ * 8;
    if (MODE == 1) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
      if (MODE == 2)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(buf)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
      else if (MODE == 5)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(buf)),
                     "l"(reinterpret_cast<uint64_t>(&tmap3)), "r"(x0), "r"(y0), "r"(z0), "r"(smem_u32(bar)) : "memory");
      else if (MODE == 6)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(buf)),
                     "l"(reinterpret_cast<uint64_t>(gmap)), "r"(x0), "r"(y0), "r"(z0), "r"(c), "r"(smem_u32(bar)) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(buf)),
                     "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(z0), "r"(c), "r"(smem_u32(bar)) : "memory");
    }
  }
  if (MODE == 4)
    asm volatile("{\n.reg .pred done;\nWAIT_%=:\nmbarrier.try_wait.parity.b64 done, [%0], %1;\n@!done bra WAIT_%=;\n}\n"
                 ::"l"(bar), "r"(0) : "memory");
  else
    asm volatile("{\n.reg .pred done;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n@!done bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 16 * 16 * PZ; i += blockDim.x) out[i] = buf[i];
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int MODE = argc > 1 ? atoi(argv[1]) : 0;
  const int SW = argc > 2 ? atoi(argv[2]) : 3;     // 0 none, 3 = 128B
  const int L2P = argc > 3 ? atoi(argv[3]) : 2;    // 0 none, 2 = 128B? (enum), 3 = 256B
  const int PZarg = argc > 4 ? atoi(argv[4]) : 15;
  const int E0 = 40, E1 = 36, E2 = 30;
  const int PZ = PZarg;
  const size_t cs = (size_t)E0 * E1 * E2;
  std::vector<double> h(3 * cs);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, 8 * h.size());
  cudaMemcpy(d, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
  cudaMalloc(&o, 8 * 16 * 16 * PZ);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  printf("entry %p q=%d\n", f, (int)q);
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)E0, (cuuint64_t)E1, (cuuint64_t)E2, 3};
  cuuint64_t str[3] = {(cuuint64_t)E0 * 8, (cuuint64_t)E0 * E1 * 8, cs * 8};
  cuuint32_t box[4] = {16, 16, (cuuint32_t)PZ, 1}, el[4] = {1, 1, 1, 1};
  CUresult r = ((EncodeTiled)f)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, el,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)SW,
                                (CUtensorMapL2promotion)L2P, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d sw %d l2p %d pz %d\n", (int)r, SW, L2P, PZ);
  CUtensorMap m3;
  cuuint64_t dims3[3] = {(cuuint64_t)E0, (cuuint64_t)E1, (cuuint64_t)E2 * 3};
  cuuint32_t box3[3] = {16, 16, (cuuint32_t)PZ};
  r = ((EncodeTiled)f)(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims3, str, box3, el,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)SW,
                       (CUtensorMapL2promotion)L2P, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode3 %d mode %d\n", (int)r, MODE);
  size_t smem = 1024 + 8 * 16 * 16 * PZ + 64;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int x0 = 9, y0 = 18, c = 2;
  const int z0 = MODE == 5 ? 8 + 2 * E2 : 8;
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &m, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  printf("sizeof map %zu align %zu host addr %p\n", sizeof(CUtensorMap), alignof(CUtensorMap), (void*)&m);
  k_probe<<<1, 128, smem>>>(m, m3, MODE, PZ, x0, y0, z0, c, d, o, gm);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<double> got(16 * 16 * PZ);
  cudaMemcpy(got.data(), o, 8 * got.size(), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int z = 0; z < PZ; ++z)
    for (int y = 0; y < 16; ++y)
      for (int x = 0; x < 16; ++x) {
        const int xs = SW == 3 ? (x ^ ((y & 7) << 1)) : x;
        const double want = h[c * cs + ((size_t)(z0 + z) * E1 + (y0 + y)) * E0 + (x0 + x)];
        const double v = got[(z * 16 + y) * 16 + xs];
        if (v != want && bad++ < 5) printf("mismatch z%d y%d x%d got %g want %g\n", z, y, x, v, want);
      }
  printf("bad=%d\n", bad);
  return 0;
}
