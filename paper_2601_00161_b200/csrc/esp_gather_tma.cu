// esp_gather_tma.cu — persistent, TMA-fed ik force gather (mesh.py:213-218
// `_gather` for the three ik fields of long_range_forces, mesh.py:336-342).
//
// Production gather for fp64, P <= 8, on the band-pruned transform path.
//
// * Fields: the inverse x pass (k_x_c2r) writes the three ik fields into a
//   ghost-padded array [3][E2][E1][E0] whose ghost planes/rows/columns hold
//   the periodic images, so every anchor tile's stencil box is one dense,
//   in-bounds box: one cp.async.bulk.tensor (TMA) per field, completing on
//   an mbarrier.  TMA boxes must start on a 16-byte boundary along x, so the
//   box is 18 columns wide from the even column at or below the tile's first
//   column (tiles are 17 - P = 9 anchors wide: every other tile starts odd).
// * Persistent CTAs (one per SM): a producer warp streams tile boxes into a
//   2-stage ring (full/empty mbarriers); NW consumer warps gather while the
//   next tile lands.  Tiles are visited z-slab-major so neighbouring tiles'
//   halo boxes are served from L2.
// * Weights are evaluated in the kernel from the binned grid coordinates u
//   (the same unrolled Horner chains as the binning pass, coefficients from
//   the constant bank; no 192 B/charge weight records): a warp takes its
//   particles in batches of 10, lane (particle, axis) evaluates one axis's
//   weights into a per-warp shared-memory slot, then the batch is gathered
//   two particles at a time.
// * Warp = 2 particles x 8 stencil rows x 2 x-parities.  Lane (p, j, e)
//   sums row y = yl + j, columns x = xl + e + 2i (i < 4), over the 8 planes.
//   Rows of 18 doubles (144 B) put row j at bank offset 2j, so the 16 lanes
//   of a particle (2j + e) hit 16 distinct 8-byte bank pairs for every load:
//   conflict-free without a swizzle.
//   The 16 lanes reduce with 4 xor-shuffle levels; one lane writes the
//   force.  No atomics, fixed order: bitwise reproducible.
//
// F_c = -q * sum (the h3 factors of mesh.py:341-342 cancel; the 1/G of the
// inverse transform is folded into the spectrum).
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "esp_internal.cuh"

namespace esp {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

constexpr int kTmaStages = 2;
#ifndef ESP_TMA_RECORDS
#define ESP_TMA_RECORDS 1   // the gathers read the weight records of the binning pass
                            // (config 4 fp64: 4.21 -> 3.54 ms against evaluating them in
                            // the batch prologue)
#endif
#ifndef ESP_TMA_UNROLL
#define ESP_TMA_UNROLL 1
#endif
constexpr int kUnroll64 = ESP_TMA_UNROLL;   // particle pairs in flight per warp (fp64)

template <int NW>
struct TmaGatherLayout {
  static constexpr int kBatch = NW > 12 ? 6 : (NW > 8 ? 8 : 10);   // particles per warp batch
  // 8-byte slots: weights, q, then ints: anchors [3 KB], ids [KB], kept list [KB]
  static constexpr int kWarpW = kBatch * 24 + kBatch + 3 * kBatch;
  static constexpr int kRow = 18;         // box columns (16 needed + alignment slack)
  __host__ __device__ static size_t box_elems(int PZ) { return (size_t)kRow * 16 * PZ; }
  __host__ __device__ static size_t bytes(int PZ) {
    size_t b = 1024;                                          // alignment slack
    b += sizeof(double) * 3 * box_elems(PZ) * kTmaStages;     // field boxes
    b += sizeof(double) * (size_t)NW * kWarpW;                // weight slots
    b += sizeof(uint64_t) * 2 * kTmaStages;                   // full / empty barriers
    return b;
  }
};

template <int P, int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
k_gather_tma(const __grid_constant__ CUtensorMap tmap, Geom g, FastTab ft,
             const double* __restrict__ tab, const double* __restrict__ brk, int n_pieces,
             int ncoef, const int* __restrict__ offsets, const double* __restrict__ U,
             long long cap, const double* __restrict__ Q, const int* __restrict__ IDX,
             double* __restrict__ forces, int xsh, const double* __restrict__ WREC,
             const int* __restrict__ PK, int id_lo, int id_hi) {
  static_assert(P <= 8, "the TMA gather covers stencils of at most 8 points");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1 KB-aligned base; offset arithmetic on smem_raw keeps the shared state
  // space visible to the compiler (LDS/STS instead of generic accesses)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const size_t box = TmaGatherLayout<NW>::box_elems(g.PZ);
  double* fbuf = reinterpret_cast<double*>(base);
  double* wslot = fbuf + 3 * box * kTmaStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(wslot + NW * TmaGatherLayout<NW>::kWarpW);
  uint64_t* empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int nxy = g.ntx * g.nty;
  const int ntiles = nxy * g.ntz;
  const unsigned box_bytes = (unsigned)(sizeof(double) * box);

  if (warp == NW) {                       // producer: one elected lane issues the TMA
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tz = t / nxy, txy = t - tz * nxy;
        const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
        const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
        if (offsets[key0] == offsets[key1]) continue;
        const int s = it % kTmaStages;
        if (it >= kTmaStages) mbar_wait(&empty[s], ((it / kTmaStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], 3 * box_bytes);
        const int tx = txy % g.ntx, ty = txy / g.ntx;
        double* dst = fbuf + (size_t)s * 3 * box;
        const int bx = (tx * g.TX + xsh) & ~1;   // TMA boxes start 16-byte aligned
#pragma unroll
        for (int c = 0; c < 3; ++c)
          tma_load_4d(dst + c * box, &tmap, &full[s], bx, ty * g.TY, tz * g.TZ, c);
        ++it;
      }
    }
    return;
  }

  const int p = lane >> 4, sub = lane & 15;
  const int j = sub >> 1, e = sub & 1;
  constexpr int R = TmaGatherLayout<NW>::kRow;
  constexpr int KB = TmaGatherLayout<NW>::kBatch;
  double* Wb = wslot + warp * TmaGatherLayout<NW>::kWarpW;        // [KB][3][8] weights
  double* s_qv = Wb + KB * 24;                                     // [KB] charges
  int* s_ai = reinterpret_cast<int*>(s_qv + KB);                   // [KB][3] anchors, [KB] ids
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tz = t / nxy, txy = t - tz * nxy;
    const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
    const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
    const long long p0 = offsets[key0], p1 = offsets[key1];
    if (p0 == p1) continue;
    const int tx = txy % g.ntx, ty = txy / g.ntx;
    // box-local column of grid anchor a: a + xsh - (box start)
    const int org0 = ((tx * g.TX + xsh) & ~1) - xsh, org1 = ty * g.TY, org2 = tz * g.TZ;
    const int s = it % kTmaStages;
    // rotate the batch order per tile so no warp always takes the extra batch
    const int wr = (warp + it) % NW;
    bool waited = false;
    const double* F = fbuf + (size_t)s * 3 * box;
    for (long long bb = p0 + (long long)wr * KB; bb < p1; bb += (long long)NW * KB) {
      const int nb = (int)min((long long)KB, p1 - bb);
#if ESP_TMA_RECORDS
      // batch prologue: the binning pass's weight records (written for the
      // spread anyway) land with cp.async; lanes < KB decode the packed
      // tile-local anchors and fetch q and the index
      {
        constexpr int kPieces = KB * 24 * 8 / 16;                 // 16 B pieces of KB records
        const char* src = reinterpret_cast<const char*>(WREC + bb * 24);
        const int avail = nb * 24 * 8;
        for (int c = lane; c < kPieces; c += 32)
          if (c * 16 < avail) {
            const unsigned dst = smem_u32(reinterpret_cast<char*>(Wb) + c * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + c * 16));
          }
        asm volatile("cp.async.commit_group;");
        if (lane < nb) {
          const int pk = PK[bb + lane];
          s_ai[lane * 3 + 0] = (pk & 0xff) + tx * g.TX - org0;
          s_ai[lane * 3 + 1] = (pk >> 8) & 0xff;
          s_ai[lane * 3 + 2] = (pk >> 16) - org2;
          s_qv[lane] = Q[bb + lane];
          s_ai[3 * KB + lane] = IDX[bb + lane];
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
#else
#error "the chunked (original-index range) gather needs the records prologue"
      // batch prologue (overlaps the tile's TMA on the first batch): lane
      // (particle, dim) evaluates the 8 weights of one axis with the unrolled
      // Horner chains of the binning pass (uniform table reads) and the
      // box-local anchor
      if (lane < 3 * KB) {
        const int pl = lane / 3, d = lane - 3 * pl;
        if (pl < nb) {
          const double u = U[d * cap + bb + pl];
          const double base = anchor_base(g, u);
          double w[P];
          stencil_weights<double, P>(ft, tab, brk, n_pieces, ncoef, u, base, g.lo, 1.0, w);
#pragma unroll
          for (int ss = 0; ss < 8; ++ss) Wb[pl * 24 + d * 8 + ss] = ss < P ? w[ss < P ? ss : 0] : 0.0;
          s_ai[pl * 3 + d] = local_anchor(g, d, base) - (d == 0 ? org0 : (d == 1 ? org1 : org2));
          if (d == 0) {
            s_qv[pl] = Q[bb + pl];
            s_ai[3 * KB + pl] = IDX[bb + pl];
          }
        }
      }
#endif
      __syncwarp();
      if (!waited) {
        mbar_wait(&full[s], (it / kTmaStages) & 1);
        waited = true;
      }
#pragma unroll kUnroll64
      // charges of this pass (original index in [id_lo, id_hi): host-buffer
      // steps gather in index ranges so each range's copy-out overlaps the
      // rest), compacted in batch order
      int* s_keep = s_ai + 4 * KB;
      int nk;
      {
        const int id = lane < nb ? IDX[bb + lane] : 0;
        const bool keep = lane < nb && id >= id_lo && id < id_hi;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) s_keep[__popc(mk & ((1u << lane) - 1u))] = lane;
        nk = __popc(mk);
      }
      __syncwarp();
      for (int pp = 0; pp < nk; pp += 2) {
        const bool live = pp + p < nk;
        const int pl = live ? s_keep[pp + p] : 0;
        double ax = 0.0, ay = 0.0, az = 0.0;
        if (live && j < P) {
          const double* W = Wb + pl * 24;
          const int xl = s_ai[pl * 3], yl = s_ai[pl * 3 + 1], zl = s_ai[pl * 3 + 2];
          const double wy = W[8 + j];
          double wx[4], wz[P];
#pragma unroll
          for (int i = 0; i < 4; ++i) wx[i] = (e + 2 * i < P) ? W[e + 2 * i] : 0.0;
#pragma unroll
          for (int k = 0; k < P; k += 2) {               // 16-byte broadcast loads
            const double2 v = *reinterpret_cast<const double2*>(W + 16 + k);
            wz[k] = v.x;
            if (k + 1 < P) wz[k + 1] = v.y;
          }
          const int row = (zl * 16 + yl + j) * R;
          const double* col[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) col[i] = F + row + min(xl + e + 2 * i, R - 1);
          double bx[2] = {0.0, 0.0}, by[2] = {0.0, 0.0}, bz[2] = {0.0, 0.0};
#pragma unroll
          for (int k = 0; k < P; ++k) {
            double rx[2] = {0.0, 0.0}, ry[2] = {0.0, 0.0}, rz[2] = {0.0, 0.0};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (2 * i < P) {                      // e + 2i < P is folded into wx
                const double* a = col[i] + k * 16 * R;
                rx[i & 1] = fma(wx[i], a[0], rx[i & 1]);
                ry[i & 1] = fma(wx[i], a[box], ry[i & 1]);
                rz[i & 1] = fma(wx[i], a[2 * box], rz[i & 1]);
              }
            }
            bx[k & 1] = fma(wz[k], rx[0] + rx[1], bx[k & 1]);
            by[k & 1] = fma(wz[k], ry[0] + ry[1], by[k & 1]);
            bz[k & 1] = fma(wz[k], rz[0] + rz[1], bz[k & 1]);
          }
          ax = (bx[0] + bx[1]) * wy;
          ay = (by[0] + by[1]) * wy;
          az = (bz[0] + bz[1]) * wy;
        }
        // transposed 16-lane reduction of (ax, ay, az): 5 double shuffles
        // instead of 12 (shuffles share the shared-memory datapath); the
        // totals land in lanes 0 / 4 / 8 of the half-warp
        const unsigned full_mask = 0xffffffffu;
        const bool h8 = sub & 8, h4 = sub & 4;
        const double r0 = __shfl_xor_sync(full_mask, h8 ? ax : az, 8);
        const double r1 = __shfl_xor_sync(full_mask, h8 ? ay : 0.0, 8);
        const double v0 = (h8 ? az : ax) + r0;
        const double v1 = (h8 ? 0.0 : ay) + r1;
        double v = (h4 ? v1 : v0) + __shfl_xor_sync(full_mask, h4 ? v0 : v1, 4);
        v += __shfl_xor_sync(full_mask, v, 2);
        v += __shfl_xor_sync(full_mask, v, 1);
        if ((sub & 3) == 0 && sub < 12 && live) {
          const double q = s_qv[pl];
          forces[3 * (long long)s_ai[3 * KB + pl] + (sub >> 2)] = -q * v;
        }
      }
      __syncwarp();                               // the batch slots are rewritten next
    }
    if (!waited) mbar_wait(&full[s], (it / kTmaStages) & 1);   // keep the phase in step
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++it;
  }
}

// fp32 fields (precision="fp32"): one particle per warp instruction.  Boxes
// are 20 floats wide (16 needed; fp32 TMA boxes start on 4-float
// boundaries); lane (row j = lane >> 2, e = lane & 3) sums row y = yl + j,
// columns xl + e + 4i (i < 2) over the 8 planes: row stride 20 floats puts
// lane (j, e) at bank 20j + e mod 32 — all 32 distinct, one wavefront per
// load.  Weights from u in fp32 (the fp32 table, fp64 coordinates and
// anchors, as the rest of the fp32 path); a transposed 32-lane reduction.
#ifndef ESP_TMA32_UNROLL
#define ESP_TMA32_UNROLL 4   // particles in flight per warp (config 4 fp32 gather: 1 -> 3.48 ms,
                             // 2 -> 3.22, 4 -> 3.03 at 12 warps; 8 -> 3.20)
#endif
constexpr int kUnroll32 = ESP_TMA32_UNROLL;
template <int NW>
struct TmaGather32Layout {
  static constexpr int kRow = 20;
  static constexpr int kBatch = 10;
  // 4-byte slots: weights, spare, anchors + ids + kept list; a multiple of 4
  // so every warp's slot starts 16-byte aligned (cp.async targets)
  static constexpr int kWarpW = (kBatch * 24 + kBatch + 5 * kBatch + 3) & ~3;
  __host__ __device__ static size_t box_elems(int PZ) { return (size_t)kRow * 16 * PZ; }
  __host__ __device__ static size_t bytes(int PZ) {
    size_t b = 1024;
    b += sizeof(float) * 3 * box_elems(PZ) * kTmaStages;
    b += sizeof(float) * (size_t)NW * kWarpW;
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint64_t) * 2 * kTmaStages;
    return b;
  }
};

template <int P, int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
k_gather_tma32(const __grid_constant__ CUtensorMap tmap, Geom g, FastTab ft,
               const float* __restrict__ tab, const double* __restrict__ brk, int n_pieces,
               int ncoef, const int* __restrict__ offsets, const double* __restrict__ U,
               long long cap, const double* __restrict__ Q, const int* __restrict__ IDX,
               double* __restrict__ forces, int xsh, const float* __restrict__ WREC,
               const int* __restrict__ PK, int id_lo, int id_hi) {
  static_assert(P <= 8, "the TMA gather covers stencils of at most 8 points");
  using LY = TmaGather32Layout<NW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const size_t box = LY::box_elems(g.PZ);
  float* fbuf = reinterpret_cast<float*>(base);
  float* wslot = fbuf + 3 * box * kTmaStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      base + ((sizeof(float) * (3 * box * kTmaStages + (size_t)NW * LY::kWarpW) + 15) & ~size_t(15)));
  uint64_t* empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nxy = g.ntx * g.nty;
  const int ntiles = nxy * g.ntz;
  const unsigned box_bytes = (unsigned)(sizeof(float) * box);
  if (warp == NW) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tz = t / nxy, txy = t - tz * nxy;
        const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
        const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
        if (offsets[key0] == offsets[key1]) continue;
        const int s = it % kTmaStages;
        if (it >= kTmaStages) mbar_wait(&empty[s], ((it / kTmaStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], 3 * box_bytes);
        const int tx = txy % g.ntx, ty = txy / g.ntx;
        float* dst = fbuf + (size_t)s * 3 * box;
        const int bx = (tx * g.TX + xsh) & ~3;   // fp32 boxes start on 4-float boundaries
#pragma unroll
        for (int c = 0; c < 3; ++c)
          tma_load_4d(dst + c * box, &tmap, &full[s], bx, ty * g.TY, tz * g.TZ, c);
        ++it;
      }
    }
    return;
  }
  const int j = lane >> 2, e = lane & 3;
  constexpr int R = LY::kRow;
  constexpr int KB = LY::kBatch;
  float* Wb = wslot + warp * LY::kWarpW;                           // [KB][3][8] weights
  int* s_ai = reinterpret_cast<int*>(Wb + KB * 24 + KB);           // [KB][3] anchors, [KB] ids
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tz = t / nxy, txy = t - tz * nxy;
    const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
    const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
    const long long p0 = offsets[key0], p1 = offsets[key1];
    if (p0 == p1) continue;
    const int tx = txy % g.ntx, ty = txy / g.ntx;
    const int org0 = ((tx * g.TX + xsh) & ~3) - xsh, org1 = ty * g.TY, org2 = tz * g.TZ;
    const int s = it % kTmaStages;
    const int wr = (warp + it) % NW;
    bool waited = false;
    const float* F = fbuf + (size_t)s * 3 * box;
    for (long long bb = p0 + (long long)wr * KB; bb < p1; bb += (long long)NW * KB) {
      const int nb = (int)min((long long)KB, p1 - bb);
#if ESP_TMA_RECORDS
      {
        constexpr int kPieces = KB * 24 * 4 / 16;                 // 16 B pieces of KB records
        const char* src = reinterpret_cast<const char*>(WREC + bb * 24);
        const int avail = nb * 24 * 4;
        for (int c = lane; c < kPieces; c += 32)
          if (c * 16 < avail) {
            const unsigned dst = smem_u32(reinterpret_cast<char*>(Wb) + c * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + c * 16));
          }
        asm volatile("cp.async.commit_group;");
        if (lane < nb) {
          const int pk = PK[bb + lane];
          s_ai[lane * 3 + 0] = (pk & 0xff) + tx * g.TX - org0;
          s_ai[lane * 3 + 1] = (pk >> 8) & 0xff;
          s_ai[lane * 3 + 2] = (pk >> 16) - org2;
          s_ai[3 * KB + lane] = IDX[bb + lane];
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      if (false) {
#else
      if (lane < 3 * KB) {
#endif
        const int pl = lane / 3, d = lane - 3 * pl;
        if (pl < nb) {
          const double u = U[d * cap + bb + pl];
          const double base = anchor_base(g, u);
          float w[P];
          stencil_weights<float, P>(ft, tab, brk, n_pieces, ncoef, u, base, g.lo, 1.0f, w);
#pragma unroll
          for (int ss = 0; ss < 8; ++ss) Wb[pl * 24 + d * 8 + ss] = ss < P ? w[ss < P ? ss : 0] : 0.0f;
          s_ai[pl * 3 + d] = local_anchor(g, d, base) - (d == 0 ? org0 : (d == 1 ? org1 : org2));
          if (d == 0) s_ai[3 * KB + pl] = IDX[bb + pl];
        }
      }
      __syncwarp();
      if (!waited) {
        mbar_wait(&full[s], (it / kTmaStages) & 1);
        waited = true;
      }
      int* s_keep = s_ai + 4 * KB;
      int nk;
      {
        const int id = lane < nb ? IDX[bb + lane] : 0;
        const bool keep = lane < nb && id >= id_lo && id < id_hi;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) s_keep[__popc(mk & ((1u << lane) - 1u))] = lane;
        nk = __popc(mk);
      }
      __syncwarp();
#pragma unroll kUnroll32
      for (int kk = 0; kk < nk; ++kk) {
        const int pl = s_keep[kk];
        float ax = 0.f, ay = 0.f, az = 0.f;
        if (j < P) {
          const float* W = Wb + pl * 24;
          const int xl = s_ai[pl * 3], yl = s_ai[pl * 3 + 1], zl = s_ai[pl * 3 + 2];
          const float wy = W[8 + j];
          float wx[2], wz[P];
#pragma unroll
          for (int i = 0; i < 2; ++i) wx[i] = (e + 4 * i < P) ? W[e + 4 * i] : 0.f;
#pragma unroll
          for (int k = 0; k < P; ++k) wz[k] = W[16 + k];
          const int row = (zl * 16 + yl + j) * R;
          const float* c0 = F + row + min(xl + e, R - 1);
          const float* c1 = F + row + min(xl + e + 4, R - 1);
#pragma unroll
          for (int k = 0; k < P; ++k) {
            const float* a = c0 + k * 16 * R;
            const float* b = c1 + k * 16 * R;
            const float rx = fmaf(wx[1], b[0], wx[0] * a[0]);
            const float ry = fmaf(wx[1], b[box], wx[0] * a[box]);
            const float rz = fmaf(wx[1], b[2 * box], wx[0] * a[2 * box]);
            ax = fmaf(wz[k], rx, ax);
            ay = fmaf(wz[k], ry, ay);
            az = fmaf(wz[k], rz, az);
          }
          ax *= wy;
          ay *= wy;
          az *= wy;
        }
        // transposed 32-lane reduction: totals in lanes 0 / 8 / 16
        const unsigned fm = 0xffffffffu;
        const bool h16 = lane & 16, h8 = lane & 8;
        const float r0 = __shfl_xor_sync(fm, h16 ? ax : az, 16);
        const float r1 = __shfl_xor_sync(fm, h16 ? ay : 0.f, 16);
        const float v0 = (h16 ? az : ax) + r0;
        const float v1 = (h16 ? 0.f : ay) + r1;
        float v = (h8 ? v1 : v0) + __shfl_xor_sync(fm, h8 ? v0 : v1, 8);
        v += __shfl_xor_sync(fm, v, 4);
        v += __shfl_xor_sync(fm, v, 2);
        v += __shfl_xor_sync(fm, v, 1);
        if ((lane & 7) == 0 && lane < 24) {
          const double q = Q[bb + pl];
          forces[3 * (long long)s_ai[3 * KB + pl] + (lane >> 3)] = -q * (double)v;
        }
      }
      __syncwarp();
    }
    if (!waited) mbar_wait(&full[s], (it / kTmaStages) & 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++it;
  }
}

// Analytic forces (mesh.py:343-349): window-gradient gather of the ONE
// ghost-padded potential field.  Same pipeline and lane map as k_gather_tma
// (fp64); each batch's weight and derivative-weight records (written by the
// binning pass of an analytic step) land with cp.async.  Per plane a lane
// forms S_w = sum_i wx_i f and S_d = sum_i wx'_i f over its 4 columns;
// A = sum_k wz S_d, B = sum_k wz S_w, C = sum_k wz' S_w give G_x = wy A,
// G_y = wy' B, G_z = wy C; F_a = -q sum_d G_d J[d][a].
template <int NW>
struct TmaGradLayout {
  static constexpr int kRow = 18;
  static constexpr int kBatch = 8;
  static constexpr int kWarpW = kBatch * 48 + kBatch + 2 * kBatch;   // w | w', q, anchors+ids
  __host__ __device__ static size_t box_elems(int PZ) { return (size_t)kRow * 16 * PZ; }
  __host__ __device__ static size_t bytes(int PZ) {
    size_t b = 1024;
    b += sizeof(double) * box_elems(PZ) * kTmaStages;
    b += sizeof(double) * (size_t)NW * kWarpW;
    b += sizeof(uint64_t) * 2 * kTmaStages;
    return b;
  }
};

template <int P, int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
k_gather_grad_tma(const __grid_constant__ CUtensorMap tmap, Geom g,
                  const int* __restrict__ offsets, const double* __restrict__ WREC,
                  const double* __restrict__ DREC, const int* __restrict__ PK,
                  const double* __restrict__ Q, const int* __restrict__ IDX, Jac J,
                  double* __restrict__ forces, int xsh) {
  static_assert(P <= 8, "the TMA gather covers stencils of at most 8 points");
  using LY = TmaGradLayout<NW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const size_t box = LY::box_elems(g.PZ);
  double* fbuf = reinterpret_cast<double*>(base);
  double* wslot = fbuf + box * kTmaStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(wslot + NW * LY::kWarpW);
  uint64_t* empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nxy = g.ntx * g.nty;
  const int ntiles = nxy * g.ntz;
  const unsigned box_bytes = (unsigned)(sizeof(double) * box);
  if (warp == NW) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tz = t / nxy, txy = t - tz * nxy;
        const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
        const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
        if (offsets[key0] == offsets[key1]) continue;
        const int s = it % kTmaStages;
        if (it >= kTmaStages) mbar_wait(&empty[s], ((it / kTmaStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], box_bytes);
        const int tx = txy % g.ntx, ty = txy / g.ntx;
        tma_load_4d(fbuf + (size_t)s * box, &tmap, &full[s], (tx * g.TX + xsh) & ~1, ty * g.TY,
                    tz * g.TZ, 0);
        ++it;
      }
    }
    return;
  }
  const int p = lane >> 4, sub = lane & 15;
  const int j = sub >> 1, e = sub & 1;
  constexpr int R = LY::kRow;
  constexpr int KB = LY::kBatch;
  double* Wb = wslot + warp * LY::kWarpW;        // [KB][3][8] weights, then [KB][3][8] derivatives
  double* Db = Wb + KB * 24;
  double* s_qv = Wb + KB * 48;
  int* s_ai = reinterpret_cast<int*>(s_qv + KB);
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tz = t / nxy, txy = t - tz * nxy;
    const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
    const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
    const long long p0 = offsets[key0], p1 = offsets[key1];
    if (p0 == p1) continue;
    const int tx = txy % g.ntx;
    const int org0 = ((tx * g.TX + xsh) & ~1) - xsh, org2 = tz * g.TZ;
    const int s = it % kTmaStages;
    const int wr = (warp + it) % NW;
    bool waited = false;
    const double* F = fbuf + (size_t)s * box;
    for (long long bb = p0 + (long long)wr * KB; bb < p1; bb += (long long)NW * KB) {
      const int nb = (int)min((long long)KB, p1 - bb);
      {
        constexpr int kPieces = KB * 24 * 8 / 16;
        const int avail = nb * 24 * 8;
        const char* sw = reinterpret_cast<const char*>(WREC + bb * 24);
        const char* sd = reinterpret_cast<const char*>(DREC + bb * 24);
        for (int c = lane; c < 2 * kPieces; c += 32) {
          const int which = c >= kPieces, piece = which ? c - kPieces : c;
          if (piece * 16 < avail) {
            const unsigned dst =
                smem_u32(reinterpret_cast<char*>(which ? Db : Wb) + piece * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"((which ? sd : sw) + piece * 16));
          }
        }
        asm volatile("cp.async.commit_group;");
        if (lane < nb) {
          const int pk = PK[bb + lane];
          s_ai[lane * 3 + 0] = (pk & 0xff) + tx * g.TX - org0;
          s_ai[lane * 3 + 1] = (pk >> 8) & 0xff;
          s_ai[lane * 3 + 2] = (pk >> 16) - org2;
          s_qv[lane] = Q[bb + lane];
          s_ai[3 * KB + lane] = IDX[bb + lane];
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      if (!waited) {
        mbar_wait(&full[s], (it / kTmaStages) & 1);
        waited = true;
      }
      for (int pp = 0; pp < nb; pp += 2) {
        const int pl = pp + p;
        const bool live = pl < nb;
        double gx = 0.0, gy = 0.0, gz = 0.0;
        if (live && j < P) {
          const double* W = Wb + pl * 24;
          const double* D = Db + pl * 24;
          const int xl = s_ai[pl * 3], yl = s_ai[pl * 3 + 1], zl = s_ai[pl * 3 + 2];
          double wx[4], dx[4], wz[P], dz[P];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            wx[i] = (e + 2 * i < P) ? W[e + 2 * i] : 0.0;
            dx[i] = (e + 2 * i < P) ? D[e + 2 * i] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < P; ++k) {
            wz[k] = W[16 + k];
            dz[k] = D[16 + k];
          }
          const int row = (zl * 16 + yl + j) * R;
          const double* col[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) col[i] = F + row + min(xl + e + 2 * i, R - 1);
          double A[2] = {0.0, 0.0}, B[2] = {0.0, 0.0}, C2[2] = {0.0, 0.0};
#pragma unroll
          for (int k = 0; k < P; ++k) {
            double sw = 0.0, sd = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (2 * i < P) {
                const double v = col[i][k * 16 * R];
                sw = fma(wx[i], v, sw);
                sd = fma(dx[i], v, sd);
              }
            }
            A[k & 1] = fma(wz[k], sd, A[k & 1]);
            B[k & 1] = fma(wz[k], sw, B[k & 1]);
            C2[k & 1] = fma(dz[k], sw, C2[k & 1]);
          }
          gx = W[8 + j] * (A[0] + A[1]);
          gy = D[8 + j] * (B[0] + B[1]);
          gz = W[8 + j] * (C2[0] + C2[1]);
        }
        const unsigned fm = 0xffffffffu;
        const bool h8 = sub & 8, h4 = sub & 4;
        const double r0 = __shfl_xor_sync(fm, h8 ? gx : gz, 8);
        const double r1 = __shfl_xor_sync(fm, h8 ? gy : 0.0, 8);
        const double v0 = (h8 ? gz : gx) + r0;
        const double v1 = (h8 ? 0.0 : gy) + r1;
        double v = (h4 ? v1 : v0) + __shfl_xor_sync(fm, h4 ? v0 : v1, 4);
        v += __shfl_xor_sync(fm, v, 2);
        v += __shfl_xor_sync(fm, v, 1);
        // lanes 0 / 4 / 8 of the half hold G_x / G_y / G_z
        const int hb = lane & 16;
        const double Gx = __shfl_sync(fm, v, hb + 0);
        const double Gy = __shfl_sync(fm, v, hb + 4);
        const double Gz = __shfl_sync(fm, v, hb + 8);
        if (sub < 3 && live) {
          const double q = s_qv[pl];
          const double j0 = sub == 0 ? J.j[0] : (sub == 1 ? J.j[1] : J.j[2]);
          const double j1 = sub == 0 ? J.j[3] : (sub == 1 ? J.j[4] : J.j[5]);
          const double j2 = sub == 0 ? J.j[6] : (sub == 1 ? J.j[7] : J.j[8]);
          forces[3 * (long long)s_ai[3 * KB + pl] + sub] = -q * ((Gx * j0 + Gy * j1) + Gz * j2);
        }
      }
      __syncwarp();
    }
    if (!waited) mbar_wait(&full[s], (it / kTmaStages) & 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++it;
  }
}

// Host side -------------------------------------------------------------------

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiled>(f);
  }();
  return fn;
}

}  // namespace

// Ghost-padded field layout for the TMA gather: axis d needs grid indices
// [lo, (n_d - 1) T_d + lo + W_d - 1], stored at padded index (index - lo).
FieldPad make_field_pad(const esp_plan* p) {
  FieldPad f;
  std::memset(&f, 0, sizeof(f));
  const int T[3] = {p->TX, p->TY, p->TZ};
  const int W[3] = {kPad, kPad, p->PZ};
  const int n[3] = {p->ntx, p->nty, p->ntz};
  for (int d = 0; d < 3; ++d) {
    f.M[d] = p->M[d];
    f.S[d] = -p->lo;
    f.E[d] = (n[d] - 1) * T[d] + W[d];
  }
  // x: shift so rows start on a 32-byte sector, columns of slack for the
  // boxes of tiles that start off a 16-byte boundary (fp64: 18-column boxes
  // from even columns; fp32: 20-column boxes from multiples of 4), pitch a
  // whole number of sectors
  const bool dp = p->precision == ESP_FP64;
  const int sec = dp ? 4 : 8, slack = dp ? 2 : 4;
  const int xsh = (sec - f.S[0] % sec) % sec;
  f.S[0] += xsh;
  f.E[0] += xsh + slack;
  f.E[0] = (f.E[0] + sec - 1) / sec * sec;
  f.cstride = (long long)f.E[0] * f.E[1] * f.E[2];
  f.enabled = 1;
  return f;
}

bool tma_gather_eligible(const esp_plan* p) {
  return p->P <= 8 && p->lo <= 0 && p->Mu[2] == p->M[2] &&
         p->zshift == 0 && p->PZ <= 16 && encode_fn() != nullptr;
}

// Tensor map over the padded fields: dims {E0, E1, E2, 3}, box {18, 16, PZ, 1},
// no swizzle (the 144-byte rows are bank-conflict free for the lane map).
cudaError_t make_field_tmap(esp_plan* p) {
  const FieldPad& f = p->fpad;
  const bool dp = p->precision == ESP_FP64;
  const cuuint64_t es = dp ? 8 : 4;
  cuuint64_t dims[4] = {(cuuint64_t)f.E[0], (cuuint64_t)f.E[1], (cuuint64_t)f.E[2], 3};
  cuuint64_t strides[3] = {(cuuint64_t)f.E[0] * es, (cuuint64_t)f.E[0] * f.E[1] * es,
                           (cuuint64_t)f.cstride * es};
  cuuint32_t box[4] = {(cuuint32_t)(dp ? TmaGatherLayout<8>::kRow : TmaGather32Layout<8>::kRow),
                       16, (cuuint32_t)p->PZ, 1};
  cuuint32_t elem[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(p->tmap),
                           dp ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           4, p->d_fpad, dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int P, int NW>
static cudaError_t tma_p(esp_plan* p, double* d_forces, cudaStream_t s, int id_lo, int id_hi) {
  Geom g = make_geom(p);
  const size_t smem = TmaGatherLayout<NW>::bytes(p->PZ);
  cudaError_t e = cudaFuncSetAttribute(k_gather_tma<P, NW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long ntiles = p->n_tiles;
  const unsigned grid = (unsigned)std::min<long long>(sms, ntiles);
  k_gather_tma<P, NW><<<grid, 32 * (NW + 1), smem, s>>>(
      *reinterpret_cast<const CUtensorMap*>(p->tmap), g, *p->h_fast, p->d_tab, p->d_breaks,
      p->n_pieces, p->ncoef, p->d_offsets, p->d_u, p->cap, p->d_q, p->d_idx, d_forces,
      p->fpad.S[0] + p->lo, reinterpret_cast<const double*>(p->d_wrec), p->d_pk, id_lo, id_hi);
  p->launches++;
  prof_mark(p, s, "gather");
  return cudaGetLastError();
}

template <int P, int NW>
static cudaError_t tma32_p(esp_plan* p, double* d_forces, cudaStream_t s, int id_lo,
                           int id_hi) {
  Geom g = make_geom(p);
  const size_t smem = TmaGather32Layout<NW>::bytes(p->PZ);
  cudaError_t e = cudaFuncSetAttribute(k_gather_tma32<P, NW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<long long>(sms, p->n_tiles);
  k_gather_tma32<P, NW><<<grid, 32 * (NW + 1), smem, s>>>(
      *reinterpret_cast<const CUtensorMap*>(p->tmap), g, *p->h_fast, p->d_tabf, p->d_breaks,
      p->n_pieces, p->ncoef, p->d_offsets, p->d_u, p->cap, p->d_q, p->d_idx, d_forces,
      p->fpad.S[0] + p->lo, reinterpret_cast<const float*>(p->d_wrec), p->d_pk, id_lo, id_hi);
  p->launches++;
  prof_mark(p, s, "gather");
  return cudaGetLastError();
}

template <int P, int NW>
static cudaError_t grad_tma_p(esp_plan* p, double* d_forces, cudaStream_t s) {
  Geom g = make_geom(p);
  const size_t smem = TmaGradLayout<NW>::bytes(p->PZ);
  cudaError_t e = cudaFuncSetAttribute(k_gather_grad_tma<P, NW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<long long>(sms, p->n_tiles);
  k_gather_grad_tma<P, NW><<<grid, 32 * (NW + 1), smem, s>>>(
      *reinterpret_cast<const CUtensorMap*>(p->tmap), g, p->d_offsets,
      reinterpret_cast<const double*>(p->d_wrec), reinterpret_cast<const double*>(p->d_drec),
      p->d_pk, p->d_q, p->d_idx, plan_jacobian(p), d_forces, p->fpad.S[0] + p->lo);
  p->launches++;
  prof_mark(p, s, "gather_grad");
  return cudaGetLastError();
}

cudaError_t launch_gather_grad_tma(esp_plan* p, double* d_forces, cudaStream_t s) {
  constexpr int NW = 12;
  if (p->precision != ESP_FP64 || !p->drec_ready || !p->records_ready)
    return cudaErrorInvalidValue;
  switch (p->P) {
    case 2: return grad_tma_p<2, NW>(p, d_forces, s);
    case 3: return grad_tma_p<3, NW>(p, d_forces, s);
    case 4: return grad_tma_p<4, NW>(p, d_forces, s);
    case 5: return grad_tma_p<5, NW>(p, d_forces, s);
    case 6: return grad_tma_p<6, NW>(p, d_forces, s);
    case 7: return grad_tma_p<7, NW>(p, d_forces, s);
    case 8: return grad_tma_p<8, NW>(p, d_forces, s);
    default: return cudaErrorInvalidValue;
  }
}

#ifndef ESP_TMA32_NW
#define ESP_TMA32_NW 12   // fp32 consumer warps (8: 3.62 ms, 12: 3.03, 16: 3.15, 20: 3.29)
#endif
#ifndef ESP_TMA_NW
#define ESP_TMA_NW 12   // consumer warps (A/B at config 4: 8 -> 4.77 ms, 12 -> 4.39, 16 -> 4.46)
#endif
cudaError_t launch_gather_tma(esp_plan* p, double* d_forces, cudaStream_t s, int id_lo,
                              int id_hi) {
  constexpr int NW = ESP_TMA_NW;
  if (p->precision != ESP_FP64) {
    constexpr int NW32 = ESP_TMA32_NW;
    switch (p->P) {
      case 2: return tma32_p<2, NW32>(p, d_forces, s, id_lo, id_hi);
      case 3: return tma32_p<3, NW32>(p, d_forces, s, id_lo, id_hi);
      case 4: return tma32_p<4, NW32>(p, d_forces, s, id_lo, id_hi);
      case 5: return tma32_p<5, NW32>(p, d_forces, s, id_lo, id_hi);
      case 6: return tma32_p<6, NW32>(p, d_forces, s, id_lo, id_hi);
      case 7: return tma32_p<7, NW32>(p, d_forces, s, id_lo, id_hi);
      case 8: return tma32_p<8, NW32>(p, d_forces, s, id_lo, id_hi);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (p->P) {
    case 2: return tma_p<2, NW>(p, d_forces, s, id_lo, id_hi);
    case 3: return tma_p<3, NW>(p, d_forces, s, id_lo, id_hi);
    case 4: return tma_p<4, NW>(p, d_forces, s, id_lo, id_hi);
    case 5: return tma_p<5, NW>(p, d_forces, s, id_lo, id_hi);
    case 6: return tma_p<6, NW>(p, d_forces, s, id_lo, id_hi);
    case 7: return tma_p<7, NW>(p, d_forces, s, id_lo, id_hi);
    case 8: return tma_p<8, NW>(p, d_forces, s, id_lo, id_hi);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace esp
