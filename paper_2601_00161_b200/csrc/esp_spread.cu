// esp_spread.cu — PSWF charge spreading (mesh.py:204-210) as a tile kernel
// plus a deterministic halo combine.
//
// Design (DESIGN.md §"spread"):
//  * CTA = one anchor tile of TX x TY columns x TZ planes (TX = TY = 17 - P),
//    whose stencils cover a padded block of 16 x 16 columns x PZ = TZ+P-1
//    planes.  Its particles are a contiguous, z-anchor-sorted range of the
//    binned arrays (esp_bin.cu).
//  * Each of the 256 threads owns one padded (x, y) column and keeps a
//    P-deep sliding window of z accumulators in registers.  Particles are
//    visited in z-anchor order; when the anchor advances the window slides
//    and the finished plane is stored (plain store, exclusive owner).  Every
//    multiply-add in the window is useful along z; along x/y a warp (8 x 4
//    columns) only visits the particles whose stencil touches it, found by a
//    ballot over a per-particle 8-bit warp mask staged with the weights.
//  * 1D weights are evaluated once per particle and dimension (unrolled
//    Horner on the reference's degree-18 piecewise table, pswf.py:238-293,
//    coefficients in the constant bank) and staged in shared memory; q is
//    folded into the x weights.
//  * The padded blocks go to a scratch buffer; k_combine sums, for every grid
//    point, the contributions of the (at most 8) covering tiles in a fixed
//    order read from precomputed per-axis tables.  No atomics: results are
//    bitwise reproducible.
#include "esp_internal.cuh"

namespace esp {

template <typename real, int P>
struct SpreadLayout {
  static constexpr int kWRow = P;  // weights per (particle, dim)
  static size_t bytes(int n_pieces, int ncoef) {
    size_t b = sizeof(real) * (size_t)n_pieces * ncoef;
    b = (b + 15) & ~size_t(15);
    b += sizeof(double) * (size_t)(n_pieces + 1);
    b = (b + 15) & ~size_t(15);
    b += sizeof(real) * 3 * (size_t)kChunk * P;
    b += sizeof(int) * 4 * (size_t)kChunk;
    return b;
  }
};

// Stage anchors, weights and warp-overlap masks of particles [c0, c0+n).
template <typename real, int P>
__device__ __forceinline__ void stage_spread(const Geom& g, const FastTab& ft,
                                             const real* s_tab, const double* s_brk,
                                             int n_pieces, int ncoef,
                                             const double* __restrict__ U,
                                             const double* __restrict__ Q, long long cap,
                                             long long c0, int n, int tx, int ty, int tz,
                                             real* s_w, int* s_anc) {
  for (int item = threadIdx.x; item < 3 * n; item += blockDim.x) {
    const int d = item / n, pl = item - d * n;   // d-major: coalesced U reads
    const double u = U[d * cap + c0 + pl];
    const double base = anchor_base(g, u);
    const int a = wrap_index((long long)base, g.M[d]);
    const int org = d == 0 ? tx * g.TX : (d == 1 ? ty * g.TY : tz * g.TZ);
    s_anc[d * kChunk + pl] = a - org;
    const real qf = d == 0 ? (real)Q[c0 + pl] : real(1);
    real w[P];
    stencil_weights<real, P>(ft, s_tab, s_brk, n_pieces, ncoef, u, base, g.lo, qf, w);
    real* dst = s_w + ((size_t)d * kChunk + pl) * P;
#pragma unroll
    for (int s = 0; s < P; ++s) dst[s] = w[s];
  }
}

template <typename real, int P>
__global__ void __launch_bounds__(kTileThreads)
k_spread_tiles(Geom g, FastTab ft, const real* __restrict__ tab,
               const double* __restrict__ brk, int n_pieces, int ncoef,
               const int* __restrict__ offsets, const double* __restrict__ U,
               const double* __restrict__ Q, long long cap, real* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tile = blockIdx.x;
  const int tz = tile % g.ntz;
  const int txy = tile / g.ntz;
  const int tx = txy % g.ntx, ty = txy / g.ntx;
  const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
  const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
  const long long p0 = offsets[key0], p1 = offsets[key1];
  if (p0 == p1) return;  // empty tile: k_combine skips it

  real* s_tab = reinterpret_cast<real*>(smem_raw);
  size_t off = sizeof(real) * (size_t)n_pieces * ncoef;
  off = (off + 15) & ~size_t(15);
  double* s_brk = reinterpret_cast<double*>(smem_raw + off);
  off += sizeof(double) * (size_t)(n_pieces + 1);
  off = (off + 15) & ~size_t(15);
  real* s_w = reinterpret_cast<real*>(smem_raw + off);
  off += sizeof(real) * 3 * (size_t)kChunk * P;
  int* s_anc = reinterpret_cast<int*>(smem_raw + off);   // [3][kChunk] + mask[kChunk]
  int* s_mask = s_anc + 3 * kChunk;

  // General table (the fast path falls back to it on exact piece-boundary ties).
  for (int i = threadIdx.x; i < n_pieces * ncoef; i += blockDim.x) s_tab[i] = tab[i];
  for (int i = threadIdx.x; i <= n_pieces; i += blockDim.x) s_brk[i] = brk[i];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
  const int cx = wx0 + (lane & 7), cy = wy0 + (lane >> 3);
  real* out = scratch + (size_t)tile * g.PZ * kPad * kPad + (size_t)cy * kPad + cx;
  const size_t plane = (size_t)kPad * kPad;

  real win[P];
#pragma unroll
  for (int s = 0; s < P; ++s) win[s] = real(0);
  int zc = 0;

  for (long long c0 = p0; c0 < p1; c0 += kChunk) {
    const int n = (int)min((long long)kChunk, p1 - c0);
    __syncthreads();
    stage_spread<real, P>(g, ft, s_tab, s_brk, n_pieces, ncoef, U, Q, cap, c0, n, tx, ty,
                          tz, s_w, s_anc);
    __syncthreads();
    for (int pl = threadIdx.x; pl < n; pl += blockDim.x) {
      const int xl = s_anc[pl], yl = s_anc[kChunk + pl];
      int m = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int ax = (w & 1) * 8, ay = (w >> 1) * 4;
        const bool hit = xl < ax + 8 && xl + P > ax && yl < ay + 4 && yl + P > ay;
        m |= (int)hit << w;
      }
      s_mask[pl] = m;
    }
    __syncthreads();
    for (int base = 0; base < n; base += 32) {
      const int pq = base + lane;
      const bool mine = pq < n && ((s_mask[pq] >> warp) & 1);
      unsigned bits = __ballot_sync(0xffffffffu, mine);
      while (bits) {
        const int pl = base + __ffs(bits) - 1;
        bits &= bits - 1;
        const int xl = s_anc[pl];
        const int yl = s_anc[kChunk + pl];
        const int zl = s_anc[2 * kChunk + pl];
        while (zc < zl) {  // slide: plane zc is final for this column
          out[(size_t)zc * plane] = win[0];
#pragma unroll
          for (int s = 0; s < P - 1; ++s) win[s] = win[s + 1];
          win[P - 1] = real(0);
          ++zc;
        }
        const int sx = cx - xl, sy = cy - yl;
        const bool in = (unsigned)sx < (unsigned)P && (unsigned)sy < (unsigned)P;
        const real* wxp = s_w + (size_t)pl * P;
        const real* wyp = s_w + ((size_t)kChunk + pl) * P;
        const real* wzp = s_w + ((size_t)2 * kChunk + pl) * P;
        const int sxc = min(max(sx, 0), P - 1), syc = min(max(sy, 0), P - 1);
        const real a = in ? wxp[sxc] * wyp[syc] : real(0);
        real wz[P];
#pragma unroll
        for (int s = 0; s < P; ++s) wz[s] = wzp[s];
#pragma unroll
        for (int s = 0; s < P; ++s) win[s] = fma(a, wz[s], win[s]);
      }
    }
  }
  while (zc < g.PZ) {
    out[(size_t)zc * plane] = win[0];
#pragma unroll
    for (int s = 0; s < P - 1; ++s) win[s] = win[s + 1];
    win[P - 1] = real(0);
    ++zc;
  }
}

template <typename real>
__global__ void k_combine(Geom g, CombineTabs ct, const int* __restrict__ offsets,
                          const real* __restrict__ scratch, real* __restrict__ grid) {
  const long long G = (long long)g.M[0] * g.M[1] * g.M[2];
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= G) return;
  const int x = (int)(gid % g.M[0]);
  const int y = (int)((gid / g.M[0]) % g.M[1]);
  const int z = (int)(gid / ((long long)g.M[0] * g.M[1]));
  const int nx = ct.cnt[0][x], ny = ct.cnt[1][y], nz = ct.cnt[2][z];
  double acc = 0.0;
  for (int a = 0; a < nz; ++a) {
    const int ez = ct.ent[2][z * kCombW + a];
    const int tz = ez & 0xffff, pz = ez >> 16;
    for (int b = 0; b < ny; ++b) {
      const int ey = ct.ent[1][y * kCombW + b];
      const int ty = ey & 0xffff, py = ey >> 16;
      for (int c = 0; c < nx; ++c) {
        const int ex = ct.ent[0][x * kCombW + c];
        const int tx = ex & 0xffff, px = ex >> 16;
        const int txy = ty * g.ntx + tx;
        const long long k0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
        const long long k1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
        if (offsets[k0] == offsets[k1]) continue;
        const long long tile = (long long)txy * g.ntz + tz;
        acc += (double)scratch[((tile * g.PZ + pz) * kPad + py) * kPad + px];
      }
    }
  }
  grid[gid] = (real)acc;
}

template <typename real, int P>
static cudaError_t spread_p(esp_plan* p, cudaStream_t s) {
  Geom g = make_geom(p);
  const real* tab = std::is_same<real, double>::value
                        ? reinterpret_cast<const real*>(p->d_tab)
                        : reinterpret_cast<const real*>(p->d_tabf);
  const size_t smem = SpreadLayout<real, P>::bytes(p->n_pieces, p->ncoef);
  static size_t attr_set = 0;  // set once per instantiation (capture-safe)
  if (smem > attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_spread_tiles<real, P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = smem;
  }
  k_spread_tiles<real, P><<<(unsigned)p->n_tiles, kTileThreads, smem, s>>>(
      g, *p->h_fast, tab, p->d_breaks, p->n_pieces, p->ncoef, p->d_offsets, p->d_u, p->d_q,
      p->cap, reinterpret_cast<real*>(p->d_scratch));
  p->launches++;
  prof_mark(p, s, "spread");
  CombineTabs ct;
  for (int d = 0; d < 3; ++d) {
    ct.ent[d] = p->d_comb_ent + kCombW * p->comb_off[d];
    ct.cnt[d] = p->d_comb_cnt + p->comb_off[d];
  }
  const int B = 256;
  k_combine<real><<<(unsigned)((p->G + B - 1) / B), B, 0, s>>>(
      g, ct, p->d_offsets, reinterpret_cast<const real*>(p->d_scratch),
      reinterpret_cast<real*>(p->d_grid));
  p->launches++;
  prof_mark(p, s, "combine");
  return cudaGetLastError();
}

template <typename real>
static cudaError_t spread_r(esp_plan* p, cudaStream_t s) {
  switch (p->P) {
    case 2: return spread_p<real, 2>(p, s);
    case 3: return spread_p<real, 3>(p, s);
    case 4: return spread_p<real, 4>(p, s);
    case 5: return spread_p<real, 5>(p, s);
    case 6: return spread_p<real, 6>(p, s);
    case 7: return spread_p<real, 7>(p, s);
    case 8: return spread_p<real, 8>(p, s);
    case 9: return spread_p<real, 9>(p, s);
    case 10: return spread_p<real, 10>(p, s);
    case 11: return spread_p<real, 11>(p, s);
    case 12: return spread_p<real, 12>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_spread(esp_plan* p, cudaStream_t s) {
  return p->precision == ESP_FP64 ? spread_r<double>(p, s) : spread_r<float>(p, s);
}

// Host-side construction of the combine tables: for each coordinate c along
// an axis, every (tile, padded index) with t*T + lo + pad == c (mod M).
void build_combine_axis(int M, int T, int E, int nt, int lo, std::vector<int>& ent,
                        std::vector<int>& cnt) {
  ent.assign((size_t)M * kCombW, 0);
  cnt.assign(M, 0);
  for (int t = 0; t < nt; ++t) {
    for (int pad = 0; pad < E; ++pad) {
      long long c = (long long)t * T + lo + pad;
      c %= M;
      if (c < 0) c += M;
      int& k = cnt[(size_t)c];
      if (k < kCombW) ent[(size_t)c * kCombW + k] = t | (pad << 16);
      ++k;
    }
  }
}

}  // namespace esp
