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
//    columns) skips particles whose stencil misses it.
//  * 1D weights are evaluated once per particle and dimension (Horner on the
//    reference's degree-18 piecewise table, pswf.py:238-293) and staged in
//    shared memory; q is folded into the x weights.
//  * The padded blocks go to a scratch buffer; k_combine sums, for every grid
//    point, the contributions of the (at most 8) covering tiles in a fixed
//    order.  No atomics: results are bitwise reproducible.
#include "esp_internal.cuh"

namespace esp {

template <typename real>
struct SpreadSmem {
  static size_t bytes(int P, int n_pieces, int ncoef) {
    size_t b = sizeof(real) * (size_t)n_pieces * ncoef;
    b = (b + 15) & ~size_t(15);
    b += sizeof(double) * (size_t)(n_pieces + 1);
    b = (b + 15) & ~size_t(15);
    b += sizeof(real) * 3 * (size_t)kChunk * P;
    b += sizeof(int) * 3 * (size_t)kChunk;
    return b;
  }
};

// Stage weights of particles [c0, c0+n) of this tile into shared memory.
// For the x dimension the charge is folded in (mul_q).
template <typename real, int P>
__device__ __forceinline__ void stage_weights(
    const Geom& g, const real* s_tab, const double* s_brk, int n_pieces, int ncoef,
    const double* __restrict__ U, const double* __restrict__ Q, long long cap,
    long long c0, int n, int tx, int ty, int tz, bool mul_q, real* s_w, int* s_anc) {
  for (int item = threadIdx.x; item < 3 * n; item += blockDim.x) {
    const int pl = item / 3, d = item - 3 * (item / 3);
    const double u = U[d * cap + c0 + pl];
    const double base = anchor_base(g, u);
    const int a = wrap_index((long long)base, g.M[d]);
    const int org = d == 0 ? tx * g.TX : (d == 1 ? ty * g.TY : tz * g.TZ);
    s_anc[d * kChunk + pl] = a - org;
    real qf = real(1);
    if (d == 0 && mul_q) qf = (real)Q[c0 + pl];
    real* w = s_w + ((size_t)d * kChunk + pl) * P;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const double t = u - (base + (double)(g.lo + s));
      w[s] = window_eval<real>(s_tab, s_brk, n_pieces, ncoef, t) * qf;
    }
  }
}

template <typename real, int P>
__global__ void __launch_bounds__(kTileThreads)
k_spread_tiles(Geom g, const real* __restrict__ tab, const double* __restrict__ brk,
               int n_pieces, int ncoef, const int* __restrict__ offsets,
               const double* __restrict__ U, const double* __restrict__ Q,
               long long cap, real* __restrict__ scratch) {
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
  int* s_anc = reinterpret_cast<int*>(smem_raw + off);

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
    stage_weights<real, P>(g, s_tab, s_brk, n_pieces, ncoef, U, Q, cap, c0, n, tx, ty,
                           tz, true, s_w, s_anc);
    __syncthreads();
    for (int pl = 0; pl < n; ++pl) {
      const int xl = s_anc[pl];
      const int yl = s_anc[kChunk + pl];
      if (xl >= wx0 + 8 || xl + P <= wx0 || yl >= wy0 + 4 || yl + P <= wy0) continue;
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
#pragma unroll
      for (int s = 0; s < P; ++s) win[s] = fma(a, wzp[s], win[s]);
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

// Candidate (tile, padded index) pairs covering coordinate c along one axis.
__device__ __forceinline__ int axis_candidates(int c, int M, int T, int E, int nt,
                                               int lo, int* tt, int* pp) {
  int cnt = 0;
  const int hi_edge = (nt - 1) * T + lo + E - 1;
  // k range such that c' = c + kM lies in [lo, hi_edge]
  int kmin = -((c - lo) / M);
  while (c + (kmin - 1) * M >= lo) --kmin;
  while (c + kmin * M < lo) ++kmin;
  for (int k = kmin; c + k * M <= hi_edge; ++k) {
    const int cp = c + k * M;
    // tiles t with t*T + lo <= cp <= t*T + lo + E - 1
    int t_hi = (cp - lo) >= 0 ? (cp - lo) / T : -1;
    int num = cp - lo - E + 1;
    int t_lo = num <= 0 ? 0 : (num + T - 1) / T;
    if (t_hi > nt - 1) t_hi = nt - 1;
    for (int t = t_lo; t <= t_hi; ++t) {
      if (cnt < 8) {
        tt[cnt] = t;
        pp[cnt] = cp - (t * T + lo);
        ++cnt;
      }
    }
  }
  return cnt;
}

template <typename real>
__global__ void k_combine(Geom g, const int* __restrict__ offsets,
                          const real* __restrict__ scratch, real* __restrict__ grid) {
  const long long G = (long long)g.M[0] * g.M[1] * g.M[2];
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= G) return;
  const int x = (int)(gid % g.M[0]);
  const int y = (int)((gid / g.M[0]) % g.M[1]);
  const int z = (int)(gid / ((long long)g.M[0] * g.M[1]));
  int xt[8], xp[8], yt[8], yp[8], zt[8], zp[8];
  const int nx = axis_candidates(x, g.M[0], g.TX, kPad, g.ntx, g.lo, xt, xp);
  const int ny = axis_candidates(y, g.M[1], g.TY, kPad, g.nty, g.lo, yt, yp);
  const int nz = axis_candidates(z, g.M[2], g.TZ, g.PZ, g.ntz, g.lo, zt, zp);
  double acc = 0.0;
  for (int a = 0; a < nz; ++a) {
    for (int b = 0; b < ny; ++b) {
      for (int c = 0; c < nx; ++c) {
        const int txy = yt[b] * g.ntx + xt[c];
        const long long k0 = (long long)txy * g.M[2] + (long long)zt[a] * g.TZ;
        const long long k1 = (long long)txy * g.M[2] + min(g.M[2], (zt[a] + 1) * g.TZ);
        if (offsets[k0] == offsets[k1]) continue;
        const long long tile = (long long)txy * g.ntz + zt[a];
        acc += (double)scratch[((tile * g.PZ + zp[a]) * kPad + yp[b]) * kPad + xp[c]];
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
  const size_t smem = SpreadSmem<real>::bytes(P, p->n_pieces, p->ncoef);
  cudaError_t e = cudaFuncSetAttribute(k_spread_tiles<real, P>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_spread_tiles<real, P><<<(unsigned)p->n_tiles, kTileThreads, smem, s>>>(
      g, tab, p->d_breaks, p->n_pieces, p->ncoef, p->d_offsets, p->d_u, p->d_q, p->cap,
      reinterpret_cast<real*>(p->d_scratch));
  p->launches++;
  prof_mark(p, s, "spread");
  const int B = 256;
  k_combine<real><<<(unsigned)((p->G + B - 1) / B), B, 0, s>>>(
      g, p->d_offsets, reinterpret_cast<const real*>(p->d_scratch),
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

}  // namespace esp
