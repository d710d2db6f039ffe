// esp_near.cu — near-field (real-space) pair sum on the B200: cell list,
// fused energy / forces / pressure pass, explicit-pair-list variant.
//
// Reference (prolate_ewald, /root/reference/pkg/src/prolate_ewald):
//   realspace.short_range          realspace.py:115-157
//   realspace.PairTable            realspace.py:29-67  (table evaluation)
//   kernel.near_field / fn_weight  kernel.py:41-97     (exact evaluation)
//   system.build_cell_list         system.py:144-222
//   system.minimum_image           system.py:75-79
//
// Cell-list path (esp_near_evaluate): particles are binned into a periodic
// lattice of cells in fractional coordinates, nc_d = floor(width_d * div /
// reach) cells along axis d (perpendicular width, so a cell is at least
// reach/div thick; div = 2 or 3, chosen per call).  A stable radix sort by
// (cell, octant of the cell) orders them; inside an octant the order is by
// original index.  Each record stores the position moved into the home cell
// image and the charge (32 B).  The tile kernel (k_near_tile) runs one CTA
// per cell and passes of 8 of its particles (one per warp): the candidate
// rows of cells within +-div are trimmed against the pass's bounding box,
// split at the periodic faces into runs with one image shift each (so no
// per-pair minimum-image rounding), and staged in shared memory with the
// shift applied.  Hits (r^2 <= reach^2) are compacted through a per-warp
// queue (ballot + popc) and evaluated 32 at a time with every lane busy.
// Full neighbour lists (each pair seen from both ends) keep every force a
// single-owner sum: no atomics, bitwise reproducible.  Energy and pressure
// take half of each directed pair and go through a fixed-order reduction.
//
// Pair values: the PairTable's low-r polynomial (Horner) and cubic splines
// (from per-knot values and second derivatives, the same pieces as the
// reference's PPoly coefficients), 1/r from a DP rsqrt; exact mode is the
// Legendre series in numpy legval's (Clenshaw) order.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "esp_internal.cuh"

using esp::set_error;

namespace {

#ifndef ESP_NEAR_HERMITE
#define ESP_NEAR_HERMITE 1
#endif
#ifndef ESP_NEAR_THREADS
#define ESP_NEAR_THREADS 256
#endif
#ifndef ESP_NEAR_MINB
#define ESP_NEAR_MINB 1
#endif
constexpr int kNearThreads = ESP_NEAR_THREADS;  // warps per cell CTA x 32
constexpr int kQueue = 64;         // per-warp compaction queue (2 x 32)
constexpr int kPolyMax = 16;
constexpr int kLegMax = 64;

struct NearConst {
  double r_c, rc2_hi, reach2, sing2, r_in, inv_dk, C0, c0rc, dk, h26;
  int use_table, n_poly, n_knots, n_leg, n_cum;
  double smooth_poly[kPolyMax];
  double fn_poly[kPolyMax];
  double leg[kLegMax];
  double cum[kLegMax];
};

struct CellGeom {
  int nc[3];
  long long ncells;
  int ortho, div;
  double eps;      // rounding margin of the row trimming (orthorhombic)
  double h[9];     // row-major, columns = cell vectors
  double hinv[9];  // row-major
  int n_rows;      // (2 div + 1)^2 candidate rows per particle
};


}  // namespace

struct esp_near {
  NearConst c{};
  double reach = 0.0;
  double volume = 1.0;
  double width[3] = {0, 0, 0};   // perpendicular widths of the bound cell
  long long cap = 0;
  int div = 2;
  int kernel = 0;             // 0: staged tile kernel, 1: per-particle rows (ESP_NEAR_KERNEL=rows)
  int octants = 1;            // cell-octant sub-order for the tile kernel (ESP_NEAR_OCT=0 off)
  int have_cell = 0;
  CellGeom g{};
  // tables
  double* d_tab = nullptr;    // [n_knots-1][10]: knot, -, smooth c0..c3, fn c0..c3
  // per-step buffers
  int* d_key = nullptr;
  int* d_key_sorted = nullptr;
  int* d_idx = nullptr;
  int* d_perm = nullptr;
  double4* d_rec_u = nullptr;   // unsorted home-image records
  double4* d_rec = nullptr;     // sorted by cell
  int* d_cell_start = nullptr;  // ncells + 1
  long long cell_cap = 0;
  double* d_part = nullptr;     // [cap][8] per-particle E, 6 virial, pair count
  double* d_red = nullptr;      // block partials
  unsigned* d_ticket = nullptr;
  void* d_sort_tmp = nullptr;
  size_t sort_bytes = 0;
  // pair-list path
  long long pair_cap = 0;
  int* d_pkey = nullptr;
  int* d_pkey_sorted = nullptr;
  long long* d_pent = nullptr;
  long long* d_pent_sorted = nullptr;
  void* d_psort_tmp = nullptr;
  size_t psort_bytes = 0;
  // enumerated pair list (esp_near_build_pairs)
  long long list_cap = 0;
  long long list_n = 0;
  unsigned long long* d_list_keys = nullptr;
  unsigned long long* d_list_keys2 = nullptr;
  long long* d_list_i = nullptr;
  long long* d_list_j = nullptr;
  void* d_list_tmp = nullptr;
  size_t list_tmp_bytes = 0;
  int launches = 0;
};

namespace {

int bits_for(long long n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

// Horner with FMA (numpy polyval order of coefficients, ascending powers).
__device__ __forceinline__ double poly_horner(double x, const double* c, int n) {
  double c0 = c[n - 1];
  for (int i = 2; i <= n; ++i) c0 = fma(c0, x, c[n - i]);
  return c0;
}

// numpy.polynomial.legendre.legval (Clenshaw, the reference's operation order).
__device__ __forceinline__ double legval_np(double x, const double* c, int n) {
  if (n == 1) return c[0];
  double c0 = c[n - 2], c1 = c[n - 1];
  if (n > 2) {
    int nd = n;
    for (int i = 3; i <= n; ++i) {
      const double tmp = c0;
      nd = nd - 1;
      c0 = __dsub_rn(c[n - i], __ddiv_rn(__dmul_rn(c1, (double)(nd - 1)), (double)nd));
      c1 = __dadd_rn(tmp, __ddiv_rn(__dmul_rn(__dmul_rn(c1, x), (double)(2 * nd - 1)),
                                    (double)nd));
    }
  }
  return __dadd_rn(c0, __dmul_rn(c1, x));
}

// Hermite-form table piece: u = (r - r_in)/dk, knot k, and the cubic from the
// knot records s0, f0 (knot k) and s1, f1 (knot k + 1).
__device__ __forceinline__ double hermite_u(const NearConst& C, double r) {
  return (r - C.r_in) * C.inv_dk;
}
__device__ __forceinline__ int hermite_knot(const NearConst& C, double u) {
  return min(max((int)u, 0), C.n_knots - 2);
}
__device__ __forceinline__ void hermite_eval(const NearConst& C, double u, int k, double rinv,
                                             double2 s0, double2 f0, double2 s1, double2 f1,
                                             double& nv, double& fv) {
  const double B = u - k, A = 1.0 - B;
  const double ca = (A * A - 1.0) * A * C.h26, cb = (B * B - 1.0) * B * C.h26;
  nv = rinv - fma(ca, s0.y, fma(cb, s1.y, fma(A, s0.x, B * s1.x)));
  fv = fma(ca, f0.y, fma(cb, f1.y, fma(A, f0.x, B * f1.x)));
}

// Near-field value N(r) and force weight F_N(r) for 0 < r <= r_c
// (realspace.py:42-67 with a table, kernel.py:41-97 without); rinv = 1/r.
// Default table (ESP_NEAR_HERMITE): per knot the value and second derivative
// of the far-field and force-weight splines (32 B; a pair reads two adjacent
// knots), which fix the same cubic pieces as the reference's PPoly
// coefficients (values agree to rounding) in 40% of the bytes.  Otherwise
// 80 B records {knot, -}, {s0, s1}, {s2, s3}, {f0, f1}, {f2, f3} with the
// scipy PPoly coefficients (highest power first).
__device__ __forceinline__ void pair_values(const NearConst& C, double r, double rinv,
                                            const double* __restrict__ tab, double& nv,
                                            double& fv) {
  if (C.use_table) {
    if (r <= C.r_in) {
      nv = rinv - poly_horner(r, C.smooth_poly, C.n_poly);
      fv = poly_horner(r, C.fn_poly, C.n_poly);
    } else if (ESP_NEAR_HERMITE) {
      // the same cubic pieces from knot values and second derivatives
      // (32 B per knot: y_s, M_s, y_f, M_f)
      const double u = hermite_u(C, r);
      const int k = hermite_knot(C, u);
      const double2* t = reinterpret_cast<const double2*>(tab + 4 * (size_t)k);
      hermite_eval(C, u, k, rinv, __ldg(t), __ldg(t + 1), __ldg(t + 2), __ldg(t + 3), nv, fv);
    } else {
      int k = (int)((r - C.r_in) * C.inv_dk);
      k = min(max(k, 0), C.n_knots - 2);
      const double2* t = reinterpret_cast<const double2*>(tab + 10 * (size_t)k);
      const double2 kn = __ldg(t), a = __ldg(t + 1), b = __ldg(t + 2), c = __ldg(t + 3),
                    d = __ldg(t + 4);
      const double s = r - kn.x;
      nv = rinv - fma(fma(fma(a.x, s, a.y), s, b.x), s, b.y);
      fv = fma(fma(fma(c.x, s, c.y), s, d.x), s, d.y);
    }
    if (r >= C.r_c) nv = 0.0;
  } else {
    const double x = fmin(__ddiv_rn(r, C.r_c), 1.0);
    double phi = __ddiv_rn(legval_np(x, C.cum, C.n_cum), C.C0);
    if (r >= C.r_c) phi = 1.0;
    nv = r < C.r_c ? __ddiv_rn(__dsub_rn(1.0, phi), r) : 0.0;
    const double psi = legval_np(x, C.leg, C.n_leg);
    fv = __dadd_rn(__dsub_rn(1.0, phi), __dmul_rn(__ddiv_rn(r, C.c0rc), psi));
  }
}

// Accumulators of one directed pair set: e, f[3], virial xx xy xz yy yz zz, count.
struct Acc {
  double e, fx, fy, fz, vxx, vxy, vxz, vyy, vyz, vzz, n;
  __device__ void zero() { e = fx = fy = fz = vxx = vxy = vxz = vyy = vyz = vzz = n = 0.0; }
};

__device__ __forceinline__ void pair_add(Acc& a, double qq, double nv, double fv, double rinv,
                                         double dx, double dy, double dz) {
  const double fmag = qq * fv * (rinv * rinv * rinv);
  a.e = fma(qq, nv, a.e);
  const double gx = fmag * dx, gy = fmag * dy, gz = fmag * dz;
  a.fx += gx;
  a.fy += gy;
  a.fz += gz;
  a.vxx = fma(gx, dx, a.vxx);
  a.vxy = fma(gx, dy, a.vxy);
  a.vxz = fma(gx, dz, a.vxz);
  a.vyy = fma(gy, dy, a.vyy);
  a.vyz = fma(gy, dz, a.vyz);
  a.vzz = fma(gz, dz, a.vzz);
  a.n += 1.0;
}

// One directed pair (i <- j) with separation d = x_i - x_j (image applied);
// pairs with r > r_c (or r = 0) contribute nothing (realspace.py:141).
__device__ __forceinline__ void pair_accumulate(const NearConst& C, Acc& a, double qi,
                                                double qj, double dx, double dy, double dz,
                                                const double* __restrict__ tab) {
  const double r2 = dx * dx + dy * dy + dz * dz;
  if (!(r2 <= C.rc2_hi) || r2 == 0.0) return;
  const double rinv = rsqrt(r2);
  const double r = r2 * rinv;
  if (!(r <= C.r_c)) return;
  double nv, fv;
  pair_values(C, r, rinv, tab, nv, fv);
  pair_add(a, qi * qj, nv, fv, rinv, dx, dy, dz);
}

// Two directed pairs per lane (queue slots lane and lane + 32), accumulated
// in that order -- the same sums, in the same order, as two single drains.
// When both pairs take the Hermite table pieces (the common case), their
// table loads are issued together so their L2 latencies overlap.
__device__ __forceinline__ void pair_accumulate2(const NearConst& C, Acc& a, double qi,
                                                 bool ua, double qa, double xa, double ya,
                                                 double za, bool ub, double qb, double xb,
                                                 double yb, double zb,
                                                 const double* __restrict__ tab) {
  const double r2a = xa * xa + ya * ya + za * za;
  const double r2b = xb * xb + yb * yb + zb * zb;
  ua = ua && r2a <= C.rc2_hi && r2a != 0.0;
  ub = ub && r2b <= C.rc2_hi && r2b != 0.0;
  const double ria = rsqrt(ua ? r2a : 1.0), rib = rsqrt(ub ? r2b : 1.0);
  const double ra = r2a * ria, rb = r2b * rib;
  ua = ua && ra <= C.r_c;
  ub = ub && rb <= C.r_c;
  if (!(ESP_NEAR_HERMITE && C.use_table && (!ua || ra > C.r_in) && (!ub || rb > C.r_in))) {
    if (ua) pair_accumulate(C, a, qi, qa, xa, ya, za, tab);
    if (ub) pair_accumulate(C, a, qi, qb, xb, yb, zb, tab);
    return;
  }
  const double uA = hermite_u(C, ra), uB = hermite_u(C, rb);
  const int kA = ua ? hermite_knot(C, uA) : 0, kB = ub ? hermite_knot(C, uB) : 0;
  const double2* tA = reinterpret_cast<const double2*>(tab + 4 * (size_t)kA);
  const double2* tB = reinterpret_cast<const double2*>(tab + 4 * (size_t)kB);
  const double2 sA0 = __ldg(tA), fA0 = __ldg(tA + 1), sA1 = __ldg(tA + 2), fA1 = __ldg(tA + 3);
  const double2 sB0 = __ldg(tB), fB0 = __ldg(tB + 1), sB1 = __ldg(tB + 2), fB1 = __ldg(tB + 3);
  if (ua) {
    double nv, fv;
    hermite_eval(C, uA, kA, ria, sA0, fA0, sA1, fA1, nv, fv);
    if (ra >= C.r_c) nv = 0.0;
    pair_add(a, qi * qa, nv, fv, ria, xa, ya, za);
  }
  if (ub) {
    double nv, fv;
    hermite_eval(C, uB, kB, rib, sB0, fB0, sB1, fB1, nv, fv);
    if (rb >= C.r_c) nv = 0.0;
    pair_add(a, qi * qb, nv, fv, rib, xb, yb, zb);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fractional coordinate s_d = (h^-1 x)_d (system.py:60-61), fixed order.
__device__ __forceinline__ double frac_coord(const CellGeom& g, int d, double x, double y,
                                             double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(g.hinv[3 * d], x), __dmul_rn(g.hinv[3 * d + 1], y)),
                   __dmul_rn(g.hinv[3 * d + 2], z));
}

// Cell of each particle and its record moved into the home image (positions
// already inside the cell, as ParticleSystem wraps them, are unchanged).
// sub = 1: the key also carries the particle's octant within its cell
// (key = cell * 8 + octant), so the tile kernel's passes of consecutive
// particles are spatially compact (tighter pass bounding boxes, fewer
// candidates); the order stays deterministic (stable sort by index).
__global__ void k_near_cells(const double* __restrict__ pos, const double* __restrict__ q,
                             long long n, CellGeom g, int* __restrict__ key,
                             int* __restrict__ idx, double4* __restrict__ rec, int sub) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
  int c[3], oct = 0;
  double img[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double s = frac_coord(g, d, x, y, z);
    double fl = floor(s);
    if (!(fabs(fl) < 1e15)) fl = 0.0;  // non-finite / huge: cell 0, no shift
    img[d] = fl;
    const double t = (s - fl) * g.nc[d];
    int cd = (int)fmin(fmax(t, 0.0), (double)(g.nc[d] - 1));
    c[d] = cd;
    oct |= (t - cd >= 0.5 ? 1 : 0) << d;
  }
  double hx = x, hy = y, hz = z;
  if (img[0] != 0.0 || img[1] != 0.0 || img[2] != 0.0) {
    hx = x - (g.h[0] * img[0] + g.h[1] * img[1] + g.h[2] * img[2]);
    hy = y - (g.h[3] * img[0] + g.h[4] * img[1] + g.h[5] * img[2]);
    hz = z - (g.h[6] * img[0] + g.h[7] * img[1] + g.h[8] * img[2]);
  }
  const int cell = (c[2] * g.nc[1] + c[1]) * g.nc[0] + c[0];
  key[i] = sub ? cell * 8 + oct : cell;
  idx[i] = (int)i;
  rec[i] = make_double4(hx, hy, hz, q ? q[i] : 0.0);
}

// Sorted records and cell start offsets (lower bound of each cell id).
__global__ void k_near_sorted(const int* __restrict__ key_sorted, const int* __restrict__ perm,
                              const double4* __restrict__ rec_u, long long n,
                              long long ncells, double4* __restrict__ rec,
                              int* __restrict__ cell_start, int sub) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  rec[k] = rec_u[perm[k]];
  const int sh = sub ? 3 : 0;   // octant bits below the cell id
  const int c = key_sorted[k] >> sh;
  const int cp = k > 0 ? (key_sorted[k - 1] >> sh) : -1;
  for (int cc = cp + 1; cc <= c; ++cc) cell_start[cc] = (int)k;
  if (k == n - 1)
    for (long long cc = c + 1; cc <= ncells; ++cc) cell_start[cc] = (int)n;
}

__global__ void k_fill_int(int* p, long long n, int v) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < n) p[k] = v;
}

// Warp-wide evaluation of up to 64 queued pairs: lane l takes slots l and
// l + 32 (in that order, as two 32-pair drains would).
__device__ __forceinline__ void drain2(const NearConst& C, Acc& a, double qi, const double* qx,
                                       const double* qy, const double* qz, const double* qqj,
                                       int lane, int cnt, const double* __restrict__ tab) {
  const int l2 = lane + 32;
  const bool ua = lane < cnt, ub = l2 < cnt;
  if (!ua) return;
  pair_accumulate2(C, a, qi, true, qqj[lane], qx[lane], qy[lane], qz[lane], ub,
                   ub ? qqj[l2] : 0.0, ub ? qx[l2] : 0.0, ub ? qy[l2] : 0.0,
                   ub ? qz[l2] : 0.0, tab);
}

// Warp-wide evaluation of the queued pairs; lanes >= cnt idle.
__device__ __forceinline__ void drain(const NearConst& C, Acc& a, double qi, const double* qx,
                                      const double* qy, const double* qz, const double* qqj,
                                      int lane, int cnt, const double* __restrict__ tab) {
  if (lane < cnt) pair_accumulate(C, a, qi, qqj[lane], qx[lane], qy[lane], qz[lane], tab);
}

// One CTA per cell; each warp takes one particle i of the cell at a time.
// Candidates come in rows of cells along x: for each (dy, dz) cell offset
// within +-div the row is trimmed (orthorhombic cells) to the x cells that
// intersect the sphere of radius reach around x_i, and split at the periodic
// face into at most three contiguous runs of the cell-sorted records, each
// with one image shift.  Hits are compacted through the warp's queue.
__global__ void __launch_bounds__(kNearThreads, ESP_NEAR_MINB)
    k_near_pairs(const __grid_constant__ NearConst C, const double4* __restrict__ rec,
                 const int* __restrict__ cell_start, const int* __restrict__ perm, CellGeom g,
                 const double* __restrict__ tab, int accumulate, double* __restrict__ forces,
                 double* __restrict__ part, unsigned long long* __restrict__ singular,
                 int n_owned) {
  __shared__ double s_q[kNearThreads / 32][4][kQueue];
  const int cell = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = cell_start[cell], i1 = cell_start[cell + 1];
  if (i0 == i1) return;
  const int nc0 = g.nc[0], nc1 = g.nc[1], nc2 = g.nc[2];
  const int cx = cell % nc0;
  const int cy = (cell / nc0) % nc1;
  const int cz = cell / (nc0 * nc1);
  const int div = g.div;
  double* qx = s_q[warp][0];
  double* qy = s_q[warp][1];
  double* qz = s_q[warp][2];
  double* qj = s_q[warp][3];
  const unsigned lt = (1u << lane) - 1u;
  const double wy = g.h[4] / nc1, wz = g.h[8] / nc2;
  const double iwx = nc0 / g.h[0];
  const double reach2 = C.reach2;
  for (int i = i0 + warp; i < i1; i += kNearThreads / 32) {
    if (perm[i] >= n_owned) {  // ghost (slab halo): partner only
      if (lane == 0)
        for (int c = 0; c < 8; ++c) part[8 * (size_t)i + c] = 0.0;
      continue;
    }
    const double4 ri = rec[i];
    Acc a;
    a.zero();
    int qn = 0;
    for (int oz = -div; oz <= div; ++oz) {
      int nz = cz + oz, sz = 0;
      if (nz < 0) { nz += nc2; sz = -1; } else if (nz >= nc2) { nz -= nc2; sz = 1; }
      double gz2 = 0.0;
      if (g.ortho) {
        const double lo = (cz + oz) * wz;
        const double gap = fmax(0.0, fmax(lo - ri.z, ri.z - (lo + wz)) - g.eps);
        gz2 = gap * gap;
        if (gz2 > reach2) continue;
      }
      for (int oy = -div; oy <= div; ++oy) {
        int ny = cy + oy, sy = 0;
        if (ny < 0) { ny += nc1; sy = -1; } else if (ny >= nc1) { ny -= nc1; sy = 1; }
        int xlo = cx - div, xhi = cx + div;
        if (g.ortho) {
          const double lo = (cy + oy) * wy;
          const double gap = fmax(0.0, fmax(lo - ri.y, ri.y - (lo + wy)) - g.eps);
          const double rest = reach2 - gz2 - gap * gap;
          if (rest < 0.0) continue;
          const double chord = sqrt(rest) + g.eps;
          xlo = max(xlo, (int)floor((ri.x - chord) * iwx));
          xhi = min(xhi, (int)floor((ri.x + chord) * iwx));
        }
        const int row = (nz * nc1 + ny) * nc0;
        // x_i minus the (y, z) part of the image shift h (sx, sy, sz)
        const double bx = ri.x - (g.h[1] * sy + g.h[2] * sz);
        const double by = ri.y - (g.h[4] * sy + g.h[5] * sz);
        const double bz = ri.z - (g.h[7] * sy + g.h[8] * sz);
        for (int sx = -1; sx <= 1; ++sx) {
          const int ra = sx < 0 ? xlo : (sx == 0 ? max(xlo, 0) : max(xlo, nc0));
          const int rb = sx < 0 ? min(xhi, -1) : (sx == 0 ? min(xhi, nc0 - 1) : xhi);
          if (ra > rb) continue;
          const int j0 = cell_start[row + ra - sx * nc0];
          const int j1 = cell_start[row + rb - sx * nc0 + 1];
          const int self = (sx | sy | sz) == 0 ? i : -1;
          const double xs = bx - g.h[0] * sx, ys = by - g.h[3] * sx, zs = bz - g.h[6] * sx;
          // software pipeline: the next batch's record is in flight while
          // this one is tested
          double2 nxy = make_double2(0.0, 0.0), nzq = nxy;
          if (j0 + lane < j1) {
            const double2* rp = reinterpret_cast<const double2*>(rec + j0 + lane);
            nxy = __ldg(rp);
            nzq = __ldg(rp + 1);
          }
          for (int jb = j0; jb < j1; jb += 32) {
            const int j = jb + lane;
            const double2 xy = nxy, zq = nzq;
            if (j + 32 < j1) {
              const double2* rp = reinterpret_cast<const double2*>(rec + j + 32);
              nxy = __ldg(rp);
              nzq = __ldg(rp + 1);
            }
            const double dx = xs - xy.x, dy = ys - xy.y, dz = zs - zq.x;
            const double r2 = dx * dx + dy * dy + dz * dz;
            const bool hit = j < j1 && r2 <= reach2 && j != self;
            if (hit && r2 < C.sing2) {
              const unsigned long long a_ = (unsigned)perm[i], b_ = (unsigned)perm[j];
              atomicMin(singular, (min(a_, b_) << 32) | max(a_, b_));
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (hit) {
              const int slot = qn + __popc(m & lt);
              qx[slot] = dx;
              qy[slot] = dy;
              qz[slot] = dz;
              qj[slot] = zq.y;
            }
            qn += __popc(m);
            if (qn >= 32) {
              __syncwarp();
              drain(C, a, ri.w, qx, qy, qz, qj, lane, 32, tab);
              __syncwarp();
              if (lane < qn - 32) {
                qx[lane] = qx[lane + 32];
                qy[lane] = qy[lane + 32];
                qz[lane] = qz[lane + 32];
                qj[lane] = qj[lane + 32];
              }
              qn -= 32;
              __syncwarp();
            }
          }
        }
      }
    }
    __syncwarp();
    drain(C, a, ri.w, qx, qy, qz, qj, lane, qn, tab);
    __syncwarp();
    const double fx = warp_sum(a.fx), fy = warp_sum(a.fy), fz = warp_sum(a.fz);
    const double e = warp_sum(a.e), vxx = warp_sum(a.vxx), vxy = warp_sum(a.vxy),
                 vxz = warp_sum(a.vxz), vyy = warp_sum(a.vyy), vyz = warp_sum(a.vyz),
                 vzz = warp_sum(a.vzz), cnt = warp_sum(a.n);
    if (lane == 0) {
      const long long oi = perm[i];
      if (accumulate) {
        forces[3 * oi] += fx;
        forces[3 * oi + 1] += fy;
        forces[3 * oi + 2] += fz;
      } else {
        forces[3 * oi] = fx;
        forces[3 * oi + 1] = fy;
        forces[3 * oi + 2] = fz;
      }
      double* pp = part + 8 * (size_t)i;
      pp[0] = 0.5 * e;
      pp[1] = 0.5 * vxx;
      pp[2] = 0.5 * vxy;
      pp[3] = 0.5 * vxz;
      pp[4] = 0.5 * vyy;
      pp[5] = 0.5 * vyz;
      pp[6] = 0.5 * vzz;
      pp[7] = cnt;
    }
  }
}

// Tile kernel (default).  One CTA per cell, passes of kTileI consecutive
// particles of the cell (one per warp).  Per pass the candidate rows are
// trimmed against the bounding box of the pass's particles (orthorhombic
// cells), split into contiguous runs of cell-sorted records with one image
// shift each, and the runs' records are staged in shared memory in chunks
// of kTileCH (image shift applied, structure of arrays), so every warp tests
// its particle against the same staged records with conflict-free loads.
// Hits go through the warp's compaction queue as in k_near_pairs; the queue
// and the accumulators persist across chunks.
#ifndef ESP_TILE_W
#define ESP_TILE_W 8
#endif
constexpr int kTileW = ESP_TILE_W;    // warps per CTA = particles per pass
constexpr int kTileI = kTileW;
#ifndef ESP_TILE_CH
#define ESP_TILE_CH 1024
#endif
constexpr int kTileCH = ESP_TILE_CH;  // staged records per chunk
#ifndef ESP_NEAR_DRAIN2
#define ESP_NEAR_DRAIN2 1             // drain 64 queued pairs (2 per lane) at a time
#endif
#ifndef ESP_NEAR_TEST2
#define ESP_NEAR_TEST2 2              // candidate batches of 32 tested per step (1 or 2)
#endif
constexpr int kTileDrain = ESP_NEAR_DRAIN2 ? 64 : 32;
constexpr int kTileTest = ESP_NEAR_TEST2;
static_assert(kTileTest >= 1 && 32 * kTileTest <= kTileDrain, "one drain per step must keep the queue below its drain threshold");
constexpr int kTileQueue = kTileDrain + 32 * kTileTest;
constexpr int kTileMaxRuns = 3 * 81;  // 3 runs per row, (2 div + 1)^2 rows, div <= 4

struct TileSmem {
  double jx[kTileCH], jy[kTileCH], jz[kTileCH], jq[kTileCH];
  int jid[kTileCH];                   // j index, bit 31 set for a shifted image
  double q[kTileW][4][kTileQueue];
  double sh[kTileMaxRuns][3];
  int j0[kTileMaxRuns];
  int pref[kTileMaxRuns + 1];
  int flag[kTileMaxRuns];             // 0x80000000 for shifted runs
  double box[6];
  int nruns;
};

__global__ void __launch_bounds__(kTileW * 32)
    k_near_tile(const __grid_constant__ NearConst C, const double4* __restrict__ rec,
                const int* __restrict__ cell_start, const int* __restrict__ perm, CellGeom g,
                const double* __restrict__ tab, int accumulate, double* __restrict__ forces,
                double* __restrict__ part, unsigned long long* __restrict__ singular,
                int n_owned) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(smem_raw);
  const int cell = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = cell_start[cell], i1 = cell_start[cell + 1];
  if (i0 == i1) return;
  const int nc0 = g.nc[0], nc1 = g.nc[1], nc2 = g.nc[2];
  const int cx = cell % nc0;
  const int cy = (cell / nc0) % nc1;
  const int cz = cell / (nc0 * nc1);
  const int div = g.div, side = 2 * div + 1, nrows = side * side;
  const double wy = g.h[4] / nc1, wz = g.h[8] / nc2, iwx = nc0 / g.h[0];
  const double reach2 = C.reach2;
  double* qx = S.q[warp][0];
  double* qy = S.q[warp][1];
  double* qz = S.q[warp][2];
  double* qj = S.q[warp][3];
  const unsigned lt = (1u << lane) - 1u;
  for (int base = i0; base < i1; base += kTileI) {
    const int ni = min(kTileI, i1 - base);
    // bounding box of the pass's particles (home-image coordinates)
    if (tid == 0) {
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (int k = 0; k < ni; ++k) {
        const double4 r = rec[base + k];
        lo[0] = fmin(lo[0], r.x); hi[0] = fmax(hi[0], r.x);
        lo[1] = fmin(lo[1], r.y); hi[1] = fmax(hi[1], r.y);
        lo[2] = fmin(lo[2], r.z); hi[2] = fmax(hi[2], r.z);
      }
      for (int d = 0; d < 3; ++d) {
        S.box[d] = lo[d];
        S.box[3 + d] = hi[d];
      }
    }
    __syncthreads();
    // candidate runs: thread t handles row t (3 run slots each)
    for (int t = tid; t < nrows; t += kTileW * 32) {
      const int oy = t % side - div, oz = t / side - div;
      int ny = cy + oy, sy = 0, nz = cz + oz, sz = 0;
      if (ny < 0) { ny += nc1; sy = -1; } else if (ny >= nc1) { ny -= nc1; sy = 1; }
      if (nz < 0) { nz += nc2; sz = -1; } else if (nz >= nc2) { nz -= nc2; sz = 1; }
      int xlo = cx - div, xhi = cx + div;
      bool keep = true;
      if (g.ortho) {
        const double ylo = (cy + oy) * wy, zlo = (cz + oz) * wz;
        const double gy = fmax(0.0, fmax(ylo - S.box[4], S.box[1] - (ylo + wy)) - g.eps);
        const double gz = fmax(0.0, fmax(zlo - S.box[5], S.box[2] - (zlo + wz)) - g.eps);
        const double rest = reach2 - gy * gy - gz * gz;
        if (rest < 0.0) {
          keep = false;
        } else {
          const double chord = sqrt(rest) + g.eps;
          xlo = max(xlo, (int)floor((S.box[0] - chord) * iwx));
          xhi = min(xhi, (int)floor((S.box[3] + chord) * iwx));
        }
      }
      const int row = (nz * nc1 + ny) * nc0;
      for (int sx = -1; sx <= 1; ++sx) {
        const int slot = 3 * t + sx + 1;
        const int ra = sx < 0 ? xlo : (sx == 0 ? max(xlo, 0) : max(xlo, nc0));
        const int rb = sx < 0 ? min(xhi, -1) : (sx == 0 ? min(xhi, nc0 - 1) : xhi);
        int len = 0, j0 = 0;
        if (keep && ra <= rb) {
          j0 = cell_start[row + ra - sx * nc0];
          len = cell_start[row + rb - sx * nc0 + 1] - j0;
        }
        S.j0[slot] = j0;
        S.pref[slot + 1] = len;  // lengths; prefix below
        S.flag[slot] = (sx | sy | sz) != 0 ? (int)0x80000000 : 0;
        S.sh[slot][0] = g.h[0] * sx + g.h[1] * sy + g.h[2] * sz;
        S.sh[slot][1] = g.h[3] * sx + g.h[4] * sy + g.h[5] * sz;
        S.sh[slot][2] = g.h[6] * sx + g.h[7] * sy + g.h[8] * sz;
      }
    }
    __syncthreads();
    const int nr = 3 * nrows;
    if (warp == 0) {
      // exclusive prefix of the run lengths: lane-contiguous blocks + warp scan
      const int per = (nr + 31) / 32;  // <= 8 (nr <= 243)
      const int a0 = lane * per, a1 = min(nr, a0 + per);
      int lens[8];
      int sum = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        lens[u] = a0 + u < a1 ? S.pref[a0 + u + 1] : 0;
        sum += lens[u];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      __syncwarp();
      int run = incl - sum;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (a0 + u < a1) {
          S.pref[a0 + u] = run;
          run += lens[u];
        }
      }
      if (lane == 31) S.pref[nr] = incl;
    }
    __syncthreads();
    const int total = S.pref[nr];
    const int i = base + warp;
    // particles with input index >= n_owned are ghosts (slab halos): partners
    // only, no sums of their own
    const bool ghost = warp < ni && perm[i] >= n_owned;
    const bool active = warp < ni && !ghost;
    if (ghost && lane == 0)
      for (int c = 0; c < 8; ++c) part[8 * (size_t)i + c] = 0.0;
    double4 ri = make_double4(0, 0, 0, 0);
    if (active) ri = rec[i];
    Acc a;
    a.zero();
    int qn = 0;
    for (int c0 = 0; c0 < total; c0 += kTileCH) {
      const int cnt = min(kTileCH, total - c0);
      // warp-per-run staging: warp w copies the parts of runs w, w + W, ...
      // that overlap this chunk (destination = run prefix - c0)
      for (int r = warp; r < nr; r += kTileW) {
        const int p0 = S.pref[r], p1 = S.pref[r + 1];
        const int a = max(p0, c0), b = min(p1, c0 + cnt);
        if (a >= b) continue;
        const int jb = S.j0[r] - p0;
        const double shx = S.sh[r][0], shy = S.sh[r][1], shz = S.sh[r][2];
        const int fl = S.flag[r];
        for (int c = a + lane; c < b; c += 32) {
          const int j = jb + c;
          const double2* rp = reinterpret_cast<const double2*>(rec + j);
          const double2 xy = __ldg(rp), zq = __ldg(rp + 1);
          const int k = c - c0;
          S.jx[k] = xy.x + shx;
          S.jy[k] = xy.y + shy;
          S.jz[k] = zq.x + shz;
          S.jq[k] = zq.y;
          S.jid[k] = j | fl;
        }
      }
      __syncthreads();
      if (active) {
        // candidates in pairs of 32-wide batches (both batches' loads and
        // tests in flight together), appended to the queue in batch order
        for (int kb = 0; kb < cnt; kb += 32 * kTileTest) {
          unsigned m[kTileTest];
          double dx[kTileTest], dy[kTileTest], dz[kTileTest], qv[kTileTest];
#pragma unroll
          for (int u = 0; u < kTileTest; ++u) {
            const int k = kb + 32 * u + lane;
            bool hit = false;
            dx[u] = dy[u] = dz[u] = qv[u] = 0.0;
            if (k < cnt) {
              dx[u] = ri.x - S.jx[k];
              dy[u] = ri.y - S.jy[k];
              dz[u] = ri.z - S.jz[k];
              qv[u] = S.jq[k];
              const int jid = S.jid[k];
              const double r2 = dx[u] * dx[u] + dy[u] * dy[u] + dz[u] * dz[u];
              hit = r2 <= reach2 && jid != i;
              if (hit && r2 < C.sing2) {
                const unsigned long long a_ = (unsigned)perm[i],
                                         b_ = (unsigned)perm[jid & 0x7fffffff];
                atomicMin(singular, (min(a_, b_) << 32) | max(a_, b_));
              }
            }
            m[u] = __ballot_sync(0xffffffffu, hit);
          }
#pragma unroll
          for (int u = 0; u < kTileTest; ++u) {
            if (m[u] & (1u << lane)) {
              const int slot = qn + __popc(m[u] & lt);
              qx[slot] = dx[u];
              qy[slot] = dy[u];
              qz[slot] = dz[u];
              qj[slot] = qv[u];
            }
            qn += __popc(m[u]);
          }
          if (qn >= kTileDrain) {
            __syncwarp();
            if (kTileDrain == 64)
              drain2(C, a, ri.w, qx, qy, qz, qj, lane, 64, tab);
            else
              drain(C, a, ri.w, qx, qy, qz, qj, lane, 32, tab);
            __syncwarp();
            for (int l = lane; l < qn - kTileDrain; l += 32) {
              qx[l] = qx[l + kTileDrain];
              qy[l] = qy[l + kTileDrain];
              qz[l] = qz[l + kTileDrain];
              qj[l] = qj[l + kTileDrain];
            }
            qn -= kTileDrain;
            __syncwarp();
          }
        }
      }
      __syncthreads();
    }
    if (active) {
      __syncwarp();
      if (kTileDrain == 64)
        drain2(C, a, ri.w, qx, qy, qz, qj, lane, qn, tab);
      else
        drain(C, a, ri.w, qx, qy, qz, qj, lane, qn, tab);
      __syncwarp();
      const double fx = warp_sum(a.fx), fy = warp_sum(a.fy), fz = warp_sum(a.fz);
      const double e = warp_sum(a.e), vxx = warp_sum(a.vxx), vxy = warp_sum(a.vxy),
                   vxz = warp_sum(a.vxz), vyy = warp_sum(a.vyy), vyz = warp_sum(a.vyz),
                   vzz = warp_sum(a.vzz), cn = warp_sum(a.n);
      if (lane == 0) {
        const long long oi = perm[i];
        if (accumulate) {
          forces[3 * oi] += fx;
          forces[3 * oi + 1] += fy;
          forces[3 * oi + 2] += fz;
        } else {
          forces[3 * oi] = fx;
          forces[3 * oi + 1] = fy;
          forces[3 * oi + 2] = fz;
        }
        double* pp = part + 8 * (size_t)i;
        pp[0] = 0.5 * e;
        pp[1] = 0.5 * vxx;
        pp[2] = 0.5 * vxy;
        pp[3] = 0.5 * vxz;
        pp[4] = 0.5 * vyy;
        pp[5] = 0.5 * vyz;
        pp[6] = 0.5 * vzz;
        pp[7] = cn;
      }
    }
    __syncthreads();
  }
}

// Explicit pair list (realspace.short_range with a caller NeighborList):
// directed entries sorted by endpoint; one warp per particle sums its entries
// in list order.  Entry e = 2 * pair + side; side 0 is particle i (+f), side 1
// particle j (-f).  Separation by minimum_image (system.py:75-79).
__global__ void k_pair_keys(const long long* __restrict__ pi, const long long* __restrict__ pj,
                            long long n_pairs, long long n, int* __restrict__ key,
                            long long* __restrict__ ent, unsigned long long* __restrict__ bad) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const long long a = pi[p], b = pj[p];
  if (a < 0 || a >= n || b < 0 || b >= n) {
    atomicMin(bad, (unsigned long long)p);
    key[2 * p] = key[2 * p + 1] = 0;
  } else {
    key[2 * p] = (int)a;
    key[2 * p + 1] = (int)b;
  }
  ent[2 * p] = 2 * p;
  ent[2 * p + 1] = 2 * p + 1;
}

__global__ void k_pair_starts(const int* __restrict__ key_sorted, long long m, long long n,
                              int* __restrict__ start) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int c = key_sorted[k];
  const int cp = k > 0 ? key_sorted[k - 1] : -1;
  for (int cc = cp + 1; cc <= c; ++cc) start[cc] = (int)k;
  if (k == m - 1)
    for (long long cc = c + 1; cc <= n; ++cc) start[cc] = (int)m;
}

__global__ void __launch_bounds__(128)
    k_pair_list(const __grid_constant__ NearConst C, const double* __restrict__ pos, const double* __restrict__ q,
                const long long* __restrict__ pi, const long long* __restrict__ pj,
                const long long* __restrict__ ent, const int* __restrict__ start, long long n,
                CellGeom g, const double* __restrict__ tab, int accumulate, double* __restrict__ forces, double* __restrict__ part,
                unsigned long long* __restrict__ singular) {
  const long long a = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (a >= n) return;
  Acc acc;
  acc.zero();
  const int e0 = start[a], e1 = start[a + 1];
  for (int k = e0 + lane; k < e1; k += 32) {
    const long long e = ent[k];
    const long long p = e >> 1;
    const long long i = pi[p], j = pj[p];
    double dr[3] = {pos[3 * i] - pos[3 * j], pos[3 * i + 1] - pos[3 * j + 1],
                    pos[3 * i + 2] - pos[3 * j + 2]};
    double s[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      s[d] = frac_coord(g, d, dr[0], dr[1], dr[2]);
      s[d] = __dsub_rn(s[d], floor(__dadd_rn(s[d], 0.5)));
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
      dr[d] = __dadd_rn(__dadd_rn(__dmul_rn(s[0], g.h[3 * d]), __dmul_rn(s[1], g.h[3 * d + 1])),
                        __dmul_rn(s[2], g.h[3 * d + 2]));
    const double r2 = dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2];
    if (r2 < C.sing2) atomicMin(singular, ((unsigned long long)i << 32) | (unsigned)j);
    Acc one;
    one.zero();
    pair_accumulate(C, one, q[i], q[j], dr[0], dr[1], dr[2], tab);
    const double sg = (e & 1) ? -1.0 : 1.0;
    acc.e += one.e;
    acc.fx += sg * one.fx;
    acc.fy += sg * one.fy;
    acc.fz += sg * one.fz;
    acc.vxx += one.vxx;
    acc.vxy += one.vxy;
    acc.vxz += one.vxz;
    acc.vyy += one.vyy;
    acc.vyz += one.vyz;
    acc.vzz += one.vzz;
    acc.n += one.n;
  }
  const double fx = warp_sum(acc.fx), fy = warp_sum(acc.fy), fz = warp_sum(acc.fz);
  const double e = warp_sum(acc.e), vxx = warp_sum(acc.vxx), vxy = warp_sum(acc.vxy),
               vxz = warp_sum(acc.vxz), vyy = warp_sum(acc.vyy), vyz = warp_sum(acc.vyz),
               vzz = warp_sum(acc.vzz), cnt = warp_sum(acc.n);
  if (lane == 0) {
    if (accumulate) {
      forces[3 * a] += fx;
      forces[3 * a + 1] += fy;
      forces[3 * a + 2] += fz;
    } else {
      forces[3 * a] = fx;
      forces[3 * a + 1] = fy;
      forces[3 * a + 2] = fz;
    }
    double* pp = part + 8 * (size_t)a;
    pp[0] = 0.5 * e;
    pp[1] = 0.5 * vxx;
    pp[2] = 0.5 * vxy;
    pp[3] = 0.5 * vxz;
    pp[4] = 0.5 * vyy;
    pp[5] = 0.5 * vyz;
    pp[6] = 0.5 * vzz;
    pp[7] = cnt;
  }
}

// Pair enumeration (system.build_cell_list, system.py:144-222): one warp per
// particle i (cell-sorted order) walks the same trimmed candidate rows as
// k_near_pairs and keeps the partners j with original index above i's and
// r^2 <= reach^2.  EMIT = false counts them; EMIT = true writes the keys
// (orig_i << 32 | orig_j) at the particle's offset.  The caller sorts the
// keys, which gives the reference's lexicographic (i, j) order.
template <bool EMIT>
__global__ void __launch_bounds__(128)
    k_pair_enum(const double4* __restrict__ rec, const int* __restrict__ cell_start,
                const int* __restrict__ key_sorted, const int* __restrict__ perm, long long n,
                CellGeom g, double reach2,
                const long long* __restrict__ offset, unsigned long long* __restrict__ out,
                long long* __restrict__ count64) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int nc0 = g.nc[0], nc1 = g.nc[1], nc2 = g.nc[2];
  const int cell = key_sorted[i];
  const int cx = cell % nc0, cy = (cell / nc0) % nc1, cz = cell / (nc0 * nc1);
  const int div = g.div;
  const double wy = g.h[4] / nc1, wz = g.h[8] / nc2, iwx = nc0 / g.h[0];
  const double4 ri = rec[i];
  const unsigned oi = (unsigned)perm[i];
  const unsigned lt = (1u << lane) - 1u;
  long long pos = EMIT ? offset[i] : 0;
  int found = 0;
  for (int oz = -div; oz <= div; ++oz) {
    int nz = cz + oz, sz = 0;
    if (nz < 0) { nz += nc2; sz = -1; } else if (nz >= nc2) { nz -= nc2; sz = 1; }
    double gz2 = 0.0;
    if (g.ortho) {
      const double lo = (cz + oz) * wz;
      const double gap = fmax(0.0, fmax(lo - ri.z, ri.z - (lo + wz)) - g.eps);
      gz2 = gap * gap;
      if (gz2 > reach2) continue;
    }
    for (int oy = -div; oy <= div; ++oy) {
      int ny = cy + oy, sy = 0;
      if (ny < 0) { ny += nc1; sy = -1; } else if (ny >= nc1) { ny -= nc1; sy = 1; }
      int xlo = cx - div, xhi = cx + div;
      if (g.ortho) {
        const double lo = (cy + oy) * wy;
        const double gap = fmax(0.0, fmax(lo - ri.y, ri.y - (lo + wy)) - g.eps);
        const double rest = reach2 - gz2 - gap * gap;
        if (rest < 0.0) continue;
        const double chord = sqrt(rest) + g.eps;
        xlo = max(xlo, (int)floor((ri.x - chord) * iwx));
        xhi = min(xhi, (int)floor((ri.x + chord) * iwx));
      }
      const int row = (nz * nc1 + ny) * nc0;
      const double bx = ri.x - (g.h[1] * sy + g.h[2] * sz);
      const double by = ri.y - (g.h[4] * sy + g.h[5] * sz);
      const double bz = ri.z - (g.h[7] * sy + g.h[8] * sz);
      for (int sx = -1; sx <= 1; ++sx) {
        const int ra = sx < 0 ? xlo : (sx == 0 ? max(xlo, 0) : max(xlo, nc0));
        const int rb = sx < 0 ? min(xhi, -1) : (sx == 0 ? min(xhi, nc0 - 1) : xhi);
        if (ra > rb) continue;
        const int j0 = cell_start[row + ra - sx * nc0];
        const int j1 = cell_start[row + rb - sx * nc0 + 1];
        const double xs = bx - g.h[0] * sx, ys = by - g.h[3] * sx, zs = bz - g.h[6] * sx;
        for (int jb = j0; jb < j1; jb += 32) {
          const int j = jb + lane;
          bool hit = false;
          unsigned oj = 0;
          if (j < j1) {
            const double2* rp = reinterpret_cast<const double2*>(rec + j);
            const double2 xy = __ldg(rp), zq = __ldg(rp + 1);
            const double dx = xs - xy.x, dy = ys - xy.y, dz = zs - zq.x;
            oj = (unsigned)perm[j];
            hit = oj > oi && dx * dx + dy * dy + dz * dz <= reach2;
          }
          const unsigned m = __ballot_sync(0xffffffffu, hit);
          if (EMIT && hit)
            out[pos + __popc(m & lt)] = ((unsigned long long)oi << 32) | oj;
          pos += __popc(m);
          found += __popc(m);
        }
      }
    }
  }
  if (!EMIT && lane == 0) count64[i] = found;
}

__global__ void k_pair_split(const unsigned long long* __restrict__ keys, long long m,
                             long long* __restrict__ pi, long long* __restrict__ pj) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const unsigned long long v = keys[k];
  pi[k] = (long long)(v >> 32);
  pj[k] = (long long)(v & 0xffffffffull);
}

constexpr int kRedBlocks = 148;
constexpr int kRedT = 256;

// Fixed-order reduction of the per-particle partials [n][8]: block b sums a
// fixed contiguous slice (thread-strided, then a fixed tree); the last block
// adds the block partials in block order.  out8 = [E, Pxx, Pxy, Pxz, Pyy,
// Pyz, Pzz] (virial / V) and the pair count (directed / 2) as int64 in
// stats[0].
__global__ void __launch_bounds__(kRedT)
    k_near_reduce(const double* __restrict__ part, long long n, double volume,
                  double* __restrict__ red, unsigned* __restrict__ ticket,
                  double* __restrict__ out7, long long* __restrict__ stats) {
  __shared__ double sh[8][kRedT];
  __shared__ bool last;
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (long long k = b0 + threadIdx.x; k < b1; k += kRedT)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] += part[8 * k + c];
#pragma unroll
  for (int c = 0; c < 8; ++c) sh[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int w = kRedT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int c = 0; c < 8; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 8) red[8 * blockIdx.x + threadIdx.x] = sh[threadIdx.x][0];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 8) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += ((volatile double*)red)[8 * b + threadIdx.x];
    if (threadIdx.x == 0) out7[0] = s;
    else if (threadIdx.x < 7) out7[threadIdx.x] = __ddiv_rn(s, volume);
    else {
      stats[0] = (long long)(0.5 * s + 0.25);
      stats[3] = (long long)(s + 0.5);  // directed count (slab ranks sum it)
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}


#define NEAR_CUDA(call)                                                            \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " +    \
                #call);                                                            \
      return e_ == cudaErrorMemoryAllocation ? ESP_ERR_OOM : ESP_ERR_CUDA;         \
    }                                                                              \
  } while (0)

int near_reserve(esp_near* p, long long n) {
  if (n <= p->cap) return ESP_OK;
  const long long cap = std::max<long long>(n, 1024);
  if (cap >= (1ll << 31)) {
    set_error("near-field particle count above 2^31");
    return ESP_ERR_CAPACITY;
  }
  cudaFree(p->d_key);
  cudaFree(p->d_key_sorted);
  cudaFree(p->d_idx);
  cudaFree(p->d_perm);
  cudaFree(p->d_rec_u);
  cudaFree(p->d_rec);
  cudaFree(p->d_part);
  cudaFree(p->d_sort_tmp);
  p->d_key = p->d_key_sorted = p->d_idx = p->d_perm = nullptr;
  p->d_rec_u = p->d_rec = nullptr;
  p->d_part = nullptr;
  p->d_sort_tmp = nullptr;
  p->cap = 0;
  NEAR_CUDA(cudaMalloc(&p->d_key, sizeof(int) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_key_sorted, sizeof(int) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_idx, sizeof(int) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_perm, sizeof(int) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_rec_u, sizeof(double4) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_rec, sizeof(double4) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_part, sizeof(double) * 8 * cap));
  size_t bytes = 0;
  NEAR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int*)nullptr, (int*)nullptr,
                                            (const int*)nullptr, (int*)nullptr, (int)cap, 0,
                                            31));
  NEAR_CUDA(cudaMalloc(&p->d_sort_tmp, bytes));
  p->sort_bytes = bytes;
  p->cap = cap;
  return ESP_OK;
}

int near_reserve_pairs(esp_near* p, long long n_pairs) {
  const long long m = 2 * n_pairs;
  if (m <= p->pair_cap) return ESP_OK;
  const long long cap = std::max<long long>(m, 4096);
  if (cap >= (1ll << 31)) {
    set_error("pair list above 2^30 pairs");
    return ESP_ERR_CAPACITY;
  }
  cudaFree(p->d_pkey);
  cudaFree(p->d_pkey_sorted);
  cudaFree(p->d_pent);
  cudaFree(p->d_pent_sorted);
  cudaFree(p->d_psort_tmp);
  p->d_pkey = p->d_pkey_sorted = nullptr;
  p->d_pent = p->d_pent_sorted = nullptr;
  p->d_psort_tmp = nullptr;
  p->pair_cap = 0;
  NEAR_CUDA(cudaMalloc(&p->d_pkey, sizeof(int) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_pkey_sorted, sizeof(int) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_pent, sizeof(long long) * cap));
  NEAR_CUDA(cudaMalloc(&p->d_pent_sorted, sizeof(long long) * cap));
  size_t bytes = 0;
  NEAR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int*)nullptr, (int*)nullptr,
                                            (const long long*)nullptr, (long long*)nullptr,
                                            (int)cap, 0, 31));
  NEAR_CUDA(cudaMalloc(&p->d_psort_tmp, bytes));
  p->psort_bytes = bytes;
  p->pair_cap = cap;
  return ESP_OK;
}

int near_reserve_cells(esp_near* p, long long need) {
  if (need <= p->cell_cap) return ESP_OK;
  cudaFree(p->d_cell_start);
  p->d_cell_start = nullptr;
  p->cell_cap = 0;
  NEAR_CUDA(cudaMalloc(&p->d_cell_start, sizeof(int) * need));
  p->cell_cap = need;
  return ESP_OK;
}

int near_reduce(esp_near* p, long long n, double* d_out7, long long* d_stats, cudaStream_t s) {
  if (n == 0) {
    NEAR_CUDA(cudaMemsetAsync(d_out7, 0, sizeof(double) * 7, s));
    NEAR_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(long long), s));
    NEAR_CUDA(cudaMemsetAsync(d_stats + 3, 0, sizeof(long long), s));
    return ESP_OK;
  }
  const int blocks = (int)std::min<long long>(kRedBlocks, (n + kRedT - 1) / kRedT);
  k_near_reduce<<<blocks, kRedT, 0, s>>>(p->d_part, n, p->volume, p->d_red, p->d_ticket,
                                         d_out7, d_stats);
  p->launches++;
  NEAR_CUDA(cudaGetLastError());
  return ESP_OK;
}

int check_plan(const esp_near* p, long long n) {
  if (!p) {
    set_error("null near-field plan");
    return ESP_ERR_PARAM;
  }
  if (!p->have_cell) {
    set_error("esp_near_set_cell has not been called");
    return ESP_ERR_MESH;
  }
  if (n < 0) {
    set_error("negative particle count");
    return ESP_ERR_PARAM;
  }
  return ESP_OK;
}

// Cell lattice with `div` cells per reach along each axis (fewer if the box
// would need more than 2^23 cells; thicker cells stay valid).
int near_layout(esp_near* p, int div) {
  CellGeom& g = p->g;
  long long nc[3], total;
  for (;;) {
    total = 1;
    for (int d = 0; d < 3; ++d) {
      nc[d] = (long long)std::floor(p->width[d] * div / p->reach);
      nc[d] = std::max<long long>(1, std::min<long long>(nc[d], 1024));
      total *= nc[d];
    }
    if (total <= (1ll << 23) || div == 1) break;
    --div;
  }
  while (total > (1ll << 23)) {
    total = 1;
    for (int d = 0; d < 3; ++d) {
      nc[d] = std::max<long long>(1, nc[d] / 2);
      total *= nc[d];
    }
  }
  const int st = near_reserve_cells(p, std::max<long long>(total + 1, p->cap + 1));
  if (st != ESP_OK) return st;
  for (int d = 0; d < 3; ++d) g.nc[d] = (int)nc[d];
  g.ncells = total;
  g.div = div;
  g.n_rows = (2 * div + 1) * (2 * div + 1);
  return ESP_OK;
}

// Automatic cells-per-reach (measured): 3 for small, dense
// orthorhombic systems (>= 24 particles per 2-per-reach cell and fewer than
// 8192 such cells: the finer trimming pays), otherwise 2.
int near_auto_div(const esp_near* p, long long n) {
  if (!p->g.ortho) return 2;
  long long c2 = 1;
  for (int d = 0; d < 3; ++d)
    c2 *= std::max<long long>(1, (long long)std::floor(p->width[d] * 2 / p->reach));
  return (c2 < 8192 && n >= 24 * c2) ? 3 : 2;
}

}  // namespace

extern "C" {

int esp_near_create(const esp_near_desc* d, esp_near** out) {
  if (!d || !out) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  *out = nullptr;
  if (!(d->r_c > 0.0)) {
    set_error("cutoff r_c must be positive");
    return ESP_ERR_PARAM;
  }
  if (d->use_table) {
    if (d->poly_order < 0 || d->poly_order + 1 > kPolyMax || d->n_knots < 2 ||
        !d->h_smooth_poly || !d->h_fn_poly || !d->h_knots || !d->h_smooth_spline ||
        !d->h_fn_spline || !(d->r_in > 0.0 && d->r_in < d->r_c)) {
      set_error("pair table shape unsupported");
      return ESP_ERR_PARAM;
    }
  }
  if (d->n_legendre < 1 || d->n_legendre > kLegMax || d->n_cumint < 1 ||
      d->n_cumint > kLegMax || !d->h_legendre || !d->h_cumint || !(d->C0 > 0.0)) {
    set_error("Legendre series shape unsupported");
    return ESP_ERR_PARAM;
  }
  if (!(d->reach >= d->r_c)) {
    set_error("cell-list reach must be at least r_c");
    return ESP_ERR_PARAM;
  }
  esp_near* p = new esp_near();
  p->div = d->cell_div > 0 ? std::min(d->cell_div, 4) : 0;   // 0: automatic
  {
    const char* k = std::getenv("ESP_NEAR_KERNEL");
    p->kernel = (k && std::strcmp(k, "rows") == 0) ? 1 : 0;
    const char* oc = std::getenv("ESP_NEAR_OCT");
    p->octants = !(oc && oc[0] == '0');
    if (cudaFuncSetAttribute(k_near_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(TileSmem)) != cudaSuccess) {
      set_error("near-field tile kernel: shared-memory opt-in failed");
      delete p;
      return ESP_ERR_CUDA;
    }
  }
  p->reach = d->reach;
  int st = near_reserve(p, std::max<long long>(d->max_particles, 1));
  if (st != ESP_OK) {
    esp_near_destroy(p);
    return st;
  }
  if (cudaMalloc(&p->d_red, sizeof(double) * 8 * kRedBlocks) != cudaSuccess ||
      cudaMalloc(&p->d_ticket, sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(p->d_ticket, 0, sizeof(unsigned)) != cudaSuccess) {
    set_error("near-field allocation failed");
    esp_near_destroy(p);
    return ESP_ERR_OOM;
  }
  NearConst& c = p->c;
  c = NearConst{};
  c.r_c = d->r_c;
  c.reach2 = d->reach * d->reach;
  c.rc2_hi = d->r_c * d->r_c * (1.0 + 1e-12);
  c.sing2 = (1e-12 * d->r_c) * (1e-12 * d->r_c);
  c.use_table = d->use_table ? 1 : 0;
  c.C0 = d->C0;
  c.c0rc = d->C0 * d->r_c;
  c.n_leg = d->n_legendre;
  c.n_cum = d->n_cumint;
  for (int k = 0; k < d->n_legendre; ++k) c.leg[k] = d->h_legendre[k];
  for (int k = 0; k < d->n_cumint; ++k) c.cum[k] = d->h_cumint[k];
  if (d->use_table) {
    c.r_in = d->r_in;
    c.n_poly = d->poly_order + 1;
    for (int k = 0; k < c.n_poly; ++k) {
      c.smooth_poly[k] = d->h_smooth_poly[k];
      c.fn_poly[k] = d->h_fn_poly[k];
    }
    c.n_knots = d->n_knots;
    c.inv_dk = (double)(d->n_knots - 1) / (d->h_knots[d->n_knots - 1] - d->h_knots[0]);
    const int nk = d->n_knots - 1;
    c.dk = (d->h_knots[nk] - d->h_knots[0]) / nk;
    c.h26 = c.dk * c.dk / 6.0;
    std::vector<double> tab;
    if (ESP_NEAR_HERMITE) {
      // per knot: value and second derivative of both splines (the cubic on
      // [x_k, x_k+1] is fixed by them; last knot from the last piece at s = h)
      tab.assign(4 * (size_t)(nk + 1), 0.0);
      const double* S = d->h_smooth_spline;
      const double* F = d->h_fn_spline;
      auto c_ = [&](const double* P, int m, int k) { return P[(size_t)m * nk + k]; };
      for (int k = 0; k <= nk; ++k) {
        for (int w = 0; w < 2; ++w) {
          const double* P = w == 0 ? S : F;
          double y, M;
          if (k < nk) {
            y = c_(P, 3, k);
            M = 2.0 * c_(P, 1, k);
          } else {
            const double h = d->h_knots[nk] - d->h_knots[nk - 1];
            y = ((c_(P, 0, nk - 1) * h + c_(P, 1, nk - 1)) * h + c_(P, 2, nk - 1)) * h +
                c_(P, 3, nk - 1);
            M = 6.0 * c_(P, 0, nk - 1) * h + 2.0 * c_(P, 1, nk - 1);
          }
          // layout per knot: y_s, M_s, y_f, M_f -> double2 {y, M} per spline;
          // loads read (s0, f0, s1, f1) as consecutive double2
          tab[4 * (size_t)k + 2 * w] = y;
          tab[4 * (size_t)k + 2 * w + 1] = M;
        }
      }
    } else {
      tab.assign(10 * (size_t)nk, 0.0);
      for (int k = 0; k < nk; ++k) {
        tab[10 * (size_t)k] = d->h_knots[k];
        for (int m = 0; m < 4; ++m) {
          tab[10 * (size_t)k + 2 + m] = d->h_smooth_spline[(size_t)m * nk + k];
          tab[10 * (size_t)k + 6 + m] = d->h_fn_spline[(size_t)m * nk + k];
        }
      }
    }
    if (cudaMalloc(&p->d_tab, sizeof(double) * tab.size()) != cudaSuccess ||
        cudaMemcpy(p->d_tab, tab.data(), sizeof(double) * tab.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess) {
      set_error("pair table upload failed");
      esp_near_destroy(p);
      return ESP_ERR_OOM;
    }
  }
  *out = p;
  return ESP_OK;
}

int esp_near_destroy(esp_near* p) {
  if (!p) return ESP_OK;
  cudaFree(p->d_tab);
  cudaFree(p->d_key);
  cudaFree(p->d_key_sorted);
  cudaFree(p->d_idx);
  cudaFree(p->d_perm);
  cudaFree(p->d_rec_u);
  cudaFree(p->d_rec);
  cudaFree(p->d_cell_start);
  cudaFree(p->d_part);
  cudaFree(p->d_red);
  cudaFree(p->d_ticket);
  cudaFree(p->d_sort_tmp);
  cudaFree(p->d_pkey);
  cudaFree(p->d_pkey_sorted);
  cudaFree(p->d_pent);
  cudaFree(p->d_pent_sorted);
  cudaFree(p->d_psort_tmp);
  cudaFree(p->d_list_keys);
  cudaFree(p->d_list_keys2);
  cudaFree(p->d_list_i);
  cudaFree(p->d_list_j);
  cudaFree(p->d_list_tmp);
  delete p;
  return ESP_OK;
}

int esp_near_reserve(esp_near* p, int64_t n_particles, int64_t n_pairs) {
  if (!p || n_particles < 0 || n_pairs < 0) {
    set_error("bad argument");
    return ESP_ERR_PARAM;
  }
  int st = near_reserve(p, n_particles);
  if (st != ESP_OK) return st;
  if (n_pairs > 0 && (st = near_reserve_pairs(p, n_pairs)) != ESP_OK) return st;
  return near_reserve_cells(p, std::max<long long>(n_particles + 1, p->g.ncells + 1));
}

int esp_near_set_cell(esp_near* p, const double* h, const double* hinv, int32_t orthorhombic,
                      double volume) {
  if (!p || !h || !hinv) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  if (!(volume > 0.0)) {
    set_error("cell volume must be positive");
    return ESP_ERR_PARAM;
  }
  CellGeom g{};
  for (int k = 0; k < 9; ++k) {
    g.h[k] = h[k];
    g.hinv[k] = hinv[k];
  }
  g.ortho = orthorhombic ? 1 : 0;
  g.eps = 1e-9 * std::max(std::max(h[0], h[4]), h[8]);
  // perpendicular width along lattice axis d: 1 / |row d of h^-1|
  for (int d = 0; d < 3; ++d) {
    const double a = hinv[3 * d], b = hinv[3 * d + 1], c = hinv[3 * d + 2];
    p->width[d] = 1.0 / std::sqrt(a * a + b * b + c * c);
    if (!(p->reach < 0.5 * p->width[d])) {
      set_error("cutoff not below half the minimum perpendicular width");
      return ESP_ERR_PARAM;
    }
  }
  p->g = g;
  p->volume = volume;
  // cell-start storage for the finest lattice the plan may pick
  int st = near_layout(p, p->div > 0 ? p->div : 3);
  if (st != ESP_OK) return st;
  if (p->div == 0 && (st = near_layout(p, 2)) != ESP_OK) return st;
  p->have_cell = 1;
  return ESP_OK;
}

int esp_near_evaluate(esp_near* p, const double* d_pos, const double* d_q, int64_t n,
                      int32_t flags, double* d_out7, double* d_forces, int64_t* d_stats,
                      void* stream) {
  return esp_near_evaluate_local(p, d_pos, d_q, n, n, flags, d_out7, d_forces, d_stats, stream);
}

int esp_near_evaluate_local(esp_near* p, const double* d_pos, const double* d_q, int64_t n,
                            int64_t n_owned, int32_t flags, double* d_out7, double* d_forces,
                            int64_t* d_stats, void* stream) {
  if (n_owned < 0 || n_owned > n) {
    set_error("n_owned must lie in [0, n]");
    return ESP_ERR_PARAM;
  }
  int st = check_plan(p, n);
  if (st != ESP_OK) return st;
  if (n > p->cap) {
    set_error("particle count exceeds the near-field plan capacity (esp_near_reserve)");
    return ESP_ERR_CAPACITY;
  }
  if (!d_out7 || !d_stats || (n > 0 && (!d_pos || !d_q)) || (n_owned > 0 && !d_forces)) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  p->launches = 0;
  if (p->div == 0) {   // automatic lattice for this particle count (storage preallocated)
    const int want = near_auto_div(p, n);
    if (want != p->g.div && (st = near_layout(p, want)) != ESP_OK) return st;
  }
  // stats[1]: first coincident pair, stats[2]: first bad pair (all ones = none)
  NEAR_CUDA(cudaMemsetAsync(d_stats + 1, 0xff, 2 * sizeof(int64_t), s));
  if (n == 0) return near_reduce(p, 0, d_out7, (long long*)d_stats, s);
  const int B = 256;
  const unsigned grid = (unsigned)((n + B - 1) / B);
  const int sub = p->kernel == 0 ? p->octants : 0;
  k_near_cells<<<grid, B, 0, s>>>(d_pos, d_q, n, p->g, p->d_key, p->d_idx, p->d_rec_u, sub);
  p->launches++;
  size_t bytes = p->sort_bytes;
  NEAR_CUDA(cub::DeviceRadixSort::SortPairs(p->d_sort_tmp, bytes, p->d_key, p->d_key_sorted,
                                            p->d_idx, p->d_perm, (int)n, 0,
                                            bits_for(p->g.ncells * (sub ? 8 : 1)), s));
  p->launches += 3;
  k_near_sorted<<<grid, B, 0, s>>>(p->d_key_sorted, p->d_perm, p->d_rec_u, n, p->g.ncells,
                                   p->d_rec, p->d_cell_start, sub);
  p->launches++;
  if (p->kernel == 1) {
    k_near_pairs<<<(unsigned)p->g.ncells, kNearThreads, 0, s>>>(
        p->c, p->d_rec, p->d_cell_start, p->d_perm, p->g, p->d_tab,
        (flags & ESP_NEAR_ACCUMULATE) ? 1 : 0, d_forces, p->d_part,
        (unsigned long long*)(d_stats + 1), (int)n_owned);
  } else {
    k_near_tile<<<(unsigned)p->g.ncells, kTileW * 32, sizeof(TileSmem), s>>>(
        p->c, p->d_rec, p->d_cell_start, p->d_perm, p->g, p->d_tab,
        (flags & ESP_NEAR_ACCUMULATE) ? 1 : 0, d_forces, p->d_part,
        (unsigned long long*)(d_stats + 1), (int)n_owned);
  }
  p->launches++;
  NEAR_CUDA(cudaGetLastError());
  return near_reduce(p, n, d_out7, (long long*)d_stats, s);
}

int esp_near_evaluate_pairs(esp_near* p, const double* d_pos, const double* d_q, int64_t n,
                            const int64_t* d_i, const int64_t* d_j, int64_t n_pairs,
                            int32_t flags, double* d_out7, double* d_forces, int64_t* d_stats,
                            void* stream) {
  int st = check_plan(p, n);
  if (st != ESP_OK) return st;
  if (n > p->cap || 2 * n_pairs > p->pair_cap || n + 1 > p->cell_cap) {
    set_error("particle or pair count exceeds the near-field plan capacity (esp_near_reserve)");
    return ESP_ERR_CAPACITY;
  }
  if (!d_out7 || !d_stats || n_pairs < 0 || (n > 0 && (!d_pos || !d_q || !d_forces)) ||
      (n_pairs > 0 && (!d_i || !d_j))) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  p->launches = 0;
  NEAR_CUDA(cudaMemsetAsync(d_stats + 1, 0xff, 2 * sizeof(int64_t), s));
  if (n == 0) return near_reduce(p, 0, d_out7, (long long*)d_stats, s);
  const long long m = 2 * n_pairs;
  if (m > 0) {
    k_pair_keys<<<(unsigned)((n_pairs + 255) / 256), 256, 0, s>>>(
        (const long long*)d_i, (const long long*)d_j, n_pairs, n, p->d_pkey, p->d_pent,
        (unsigned long long*)(d_stats + 2));
    p->launches++;
    size_t bytes = p->psort_bytes;
    NEAR_CUDA(cub::DeviceRadixSort::SortPairs(p->d_psort_tmp, bytes, p->d_pkey,
                                              p->d_pkey_sorted, p->d_pent, p->d_pent_sorted,
                                              (int)m, 0, bits_for(n + 1), s));
    p->launches += 3;
    // particle segment starts reuse the cell-start buffer (n + 1 entries)
    k_pair_starts<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(p->d_pkey_sorted, m, n,
                                                             p->d_cell_start);
  } else {
    k_fill_int<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(p->d_cell_start, n + 1, 0);
  }
  p->launches++;
  k_pair_list<<<(unsigned)((n * 32 + 127) / 128), 128, 0, s>>>(
      p->c, d_pos, d_q, (const long long*)d_i, (const long long*)d_j, p->d_pent_sorted,
      p->d_cell_start, n, p->g, p->d_tab, (flags & ESP_NEAR_ACCUMULATE) ? 1 : 0,
      d_forces, p->d_part, (unsigned long long*)(d_stats + 1));
  p->launches++;
  NEAR_CUDA(cudaGetLastError());
  return near_reduce(p, n, d_out7, (long long*)d_stats, s);
}

int esp_near_build_pairs(esp_near* p, const double* d_pos, int64_t n, int64_t* n_pairs,
                         void* stream) {
  int st = check_plan(p, n);
  if (st != ESP_OK) return st;
  if (!n_pairs || (n > 0 && !d_pos)) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  if ((st = near_reserve(p, n)) != ESP_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  *n_pairs = 0;
  p->list_n = 0;
  if (n < 2) return ESP_OK;
  const int B = 256;
  const unsigned grid = (unsigned)((n + B - 1) / B);
  k_near_cells<<<grid, B, 0, s>>>(d_pos, nullptr, n, p->g, p->d_key, p->d_idx, p->d_rec_u, 0);
  size_t bytes = p->sort_bytes;
  NEAR_CUDA(cub::DeviceRadixSort::SortPairs(p->d_sort_tmp, bytes, p->d_key, p->d_key_sorted,
                                            p->d_idx, p->d_perm, (int)n, 0,
                                            bits_for(p->g.ncells), s));
  k_near_sorted<<<grid, B, 0, s>>>(p->d_key_sorted, p->d_perm, p->d_rec_u, n, p->g.ncells,
                                   p->d_rec, p->d_cell_start, 0);
  // per-particle counts and their exclusive prefix (n + 1 entries)
  long long *d_cnt = nullptr, *d_off = nullptr;
  NEAR_CUDA(cudaMallocAsync(&d_cnt, sizeof(long long) * (n + 1), s));
  NEAR_CUDA(cudaMallocAsync(&d_off, sizeof(long long) * (n + 1), s));
  NEAR_CUDA(cudaMemsetAsync(d_cnt + n, 0, sizeof(long long), s));
  const unsigned wgrid = (unsigned)((n * 32 + 127) / 128);
  k_pair_enum<false><<<wgrid, 128, 0, s>>>(p->d_rec, p->d_cell_start, p->d_key_sorted,
                                            p->d_perm, n, p->g, p->reach * p->reach, nullptr,
                                            nullptr, d_cnt);
  NEAR_CUDA(cudaGetLastError());
  size_t sb = 0;
  NEAR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, d_cnt, d_off, (int)(n + 1), s));
  void* tmp = nullptr;
  NEAR_CUDA(cudaMallocAsync(&tmp, sb, s));
  NEAR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, sb, d_cnt, d_off, (int)(n + 1), s));
  long long m = 0;
  NEAR_CUDA(cudaMemcpyAsync(&m, d_off + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
  NEAR_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(d_cnt, s);
  if (m >= (1ll << 31)) {
    cudaFreeAsync(d_off, s);
    set_error("pair list above 2^31 pairs");
    return ESP_ERR_CAPACITY;
  }
  if (m > 0) {
    if (m > p->list_cap) {
      cudaFree(p->d_list_keys);
      cudaFree(p->d_list_keys2);
      cudaFree(p->d_list_i);
      cudaFree(p->d_list_j);
      cudaFree(p->d_list_tmp);
      p->d_list_keys = p->d_list_keys2 = nullptr;
      p->d_list_i = p->d_list_j = nullptr;
      p->d_list_tmp = nullptr;
      p->list_cap = 0;
      NEAR_CUDA(cudaMalloc(&p->d_list_keys, sizeof(unsigned long long) * m));
      NEAR_CUDA(cudaMalloc(&p->d_list_keys2, sizeof(unsigned long long) * m));
      NEAR_CUDA(cudaMalloc(&p->d_list_i, sizeof(long long) * m));
      NEAR_CUDA(cudaMalloc(&p->d_list_j, sizeof(long long) * m));
      size_t tb = 0;
      NEAR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, (const unsigned long long*)nullptr,
                                               (unsigned long long*)nullptr, (int)m, 0, 64));
      NEAR_CUDA(cudaMalloc(&p->d_list_tmp, tb));
      p->list_tmp_bytes = tb;
      p->list_cap = m;
    }
    k_pair_enum<true><<<wgrid, 128, 0, s>>>(p->d_rec, p->d_cell_start, p->d_key_sorted,
                                             p->d_perm, n, p->g, p->reach * p->reach, d_off,
                                             p->d_list_keys, nullptr);
    const int hb = bits_for(n);
    size_t tb = p->list_tmp_bytes;
    NEAR_CUDA(cub::DeviceRadixSort::SortKeys(p->d_list_tmp, tb, p->d_list_keys,
                                             p->d_list_keys2, (int)m, 0, 32 + hb, s));
    k_pair_split<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(p->d_list_keys2, m, p->d_list_i,
                                                             p->d_list_j);
    NEAR_CUDA(cudaGetLastError());
  }
  cudaFreeAsync(d_off, s);
  NEAR_CUDA(cudaStreamSynchronize(s));
  *n_pairs = m;
  p->list_n = m;
  return ESP_OK;
}

int esp_near_copy_pairs(esp_near* p, int64_t* d_i, int64_t* d_j, void* stream) {
  if (!p || (p->list_n > 0 && (!d_i || !d_j))) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  if (p->list_n == 0) return ESP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  NEAR_CUDA(cudaMemcpyAsync(d_i, p->d_list_i, sizeof(int64_t) * p->list_n,
                            cudaMemcpyDeviceToDevice, s));
  NEAR_CUDA(cudaMemcpyAsync(d_j, p->d_list_j, sizeof(int64_t) * p->list_n,
                            cudaMemcpyDeviceToDevice, s));
  return ESP_OK;
}

int esp_near_info(const esp_near* p, int64_t* info8) {
  if (!p || !info8) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  info8[0] = p->g.nc[0];
  info8[1] = p->g.nc[1];
  info8[2] = p->g.nc[2];
  info8[3] = p->g.n_rows;
  info8[4] = p->cap;
  info8[5] = p->launches;
  info8[6] = p->g.div;
  info8[7] = p->c.use_table;
  return ESP_OK;
}

}  // extern "C"
