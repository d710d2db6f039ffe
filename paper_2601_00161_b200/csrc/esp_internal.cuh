// esp_internal.cuh — shared structs and device helpers for the B200 ESP
// k-space path.  See DESIGN.md for the data layout and kernel roofline notes.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/esp_b200.h"

namespace esp {

constexpr int kPad = 16;          // padded columns per tile along x and y
constexpr int kTileThreads = 256; // threads per gather CTA
constexpr int kSpreadThreads = 128; // spread CTA: 4 warps x 8x8 columns, 2 per lane
constexpr int kChunk = 256;       // particles staged per CTA pass (spread)
constexpr int kGChunk = 64;       // particles staged per CTA pass (gather)
constexpr int kMaxCoef = 25;      // window table degree + 1 (reference: 19)
constexpr int kMaxPieces = 64;    // window pieces (P * pieces-per-unit)
constexpr int kRedThreads = 256;
constexpr long long kSortThreshold = 500000;   // radix-sort binning above this N

// Grid/tile geometry passed by value to every kernel.
struct Geom {
  int M[3];             // local tile-grid counts (== Mu except for z slabs)
  int Mu[3];            // global grid counts: coordinates and periodic wrap
  int zshift;           // slab plans: local plane = global plane - zshift
  int P, lo, odd, ortho;
  double spacing[3];
  double hinv[9];       // row-major inverse cell matrix (triclinic u)
  int TX, TY, TZ, PZ;   // anchor-cell tile and padded z extent (gather tiles)
  int ntx, nty, ntz;
  int TZS, PZS, ntzs;   // spread tiles: deeper in z (less scratch halo)
  long long n_keys;     // ntx * nty * Mz  (key = (ty*ntx+tx)*Mz + az)
};

// Window table (device pointers).
struct Table {
  const double* coef;   // n_pieces * ncoef, highest power first
  const double* dcoef;  // derivative table
  const double* breaks; // n_pieces + 1
  int n_pieces, ncoef;
};

// Grid coordinate u_d of a Cartesian position (mesh.py:160 for orthorhombic
// cells: u = x / h_d, IEEE division; triclinic: M_d * (h^-1 r)_d with the
// oracle's fixed operation order).  No FMA contraction, so the anchors agree
// bit-for-bit with the CPU reference.
__device__ __forceinline__ void grid_coords(const Geom& g, double x, double y,
                                            double z, double u[3]) {
  if (g.ortho) {
    u[0] = __ddiv_rn(x, g.spacing[0]);
    u[1] = __ddiv_rn(y, g.spacing[1]);
    u[2] = __ddiv_rn(z, g.spacing[2]);
  } else {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double s = __dadd_rn(__dadd_rn(__dmul_rn(g.hinv[3 * d + 0], x),
                                     __dmul_rn(g.hinv[3 * d + 1], y)),
                           __dmul_rn(g.hinv[3 * d + 2], z));
      u[d] = __dmul_rn(s, (double)g.Mu[d]);
    }
  }
}

// One component u_d of grid_coords (same operations, same order).
__device__ __forceinline__ double grid_coord(const Geom& g, int d, double x, double y,
                                             double z) {
  if (g.ortho) return __ddiv_rn(d == 0 ? x : (d == 1 ? y : z), g.spacing[d]);
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(g.hinv[3 * d + 0], x),
                                       __dmul_rn(g.hinv[3 * d + 1], y)),
                             __dmul_rn(g.hinv[3 * d + 2], z));
  return __dmul_rn(s, (double)g.Mu[d]);
}

// Stencil anchor: np.round (half-to-even) for odd P, np.floor for even P
// (mesh.py:161-168).
// Non-finite or huge coordinates are clamped (fmax/fmin drop NaN) so that
// every pass derives the same in-range anchor; finite |u| < 4e15 is unchanged.
// The reference's int64 cast is undefined there too (mesh.py:160-168).
__device__ __forceinline__ double anchor_base(const Geom& g, double u) {
  const double b = g.odd ? rint(u) : floor(u);
  return fmin(fmax(b, -4.0e15), 4.0e15);
}

__device__ __forceinline__ int wrap_index(long long v, int M) {
  long long r = v % M;
  return (int)(r < 0 ? r + M : r);
}

// Local anchor index of a stencil base along axis d: the periodic global
// anchor, shifted into the slab's local planes for z.
__device__ __forceinline__ int local_anchor(const Geom& g, int d, double base) {
  const int a = wrap_index((long long)base, g.Mu[d]);
  if (d != 2 || g.zshift == 0 && g.M[2] == g.Mu[2]) return a;
  // slab plans: a charge outside the slab (a caller error) is clamped onto
  // the local planes so that keys and tile offsets stay in range
  return min(max(a - g.zshift, 0), g.M[2] - 1);
}

// Periodic wrap for indices a few periods from [0, M): no division.
__device__ __forceinline__ int wrap_near(int v, int M) {
  while (v < 0) v += M;
  while (v >= M) v -= M;
  return v;
}

// W(t) from the piecewise table (pswf.py:253-258 semantics: zero outside
// [breaks[0], breaks[n]]; interval search as scipy PPoly, right end closed).
template <typename real>
__device__ __forceinline__ real window_eval(const real* __restrict__ coef,
                                            const double* __restrict__ breaks,
                                            int n_pieces, int ncoef, double t) {
  const double b0 = breaks[0], bn = breaks[n_pieces];
  if (!(t >= b0 && t <= bn)) return real(0);
  const double width = (bn - b0) / n_pieces;
  int j = (int)floor((t - b0) / width);
  j = j < 0 ? 0 : (j > n_pieces - 1 ? n_pieces - 1 : j);
  if (t < breaks[j] && j > 0) --j;
  else if (j + 1 < n_pieces && t >= breaks[j + 1]) ++j;
  const real s = (real)(t - breaks[j]);
  const real* c = coef + j * ncoef;
  real acc = c[0];
  for (int m = 1; m < ncoef; ++m) acc = fma(acc, s, c[m]);
  return acc;
}

// numpy.polynomial.legendre.legval (Clenshaw recursion, same operation order;
// used for Fhat and dterm in the mode setup, mesh.py:269-275).
__device__ __forceinline__ double legval(double x, const double* c, int n) {
  if (n == 1) return c[0];
  double c0, c1;
  if (n == 2) {
    c0 = c[0];
    c1 = c[1];
  } else {
    int nd = n;
    c0 = c[n - 2];
    c1 = c[n - 1];
    for (int i = 3; i <= n; ++i) {
      double tmp = c0;
      nd = nd - 1;
      c0 = __dsub_rn(c[n - i], __ddiv_rn(__dmul_rn(c1, (double)(nd - 1)), (double)nd));
      c1 = __dadd_rn(tmp, __ddiv_rn(__dmul_rn(__dmul_rn(c1, x), (double)(2 * nd - 1)),
                                    (double)nd));
    }
  }
  return __dadd_rn(c0, __dmul_rn(c1, x));
}

// Fast path for the common table shape (one degree-18 piece per unit
// interval, P <= 12): the coefficients travel as a kernel parameter, so the
// unrolled Horner chains read them straight from the constant bank (no
// shared-memory loads).  Stencil offset s always falls in piece P-1-s; the
// rare tie on a piece boundary drops to the general search.
constexpr int kFastNC = 19;
constexpr int kFastMaxP = 12;
struct FastTab {
  double c[kFastMaxP * kFastNC];
  float cf[kFastMaxP * kFastNC];
  double brk[kFastMaxP + 1];
  int enabled;
};

template <typename real> __device__ __forceinline__ const real* fast_coef(const FastTab& t);
template <> __device__ __forceinline__ const double* fast_coef<double>(const FastTab& t) { return t.c; }
template <> __device__ __forceinline__ const float* fast_coef<float>(const FastTab& t) { return t.cf; }

// Out-of-line general table evaluation: only reached on exact piece-boundary
// ties, so it must not bloat the unrolled fast path (I-cache).
template <typename real>
__device__ __noinline__ real window_eval_slow(const real* __restrict__ coef,
                                              const double* __restrict__ breaks,
                                              int n_pieces, int ncoef, double t) {
  return window_eval<real>(coef, breaks, n_pieces, ncoef, t);
}

// w[s] = qf * W(u - (base + lo + s)), s = 0..P-1.
// Fast table (P unit-width pieces, checked at plan creation): stencil offset s
// falls in piece P-1-s, and because the pieces are one grid spacing wide the
// offset inside the piece, x = u - base - lo - brk[P-1], is the same for all
// P weights — one subtraction and one range test per axis, then P
// straight-line Horner chains that share x (coefficients are kernel-parameter
// constants).  A tie on a piece boundary (rounding) drops to the general
// search for all P weights.
template <typename real, int P>
__device__ __forceinline__ void stencil_weights(const FastTab& ft, const real* s_tab,
                                                const double* s_brk, int n_pieces,
                                                int ncoef, double u, double base, int lo,
                                                real qf, real* w) {
  if (ft.enabled) {
    const double t0 = u - (base + (double)lo);       // s = 0: piece P - 1
    const double xd = t0 - ft.brk[P - 1];
    if (xd >= 0.0 && t0 < ft.brk[P]) {
      const real* C = fast_coef<real>(ft);
      const real x = (real)xd;
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const int j = P - 1 - s;
        real acc = C[j * kFastNC];
#pragma unroll
        for (int m = 1; m < kFastNC; ++m) acc = fma(acc, x, C[j * kFastNC + m]);
        w[s] = acc * qf;
      }
      return;
    }
  }
#pragma unroll 1
  for (int s = 0; s < P; ++s) {
    const double t = u - (base + (double)(lo + s));
    w[s] = window_eval_slow<real>(s_tab, s_brk, n_pieces, ncoef, t) * qf;
  }
}

// Per-axis candidate (tile, padded index) pairs for the deterministic halo
// combine, precomputed at plan creation: entry [c*kCombW + k] =
// tile | pad << 16, count in cnt[c].
constexpr int kCombW = 8;
// Per-particle weight record: 3 dims x RS weights (RS = 8 for P <= 8, else 12).
__host__ __device__ constexpr int rec_stride(int P) { return P <= 8 ? 8 : 12; }
struct CombineTabs {
  const int* ent[3];
  const int* cnt[3];
};

// Grid value at (x, y, z): the sum of the (at most 8) spread tile blocks
// covering it, in a fixed (z, y, x) order (bitwise reproducible).  Used by
// k_combine and, on the fused-transform path, by the x transform's loads.
// Scratch layout of the spread's padded tile blocks: [tz][pz][ty][py][tx][px]
// (px fastest, 16 wide).  One padded row of every tile along x is one
// contiguous run of ntx * 16 values, so the combine's loads for a grid row
// (own columns and the left neighbour's halo) stream through contiguous
// memory instead of 72 / 56-byte pieces of blocks 80 KB apart.
struct ScrLayout {
  long long row;     // ntx * 16: stride of py
  long long plane;   // nty * 16 * row: stride of pz
};
__host__ __device__ __forceinline__ ScrLayout scr_layout(const Geom& g) {
  ScrLayout L;
  L.row = (long long)g.ntx * kPad;
  L.plane = (long long)g.nty * kPad * L.row;
  return L;
}
// element (pz, py, px) of tile (tx, ty, tz)
__host__ __device__ __forceinline__ long long scr_index(const Geom& g, const ScrLayout& L,
                                                       int tx, int ty, int tz, int pz, int py,
                                                       int px) {
  return ((long long)tz * g.PZS + pz) * L.plane + ((long long)ty * kPad + py) * L.row +
         (long long)tx * kPad + px;
}

template <typename real>
__device__ __forceinline__ double combine_at(const Geom& g, const CombineTabs& ct,
                                             const real* __restrict__ scratch, int x, int y,
                                             int z) {
  const int nx = ct.cnt[0][x], ny = ct.cnt[1][y], nz = ct.cnt[2][z];
  const ScrLayout L = scr_layout(g);
  double acc = 0.0;
  if (nx <= 2 && ny <= 2 && nz <= 2) {
    // common case (each axis covered by <= 2 tiles): issue all <= 8 loads
    // before summing, in the same fixed (z, y, x) order
    long long addr[8];
    bool use[8];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int ez = ct.ent[2][z * kCombW + (a < nz ? a : 0)];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int ey = ct.ent[1][y * kCombW + (b < ny ? b : 0)];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int ex = ct.ent[0][x * kCombW + (c < nx ? c : 0)];
          const int i = (a * 2 + b) * 2 + c;
          addr[i] = scr_index(g, L, ex & 0xffff, ey & 0xffff, ez & 0xffff, ez >> 16, ey >> 16,
                              ex >> 16);
          use[i] = a < nz && b < ny && c < nx;
        }
      }
    }
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = use[i] ? (double)scratch[addr[i]] : 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (use[i]) acc += v[i];
  } else {
    for (int a = 0; a < nz; ++a) {
      const int ez = ct.ent[2][z * kCombW + a];
      for (int b = 0; b < ny; ++b) {
        const int ey = ct.ent[1][y * kCombW + b];
        for (int c = 0; c < nx; ++c) {
          const int ex = ct.ent[0][x * kCombW + c];
          acc += (double)scratch[scr_index(g, L, ex & 0xffff, ey & 0xffff, ez & 0xffff,
                                           ez >> 16, ey >> 16, ex >> 16)];
        }
      }
    }
  }
  return acc;
}

// Ghost-padded layout of the three ik fields for the TMA gather
// (esp_gather_tma.cu): component c, grid point (x, y, z) lives at
// c*cstride + ((z + S2)*E1 + (y + S1))*E0 + (x + S0); the ghost entries hold
// the periodic images, so every tile's stencil box is in bounds.
struct FieldPad {
  int enabled;
  int S[3];
  int E[3];
  int M[3];
  long long cstride;
};

// du/dr (grid units per length) of the gradient gathers: F_a = -q sum_d G_d J[d][a].
struct Jac {
  double j[9];
};

template <typename T> struct Cplx;
template <> struct Cplx<double> { using type = double2; };
template <> struct Cplx<float> { using type = float2; };

}  // namespace esp

// ---------------------------------------------------------------------------
// Host-side plan object.
struct esp_plan {
  // static description
  int M[3];
  int Mu[3];              // global grid counts (slab plans: Mu[2] != M[2])
  int zshift;             // slab plans: z0 + lo
  long long G, Hx, H;
  int P, lo, odd, precision, deterministic;
  long long cap;
  int n_pieces, ncoef;
  double kmax, r_c, split_c, split_lambda0, split_C0;
  int n_leg, n_legd;
  // tiles
  int TX, TY, TZ, PZ, ntx, nty, ntz;
  int TZS, PZS, ntzs;
  long long n_tiles, n_tiles_s, n_keys;
  // cell
  int have_cell;
  int ortho;
  double spacing[3], hinv[9], hmat[9], volume, h3, grad_scale[3];
  int band[3];
  int nbx, nby, nbz;
  long long nbox, n_modes;
  int n_red_blocks;
  // band-pruned fused transforms (esp_fft.cu); null -> cuFFT path
  void* fused;
  double* d_partials_fft;
  int n_red_blocks_fft;
  // device buffers
  double *d_tab, *d_dtab, *d_breaks;
  float *d_tabf, *d_dtabf;
  double *d_leg, *d_legd;
  int *d_key, *d_slot, *d_counts, *d_offsets, *d_bkey;
  double *d_u, *d_q;      // binned (canonical) particle data: u[3][cap], q[cap]
  int* d_idx;
  double *d_u_tmp, *d_q_tmp;
  int* d_idx_tmp;
  void* d_drec;           // per binned particle: window-derivative weights (analytic)
  void* d_wrec;           // per binned particle: 24 window weights (x|y|z, q folded
                          // into x by the spread), precision of the plan
  int* d_pk;              // per binned particle: tile-local anchor x | y<<8 | z<<16
  void* d_cub;
  size_t cub_bytes;
  void* d_sort_tmp;       // CUB radix-sort temp (large-N binning path)
  size_t sort_bytes;
  long long sort_threshold;
  void* d_scratch;
  void* d_grid;
  void* d_spec;
  void* d_ikspec;
  void* d_fields;
  double* d_axis_k;       // 9 arrays: K[a*3+d] at offset koff[d]
  double* d_axis_w;       // 3 arrays
  long long koff[3];      // offsets of axis d inside each block of length Msum
  int* d_box_iy;
  int* d_box_iz;
  double *d_modeA, *d_modeB;
  double* d_partials;
  int* d_err;
  double* d_err_out7;     // sink for reductions run only to write spectra
  int* d_comb_ent;        // combine candidate tables (3 axes)
  int* d_comb_cnt;
  long long comb_off[3];
  int comb_max[3];        // most tiles covering one coordinate, per axis
  int* d_zlist = nullptr; // z planes covered by one z tile (n_z_single of them), then the rest
  int n_z_single = 0;
  esp::FastTab* h_fast;   // host copy of the fast window table (kernel param)
  esp::FastTab* h_fast_d = nullptr;   // derivative window table (analytic gather)
  int need_records = 0; // next radix binning writes the weight records in its gather pass
                        // (else: records-free gather, records by ensure_records)
  int records_ready = 0;  // wrec / pk hold the last binning's records
  int want_drec = 0;    // next binning also writes derivative records (analytic step)
  int drec_ready = 0;   // d_drec holds the last binning's derivative records
  cufftHandle fwd, inv3, inv1;
  int have_fwd, have_inv3, have_inv1;
  long long fwd_count, inv_count;
  long long last_n;
  int have_bins, have_spec, have_ik;
  int ik_zeroed;          // ik spectra already zeroed on the side stream
  cudaStream_t side;      // fork/join stream (captured as a parallel graph branch)
  cudaEvent_t ev_fork, ev_join;
  int have_side;
  int launches;
  // profiling: events recorded after each stage kernel when enabled
  int profiling;
  int n_ev;
  cudaEvent_t q_ready = nullptr;   // esp_set_charges_event: wait before reading q
  // radix binning with late charges: the caller's q, binned by ensure_records
  // after the records pass (k_bin_charges) once q_deferred_ev has fired
  const double* q_deferred = nullptr;
  cudaEvent_t q_deferred_ev = nullptr;
  cudaEvent_t ev[48];
  const char* ev_name[48];
  // TMA gather (esp_gather_tma.cu): ghost-padded ik fields and their tensor map
  void* d_fpad = nullptr;
  esp::FieldPad fpad{};
  int fpad_written = 0;   // the last fused inverse wrote d_fpad (not d_fields)
  // esp_evaluate on the band-pruned transforms: the spread leaves its tile
  // blocks in d_scratch and the forward x pass sums them (k_x_comb_r2c);
  // d_grid is then not written by that step
  int grid_in_scratch = 0;
  alignas(64) unsigned char tmap[128];
  // esp_set_host_forces: the next force step copies its forces to this pinned
  // host buffer in `host_chunks` index ranges, each as soon as it is gathered
  double* host_forces = nullptr;
  int host_chunks = 0;
  cudaEvent_t ev_chunk[8] = {};
  int have_ev_chunk = 0;
};

namespace esp {

Geom make_geom(const esp_plan* p);

// Launchers (each returns cudaError_t of the launch).
cudaError_t launch_bin(esp_plan* p, const double* d_pos, const double* d_q,
                       long long n, cudaStream_t s);
// Weight records of the current bins, if the binning pass skipped them (the
// record consumers: cp.async gathers, the tiny-grid spread, local pressure).
cudaError_t ensure_records(esp_plan* p, cudaStream_t s);
// The spread will run k_spread_warp (weights from u, no records).
bool spread_uses_warp(const esp_plan* p);
// Tiles into the scratch blocks, then (with_combine) the halo combine into
// d_grid.
cudaError_t launch_spread(esp_plan* p, cudaStream_t s, bool with_combine = true);
CombineTabs combine_tabs(const esp_plan* p);
// The fused transforms' forward x pass can sum the spread's tile blocks itself
// (no k_combine, no grid round trip): separate x and y passes, one GPU.
bool fused_x_combines(const esp_plan* p);
cudaError_t launch_scale_reduce(esp_plan* p, double* d_out7, int write_ik,
                                cudaStream_t s);
// Output placement of the 3 gathered values of particle id:
// out[id*stride + m[c]] (and out[id*stride + m2[c]] when m2[c] >= 0).
struct OutMap {
  int stride;
  int m[3];
  int m2[3];
};
cudaError_t launch_gather_ik(esp_plan* p, double* d_forces, cudaStream_t s,
                             const void* fields = nullptr,
                             OutMap om = OutMap{3, {0, 1, 2}, {-1, -1, -1}});
cudaError_t launch_gather_grad(esp_plan* p, double* d_forces, cudaStream_t s);
// Persistent TMA-fed ik gather from the ghost-padded fields (fp64, P <= 8).
FieldPad make_field_pad(const esp_plan* p);
bool tma_gather_eligible(const esp_plan* p);
cudaError_t make_field_tmap(esp_plan* p);
// Charges with original index in [id_lo, id_hi) only (host-buffer steps
// gather in index ranges to overlap each range's copy-out).
cudaError_t launch_gather_tma(esp_plan* p, double* d_forces, cudaStream_t s, int id_lo = 0,
                              int id_hi = 0x7fffffff);
// Analytic (window-gradient) forces from the ghost-padded potential field
// (fp64), reading the binning pass's weight and derivative-weight records.
cudaError_t launch_gather_grad_tma(esp_plan* p, double* d_forces, cudaStream_t s);
Jac plan_jacobian(const esp_plan* p);
// Fused band-pruned forward transform + scale/reduce (+ ik spectra and the
// inverse transforms into d_fields when want_ik).  Requires p->fused.
cudaError_t launch_fused_fft(esp_plan* p, int want_ik, double* d_out7, cudaStream_t s);
int fused_reduce_blocks(const esp_plan* p);
cudaError_t slab_forward(esp_plan* p, const esp_slab_desc* d, const void* own, cudaStream_t s);
cudaError_t slab_reduce(esp_plan* p, const esp_slab_desc* d, const void* recv, int want_ik,
                        double* d_out7, cudaStream_t s);
cudaError_t slab_inverse(esp_plan* p, const esp_slab_desc* d, const void* recv, void* fields,
                         cudaStream_t s);
void slab_by_split(int nby, int R, int* by_start);
int fused_ldx(const esp_plan* p);
cudaError_t launch_mode_setup(esp_plan* p, double what_zero, cudaStream_t s);
void build_combine_axis(int M, int T, int E, int nt, int lo, std::vector<int>& ent,
                        std::vector<int>& cnt);

void set_error(const std::string& msg);

// Record a profiling event named `name` on stream s (no-op unless enabled).
inline void prof_mark(esp_plan* p, cudaStream_t s, const char* name) {
  if (!p->profiling || p->n_ev >= 48) return;
  cudaEventRecord(p->ev[p->n_ev], s);
  p->ev_name[p->n_ev] = name;
  p->n_ev++;
}

}  // namespace esp

// esp_fft.cu: fused transform state (nullptr when a grid length has a prime
// factor other than 2 or 3, or for slab plans).
void* esp_fused_fft_create(esp_plan* p);
void esp_fused_fft_destroy(void* f);
bool esp_fused_fft_matches(const void* f, const esp_plan* p);   // same in-band box
