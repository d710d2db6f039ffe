// esp_bin.cu — per-step particle binning for the tile kernels.
//
// The reference materialises (N, P^3) flat indices and weights and scatters
// them with np.bincount (mesh.py:193-210).  Here particles are binned once
// per step by anchor cell: key = (ty*ntx + tx)*Mz + az, where (tx, ty) is the
// x-y tile of the anchor column and az its z anchor.  A spread/gather CTA then
// owns a contiguous key range, i.e. its particles sorted by z anchor, which is
// what the sliding-window accumulation needs.
//
// Passes: count (atomic slot per key) -> exclusive scan (CUB) -> scatter ->
// canonicalise (deterministic mode: order inside each key segment by
// original particle index, so every grid sum has a fixed operation order and
// the result is bitwise reproducible run to run).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>

#include "esp_internal.cuh"

namespace esp {

// One dimension of a particle's record (three threads per particle: the
// binning kernels run 96-thread blocks = 32 particles x 3 dimensions, so each
// thread carries one copy of the 8 unrolled Horner chains).  The packed
// anchor is written bytewise: x -> byte 0, y -> byte 1, z -> bytes 2-3.
template <typename real, int P>
__device__ __forceinline__ void record_dim_compute(const Geom& g, const FastTab& ft,
                                                   const real* __restrict__ tab,
                                                   const double* __restrict__ brk,
                                                   int n_pieces, int ncoef, int d, double u,
                                                   real (&w)[P], int& a) {
  const double base = anchor_base(g, u);
  stencil_weights<real, P>(ft, tab, brk, n_pieces, ncoef, u, base, g.lo, real(1), w);
  a = local_anchor(g, d, base);
}

template <typename real, int P>
__device__ __forceinline__ void record_dim_store(const Geom& g, int key, int d,
                                                 const real (&w)[P], int a, long long dst,
                                                 real* __restrict__ wrec,
                                                 int* __restrict__ pk) {
  constexpr int RS = rec_stride(P);
  real* out = wrec + dst * (3 * RS) + d * RS;
#pragma unroll
  for (int s = 0; s < RS; ++s) out[s] = s < P ? w[s < P ? s : 0] : real(0);
  unsigned char* pb = reinterpret_cast<unsigned char*>(pk + dst);
  if (d == 2) {
    *reinterpret_cast<unsigned short*>(pb + 2) = (unsigned short)a;   // absolute z
  } else {
    const int txy = key / g.M[2];
    const int org = d == 0 ? (txy % g.ntx) * g.TX : (txy / g.ntx) * g.TY;
    pb[d] = (unsigned char)(a - org);
  }
}

// Derivative-weight row of one dimension (analytic forces): computed in the
// binning pass when the step needs it, so the gradient gather needs no
// separate pass over the particles.
template <typename real, int P>
__device__ __forceinline__ void drec_dim_store(const Geom& g, const FastTab& ftd,
                                               const real* __restrict__ dtab,
                                               const double* __restrict__ brk, int n_pieces,
                                               int ncoef, int d, double u, long long dst,
                                               real* __restrict__ drec) {
  constexpr int RS = rec_stride(P);
  const double base = anchor_base(g, u);
  real w[P];
  stencil_weights<real, P>(ftd, dtab, brk, n_pieces, ncoef, u, base, g.lo, real(1), w);
  real* out = drec + dst * (3 * RS) + d * RS;
#pragma unroll
  for (int s = 0; s < RS; ++s) out[s] = s < P ? w[s < P ? s : 0] : real(0);
}

template <typename real, int P>
__device__ __forceinline__ void write_record_dim(const Geom& g, const FastTab& ft,
                                                 const real* __restrict__ tab,
                                                 const double* __restrict__ brk,
                                                 int n_pieces, int ncoef, int key, int d,
                                                 double u, long long dst,
                                                 real* __restrict__ wrec,
                                                 int* __restrict__ pk) {
  real w[P];
  int a;
  record_dim_compute<real, P>(g, ft, tab, brk, n_pieces, ncoef, d, u, w, a);
  record_dim_store<real, P>(g, key, d, w, a, dst, wrec, pk);
}

constexpr int kBinPerBlock = 32;   // particles per 96-thread binning block

__global__ void k_bin_count(const double* __restrict__ pos, long long n, Geom g,
                            int* __restrict__ key, int* __restrict__ slot,
                            int* __restrict__ counts) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u[3];
  grid_coords(g, pos[3 * i + 0], pos[3 * i + 1], pos[3 * i + 2], u);
  int a[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    a[d] = local_anchor(g, d, anchor_base(g, u[d]));
  }
  const int tx = a[0] / g.TX, ty = a[1] / g.TY;
  const int k = (ty * g.ntx + tx) * g.M[2] + a[2];
  key[i] = k;
  slot[i] = atomicAdd(&counts[k], 1);
}

// Large-N path: key per particle (histogram for the tile offsets) and the
// identity permutation as sort payload.
__global__ void k_bin_keys(const double* __restrict__ pos, long long n, Geom g,
                           int* __restrict__ key, int* __restrict__ val,
                           int* __restrict__ counts) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u[3];
  grid_coords(g, pos[3 * i + 0], pos[3 * i + 1], pos[3 * i + 2], u);
  int a[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    a[d] = local_anchor(g, d, anchor_base(g, u[d]));
  }
  const int k = ((a[1] / g.TY) * g.ntx + a[0] / g.TX) * g.M[2] + a[2];
  key[i] = k;
  val[i] = (int)i;
  atomicAdd(&counts[k], 1);
}

// After the stable radix sort: gather each particle into its binned slot and
// write its weight record.  Reads are random, writes contiguous per block.
template <typename real, int P, bool DREC>
__global__ void __launch_bounds__(3 * kBinPerBlock)
k_bin_sorted(Geom g, FastTab ft, const real* __restrict__ tab, const double* __restrict__ brk,
             int n_pieces, int ncoef, long long n, long long cap,
             const int* __restrict__ skey, const int* __restrict__ sval,
             const double* __restrict__ pos, const double* __restrict__ q,
             double* __restrict__ u_out, double* __restrict__ q_out,
             int* __restrict__ idx_out, real* __restrict__ wrec, int* __restrict__ pk,
             FastTab ftd, const real* __restrict__ dtab, real* __restrict__ drec) {
  // The block's 32 records (and packed anchors) are assembled in shared
  // memory and written out as one contiguous run.
  constexpr int RS = rec_stride(P);
  __shared__ __align__(16) real s_rec[kBinPerBlock * 3 * RS];
  __shared__ __align__(16) real s_drec[DREC ? kBinPerBlock * 3 * RS : 2];
  __shared__ int s_pk[kBinPerBlock];
  const int d = threadIdx.x / kBinPerBlock, l = threadIdx.x % kBinPerBlock;
  const long long j0 = (long long)blockIdx.x * kBinPerBlock;
  const long long j = j0 + l;
  const int nb = (int)min((long long)kBinPerBlock, n - j0);
  if (l < nb) {
    const int i = sval[j];
    const long long i3 = 3 * (long long)i;
    const double u = grid_coord(g, d, pos[i3], pos[i3 + 1], pos[i3 + 2]);
    u_out[d * cap + j] = u;
    if (d == 0) {
      q_out[j] = q[i];
      idx_out[j] = i;
    }
    real w[P];
    int a;
    record_dim_compute<real, P>(g, ft, tab, brk, n_pieces, ncoef, d, u, w, a);
#pragma unroll
    for (int t = 0; t < RS; ++t) s_rec[(l * 3 + d) * RS + t] = t < P ? w[t < P ? t : 0] : real(0);
    if (DREC) {   // derivative row staged like the weights, written contiguously below
      real dw[P];
      stencil_weights<real, P>(ftd, dtab, brk, n_pieces, ncoef, u, anchor_base(g, u), g.lo,
                               real(1), dw);
#pragma unroll
      for (int t = 0; t < RS; ++t)
        s_drec[(l * 3 + d) * RS + t] = t < P ? dw[t < P ? t : 0] : real(0);
    }
    unsigned char* pb = reinterpret_cast<unsigned char*>(s_pk + l);
    if (d == 2) {
      *reinterpret_cast<unsigned short*>(pb + 2) = (unsigned short)a;   // absolute z
    } else {
      const int txy = skey[j] / g.M[2];
      const int org = d == 0 ? (txy % g.ntx) * g.TX : (txy / g.ntx) * g.TY;
      pb[d] = (unsigned char)(a - org);
    }
  }
  __syncthreads();
  real* dst = wrec + j0 * (3 * RS);
  for (int t = threadIdx.x; t < nb * 3 * RS; t += 3 * kBinPerBlock) dst[t] = s_rec[t];
  for (int t = threadIdx.x; t < nb; t += 3 * kBinPerBlock) pk[j0 + t] = s_pk[t];
  if (DREC) {
    real* ddst = drec + j0 * (3 * RS);
    for (int t = threadIdx.x; t < nb * 3 * RS; t += 3 * kBinPerBlock) ddst[t] = s_drec[t];
  }
}

// Records-free sorted pass (the step's spread and gather evaluate their
// weights from u): gather each particle into its binned slot — grid
// coordinates (SoA), charge and original index, one thread per particle.
__global__ void k_bin_gather(Geom g, long long n, long long cap, const int* __restrict__ sval,
                             const double* __restrict__ pos, const double* __restrict__ q,
                             double* __restrict__ u_out, double* __restrict__ q_out,
                             int* __restrict__ idx_out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int i = sval[j];
  double u[3];
  grid_coords(g, pos[3 * (long long)i], pos[3 * (long long)i + 1], pos[3 * (long long)i + 2], u);
  u_out[j] = u[0];
  u_out[cap + j] = u[1];
  u_out[2 * cap + j] = u[2];
  if (q) q_out[j] = q[i];
  idx_out[j] = i;
}

// Charges into binned order, for steps whose charges arrive late (the
// host-buffer step copies them on a side stream): run after the records pass,
// just before the spread, so the copy hides behind sort, gather and records.
__global__ void k_bin_charges(long long n, const int* __restrict__ idx,
                              const double* __restrict__ q, double* __restrict__ q_out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j < n) q_out[j] = q[idx[j]];
}

// Weight records from the binned grid coordinates (deferred records:
// ensure_records), three threads per particle; key = the sorted bin key.
template <typename real, int P, bool DREC>
__global__ void __launch_bounds__(3 * kBinPerBlock)
k_bin_records_u(Geom g, FastTab ft, const real* __restrict__ tab, const double* __restrict__ brk,
                int n_pieces, int ncoef, long long n, long long cap,
                const int* __restrict__ skey, const double* __restrict__ U,
                real* __restrict__ wrec, int* __restrict__ pk, FastTab ftd,
                const real* __restrict__ dtab, real* __restrict__ drec) {
  // the block's 32 records (and, for analytic steps, derivative records) are
  // assembled in shared memory and written as contiguous runs (coalesced)
  constexpr int RS = rec_stride(P);
  __shared__ __align__(16) real s_rec[kBinPerBlock * 3 * RS];
  __shared__ __align__(16) real s_drec[DREC ? kBinPerBlock * 3 * RS : 2];
  __shared__ int s_pk[kBinPerBlock];
  const int d = threadIdx.x / kBinPerBlock, l = threadIdx.x % kBinPerBlock;
  // grid-stride over 32-charge groups; the next group's coordinate and key
  // are loaded before this group's weights are evaluated (each thread has one
  // load per group: without the prefetch its latency is fully exposed)
  const long long ngroups = (n + kBinPerBlock - 1) / kBinPerBlock;
  double u_next = 0.0;
  int key_next = 0;
  auto prefetch = [&](long long grp) {
    const long long jn = grp * kBinPerBlock + l;
    if (jn < n) {
      u_next = U[d * cap + jn];
      if (d < 2) key_next = skey[jn];
    }
  };
  long long grp = blockIdx.x;
  if (grp < ngroups) prefetch(grp);
  for (; grp < ngroups; grp += gridDim.x) {
    const double u = u_next;
    const int key = key_next;
    if (grp + gridDim.x < ngroups) prefetch(grp + gridDim.x);
    const long long j0 = grp * kBinPerBlock;
    const int nb = (int)min((long long)kBinPerBlock, n - j0);
    if (l < nb) {
      real w[P];
      int a;
      record_dim_compute<real, P>(g, ft, tab, brk, n_pieces, ncoef, d, u, w, a);
#pragma unroll
      for (int t = 0; t < RS; ++t) s_rec[(l * 3 + d) * RS + t] = t < P ? w[t < P ? t : 0] : real(0);
      if (DREC) {
        real dw[P];
        stencil_weights<real, P>(ftd, dtab, brk, n_pieces, ncoef, u, anchor_base(g, u), g.lo,
                                 real(1), dw);
#pragma unroll
        for (int t = 0; t < RS; ++t)
          s_drec[(l * 3 + d) * RS + t] = t < P ? dw[t < P ? t : 0] : real(0);
      }
      unsigned char* pb = reinterpret_cast<unsigned char*>(s_pk + l);
      if (d == 2) {
        *reinterpret_cast<unsigned short*>(pb + 2) = (unsigned short)a;   // absolute z
      } else {
        const int txy = key / g.M[2];
        const int org = d == 0 ? (txy % g.ntx) * g.TX : (txy / g.ntx) * g.TY;
        pb[d] = (unsigned char)(a - org);
      }
    }
    __syncthreads();
    real* dst = wrec + j0 * (3 * RS);
    for (int t = threadIdx.x; t < nb * 3 * RS; t += 3 * kBinPerBlock) dst[t] = s_rec[t];
    for (int t = threadIdx.x; t < nb; t += 3 * kBinPerBlock) pk[j0 + t] = s_pk[t];
    if (DREC) {
      real* ddst = drec + j0 * (3 * RS);
      for (int t = threadIdx.x; t < nb * 3 * RS; t += 3 * kBinPerBlock) ddst[t] = s_drec[t];
    }
    __syncthreads();   // the staging rows are rewritten by the next group
  }
}

// Small key spaces (<= kScanMax keys, e.g. config 1's 4096): every scatter
// CTA scans the key counts in shared memory itself (CTA 0 also publishes the
// offsets), so the separate device-wide scan launch disappears from the step.
constexpr int kScanT = 256;
constexpr int kScanMax = 8192;

__global__ void __launch_bounds__(kScanT)
    k_bin_scatter_scan(const double* __restrict__ pos, const double* __restrict__ q,
                       long long n, Geom g, const int* __restrict__ key,
                       const int* __restrict__ slot, const int* __restrict__ counts, int nk1,
                       int* __restrict__ offsets_out, long long cap,
                       double* __restrict__ u_out, double* __restrict__ q_out,
                       int* __restrict__ idx_out, int* __restrict__ key_out) {
  __shared__ int s_off[kScanMax];
  __shared__ int s_wsum[kScanT / 32];
  const int per = (nk1 + kScanT - 1) / kScanT;
  const int a0 = threadIdx.x * per;
  for (int k = threadIdx.x; k < nk1; k += kScanT) s_off[k] = counts[k];
  __syncthreads();
  int sum = 0;
  for (int k = 0; k < per; ++k)
    if (a0 + k < nk1) sum += s_off[a0 + k];
  // exclusive block scan of the per-thread sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += s_wsum[w];
  int run = wbase + incl - sum;
  for (int k = 0; k < per; ++k) {
    if (a0 + k < nk1) {
      const int c = s_off[a0 + k];
      s_off[a0 + k] = run;
      run += c;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < nk1; k += kScanT) offsets_out[k] = s_off[k];
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u[3];
  grid_coords(g, pos[3 * i + 0], pos[3 * i + 1], pos[3 * i + 2], u);
  const int k = key[i];
  const long long dst = (long long)s_off[k] + slot[i];
  u_out[dst] = u[0];
  u_out[cap + dst] = u[1];
  u_out[2 * cap + dst] = u[2];
  q_out[dst] = q[i];
  idx_out[dst] = (int)i;
  if (key_out) key_out[dst] = k;
}

// Scatter to key segments.  Writes grid coordinates u (SoA), charge and the
// original index.  In deterministic mode the destination is a temporary and
// k_bin_canon fixes the intra-segment order.
__global__ void k_bin_scatter(const double* __restrict__ pos,
                              const double* __restrict__ q, long long n, Geom g,
                              const int* __restrict__ key,
                              const int* __restrict__ slot,
                              const int* __restrict__ offsets, long long cap,
                              double* __restrict__ u_out, double* __restrict__ q_out,
                              int* __restrict__ idx_out, int* __restrict__ key_out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u[3];
  grid_coords(g, pos[3 * i + 0], pos[3 * i + 1], pos[3 * i + 2], u);
  const int k = key[i];
  const long long dst = (long long)offsets[k] + slot[i];
  u_out[dst] = u[0];
  u_out[cap + dst] = u[1];
  u_out[2 * cap + dst] = u[2];
  q_out[dst] = q[i];
  idx_out[dst] = (int)i;
  if (key_out) key_out[dst] = k;
}

// Deterministic order inside each key segment: rank by original index; then
// the particle's record at its final position (3 threads per particle).
template <typename real, int P>
__global__ void __launch_bounds__(3 * kBinPerBlock)
k_bin_canon(Geom g, FastTab ft, const real* __restrict__ tab, const double* __restrict__ brk,
            int n_pieces, int ncoef, long long n, long long cap,
            const int* __restrict__ key_tmp, const int* __restrict__ offsets,
            const double* __restrict__ u_tmp, const double* __restrict__ q_tmp,
            const int* __restrict__ idx_tmp, double* __restrict__ u_out,
            double* __restrict__ q_out, int* __restrict__ idx_out, real* __restrict__ wrec,
            int* __restrict__ pk, FastTab ftd, const real* __restrict__ dtab,
            real* __restrict__ drec) {
  __shared__ long long s_dst[kBinPerBlock];
  __shared__ int s_rank[3][kBinPerBlock];
  const int d = threadIdx.x / kBinPerBlock, l = threadIdx.x % kBinPerBlock;
  const long long j = (long long)blockIdx.x * kBinPerBlock + l;
  const bool live = j < n;
  // rank by original index: the particle's three threads each count a third
  // of its key segment (loads issued in batches of 8), then warp 0 combines
  int s0 = 0;
  int me = 0;
  if (live) {
    const int k = key_tmp[j];
    s0 = offsets[k];
    const int s1 = offsets[k + 1];
    me = idx_tmp[j];
    const int len = s1 - s0, part = (len + 2) / 3;
    const int b0 = s0 + d * part, b1 = min(s1, b0 + part);
    int rank = 0;
    int t = b0;
    for (; t + 8 <= b1; t += 8) {
      int v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = idx_tmp[t + i];
#pragma unroll
      for (int i = 0; i < 8; ++i) rank += (v[i] < me);
    }
    for (; t < b1; ++t) rank += (idx_tmp[t] < me);
    s_rank[d][l] = rank;
  }
  __syncthreads();
  if (d == 0 && live) {
    const long long dst = (long long)s0 + s_rank[0][l] + s_rank[1][l] + s_rank[2][l];
    s_dst[l] = dst;
    q_out[dst] = q_tmp[j];
    idx_out[dst] = me;
  }
  // the record (weights, anchor) does not depend on the rank: warps 1-2 and
  // warp 0 after its rank compute it before the barrier
  double u = 0.0;
  int key = 0, a = 0;
  real w[P];
  if (live) {
    u = u_tmp[d * cap + j];
    key = key_tmp[j];
    record_dim_compute<real, P>(g, ft, tab, brk, n_pieces, ncoef, d, u, w, a);
  }
  __syncthreads();
  if (!live) return;
  const long long dst = s_dst[l];
  u_out[d * cap + dst] = u;
  record_dim_store<real, P>(g, key, d, w, a, dst, wrec, pk);
  if (drec) drec_dim_store<real, P>(g, ftd, dtab, brk, n_pieces, ncoef, d, u, dst, drec);
}

// Non-deterministic mode: records straight after the atomic-slot scatter.
template <typename real, int P>
__global__ void __launch_bounds__(3 * kBinPerBlock)
k_bin_records(Geom g, FastTab ft, const real* __restrict__ tab, const double* __restrict__ brk,
              int n_pieces, int ncoef, long long n, long long cap,
              const int* __restrict__ key, const int* __restrict__ slot,
              const int* __restrict__ offsets, const double* __restrict__ u_in,
              real* __restrict__ wrec, int* __restrict__ pk) {
  const int d = threadIdx.x / kBinPerBlock;
  const long long i = (long long)blockIdx.x * kBinPerBlock + (threadIdx.x % kBinPerBlock);
  if (i >= n) return;
  const int k = key[i];
  const long long dst = (long long)offsets[k] + slot[i];
  write_record_dim<real, P>(g, ft, tab, brk, n_pieces, ncoef, k, d, u_in[d * cap + dst], dst,
                            wrec, pk);
}

template <typename real, int P>
static void launch_tail(esp_plan* p, const Geom& g, long long n, unsigned grid, int B,
                        cudaStream_t s) {
  const real* tab = std::is_same<real, double>::value
                        ? reinterpret_cast<const real*>(p->d_tab)
                        : reinterpret_cast<const real*>(p->d_tabf);
  real* wrec = reinterpret_cast<real*>(p->d_wrec);
  const real* dtab = std::is_same<real, double>::value
                         ? reinterpret_cast<const real*>(p->d_dtab)
                         : reinterpret_cast<const real*>(p->d_dtabf);
  // derivative records in the same pass when the step's forces are analytic
  real* drec = p->want_drec && p->deterministic && P <= 8 && p->h_fast_d->enabled
                   ? reinterpret_cast<real*>(p->d_drec)
                   : nullptr;
  p->drec_ready = drec != nullptr;
  const unsigned g3 = (unsigned)((n + kBinPerBlock - 1) / kBinPerBlock);
  if (p->deterministic) {
    k_bin_canon<real, P><<<g3, 3 * kBinPerBlock, 0, s>>>(g, *p->h_fast, tab, p->d_breaks, p->n_pieces,
                                           p->ncoef, n, p->cap, p->d_bkey, p->d_offsets,
                                           p->d_u_tmp, p->d_q_tmp, p->d_idx_tmp, p->d_u,
                                           p->d_q, p->d_idx, wrec, p->d_pk, *p->h_fast_d, dtab,
                                           drec);
  } else {
    k_bin_records<real, P><<<g3, 3 * kBinPerBlock, 0, s>>>(g, *p->h_fast, tab, p->d_breaks, p->n_pieces,
                                             p->ncoef, n, p->cap, p->d_key, p->d_slot,
                                             p->d_offsets, p->d_u, wrec, p->d_pk);
  }
}

template <typename real>
static cudaError_t launch_tail_r(esp_plan* p, const Geom& g, long long n, unsigned grid,
                                 int B, cudaStream_t s) {
  switch (p->P) {
    case 2: launch_tail<real, 2>(p, g, n, grid, B, s); break;
    case 3: launch_tail<real, 3>(p, g, n, grid, B, s); break;
    case 4: launch_tail<real, 4>(p, g, n, grid, B, s); break;
    case 5: launch_tail<real, 5>(p, g, n, grid, B, s); break;
    case 6: launch_tail<real, 6>(p, g, n, grid, B, s); break;
    case 7: launch_tail<real, 7>(p, g, n, grid, B, s); break;
    case 8: launch_tail<real, 8>(p, g, n, grid, B, s); break;
    case 9: launch_tail<real, 9>(p, g, n, grid, B, s); break;
    case 10: launch_tail<real, 10>(p, g, n, grid, B, s); break;
    case 11: launch_tail<real, 11>(p, g, n, grid, B, s); break;
    case 12: launch_tail<real, 12>(p, g, n, grid, B, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <typename real, int P>
static void launch_sorted(esp_plan* p, const Geom& g, const double* d_pos, const double* d_q,
                          long long n, unsigned grid, int B, cudaStream_t s) {
  const real* tab = std::is_same<real, double>::value
                        ? reinterpret_cast<const real*>(p->d_tab)
                        : reinterpret_cast<const real*>(p->d_tabf);
  const real* dtab = std::is_same<real, double>::value
                         ? reinterpret_cast<const real*>(p->d_dtab)
                         : reinterpret_cast<const real*>(p->d_dtabf);
  real* drec = p->want_drec && P <= 8 && p->h_fast_d->enabled
                   ? reinterpret_cast<real*>(p->d_drec)
                   : nullptr;
  p->drec_ready = drec != nullptr;
  const unsigned g3 = (unsigned)((n + kBinPerBlock - 1) / kBinPerBlock);
  if (drec)
    k_bin_sorted<real, P, true><<<g3, 3 * kBinPerBlock, 0, s>>>(
        g, *p->h_fast, tab, p->d_breaks, p->n_pieces, p->ncoef, n, p->cap, p->d_bkey,
        p->d_idx_tmp, d_pos, d_q, p->d_u, p->d_q, p->d_idx, reinterpret_cast<real*>(p->d_wrec),
        p->d_pk, *p->h_fast_d, dtab, drec);
  else
    k_bin_sorted<real, P, false><<<g3, 3 * kBinPerBlock, 0, s>>>(
        g, *p->h_fast, tab, p->d_breaks, p->n_pieces, p->ncoef, n, p->cap, p->d_bkey,
        p->d_idx_tmp, d_pos, d_q, p->d_u, p->d_q, p->d_idx, reinterpret_cast<real*>(p->d_wrec),
        p->d_pk, *p->h_fast_d, dtab, nullptr);
}

template <typename real>
static cudaError_t launch_sorted_r(esp_plan* p, const Geom& g, const double* d_pos,
                                   const double* d_q, long long n, unsigned grid, int B,
                                   cudaStream_t s) {
  switch (p->P) {
    case 2: launch_sorted<real, 2>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 3: launch_sorted<real, 3>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 4: launch_sorted<real, 4>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 5: launch_sorted<real, 5>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 6: launch_sorted<real, 6>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 7: launch_sorted<real, 7>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 8: launch_sorted<real, 8>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 9: launch_sorted<real, 9>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 10: launch_sorted<real, 10>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 11: launch_sorted<real, 11>(p, g, d_pos, d_q, n, grid, B, s); break;
    case 12: launch_sorted<real, 12>(p, g, d_pos, d_q, n, grid, B, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int key_bits(long long n_keys) {
  int b = 1;
  while ((1ll << b) < n_keys) ++b;
  return b;
}

size_t sort_temp_bytes(long long cap, long long n_keys) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int*)nullptr, (int*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, (int)cap, 0,
                                  key_bits(n_keys));
  return bytes;
}

cudaError_t launch_bin(esp_plan* p, const double* d_pos, const double* d_q,
                       long long n, cudaStream_t s) {
  Geom g = make_geom(p);
  cudaError_t e = cudaMemsetAsync(p->d_counts, 0, sizeof(int) * (p->n_keys + 1), s);
  if (e != cudaSuccess) return e;
  const int B = 256;
  const unsigned grid = (unsigned)((n + B - 1) / B);
  if (n >= p->sort_threshold && p->d_sort_tmp) {
    // stable LSD radix sort of (key, index): deterministic intra-key order
    k_bin_keys<<<grid, B, 0, s>>>(d_pos, n, g, p->d_key, p->d_slot, p->d_counts);
    p->launches++;
    prof_mark(p, s, "bin_keys");
    size_t bytes = p->cub_bytes;
    e = cub::DeviceScan::ExclusiveSum(p->d_cub, bytes, p->d_counts, p->d_offsets,
                                      (int)(p->n_keys + 1), s);
    if (e != cudaSuccess) return e;
    p->launches++;
    size_t sbytes = p->sort_bytes;
    e = cub::DeviceRadixSort::SortPairs(p->d_sort_tmp, sbytes, p->d_key, p->d_bkey, p->d_slot,
                                        p->d_idx_tmp, (int)n, 0, key_bits(p->n_keys), s);
    if (e != cudaSuccess) return e;
    p->launches += 3;
    prof_mark(p, s, "bin_sort");
    p->q_deferred = nullptr;
    if (p->q_ready && !p->need_records) {
      // charges still in flight on another stream (host-buffer step): bin
      // them after the records pass (ensure_records), not here
      p->q_deferred = d_q;
      p->q_deferred_ev = p->q_ready;
      p->q_ready = nullptr;
    } else if (p->q_ready) {
      e = cudaStreamWaitEvent(s, p->q_ready, 0);
      p->q_ready = nullptr;
      if (e != cudaSuccess) return e;
    }
    if (p->need_records) {
      e = p->precision == ESP_FP64 ? launch_sorted_r<double>(p, g, d_pos, d_q, n, grid, B, s)
                                   : launch_sorted_r<float>(p, g, d_pos, d_q, n, grid, B, s);
      p->records_ready = 1;
    } else {
      k_bin_gather<<<grid, B, 0, s>>>(g, n, p->cap, p->d_idx_tmp, d_pos,
                                      p->q_deferred ? nullptr : d_q, p->d_u, p->d_q, p->d_idx);
      e = cudaGetLastError();
      p->records_ready = 0;
      p->drec_ready = 0;
    }
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, p->records_ready ? "bin_gather_weights" : "bin_gather");
    return cudaGetLastError();
  }
  if (n > 0) {
    k_bin_count<<<grid, B, 0, s>>>(d_pos, n, g, p->d_key, p->d_slot, p->d_counts);
    p->launches++;
    prof_mark(p, s, "bin_count");
  }
  static const bool no_fuse_scan = std::getenv("ESP_BIN_NO_FUSED_SCAN") != nullptr;
  const bool fused_scan = n > 0 && p->deterministic && !no_fuse_scan &&
                          p->n_keys + 1 <= kScanMax && B == kScanT;
  if (!fused_scan) {
    size_t bytes = p->cub_bytes;
    e = cub::DeviceScan::ExclusiveSum(p->d_cub, bytes, p->d_counts, p->d_offsets,
                                      (int)(p->n_keys + 1), s);
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "bin_scan");
  }
  if (n == 0) return cudaGetLastError();
  if (p->q_ready) {  // charges copied on another stream (host-buffer step)
    e = cudaStreamWaitEvent(s, p->q_ready, 0);
    p->q_ready = nullptr;
    if (e != cudaSuccess) return e;
  }
  if (fused_scan) {
    k_bin_scatter_scan<<<grid, kScanT, 0, s>>>(d_pos, d_q, n, g, p->d_key, p->d_slot,
                                               p->d_counts, (int)(p->n_keys + 1),
                                               p->d_offsets, p->cap, p->d_u_tmp, p->d_q_tmp,
                                               p->d_idx_tmp, p->d_bkey);
    prof_mark(p, s, "bin_scatter");
    p->launches += 1;
  } else if (p->deterministic) {
    k_bin_scatter<<<grid, B, 0, s>>>(d_pos, d_q, n, g, p->d_key, p->d_slot,
                                     p->d_offsets, p->cap, p->d_u_tmp, p->d_q_tmp,
                                     p->d_idx_tmp, p->d_bkey);
    prof_mark(p, s, "bin_scatter");
    p->launches += 1;
  } else {
    k_bin_scatter<<<grid, B, 0, s>>>(d_pos, d_q, n, g, p->d_key, p->d_slot,
                                     p->d_offsets, p->cap, p->d_u, p->d_q, p->d_idx,
                                     nullptr);
    p->launches++;
    prof_mark(p, s, "bin_scatter");
  }
  e = p->precision == ESP_FP64 ? launch_tail_r<double>(p, g, n, grid, B, s)
                               : launch_tail_r<float>(p, g, n, grid, B, s);
  if (e != cudaSuccess) return e;
  p->records_ready = 1;
  p->launches++;
  prof_mark(p, s, p->deterministic ? "bin_canon_weights" : "bin_weights");
  return cudaGetLastError();
}

template <typename real, int P>
static cudaError_t records_p(esp_plan* p, cudaStream_t s) {
  const Geom g = make_geom(p);
  const real* tab = std::is_same<real, double>::value
                        ? reinterpret_cast<const real*>(p->d_tab)
                        : reinterpret_cast<const real*>(p->d_tabf);
  // grid-stride groups: a few waves of CTAs, so every thread prefetches
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long ngroups = (p->last_n + kBinPerBlock - 1) / kBinPerBlock;
  const unsigned g3 = (unsigned)std::max<long long>(1, std::min<long long>(ngroups, (long long)nsm * 64));
  const real* dtab = std::is_same<real, double>::value
                         ? reinterpret_cast<const real*>(p->d_dtab)
                         : reinterpret_cast<const real*>(p->d_dtabf);
  // derivative records too when the step's forces are analytic
  const bool drec = p->want_drec && P <= 8 && p->h_fast_d->enabled;
  if (drec)
    k_bin_records_u<real, P, true><<<g3, 3 * kBinPerBlock, 0, s>>>(
        g, *p->h_fast, tab, p->d_breaks, p->n_pieces, p->ncoef, p->last_n, p->cap, p->d_bkey,
        p->d_u, reinterpret_cast<real*>(p->d_wrec), p->d_pk, *p->h_fast_d, dtab,
        reinterpret_cast<real*>(p->d_drec));
  else
    k_bin_records_u<real, P, false><<<g3, 3 * kBinPerBlock, 0, s>>>(
        g, *p->h_fast, tab, p->d_breaks, p->n_pieces, p->ncoef, p->last_n, p->cap, p->d_bkey,
        p->d_u, reinterpret_cast<real*>(p->d_wrec), p->d_pk, *p->h_fast_d, dtab, nullptr);
  p->drec_ready = drec;
  p->launches++;
  prof_mark(p, s, "bin_records");
  return cudaGetLastError();
}

template <typename real>
static cudaError_t records_r(esp_plan* p, cudaStream_t s) {
  switch (p->P) {
    case 2: return records_p<real, 2>(p, s);
    case 3: return records_p<real, 3>(p, s);
    case 4: return records_p<real, 4>(p, s);
    case 5: return records_p<real, 5>(p, s);
    case 6: return records_p<real, 6>(p, s);
    case 7: return records_p<real, 7>(p, s);
    case 8: return records_p<real, 8>(p, s);
    case 9: return records_p<real, 9>(p, s);
    case 10: return records_p<real, 10>(p, s);
    case 11: return records_p<real, 11>(p, s);
    case 12: return records_p<real, 12>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t ensure_records(esp_plan* p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (!p->records_ready && p->last_n > 0) {
    e = p->precision == ESP_FP64 ? records_r<double>(p, s) : records_r<float>(p, s);
    if (e == cudaSuccess) p->records_ready = 1;
  }
  if (e == cudaSuccess && p->q_deferred) {
    // late charges (launch_bin): wait for their copy, then bin them
    const double* q = p->q_deferred;
    p->q_deferred = nullptr;
    e = cudaStreamWaitEvent(s, p->q_deferred_ev, 0);
    if (e != cudaSuccess) return e;
    if (p->last_n > 0) {
      const int B = 256;
      k_bin_charges<<<(unsigned)((p->last_n + B - 1) / B), B, 0, s>>>(p->last_n, p->d_idx, q,
                                                                      p->d_q);
      p->launches++;
      prof_mark(p, s, "bin_charges");
      e = cudaGetLastError();
    }
  }
  return e;
}

size_t scan_temp_bytes(long long n_items) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int*)nullptr, (int*)nullptr,
                                (int)n_items);
  return bytes;
}

}  // namespace esp
