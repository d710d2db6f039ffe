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

#include "esp_internal.cuh"

namespace esp {

// Window weights and tile-local anchors of one binned particle, written once
// per step and read by both the spread and the gather kernels.
template <typename real, int P>
__device__ __forceinline__ void write_record(const Geom& g, const FastTab& ft,
                                             const real* __restrict__ tab,
                                             const double* __restrict__ brk,
                                             int n_pieces, int ncoef, int key,
                                             const double u[3], long long dst,
                                             real* __restrict__ wrec,
                                             int* __restrict__ pk) {
  const int az = key % g.M[2];
  const int txy = key / g.M[2];
  // x, y relative to the tile; z absolute (spread and gather tiles differ in z)
  const int org[3] = {(txy % g.ntx) * g.TX, (txy / g.ntx) * g.TY, 0};
  constexpr int RS = rec_stride(P);
  real* out = wrec + dst * (3 * RS);
  int packed = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double base = anchor_base(g, u[d]);
    const int a = local_anchor(g, d, base);
    packed |= (a - org[d]) << (8 * d);
    real w[P];
    stencil_weights<real, P>(ft, tab, brk, n_pieces, ncoef, u[d], base, g.lo, real(1), w);
#pragma unroll
    for (int s = 0; s < RS; ++s) out[d * RS + s] = s < P ? w[s < P ? s : 0] : real(0);
  }
  pk[dst] = packed;
}

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
    double b = anchor_base(g, u[d]);
    // Clamp pathological (non-finite / huge) coordinates into range; the
    // reference's int64 cast would be undefined there as well.
    b = fmin(fmax(b, -4.0e15), 4.0e15);
    a[d] = local_anchor(g, d, b);
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
    double b = anchor_base(g, u[d]);
    b = fmin(fmax(b, -4.0e15), 4.0e15);
    a[d] = local_anchor(g, d, b);
  }
  const int k = ((a[1] / g.TY) * g.ntx + a[0] / g.TX) * g.M[2] + a[2];
  key[i] = k;
  val[i] = (int)i;
  atomicAdd(&counts[k], 1);
}

// After the stable radix sort: gather each particle into its binned slot and
// write its weight record.  Reads are random, writes coalesced.
template <typename real, int P>
__global__ void k_bin_sorted(Geom g, FastTab ft, const real* __restrict__ tab,
                             const double* __restrict__ brk, int n_pieces, int ncoef,
                             long long n, long long cap, const int* __restrict__ skey,
                             const int* __restrict__ sval, const double* __restrict__ pos,
                             const double* __restrict__ q, double* __restrict__ u_out,
                             double* __restrict__ q_out, int* __restrict__ idx_out,
                             real* __restrict__ wrec, int* __restrict__ pk) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int i = sval[j];
  double u[3];
  grid_coords(g, pos[3 * (long long)i + 0], pos[3 * (long long)i + 1],
              pos[3 * (long long)i + 2], u);
  u_out[j] = u[0];
  u_out[cap + j] = u[1];
  u_out[2 * cap + j] = u[2];
  q_out[j] = q[i];
  idx_out[j] = i;
  write_record<real, P>(g, ft, tab, brk, n_pieces, ncoef, skey[j], u, j, wrec, pk);
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
// the particle's weight record at its final position.
template <typename real, int P>
__global__ void k_bin_canon(Geom g, FastTab ft, const real* __restrict__ tab,
                            const double* __restrict__ brk, int n_pieces, int ncoef,
                            long long n, long long cap,
                            const int* __restrict__ key_tmp,
                            const int* __restrict__ offsets,
                            const double* __restrict__ u_tmp,
                            const double* __restrict__ q_tmp,
                            const int* __restrict__ idx_tmp,
                            double* __restrict__ u_out, double* __restrict__ q_out,
                            int* __restrict__ idx_out, real* __restrict__ wrec,
                            int* __restrict__ pk) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int k = key_tmp[j];
  const int s0 = offsets[k], s1 = offsets[k + 1];
  const int me = idx_tmp[j];
  int rank = 0;
  for (int t = s0; t < s1; ++t) rank += (idx_tmp[t] < me);
  const long long dst = (long long)s0 + rank;
  const double u[3] = {u_tmp[j], u_tmp[cap + j], u_tmp[2 * cap + j]};
  u_out[dst] = u[0];
  u_out[cap + dst] = u[1];
  u_out[2 * cap + dst] = u[2];
  q_out[dst] = q_tmp[j];
  idx_out[dst] = me;
  write_record<real, P>(g, ft, tab, brk, n_pieces, ncoef, k, u, dst, wrec, pk);
}

// Non-deterministic mode: records straight after the atomic-slot scatter.
template <typename real, int P>
__global__ void k_bin_records(Geom g, FastTab ft, const real* __restrict__ tab,
                              const double* __restrict__ brk, int n_pieces, int ncoef,
                              long long n, long long cap, const int* __restrict__ key,
                              const int* __restrict__ slot, const int* __restrict__ offsets,
                              const double* __restrict__ u_in, real* __restrict__ wrec,
                              int* __restrict__ pk) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = key[i];
  const long long dst = (long long)offsets[k] + slot[i];
  const double u[3] = {u_in[dst], u_in[cap + dst], u_in[2 * cap + dst]};
  write_record<real, P>(g, ft, tab, brk, n_pieces, ncoef, k, u, dst, wrec, pk);
}

template <typename real, int P>
static void launch_tail(esp_plan* p, const Geom& g, long long n, unsigned grid, int B,
                        cudaStream_t s) {
  const real* tab = std::is_same<real, double>::value
                        ? reinterpret_cast<const real*>(p->d_tab)
                        : reinterpret_cast<const real*>(p->d_tabf);
  real* wrec = reinterpret_cast<real*>(p->d_wrec);
  if (p->deterministic) {
    k_bin_canon<real, P><<<grid, B, 0, s>>>(g, *p->h_fast, tab, p->d_breaks, p->n_pieces,
                                           p->ncoef, n, p->cap, p->d_bkey, p->d_offsets,
                                           p->d_u_tmp, p->d_q_tmp, p->d_idx_tmp, p->d_u,
                                           p->d_q, p->d_idx, wrec, p->d_pk);
  } else {
    k_bin_records<real, P><<<grid, B, 0, s>>>(g, *p->h_fast, tab, p->d_breaks, p->n_pieces,
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
  k_bin_sorted<real, P><<<grid, B, 0, s>>>(g, *p->h_fast, tab, p->d_breaks, p->n_pieces,
                                          p->ncoef, n, p->cap, p->d_bkey, p->d_idx_tmp, d_pos,
                                          d_q, p->d_u, p->d_q, p->d_idx,
                                          reinterpret_cast<real*>(p->d_wrec), p->d_pk);
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
  if (n >= kSortThreshold && p->d_sort_tmp) {
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
    e = p->precision == ESP_FP64 ? launch_sorted_r<double>(p, g, d_pos, d_q, n, grid, B, s)
                                 : launch_sorted_r<float>(p, g, d_pos, d_q, n, grid, B, s);
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "bin_gather_weights");
    return cudaGetLastError();
  }
  if (n > 0) {
    k_bin_count<<<grid, B, 0, s>>>(d_pos, n, g, p->d_key, p->d_slot, p->d_counts);
    p->launches++;
    prof_mark(p, s, "bin_count");
  }
  size_t bytes = p->cub_bytes;
  e = cub::DeviceScan::ExclusiveSum(p->d_cub, bytes, p->d_counts, p->d_offsets,
                                    (int)(p->n_keys + 1), s);
  if (e != cudaSuccess) return e;
  p->launches++;
  prof_mark(p, s, "bin_scan");
  if (n == 0) return cudaGetLastError();
  if (p->deterministic) {
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
  p->launches++;
  prof_mark(p, s, p->deterministic ? "bin_canon_weights" : "bin_weights");
  return cudaGetLastError();
}

size_t scan_temp_bytes(long long n_items) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int*)nullptr, (int*)nullptr,
                                (int)n_items);
  return bytes;
}

}  // namespace esp
