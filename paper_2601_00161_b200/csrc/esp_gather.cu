// esp_gather.cu — force interpolation (mesh.py:213-218 `_gather`, used by
// long_range_forces ik mode, mesh.py:336-342).
//
// k_gather_warp (P <= 8, the production path): CTA = one anchor tile (the
// spread's decomposition).  The CTA stages the padded field tile — the three
// ik fields on 16 x 16 columns x PZ planes — in shared memory once; a warp
// then handles 2 particles at a time, lane (p, h, k) summing the rows of
// parity h of particle p's stencil plane k (x rows at immediate offsets),
// and the 16 lanes of a particle reduce with 4 xor-shuffle levels.  Odd
// plane strides keep every LDS phase bank-conflict free; weight records
// arrive through a per-warp cp.async ring.  Each particle is owned by one
// lane group: no atomics, fixed reduction order, bitwise reproducible.
//
// k_gather_ik (P > 8): column-owner variant — each thread holds a P-deep
// sliding window of the three fields of one padded column in registers and
// warps reduce per-particle partials.
//
// F_c = -q * sum (the h3 factors of mesh.py:341-342 cancel; the 1/G of the
// inverse transform is folded into the spectrum).
#include "esp_internal.cuh"

namespace esp {

// Asynchronous global -> shared copy of one real (cp.async, 4 or 8 bytes):
// the field-tile staging issues every plane's loads without waiting on any.
template <typename real>
__device__ __forceinline__ void cp_async_real(real* dst_smem, const real* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  if (sizeof(real) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src));
}

template <typename real, int P>
__device__ __forceinline__ void stage_weights_g(
    const Geom& g, const real* s_tab, const double* s_brk, int n_pieces, int ncoef,
    const double* __restrict__ U, long long cap, long long c0, int n, int tx, int ty,
    int tz, real* s_w, int* s_anc) {
  for (int item = threadIdx.x; item < 3 * n; item += blockDim.x) {
    const int pl = item / 3, d = item - 3 * (item / 3);
    const double u = U[d * cap + c0 + pl];
    const double base = anchor_base(g, u);
    const int a = local_anchor(g, d, base);
    const int org = d == 0 ? tx * g.TX : (d == 1 ? ty * g.TY : tz * g.TZ);
    s_anc[d * kChunk + pl] = a - org;
    real* w = s_w + ((size_t)d * kChunk + pl) * P;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const double t = u - (base + (double)(g.lo + s));
      w[s] = window_eval<real>(s_tab, s_brk, n_pieces, ncoef, t);
    }
  }
}

// Sum (v0, v1, v2) over the 32 lanes.  Afterwards lane 0 holds comp 0, lane 8
// comp 1, lane 16 comp 2.
template <typename real>
__device__ __forceinline__ real warp_reduce3(real v0, real v1, real v2, int lane) {
  const unsigned full = 0xffffffffu;
  const real v3 = real(0);
  const bool hi = lane & 16;
  real r0 = __shfl_xor_sync(full, hi ? v0 : v2, 16);
  real r1 = __shfl_xor_sync(full, hi ? v1 : v3, 16);
  real k0 = (hi ? v2 : v0) + r0;
  real k1 = (hi ? v3 : v1) + r1;
  const bool b3 = lane & 8;
  real r = __shfl_xor_sync(full, b3 ? k0 : k1, 8);
  real k = (b3 ? k1 : k0) + r;
  k += __shfl_xor_sync(full, k, 4);
  k += __shfl_xor_sync(full, k, 2);
  k += __shfl_xor_sync(full, k, 1);
  return k;
}


template <typename real> struct Vec16;
template <> struct Vec16<double> {
  using type = double2;
  __device__ static void split(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
};
template <> struct Vec16<float> {
  using type = float4;
  __device__ static void split(const float4& v, float* o) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
};

template <typename real> struct Real2;
template <> struct Real2<double> { using type = double2; };
template <> struct Real2<float> { using type = float2; };

template <typename real, int P>
struct GatherLayout {
  // (f_x, f_y) pairs: rows of 16, plane stride 257 (odd): the 8 planes read by
  // one LDS.128 phase fall in 8 distinct bank groups.
  static constexpr int kPlane = kPad * kPad + 1;
  // f_z: rows of 24 (= 8 mod 16), plane stride 385 (= 1 mod 16): the 16 lanes
  // of one LDS.64 phase (8 planes x 2 adjacent rows) hit 16 distinct banks.
  static constexpr int kRowZ = 24;
  static constexpr int kPlaneZ = kPad * kRowZ + 1;
  static constexpr int kRing = (kTileThreads / 32) * 2 * 2 * 3 * rec_stride(P);  // warps x bufs x pair
  __host__ __device__ static size_t fields_bytes(int PZ) {
    size_t b = 2 * sizeof(real) * (size_t)PZ * kPlane;   // (f_x, f_y) pairs
    b = (b + 15) & ~size_t(15);
    b += sizeof(real) * (size_t)PZ * kPlaneZ;           // f_z
    return (b + 15) & ~size_t(15);
  }
  static size_t bytes(int PZ) { return fields_bytes(PZ) + sizeof(real) * (size_t)kRing; }
};

// Warp = 2 particles x 8 stencil planes x 2 row parities.  Lane (p, h, k)
// sums rows j = h, h+2, .. of particle p's stencil on plane zl+k (x contiguous,
// immediate smem offsets), weights by wz[k], and the 16 lanes of a particle
// reduce with 4 xor-shuffle levels.  Weights and anchors come from the
// per-particle records of the binning pass; the field tile is the only
// shared-memory data.  Strides make every LDS phase bank-conflict free.
template <typename real, int P>
__global__ void __launch_bounds__(kTileThreads, 2)
k_gather_warp(Geom g, const int* __restrict__ offsets, const real* __restrict__ wrec,
              const int* __restrict__ PK, const double* __restrict__ Q,
              const int* __restrict__ IDX, const real* __restrict__ fld, long long G,
              double* __restrict__ forces, OutMap om) {
  static_assert(P <= 8, "warp gather covers at most 8 stencil planes");
  using R2 = typename Real2<real>::type;
  constexpr int kPlane = GatherLayout<real, P>::kPlane;
  constexpr int kRowZ = GatherLayout<real, P>::kRowZ;
  constexpr int kPlaneZ = GatherLayout<real, P>::kPlaneZ;
  constexpr int RS = rec_stride(P);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // z-slab-major tile order: CTAs running together cover one slab of tiles,
  // whose halo planes (3 fields x PZ planes x the whole x-y plane) stay in L2
  const int nxy = g.ntx * g.nty;
  const int tz = blockIdx.x / nxy;
  const int txy = blockIdx.x - tz * nxy;
  const int tx = txy % g.ntx, ty = txy / g.ntx;
  const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
  const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
  const long long p0 = offsets[key0], p1 = offsets[key1];
  if (p0 == p1) return;

  R2* s_f01 = reinterpret_cast<R2*>(smem_raw);
  size_t off = 2 * sizeof(real) * (size_t)g.PZ * kPlane;
  off = (off + 15) & ~size_t(15);
  real* s_f2 = reinterpret_cast<real*>(smem_raw + off);

  // Stage the padded field tile.  blockDim == 256 == one 16x16 plane, so
  // each thread owns one (x, y) column: wrap it once, then walk the planes.
  {
    const real* f0 = fld;
    const real* f1 = fld + G;
    const real* f2 = fld + 2 * G;
    const long long Mxy = (long long)g.M[0] * g.M[1];
    const int r = threadIdx.x;
    const int gx = wrap_near(tx * g.TX + g.lo + (r & 15), g.M[0]);
    const int gy = wrap_near(ty * g.TY + g.lo + (r >> 4), g.M[1]);
    const long long col = (long long)gy * g.M[0] + gx;
    int gz = wrap_near(tz * g.TZ + g.lo, g.M[2]);
    for (int pz = 0; pz < g.PZ; ++pz) {
      const long long o = gz * Mxy + col;
      real* d01 = reinterpret_cast<real*>(s_f01 + pz * kPlane + r);
      cp_async_real(d01, f0 + o);
      cp_async_real(d01 + 1, f1 + o);
      cp_async_real(s_f2 + pz * kPlaneZ + (r >> 4) * kRowZ + (r & 15), f2 + o);
      gz = gz + 1 == g.M[2] ? 0 : gz + 1;
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 4, h = (lane >> 3) & 1, k = lane & 7;
  constexpr int kStep = (kTileThreads / 32) * 2;
  constexpr int kRec = 3 * RS;                              // reals per record
  constexpr int kChunks = (2 * kRec * (int)sizeof(real)) / 16;   // 16 B pieces per pair
  real* ring = reinterpret_cast<real*>(smem_raw + GatherLayout<real, P>::fields_bytes(g.PZ)) +
               (size_t)warp * 2 * 2 * kRec;
  // Records of particle pair `pb` -> ring buffer `b` (cp.async, 16 B pieces).
  auto fetch = [&](long long pb, int b) {
    if (lane < kChunks) {
      const long long first = pb;
      const int avail = (int)min((long long)2, p1 - first);
      const int bytes_needed = avail * kRec * (int)sizeof(real);
      if (lane * 16 < bytes_needed) {
        const char* src = reinterpret_cast<const char*>(wrec + first * kRec) + lane * 16;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(
            reinterpret_cast<char*>(ring + (size_t)b * 2 * kRec) + lane * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  long long pb = p0 + warp * 2;
  int buf = 0;
  if (pb < p1) fetch(pb, 0);
  int pk_n = 0;
  double q_n = 0.0;
  int id_n = 0;
  if (pb + slot < p1) {
    pk_n = PK[pb + slot];
    q_n = Q[pb + slot];
    id_n = IDX[pb + slot];
  }
  for (; pb < p1; pb += kStep, buf ^= 1) {
    const long long pl = pb + slot;
    const bool live = pl < p1 && k < P;
    const int pk_c = pk_n;
    const double q_c = q_n;
    const int id_c = id_n;
    const long long nx = pb + kStep;
    if (nx < p1) {
      fetch(nx, buf ^ 1);
      if (nx + slot < p1) {          // scalars of the next pair, consumed next iteration
        pk_n = PK[nx + slot];
        q_n = Q[nx + slot];
        id_n = IDX[nx + slot];
      }
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncwarp();
    real ax = 0, ay = 0, az = 0;
    if (live) {
      const int pk = pk_c;
      const int xl = pk & 0xff, yl = (pk >> 8) & 0xff, zl = (pk >> 16) - tz * g.TZ;
      const real* W = ring + ((size_t)buf * 2 + slot) * kRec;
      real wx[RS], wy[RS];
      // 16-byte loads of the x and y weight rows (records are 16 B aligned)
      using V = typename Vec16<real>::type;
      constexpr int kPer = 16 / (int)sizeof(real);
#pragma unroll
      for (int c = 0; c < RS / kPer; ++c) {
        const V a = reinterpret_cast<const V*>(W)[c];
        const V b = reinterpret_cast<const V*>(W + RS)[c];
        Vec16<real>::split(a, wx + c * kPer);
        Vec16<real>::split(b, wy + c * kPer);
      }
      const real wzk = W[2 * RS + k];
      const R2* rowp = s_f01 + (zl + k) * kPlane + (yl + h) * kPad + xl;
      const real* rowz = s_f2 + (zl + k) * kPlaneZ + (yl + h) * kRowZ + xl;
#pragma unroll
      for (int jj = 0; jj < (P + 1) / 2; ++jj) {
        const int j = 2 * jj;                 // row j + h of the stencil
        const bool odd_row = j + 1 < P;       // compile-time after unrolling
        if (odd_row || h == 0) {
          const real wy_ = (odd_row && h) ? wy[odd_row ? j + 1 : j] : wy[j];
          real rx = 0, ry = 0, rz = 0;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const R2 v = rowp[j * kPad + i];
            const real vz = rowz[j * kRowZ + i];
            rx = fma(wx[i], v.x, rx);
            ry = fma(wx[i], v.y, ry);
            rz = fma(wx[i], vz, rz);
          }
          ax = fma(wy_, rx, ax);
          ay = fma(wy_, ry, ay);
          az = fma(wy_, rz, az);
        }
      }
      ax *= wzk;
      ay *= wzk;
      az *= wzk;
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      ax += __shfl_xor_sync(0xffffffffu, ax, o);
      ay += __shfl_xor_sync(0xffffffffu, ay, o);
      az += __shfl_xor_sync(0xffffffffu, az, o);
    }
    __syncwarp();   // the ring slot is refilled two iterations later
    if ((lane & 15) == 0 && pl < p1) {
      const double q = q_c;
      double* f = forces + (long long)id_c * om.stride;
      const double v[3] = {-q * (double)ax, -q * (double)ay, -q * (double)az};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        f[om.m[c]] = v[c];
        if (om.m2[c] >= 0) f[om.m2[c]] = v[c];
      }
    }
  }
}

// Window-gradient gather (analytic differentiation, mesh.py:343-349): one
// field, three derivative sums G_d = sum w..w'_d..w f over the stencil (the
// derivative on axis d), F_a = -q sum_d G_d J[d][a] with J = du/dr.
// Same lane mapping and conflict-free strides as k_gather_warp's f_z tile.

template <typename real, int P>
__global__ void __launch_bounds__(kTileThreads, 2)
k_gather_grad(Geom g, const int* __restrict__ offsets, const real* __restrict__ wrec,
              const real* __restrict__ drec, const int* __restrict__ PK,
              const double* __restrict__ Q, const int* __restrict__ IDX,
              const real* __restrict__ fld, Jac J, double* __restrict__ forces) {
  static_assert(P <= 8, "gradient gather covers at most 8 stencil planes");
  constexpr int kRowZ = GatherLayout<real, P>::kRowZ;
  constexpr int kPlaneZ = GatherLayout<real, P>::kPlaneZ;
  constexpr int RS = rec_stride(P);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nxy = g.ntx * g.nty;                    // z-slab-major (see k_gather_warp)
  const int tz = blockIdx.x / nxy;
  const int txy = blockIdx.x - tz * nxy;
  const int tx = txy % g.ntx, ty = txy / g.ntx;
  const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
  const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
  const long long p0 = offsets[key0], p1 = offsets[key1];
  if (p0 == p1) return;
  real* s_f = reinterpret_cast<real*>(smem_raw);
  {
    const long long Mxy = (long long)g.M[0] * g.M[1];
    const int r = threadIdx.x;
    const int gx = wrap_near(tx * g.TX + g.lo + (r & 15), g.M[0]);
    const int gy = wrap_near(ty * g.TY + g.lo + (r >> 4), g.M[1]);
    const long long col = (long long)gy * g.M[0] + gx;
    int gz = wrap_near(tz * g.TZ + g.lo, g.M[2]);
    for (int pz = 0; pz < g.PZ; ++pz) {
      cp_async_real(s_f + pz * kPlaneZ + (r >> 4) * kRowZ + (r & 15), fld + gz * Mxy + col);
      gz = gz + 1 == g.M[2] ? 0 : gz + 1;
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 4, h = (lane >> 3) & 1, k = lane & 7;
  constexpr int kStep = (kTileThreads / 32) * 2;
  constexpr int kRec = 3 * RS;                                  // reals per record
  constexpr int kChunks = (2 * kRec * (int)sizeof(real)) / 16;  // 16 B pieces per pair
  // per warp: 2 buffers x (W records of the pair | D records of the pair)
  real* ring = reinterpret_cast<real*>(
                   smem_raw + ((sizeof(real) * (size_t)g.PZ * kPlaneZ + 15) & ~size_t(15))) +
               (size_t)warp * 2 * 4 * kRec;
  auto fetch = [&](long long pb, int b) {
    const int avail = (int)min((long long)2, p1 - pb);
    const int bytes_needed = avail * kRec * (int)sizeof(real);
    for (int c = lane; c < 2 * kChunks; c += 32) {
      const int which = c >= kChunks;          // 0: W records, 1: D records
      const int piece = which ? c - kChunks : c;
      if (piece * 16 < bytes_needed) {
        const real* srcb = which ? drec : wrec;
        const char* src = reinterpret_cast<const char*>(srcb + pb * kRec) + piece * 16;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(
            reinterpret_cast<char*>(ring + ((size_t)b * 4 + 2 * which) * kRec) + piece * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  long long pb = p0 + warp * 2;
  int buf = 0;
  if (pb < p1) fetch(pb, 0);
  // the pair's scalars (anchor, charge, index) one iteration ahead
  int pk_n = 0, id_n = 0;
  double q_n = 0.0;
  if (pb + slot < p1) {
    pk_n = PK[pb + slot];
    q_n = Q[pb + slot];
    id_n = IDX[pb + slot];
  }
  for (; pb < p1; pb += kStep, buf ^= 1) {
    const long long pl = pb + slot;
    const bool live = pl < p1 && k < P;
    const long long nx = pb + kStep;
    const int pk = pk_n, id_c = id_n;
    const double q_c = q_n;
    if (nx < p1) {
      fetch(nx, buf ^ 1);
      if (nx + slot < p1) {
        pk_n = PK[nx + slot];
        q_n = Q[nx + slot];
        id_n = IDX[nx + slot];
      }
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncwarp();
    real gx = 0, gy = 0, gz = 0;
    if (live) {
      const int xl = pk & 0xff, yl = (pk >> 8) & 0xff, zl = (pk >> 16) - tz * g.TZ;
      const real* W = ring + ((size_t)buf * 4 + slot) * kRec;
      const real* D = ring + ((size_t)buf * 4 + 2 + slot) * kRec;
      real wx[RS], dx[RS], wy[RS], dy[RS];
      // 16-byte loads of the weight rows (records are 16 B aligned)
      using V = typename Vec16<real>::type;
      constexpr int kPer = 16 / (int)sizeof(real);
#pragma unroll
      for (int c = 0; c < RS / kPer; ++c) {
        Vec16<real>::split(reinterpret_cast<const V*>(W)[c], wx + c * kPer);
        Vec16<real>::split(reinterpret_cast<const V*>(D)[c], dx + c * kPer);
        Vec16<real>::split(reinterpret_cast<const V*>(W + RS)[c], wy + c * kPer);
        Vec16<real>::split(reinterpret_cast<const V*>(D + RS)[c], dy + c * kPer);
      }
      const real wzk = W[2 * RS + k], dzk = D[2 * RS + k];
      const real* row = s_f + (zl + k) * kPlaneZ + (yl + h) * kRowZ + xl;
      real ax = 0, ay = 0, az = 0;
#pragma unroll
      for (int jj = 0; jj < (P + 1) / 2; ++jj) {
        const int j = 2 * jj;
        const bool odd_row = j + 1 < P;
        if (odd_row || h == 0) {
          const real wy_ = (odd_row && h) ? wy[odd_row ? j + 1 : j] : wy[j];
          const real dy_ = (odd_row && h) ? dy[odd_row ? j + 1 : j] : dy[j];
          real r0 = 0, r1 = 0;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const real v = row[j * kRowZ + i];
            r0 = fma(wx[i], v, r0);
            r1 = fma(dx[i], v, r1);
          }
          ax = fma(wy_, r1, ax);     // d/dx
          ay = fma(dy_, r0, ay);     // d/dy
          az = fma(wy_, r0, az);     // d/dz (plane weight below)
        }
      }
      gx = ax * wzk;
      gy = ay * wzk;
      gz = az * dzk;
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      gx += __shfl_xor_sync(0xffffffffu, gx, o);
      gy += __shfl_xor_sync(0xffffffffu, gy, o);
      gz += __shfl_xor_sync(0xffffffffu, gz, o);
    }
    __syncwarp();   // the ring slot is refilled next iteration
    if ((lane & 15) == 0 && pl < p1) {
      const double q = q_c;
      const double G3[3] = {(double)gx, (double)gy, (double)gz};
      double* f = forces + (long long)id_c * 3;
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2)
        f[a2] = -q * ((G3[0] * J.j[0 * 3 + a2] + G3[1] * J.j[1 * 3 + a2]) + G3[2] * J.j[2 * 3 + a2]);
    }
  }
}

// Window-derivative records dW/dt of every binned particle (analytic mode).
// Window-derivative weights for the analytic gather: one thread per
// (particle, axis), unrolled Horner on the derivative table (FastTab) like the
// binning pass's weight records.
template <typename real, int P>
__global__ void k_dweights(Geom g, FastTab ft, const real* __restrict__ dtab,
                           const double* __restrict__ brk, int n_pieces, int ncoef,
                           long long n, long long cap, const double* __restrict__ U,
                           real* __restrict__ drec) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 3 * n) return;
  const long long j = t / 3;
  const int d = (int)(t - 3 * j);
  constexpr int RS = rec_stride(P);
  const double u = U[d * cap + j];
  const double base = anchor_base(g, u);
  real w[P];
  stencil_weights<real, P>(ft, dtab, brk, n_pieces, ncoef, u, base, g.lo, real(1), w);
  real* out = drec + j * (3 * RS) + d * RS;
#pragma unroll
  for (int s = 0; s < RS; ++s) out[s] = s < P ? w[s] : real(0);
}

template <typename real, int P>
__global__ void __launch_bounds__(kTileThreads)
k_gather_ik(Geom g, const real* __restrict__ tab, const double* __restrict__ brk,
            int n_pieces, int ncoef, const int* __restrict__ offsets,
            const double* __restrict__ U, const double* __restrict__ Q,
            const int* __restrict__ IDX, long long cap, const real* __restrict__ fld,
            long long G, double* __restrict__ forces, OutMap om) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tile = blockIdx.x;
  const int tz = tile % g.ntz;
  const int txy = tile / g.ntz;
  const int tx = txy % g.ntx, ty = txy / g.ntx;
  const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZ;
  const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZ);
  const long long p0 = offsets[key0], p1 = offsets[key1];
  if (p0 == p1) return;

  real* s_tab = reinterpret_cast<real*>(smem_raw);
  size_t off = sizeof(real) * (size_t)n_pieces * ncoef;
  off = (off + 15) & ~size_t(15);
  double* s_brk = reinterpret_cast<double*>(smem_raw + off);
  off += sizeof(double) * (size_t)(n_pieces + 1);
  off = (off + 15) & ~size_t(15);
  real* s_w = reinterpret_cast<real*>(smem_raw + off);
  off += sizeof(real) * 3 * (size_t)kChunk * P;
  off = (off + 15) & ~size_t(15);
  double* s_acc = reinterpret_cast<double*>(smem_raw + off);
  off += sizeof(double) * (size_t)kChunk * 8 * 3;
  int* s_anc = reinterpret_cast<int*>(smem_raw + off);

  for (int i = threadIdx.x; i < n_pieces * ncoef; i += blockDim.x) s_tab[i] = tab[i];
  for (int i = threadIdx.x; i <= n_pieces; i += blockDim.x) s_brk[i] = brk[i];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
  const int cx = wx0 + (lane & 7), cy = wy0 + (lane >> 3);
  const int gx = wrap_index((long long)tx * g.TX + g.lo + cx, g.M[0]);
  const int gy = wrap_index((long long)ty * g.TY + g.lo + cy, g.M[1]);
  const long long colbase = (long long)gy * g.M[0] + gx;
  const long long plane = (long long)g.M[0] * g.M[1];
  const int zorg = tz * g.TZ + g.lo;
  const real* f0 = fld;
  const real* f1 = fld + G;
  const real* f2 = fld + 2 * G;

  real w0[P], w1[P], w2[P];
  int zc = -1;

  for (long long c0 = p0; c0 < p1; c0 += kChunk) {
    const int n = (int)min((long long)kChunk, p1 - c0);
    __syncthreads();
    stage_weights_g<real, P>(g, s_tab, s_brk, n_pieces, ncoef, U, cap, c0, n, tx, ty,
                             tz, s_w, s_anc);
    for (int i = threadIdx.x; i < n * 24; i += blockDim.x) s_acc[i] = 0.0;
    __syncthreads();
    for (int pl = 0; pl < n; ++pl) {
      const int xl = s_anc[pl];
      const int yl = s_anc[kChunk + pl];
      if (xl >= wx0 + 8 || xl + P <= wx0 || yl >= wy0 + 4 || yl + P <= wy0) continue;
      const int zl = s_anc[2 * kChunk + pl];
      if (zc < 0 || zl - zc >= P) {
        zc = zl;
#pragma unroll
        for (int s = 0; s < P; ++s) {
          const long long o = (long long)wrap_index(zorg + zc + s, g.M[2]) * plane + colbase;
          w0[s] = f0[o];
          w1[s] = f1[o];
          w2[s] = f2[o];
        }
      } else {
        while (zc < zl) {
#pragma unroll
          for (int s = 0; s < P - 1; ++s) {
            w0[s] = w0[s + 1];
            w1[s] = w1[s + 1];
            w2[s] = w2[s + 1];
          }
          const long long o =
              (long long)wrap_index(zorg + zc + P, g.M[2]) * plane + colbase;
          w0[P - 1] = f0[o];
          w1[P - 1] = f1[o];
          w2[P - 1] = f2[o];
          ++zc;
        }
      }
      const int sx = cx - xl, sy = cy - yl;
      const bool in = (unsigned)sx < (unsigned)P && (unsigned)sy < (unsigned)P;
      const real* wxp = s_w + (size_t)pl * P;
      const real* wyp = s_w + ((size_t)kChunk + pl) * P;
      const real* wzp = s_w + ((size_t)2 * kChunk + pl) * P;
      const int sxc = min(max(sx, 0), P - 1), syc = min(max(sy, 0), P - 1);
      const real a = in ? wxp[sxc] * wyp[syc] : real(0);
      real t0 = real(0), t1 = real(0), t2 = real(0);
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const real wz = wzp[s];
        t0 = fma(wz, w0[s], t0);
        t1 = fma(wz, w1[s], t1);
        t2 = fma(wz, w2[s], t2);
      }
      const real v = warp_reduce3<real>(a * t0, a * t1, a * t2, lane);
      if ((lane & 7) == 0 && lane < 24) s_acc[((size_t)pl * 8 + warp) * 3 + (lane >> 3)] = (double)v;
    }
    __syncthreads();
    for (int pl = threadIdx.x; pl < n; pl += blockDim.x) {
      const double q = Q[c0 + pl];
      const long long id = IDX[c0 + pl];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += s_acc[((size_t)pl * 8 + w) * 3 + c];
        forces[id * om.stride + om.m[c]] = -q * s;
        if (om.m2[c] >= 0) forces[id * om.stride + om.m2[c]] = -q * s;
      }
    }
  }
}

template <typename real>
static size_t gather_smem(int P, int n_pieces, int ncoef) {
  size_t b = sizeof(real) * (size_t)n_pieces * ncoef;
  b = (b + 15) & ~size_t(15);
  b += sizeof(double) * (size_t)(n_pieces + 1);
  b = (b + 15) & ~size_t(15);
  b += sizeof(real) * 3 * (size_t)kChunk * P;
  b = (b + 15) & ~size_t(15);
  b += sizeof(double) * (size_t)kChunk * 8 * 3;
  b += sizeof(int) * 3 * (size_t)kChunk;
  return b;
}

template <typename real, int P>
static cudaError_t gather_p(esp_plan* p, double* d_forces, cudaStream_t s, OutMap om) {
  Geom g = make_geom(p);
  if constexpr (P <= 8) {
    const size_t smem = GatherLayout<real, P>::bytes(p->PZ);
    // the opt-in is per device: set it on every call (host-only, capture-safe)
    cudaError_t e = cudaFuncSetAttribute(k_gather_warp<real, P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_gather_warp<real, P><<<(unsigned)p->n_tiles, kTileThreads, smem, s>>>(
        g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec), p->d_pk, p->d_q, p->d_idx,
        reinterpret_cast<const real*>(p->d_fields), p->G, d_forces, om);
    p->launches++;
    prof_mark(p, s, "gather");
    return cudaGetLastError();
  }
  const real* tab = std::is_same<real, double>::value
                        ? reinterpret_cast<const real*>(p->d_tab)
                        : reinterpret_cast<const real*>(p->d_tabf);
  const size_t smem = gather_smem<real>(P, p->n_pieces, p->ncoef);
  // the opt-in is per device: set it on every call (host-only, capture-safe)
  cudaError_t e = cudaFuncSetAttribute(k_gather_ik<real, P>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_gather_ik<real, P><<<(unsigned)p->n_tiles, kTileThreads, smem, s>>>(
      g, tab, p->d_breaks, p->n_pieces, p->ncoef, p->d_offsets, p->d_u, p->d_q,
      p->d_idx, p->cap, reinterpret_cast<const real*>(p->d_fields), p->G, d_forces, om);
  p->launches++;
  prof_mark(p, s, "gather");
  return cudaGetLastError();
}

template <typename real>
static cudaError_t gather_r(esp_plan* p, double* d_forces, cudaStream_t s, OutMap om) {
  switch (p->P) {
    case 2: return gather_p<real, 2>(p, d_forces, s, om);
    case 3: return gather_p<real, 3>(p, d_forces, s, om);
    case 4: return gather_p<real, 4>(p, d_forces, s, om);
    case 5: return gather_p<real, 5>(p, d_forces, s, om);
    case 6: return gather_p<real, 6>(p, d_forces, s, om);
    case 7: return gather_p<real, 7>(p, d_forces, s, om);
    case 8: return gather_p<real, 8>(p, d_forces, s, om);
    case 9: return gather_p<real, 9>(p, d_forces, s, om);
    case 10: return gather_p<real, 10>(p, d_forces, s, om);
    case 11: return gather_p<real, 11>(p, d_forces, s, om);
    case 12: return gather_p<real, 12>(p, d_forces, s, om);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gather_ik(esp_plan* p, double* d_forces, cudaStream_t s,
                             const void* fields, OutMap om) {
  const cudaError_t er = ensure_records(p, s);
  if (er != cudaSuccess) return er;
  void* saved = p->d_fields;
  if (fields) p->d_fields = const_cast<void*>(fields);
  cudaError_t e = p->precision == ESP_FP64 ? gather_r<double>(p, d_forces, s, om)
                                           : gather_r<float>(p, d_forces, s, om);
  p->d_fields = saved;
  return e;
}

template <typename real, int P>
static cudaError_t grad_p(esp_plan* p, double* d_forces, cudaStream_t s) {
  if constexpr (P > 8) {
    return cudaErrorNotSupported;
  } else {
    Geom g = make_geom(p);
    const real* dtab = std::is_same<real, double>::value
                           ? reinterpret_cast<const real*>(p->d_dtab)
                           : reinterpret_cast<const real*>(p->d_dtabf);
    const int B = 256;
    const long long n = p->last_n;
    if (!p->drec_ready) {   // not produced by the binning pass of this step
      k_dweights<real, P><<<(unsigned)((3 * n + B - 1) / B), B, 0, s>>>(
          g, *p->h_fast_d, dtab, p->d_breaks, p->n_pieces, p->ncoef, n, p->cap, p->d_u,
          reinterpret_cast<real*>(p->d_drec));
      p->launches++;
      prof_mark(p, s, "dweights");
    }
    const Jac J = plan_jacobian(p);
    constexpr int RS = rec_stride(P);
    const size_t smem = ((sizeof(real) * (size_t)p->PZ * GatherLayout<real, P>::kPlaneZ + 15) &
                         ~size_t(15)) +
                        sizeof(real) * (size_t)(kTileThreads / 32) * 2 * 4 * 3 * RS;
    // the opt-in is per device: set it on every call (host-only, capture-safe)
    cudaError_t e = cudaFuncSetAttribute(k_gather_grad<real, P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_gather_grad<real, P><<<(unsigned)p->n_tiles, kTileThreads, smem, s>>>(
        g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec),
        reinterpret_cast<const real*>(p->d_drec), p->d_pk, p->d_q, p->d_idx,
        reinterpret_cast<const real*>(p->d_fields), J, d_forces);
    p->launches++;
    prof_mark(p, s, "gather_grad");
    return cudaGetLastError();
  }
}

template <typename real>
static cudaError_t grad_r(esp_plan* p, double* d_forces, cudaStream_t s) {
  switch (p->P) {
    case 2: return grad_p<real, 2>(p, d_forces, s);
    case 3: return grad_p<real, 3>(p, d_forces, s);
    case 4: return grad_p<real, 4>(p, d_forces, s);
    case 5: return grad_p<real, 5>(p, d_forces, s);
    case 6: return grad_p<real, 6>(p, d_forces, s);
    case 7: return grad_p<real, 7>(p, d_forces, s);
    case 8: return grad_p<real, 8>(p, d_forces, s);
    default: return cudaErrorNotSupported;
  }
}

Jac plan_jacobian(const esp_plan* p) {
  Jac J;
  for (int d = 0; d < 3; ++d)
    for (int a = 0; a < 3; ++a)
      J.j[d * 3 + a] = p->ortho ? (d == a ? 1.0 / p->spacing[d] : 0.0)
                                : (double)p->Mu[d] * p->hinv[d * 3 + a];
  return J;
}

cudaError_t launch_gather_grad(esp_plan* p, double* d_forces, cudaStream_t s) {
  const cudaError_t er = ensure_records(p, s);
  if (er != cudaSuccess) return er;
  return p->precision == ESP_FP64 ? grad_r<double>(p, d_forces, s)
                                  : grad_r<float>(p, d_forces, s);
}

}  // namespace esp
