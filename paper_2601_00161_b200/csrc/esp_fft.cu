// esp_fft.cu — band-pruned, fused 3D transforms for the k-space step.
//
// The far field only ever uses modes inside the box |m_d| <= band_d (the
// mask |k| <= kmax lies inside it, mesh.py:248-249).  The forward transform
// therefore keeps only in-band outputs after each 1D stage, and its last
// stage (along z) is fused with the deconvolution scaling + energy/pressure
// reduction (mesh.py:285-312), the ik spectra (mesh.py:333-341) and the
// first inverse stage:
//
//   P1  x rows:  real -> complex (two rows per complex FFT), keep kx <= band;
//                in esp_evaluate the rows are summed straight from the
//                spread's tile blocks (k_x_bulk_r2c: scratch rows staged by
//                cp.async.bulk on an mbarrier; k_x_comb_r2c: register-staged)
//   P2  y lines: C2C, keep |ky| <= band
//   P3a z lines: C2C; reduce E, P_ab over the retained modes; write the box
//                spectrum
//   P3b z lines: build i k_d A X h3/G on the box, inverse C2C along z
//   P4  y lines: inverse C2C of the three ik pencils, zero-padded in ky
//   P5  x rows:  complex -> real (two rows per complex FFT), zero-padded in kx
//
// The pressure-only path is P1-P3a: one forward transform whose last pass is
// the fused scaling/reduction.  Intermediate arrays keep kx in a column pitch
// `ldx` rounded up to 8 so that every 8 (fp64) / 16 (fp32) consecutive lines
// a CTA reads form full 128-byte segments.
//
// Line transforms: compile-time length N, mixed-radix (8, 6, 4, 3, 2)
// Stockham auto-sort stages executed in place in shared memory through
// registers (load R inputs -> barrier -> twiddle, DFT, store; the forward y
// pass gives each warp whole lines and synchronises per warp, fft_lines).  Shared rows
// use pitch N + N/8 + 1 and index i + i/8 so that strided butterflies and
// the line-transposing loads are bank-conflict free; per-stage twiddle
// tables are laid out [t-1][k] so a warp reads consecutive entries.
// Grids whose lengths are not in ESP_FFT_SIZES use the cuFFT path.
//
// Small square planes (Mx == My <= 64) run P1+P2 and P4+P5 as one kernel
// per z plane (k_xy_fwd, k_yx_inv).  The distributed z-slab decomposition
// (esp_slab_*) reuses P1-P5 with the transposes fused into P2 and P3b: their
// stores go straight into the destination rank's receive buffer (SlabMap).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "esp_internal.cuh"

#define ESP_FFT_SIZES(X) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384)

namespace esp {
namespace fft {

template <typename real> struct Cx;
template <> struct Cx<double> { using t = double2; };
template <> struct Cx<float> { using t = float2; };

__host__ __device__ constexpr int pick_radix(int n) {
  return n % 8 == 0 ? 8 : n % 6 == 0 ? 6 : n % 4 == 0 ? 4 : n % 3 == 0 ? 3 : 2;
}
// twiddle entries needed by the stages that start at span Ns
__host__ __device__ constexpr int tw_from(int N, int Ns) {
  return Ns >= N ? 0
                 : (Ns > 1 ? (pick_radix(N / Ns) - 1) * Ns : 0) +
                       tw_from(N, Ns * pick_radix(N / Ns));
}
__host__ __device__ constexpr int tw_total(int N) { return tw_from(N, 1); }
__host__ __device__ constexpr int tw_offset(int N, int Ns) { return tw_total(N) - tw_from(N, Ns); }
__host__ __device__ constexpr int pitch(int N) { return N + N / 8 + 1; }
__device__ __forceinline__ int pidx(int i) { return i + (i >> 3); }

__host__ __device__ constexpr int pow2_floor(int v) {
  int p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}
// CTA shapes.  x rows: kThreadsX threads transform pairs_x(N) row pairs.
// y/z lines: lines_yz consecutive kx columns (one 128-byte segment per row)
// with threads_yz(N) threads, so that small grids still launch several CTAs
// per SM.
constexpr int kThreadsX = 128;
// resident CTAs per SM the register allocation is sized for (A/B knobs)
#ifndef ESP_YZ_MINB
#define ESP_YZ_MINB 3
#endif
#ifndef ESP_X_MINB
#define ESP_X_MINB 8   // config 4: inverse x 0.667 -> 0.630 ms against 6
#endif
// x rows: ~1024 elements per CTA on large grids; small grids (L2-resident)
// take fewer rows per CTA so that every SM gets work.
__host__ __device__ constexpr int pairs_x(int N) {
  return N >= 128 ? (N >= 1024 ? 1 : 1024 / N) : 256 / N;
}
// y/z lines: one 128-byte segment of consecutive kx per row on large grids;
// 2 lines on small grids.
#ifndef ESP_YZ_SEG
#define ESP_YZ_SEG 128   // bytes of consecutive kx per row and CTA on large grids
#endif
template <typename real>
__host__ __device__ constexpr int lines_yz(int N) {
  return N > 128 ? ESP_YZ_SEG / (2 * (int)sizeof(real)) : 2;
}
template <typename real>
__host__ __device__ constexpr int threads_yz(int N) {
  return lines_yz<real>(N) * N / 8 < 32 ? 32
         : lines_yz<real>(N) * N / 8 > 256 ? 256
                                           : lines_yz<real>(N) * N / 8;
}

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <typename C>
__device__ __forceinline__ C cadd(C a, C b) {
  C r;
  r.x = a.x + b.x;
  r.y = a.y + b.y;
  return r;
}
template <typename C>
__device__ __forceinline__ C csub(C a, C b) {
  C r;
  r.x = a.x - b.x;
  r.y = a.y - b.y;
  return r;
}
// a * (SIGN i): -i for the forward sign, +i for the inverse
template <int SIGN, typename C>
__device__ __forceinline__ C cmuli(C a) {
  C r;
  if (SIGN < 0) {
    r.x = a.y;
    r.y = -a.x;
  } else {
    r.x = -a.y;
    r.y = a.x;
  }
  return r;
}

// In-register DFT of radix R with kernel e^{SIGN 2 pi i jk/R}.
template <int R, int SIGN, typename C>
__device__ __forceinline__ void dft(C* v) {
  using real = decltype(v[0].x);
  if constexpr (R == 2) {
    const C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 3) {
    const real c1 = real(-0.5), s1 = real(SIGN) * real(0.86602540378443864676);
    const C a = v[0], b = v[1], c = v[2];
    const C t1 = cadd(b, c), t2 = csub(b, c);
    C m1, m2;
    m1.x = a.x + c1 * t1.x;
    m1.y = a.y + c1 * t1.y;
    m2.x = -s1 * t2.y;
    m2.y = s1 * t2.x;
    v[0] = cadd(a, t1);
    v[1] = cadd(m1, m2);
    v[2] = csub(m1, m2);
  } else if constexpr (R == 4) {
    const C a = v[0], b = v[1], c = v[2], d = v[3];
    const C t0 = cadd(a, c), t1 = csub(a, c), t2 = cadd(b, d), t3 = cmuli<SIGN>(csub(b, d));
    v[0] = cadd(t0, t2);
    v[1] = cadd(t1, t3);
    v[2] = csub(t0, t2);
    v[3] = csub(t1, t3);
  } else if constexpr (R == 6) {
    C e[3] = {v[0], v[2], v[4]}, o[3] = {v[1], v[3], v[5]};
    dft<3, SIGN>(e);
    dft<3, SIGN>(o);
    const real h = real(0.86602540378443864676) * real(SIGN);
    C w1, w2;
    w1.x = real(0.5);
    w1.y = h;
    w2.x = real(-0.5);
    w2.y = h;
    o[1] = cmul(o[1], w1);
    o[2] = cmul(o[2], w2);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 3] = csub(e[k], o[k]);
    }
  } else if constexpr (R == 8) {
    C e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft<4, SIGN>(e);
    dft<4, SIGN>(o);
    const real h = real(0.70710678118654752440);
    C w1, w3;
    w1.x = h;
    w1.y = real(SIGN) * h;
    w3.x = -h;
    w3.y = real(SIGN) * h;
    o[1] = cmul(o[1], w1);
    o[2] = cmuli<SIGN>(o[2]);
    o[3] = cmul(o[3], w3);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    }
  }
}

// One Stockham stage over L lines of length N, in place through registers.
// Enters with the buffer complete; leaves after a barrier.
template <int R, int N, int Ns, int L, int NT, int SIGN, typename C>
__device__ __forceinline__ void stage_ip(C* buf, const C* __restrict__ tw) {
  constexpr int nb = N / R, total = L * nb, iters = (total + NT - 1) / NT, LP = pitch(N);
  constexpr int toff = tw_offset(N, Ns);
  C v[iters][R];
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int idx = threadIdx.x + it * NT;
    if (total % NT == 0 || idx < total) {
      const int line = idx / nb, j = idx - line * nb;
      const C* in = buf + line * LP;
#pragma unroll
      for (int t = 0; t < R; ++t) v[it][t] = in[pidx(j + t * nb)];
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int idx = threadIdx.x + it * NT;
    if (total % NT == 0 || idx < total) {
      const int line = idx / nb, j = idx - line * nb;
      const int k = j % Ns;
      if constexpr (Ns > 1) {
#pragma unroll
        for (int t = 1; t < R; ++t) {
          C w = __ldg(tw + toff + (t - 1) * Ns + k);
          if (SIGN > 0) w.y = -w.y;
          v[it][t] = cmul(v[it][t], w);
        }
      }
      dft<R, SIGN>(v[it]);
      C* out = buf + line * LP;
      const int base = (j / Ns) * Ns * R + k;
#pragma unroll
      for (int t = 0; t < R; ++t) out[pidx(base + t * Ns)] = v[it][t];
    }
  }
  __syncthreads();
}

template <int N, int Ns, int L, int NT, int SIGN, typename C>
__device__ __forceinline__ void fft_ip(C* buf, const C* tw) {
  if constexpr (Ns < N) {
    constexpr int R = pick_radix(N / Ns);
    stage_ip<R, N, Ns, L, NT, SIGN>(buf, tw);
    fft_ip<N, Ns * R, L, NT, SIGN>(buf, tw);
  }
}

// Line groups of the y / z passes: when the CTA's warps divide its lines, a
// warp owns whole lines and runs their stages back to back with warp-level
// synchronisation only — the stages of different lines no longer meet at a
// CTA barrier (six per transform), so one line's shared-memory and twiddle
// latencies overlap another's butterflies.  One CTA barrier closes the
// transform for the stores that follow.
#ifndef ESP_FFT_WARPLINES
#define ESP_FFT_WARPLINES 1
#endif
template <int R, int N, int Ns, int L, int NT, int SIGN, typename C>
__device__ __forceinline__ void stage_ip_w(C* buf, const C* __restrict__ tw) {
  constexpr int nb = N / R, NW = NT / 32, LW = L / NW, iters = (nb + 31) / 32, LP = pitch(N);
  constexpr int toff = tw_offset(N, Ns);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int lw = 0; lw < LW; ++lw) {
    C* line = buf + (warp * LW + lw) * LP;
    C v[iters][R];
#pragma unroll
    for (int it = 0; it < iters; ++it) {
      const int j = lane + it * 32;
      if (nb % 32 == 0 || j < nb) {
#pragma unroll
        for (int t = 0; t < R; ++t) v[it][t] = line[pidx(j + t * nb)];
      }
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < iters; ++it) {
      const int j = lane + it * 32;
      if (nb % 32 == 0 || j < nb) {
        const int k = j % Ns;
        if constexpr (Ns > 1) {
#pragma unroll
          for (int t = 1; t < R; ++t) {
            C w = __ldg(tw + toff + (t - 1) * Ns + k);
            if (SIGN > 0) w.y = -w.y;
            v[it][t] = cmul(v[it][t], w);
          }
        }
        dft<R, SIGN>(v[it]);
        const int base = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int t = 0; t < R; ++t) line[pidx(base + t * Ns)] = v[it][t];
      }
    }
    __syncwarp();
  }
}

template <int N, int Ns, int L, int NT, int SIGN, typename C>
__device__ __forceinline__ void fft_ip_w(C* buf, const C* tw) {
  if constexpr (Ns < N) {
    constexpr int R = pick_radix(N / Ns);
    stage_ip_w<R, N, Ns, L, NT, SIGN>(buf, tw);
    fft_ip_w<N, Ns * R, L, NT, SIGN>(buf, tw);
  }
}

// L lines of length N in place; enters after a CTA barrier, leaves after one.
// WL: warp-owned lines.  Measured at config 4 (ms, CTA-barrier stages -> warp
// lines at 3 -> at 2 CTAs per SM): forward y 0.132 -> 0.121 -> 0.097, z +
// reduce 0.103 -> 0.102 -> 0.100, ik + inverse z 0.224 -> 0.221 -> 0.252,
// inverse y 0.362 -> 0.384 -> 0.377 — the store-heavy inverse passes want the
// third CTA more than the loose stages, so only the forward y pass takes it.
template <int N, int L, int NT, int SIGN, bool WL, typename C>
__device__ __forceinline__ void fft_lines(C* buf, const C* tw) {
  if constexpr (WL && ESP_FFT_WARPLINES && NT % 32 == 0 && L % (NT / 32) == 0) {
    fft_ip_w<N, 1, L, NT, SIGN>(buf, tw);
    __syncthreads();
  } else {
    fft_ip<N, 1, L, NT, SIGN>(buf, tw);
  }
}

// Twiddle tables live in global memory in the plan's precision and are read
// through L1 (a warp reads consecutive entries).

// in-band index -> mode and mode -> in-band index along y/z (band box is
// [0..b] U [N-b..N-1], or the whole axis when nb == N)
__device__ __forceinline__ int band_mode(int bi, int nb, int N) {
  return (nb == N || bi <= (nb - 1) / 2) ? bi : bi + N - nb;
}
__device__ __forceinline__ int band_index(int m, int nb, int N) {
  if (nb == N) return m;
  const int b = (nb - 1) / 2;
  return m <= b ? m : (m >= N - b ? m - (N - nb) : -1);
}

// ---------------------------------------------------------------------------
// P1: x rows, real -> complex, two rows per transform; out[row][kx], kx < ldx
// (zeros for kx >= nbx).
template <typename real, int N>
__global__ void __launch_bounds__(kThreadsX, ESP_X_MINB)
k_x_r2c(const real* __restrict__ grid, typename Cx<real>::t* __restrict__ out,
        const typename Cx<real>::t* __restrict__ tw, long long nrows, int ldx, int nbx) {
  using C = typename Cx<real>::t;
  constexpr int PP = pairs_x(N), LP = pitch(N), NT = kThreadsX;
  __shared__ C buf[PP * LP];
  const long long r0 = 2LL * blockIdx.x * PP;
  constexpr int nld = (PP * N + NT - 1) / NT;
  real va[nld], vb[nld];
#pragma unroll
  for (int it = 0; it < nld; ++it) {
    const int e = threadIdx.x + it * NT;
    const int l = e / N, i = e - l * N;
    const long long ra = r0 + 2 * l;
    const bool in = (PP * N) % NT == 0 || e < PP * N;
    va[it] = in && ra < nrows ? __ldcs(grid + ra * N + i) : real(0);
    vb[it] = in && ra + 1 < nrows ? __ldcs(grid + (ra + 1) * N + i) : real(0);
  }
#pragma unroll
  for (int it = 0; it < nld; ++it) {
    const int e = threadIdx.x + it * NT;
    if ((PP * N) % NT == 0 || e < PP * N) {
      const int l = e / N, i = e - l * N;
      C z;
      z.x = va[it];
      z.y = vb[it];
      buf[l * LP + pidx(i)] = z;
    }
  }
  __syncthreads();
  fft_ip<N, 1, PP, NT, -1>(buf, tw);
  for (int e = threadIdx.x; e < PP * ldx; e += NT) {
    const int l = e / ldx, k = e - l * ldx;
    const long long ra = r0 + 2 * l;
    C A, B;
    A.x = A.y = B.x = B.y = real(0);
    if (k < nbx) {
      const C zk = buf[l * LP + pidx(k)], zm = buf[l * LP + pidx((N - k) % N)];
      A.x = real(0.5) * (zk.x + zm.x);   // (Zk + conj Zm) / 2
      A.y = real(0.5) * (zk.y - zm.y);
      B.x = real(0.5) * (zk.y + zm.y);   // (Zk - conj Zm) / 2i
      B.y = real(-0.5) * (zk.x - zm.x);
    }
    if (ra < nrows) out[ra * ldx + k] = A;
    if (ra + 1 < nrows) out[(ra + 1) * ldx + k] = B;
  }
}

// P1 with the spread's halo combine folded in (single-GPU esp_evaluate): the
// CTA's rows are summed straight from the spread scratch ([tz][pz][ty][py][tx][px],
// scr_index) instead of being read from a combined grid, so the grid is never
// written or re-read (config 4: k_combine 0.70 ms + k_x_r2c 0.17 ms -> one
// pass over the scratch).  Per row the <= 4 covering scratch rows (z tile x
// y tile) are looked up once per CTA into shared memory; per thread the <= 2
// covering x entries of its (at most 3) columns are looked up once.  Every
// point adds its <= 8 contributions in k_combine's (z, y, x) order, so the
// sums are bitwise those of combine_at; coordinates covered by more than two
// tiles on an axis (the periodic wrap of a partial last tile) call
// combine_at itself.
__host__ __device__ constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }

template <typename real, int N>
__global__ void __launch_bounds__(kThreadsX, ESP_X_MINB)
k_x_comb_r2c(Geom g, CombineTabs ct, const real* __restrict__ scratch,
             typename Cx<real>::t* __restrict__ out,
             const typename Cx<real>::t* __restrict__ tw, long long nrows, int ldx, int nbx) {
  using C = typename Cx<real>::t;
  constexpr int PP = pairs_x(N), LP = pitch(N), NT = kThreadsX, NR = 2 * PP;
  constexpr int XP = N / gcd_c(N, NT);   // distinct columns per thread
  static_assert(NR * 6 <= NT, "row-base setup: one thread per (row, z tile, y tile)");
  __shared__ C buf[PP * LP];
  // scratch row bases of (z tile a < 2, y tile b < 3): slots a * 2 + b for
  // b < 2, 4 + a for the third y tile of a wrapped coordinate; -1 unused
  __shared__ long long s_rb[NR][6];
  __shared__ int s_yz[NR][2];
  const long long r0 = 2LL * blockIdx.x * PP;
  const ScrLayout SL = scr_layout(g);
  bool slow = false;
  if (threadIdx.x < NR * 6) {
    const int rr = threadIdx.x / 6, slot = threadIdx.x - rr * 6;
    const int a = slot < 4 ? slot >> 1 : slot - 4, b = slot < 4 ? slot & 1 : 2;
    const long long ra = r0 + rr;
    long long v = -1;
    if (ra < nrows) {
      const int z = (int)(ra / g.M[1]), y = (int)(ra - (long long)z * g.M[1]);
      const int nz = ct.cnt[2][z], ny = ct.cnt[1][y];
      slow = nz > 2 || ny > 3;
      if (!slow && a < nz && b < ny) {
        const int ez = ct.ent[2][z * kCombW + a], ey = ct.ent[1][y * kCombW + b];
        v = scr_index(g, SL, 0, ey & 0xffff, ez & 0xffff, ez >> 16, ey >> 16, 0);
      }
      if (slot == 0) {
        s_yz[rr][0] = y;
        s_yz[rr][1] = z;
      }
    } else if (slot == 0) {
      s_yz[rr][0] = -1;
    }
    s_rb[rr][slot] = v;
  }
  int xo[XP][3];
#pragma unroll
  for (int k = 0; k < XP; ++k) {
    const int i = (threadIdx.x + k * NT) % N;
    const int nx = ct.cnt[0][i];
    slow = slow || nx > 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int ex = ct.ent[0][i * kCombW + (c < nx ? c : 0)];
      xo[k][c] = c < nx ? (ex & 0xffff) * kPad + (ex >> 16) : -1;
    }
  }
  // CTA-uniform: a coordinate of this CTA covered by more tiles than the
  // straight-line path handles (tiny grids whose tiles wrap more than once)
  const bool general = __syncthreads_or(slow) != 0;
  constexpr int nld = (PP * N + NT - 1) / NT;
  if (!general) {
    // the 8 common loads of a point are unconditional (unused slots re-read a
    // valid address and are not added), so they batch up; third tiles
    // (periodic wrap) are rare and loaded where they are added.  Measured at
    // config 4 (x pass ms): this form at 8 CTAs per SM 0.68-0.70; the loads of
    // both rows of a pair (16) or of 2-3 pairs issued before the first sum at
    // 8 / 5 / 4 CTAs per SM 0.78 / 1.08 / 1.22 (spills, then fewer warps):
    // resident warps matter more than loads in flight per thread.
#pragma unroll
    for (int it = 0; it < nld; ++it) {
      const int e = threadIdx.x + it * NT;
      if ((PP * N) % NT != 0 && e >= PP * N) break;
      const int l = e / N, i = e - l * N;
      const int k = it % XP;
      const int x0 = xo[k][0], x1 = xo[k][1] >= 0 ? xo[k][1] : xo[k][0], x2 = xo[k][2];
      const bool two = xo[k][1] >= 0;
      real v2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = 2 * l + h;
        real v[8];
        long long bs[4];
#pragma unroll
        for (int ab = 0; ab < 4; ++ab) {
          bs[ab] = s_rb[rr][ab];
          const real* src = scratch + (bs[ab] >= 0 ? bs[ab] : 0);
          v[2 * ab] = src[x0];
          v[2 * ab + 1] = src[x1];
        }
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int ab = a * 2 + b;
            if (bs[ab] >= 0) {
              acc += (double)v[2 * ab];
              if (two) acc += (double)v[2 * ab + 1];
              if (x2 >= 0) acc += (double)scratch[bs[ab] + x2];
            }
          }
          const long long b3 = s_rb[rr][4 + a];
          if (b3 >= 0) {
            acc += (double)scratch[b3 + x0];
            if (two) acc += (double)scratch[b3 + x1];
            if (x2 >= 0) acc += (double)scratch[b3 + x2];
          }
        }
        v2[h] = (real)acc;
      }
      C z;
      z.x = v2[0];
      z.y = v2[1];
      buf[l * LP + pidx(i)] = z;
    }
  } else {
    for (int e = threadIdx.x; e < PP * N; e += NT) {
      const int l = e / N, i = e - l * N;
      C z;
      z.x = s_yz[2 * l][0] < 0
                ? real(0)
                : (real)combine_at(g, ct, scratch, i, s_yz[2 * l][0], s_yz[2 * l][1]);
      z.y = s_yz[2 * l + 1][0] < 0
                ? real(0)
                : (real)combine_at(g, ct, scratch, i, s_yz[2 * l + 1][0], s_yz[2 * l + 1][1]);
      buf[l * LP + pidx(i)] = z;
    }
  }
  __syncthreads();
  fft_ip<N, 1, PP, NT, -1>(buf, tw);
  for (int e = threadIdx.x; e < PP * ldx; e += NT) {
    const int l = e / ldx, k = e - l * ldx;
    const long long ra = r0 + 2 * l;
    C A, B;
    A.x = A.y = B.x = B.y = real(0);
    if (k < nbx) {
      const C zk = buf[l * LP + pidx(k)], zm = buf[l * LP + pidx((N - k) % N)];
      A.x = real(0.5) * (zk.x + zm.x);   // (Zk + conj Zm) / 2
      A.y = real(0.5) * (zk.y - zm.y);
      B.x = real(0.5) * (zk.y + zm.y);   // (Zk - conj Zm) / 2i
      B.y = real(-0.5) * (zk.x - zm.x);
    }
    if (ra < nrows) out[ra * ldx + k] = A;
    if (ra + 1 < nrows) out[(ra + 1) * ldx + k] = B;
  }
}

// The same pass with the scratch rows staged by the copy engine (large grids:
// N a multiple of 64, >= 192; one row pair per CTA; every coordinate covered
// by <= 3 x, <= 3 y and <= 2 z tiles).  A grid row's <= 4 covering scratch
// rows are contiguous runs of ntx * 16 values (scr_index), so one thread
// issues one cp.async.bulk per run, completing on an mbarrier: no registers
// hold loads in flight.  The sums then read shared memory, in k_combine's
// (z, y, x) order (bitwise the same); third y tiles (periodic wrap) come from
// global memory where they are added.  Config 4: 0.66 ms against 0.68 for the
// register-staged pass.  A persistent 2-stage ring of this kernel (two CTAs
// per SM, the next pair's copies issued before the current pair's sums) is
// slower, 0.85 ms: one 384-point line takes ~5 us through its six barriers,
// so the pass needs many lines in flight per SM, which the 44 KB of staging
// per pair caps at four here.
__device__ __forceinline__ unsigned bulk_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAITX_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra WAITX_%=;\n"
      "}\n" ::"r"(bulk_smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// threads per CTA: 128 on rows that are a multiple of 128, else 64
__host__ __device__ constexpr int threads_xb(int N) { return N % 128 == 0 ? 128 : 64; }
// ZT: z tiles covering the planes of this launch.  Most planes lie under one
// z tile (25 of 32 at config 4) and need 4 staged rows per pair, not 8: they
// get their own launch (zlist: the plane list of the class, My even), which
// fits seven CTAs per SM instead of four.
template <typename real, int N, int ZT>
__global__ void __launch_bounds__(threads_xb(N), (ZT == 1 ? 7 : 4) * (128 / threads_xb(N)))
k_x_bulk_r2c(Geom g, CombineTabs ct, const real* __restrict__ scratch,
             typename Cx<real>::t* __restrict__ out,
             const typename Cx<real>::t* __restrict__ tw, long long nrows, int ldx, int nbx,
             const int* __restrict__ zlist) {
  using C = typename Cx<real>::t;
  constexpr int LP = pitch(N), NT = threads_xb(N), NR = 2;
  static_assert(N % NT == 0, "a thread owns N / NT columns");
  constexpr int XC = N / NT;
  extern __shared__ __align__(128) unsigned char xb_sm[];
  const ScrLayout SL = scr_layout(g);
  const int row_elems = (int)SL.row;                     // ntx * 16
  constexpr int NS = 2 * ZT;                             // staged rows per grid row
  real* stage = reinterpret_cast<real*>(xb_sm);          // [2 rows][NS slots][row_elems]
  C* buf = reinterpret_cast<C*>(xb_sm +
                                (((size_t)2 * NS * row_elems * sizeof(real) + 15) & ~size_t(15)));
  __shared__ long long s_rb[NR][6];   // slots a * 2 + b (z tile a, y tile b < 2), 4 + a: third y tile
  __shared__ __align__(8) uint64_t bar;
  // row pair -> first row: pairs of the listed planes (My even)
  const int ppp = g.M[1] / 2;                            // pairs per plane
  const long long r0 = zlist ? (long long)zlist[blockIdx.x / ppp] * g.M[1] +
                                   2LL * (blockIdx.x % ppp)
                             : 2LL * blockIdx.x;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bulk_smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < NR * 6) {
    const int rr = threadIdx.x / 6, slot = threadIdx.x - rr * 6;
    const int a = slot < 4 ? slot >> 1 : slot - 4, b = slot < 4 ? slot & 1 : 2;
    const long long ra = r0 + rr;
    long long v = -1;
    if (ra < nrows) {
      const int z = (int)(ra / g.M[1]), y = (int)(ra - (long long)z * g.M[1]);
      const int nz = ct.cnt[2][z], ny = ct.cnt[1][y];
      if (a < nz && b < ny) {
        const int ez = ct.ent[2][z * kCombW + a], ey = ct.ent[1][y * kCombW + b];
        v = scr_index(g, SL, 0, ey & 0xffff, ez & 0xffff, ez >> 16, ey >> 16, 0);
      }
    }
    s_rb[rr][slot] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned row_bytes = (unsigned)(row_elems * sizeof(real));
    unsigned total = 0;
#pragma unroll
    for (int s8 = 0; s8 < 2 * NS; ++s8)
      if (s_rb[s8 / NS][s8 % NS] >= 0) total += row_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     bulk_smem_u32(&bar)),
                 "r"(total)
                 : "memory");
#pragma unroll
    for (int s8 = 0; s8 < 2 * NS; ++s8) {
      const long long b = s_rb[s8 / NS][s8 % NS];
      if (b >= 0)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(bulk_smem_u32(stage + (size_t)s8 * row_elems)),
            "l"(scratch + b), "r"(row_bytes), "r"(bulk_smem_u32(&bar))
            : "memory");
    }
  }
  // the covering x entries of this thread's columns: looked up while the
  // copies are in flight
  int xo[XC][3];
#pragma unroll
  for (int k = 0; k < XC; ++k) {
    const int i = threadIdx.x + k * NT;
    const int nx = ct.cnt[0][i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int ex = ct.ent[0][i * kCombW + (c < nx ? c : 0)];
      xo[k][c] = c < nx ? (ex & 0xffff) * kPad + (ex >> 16) : -1;
    }
  }
  bulk_mbar_wait(&bar, 0);
#pragma unroll
  for (int k = 0; k < XC; ++k) {
    const int i = threadIdx.x + k * NT;
    const int x0 = xo[k][0], x1 = xo[k][1], x2 = xo[k][2];
    real v2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < ZT; ++a) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int ab = a * 2 + b;
          if (s_rb[h][ab] >= 0) {
            const real* row = stage + (size_t)(h * NS + ab) * row_elems;
            acc += (double)row[x0];
            if (x1 >= 0) acc += (double)row[x1];
            if (x2 >= 0) acc += (double)row[x2];
          }
        }
        const long long b3 = s_rb[h][4 + a];
        if (b3 >= 0) {
          acc += (double)scratch[b3 + x0];
          if (x1 >= 0) acc += (double)scratch[b3 + x1];
          if (x2 >= 0) acc += (double)scratch[b3 + x2];
        }
      }
      v2[h] = (real)acc;
    }
    C z;
    z.x = v2[0];
    z.y = v2[1];
    buf[pidx(i)] = z;
  }
  __syncthreads();
  fft_ip<N, 1, 1, NT, -1>(buf, tw);
  for (int k = threadIdx.x; k < ldx; k += NT) {
    C A, B;
    A.x = A.y = B.x = B.y = real(0);
    if (k < nbx) {
      const C zk = buf[pidx(k)], zm = buf[pidx((N - k) % N)];
      A.x = real(0.5) * (zk.x + zm.x);   // (Zk + conj Zm) / 2
      A.y = real(0.5) * (zk.y - zm.y);
      B.x = real(0.5) * (zk.y + zm.y);   // (Zk - conj Zm) / 2i
      B.y = real(-0.5) * (zk.x - zm.x);
    }
    if (r0 < nrows) out[r0 * ldx + k] = A;
    if (r0 + 1 < nrows) out[(r0 + 1) * ldx + k] = B;
  }
}

// Distributed (z-slab) layout of the fused transforms.  R == 0: one GPU.
// Otherwise the in-band ky rows are split over the R ranks (by_start) and
// the z planes too (z_start); the forward y pass and the ik pass store
// straight into the destination rank's receive buffer (peers[r], reachable
// over NVLink peer memory): forward buffers are [Mz][ny_r][ldx], backward
// buffers [3][nz_r][nby][ldx].
constexpr int kMaxRanks = 8;
struct SlabMap {
  int R;
  int z0;                          // this rank's first global plane (forward pass)
  int by_start[kMaxRanks + 1];
  int z_start[kMaxRanks + 1];
  void* peers[kMaxRanks];
};

__device__ __forceinline__ int slab_owner(const int* start, int R, int v) {
  int r = 0;
  while (r + 1 < R && v >= start[r + 1]) ++r;
  return r;
}

// P2: y lines (z, kx) for kx < ldx: forward C2C, keep the nby in-band ky.
// in[(z*N + y)*ldx + kx] -> out[(z*nby + by)*ldx + kx].
template <typename real, int N>
__global__ void __launch_bounds__(threads_yz<real>(N), ESP_FFT_WARPLINES ? 2 : ESP_YZ_MINB)
k_y_fwd(const typename Cx<real>::t* __restrict__ in, typename Cx<real>::t* __restrict__ out,
        const typename Cx<real>::t* __restrict__ tw, long long nlines, int ldx, int nby,
        SlabMap smap) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N), LP = pitch(N), NT = threads_yz<real>(N);
  constexpr int YS = NT / L, nld = N / YS;
  static_assert(NT % L == 0 && N % YS == 0, "CTA shape");
  extern __shared__ __align__(16) unsigned char sm[];
  C* buf = reinterpret_cast<C*>(sm);
  const int l = threadIdx.x % L;           // fixed line per thread
  const long long line = (long long)blockIdx.x * L + l;
  const bool valid = line < nlines;
  const long long z = valid ? line / ldx : 0, kx = valid ? line - z * ldx : 0;
  const C* src = in + z * N * ldx + kx;
  C v[nld];
#pragma unroll
  for (int it = 0; it < nld; ++it) {
    const int y = threadIdx.x / L + it * YS;
    if (valid) v[it] = __ldcs(src + (long long)y * ldx);
    else v[it].x = v[it].y = real(0);
  }
#pragma unroll
  for (int it = 0; it < nld; ++it) buf[l * LP + pidx(threadIdx.x / L + it * YS)] = v[it];
  __syncthreads();
  fft_lines<N, L, NT, -1, true>(buf, tw);
  if (!valid) return;
  if (smap.R == 0) {
    C* dst = out + z * (long long)nby * ldx + kx;
    for (int by = threadIdx.x / L; by < nby; by += YS)
      dst[(long long)by * ldx] = buf[l * LP + pidx(band_mode(by, nby, N))];
  } else {   // transpose into the ky owner's buffer: [Mz][ny_r][ldx]
    const long long zg = smap.z0 + z;
    for (int by = threadIdx.x / L; by < nby; by += YS) {
      const int r = slab_owner(smap.by_start, smap.R, by);
      const int ny_r = smap.by_start[r + 1] - smap.by_start[r];
      C* dst = reinterpret_cast<C*>(smap.peers[r]);
      dst[(zg * ny_r + (by - smap.by_start[r])) * ldx + kx] =
          buf[l * LP + pidx(band_mode(by, nby, N))];
    }
  }
}

struct FusedArgs {
  int M[3];
  int nbx, nby, nbz, ldx;
  long long Hx;
  long long Msum;
  long long koff[3];
  const double* axis_k;
  const double* modeA;
  const double* modeB;
  double ik_scale;
  double escale, pscale;
  int by0, npy;        // pencil rows by0 .. by0+npy-1 of the in-band box (one GPU: 0, nby)
  int potential;       // 1: one potential spectrum A X h3/G (analytic forces) instead of ik x3
};

// Deterministic two-level completion of a per-block reduction: block b has
// written partials[b][0..6].  The last block to finish in each group of 32
// sums the group's partials in block order (lane j <- block 32g + j, then a
// fixed xor tree) into the group slot; the last group to finish sums the
// group slots the same way and writes out7.  Counters re-arm themselves.
// Layout (fixed by the allocated capacity, so launches of any size share
// it): partials [cap][8] | group sums [cap_groups][8] | counters.
__device__ __forceinline__ void tree_finish(double* partials, double* gsum, int* counters,
                                            double* out7, double escale, double pscale) {
  __shared__ int s_flag;
  const int nb = gridDim.x, g = blockIdx.x >> 5, ng = (nb + 31) >> 5;
  const int gsize = min(32, nb - (g << 5));
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_flag = atomicAdd(counters + g, 1) == gsize - 1;
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  const int lane = threadIdx.x;
  if (lane < 32) {
    double v[7];
#pragma unroll
    for (int i = 0; i < 7; ++i)
      v[i] = lane < gsize ? __ldcg(partials + (size_t)((g << 5) + lane) * 8 + i) : 0.0;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < 7; ++i) gsum[(size_t)g * 8 + i] = v[i];
      counters[g] = 0;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_flag = atomicAdd(counters + ng, 1) == ng - 1;
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  if (lane < 32) {
    double v[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) v[i] = 0.0;
    for (int j = lane; j < ng; j += 32) {
#pragma unroll
      for (int i = 0; i < 7; ++i) v[i] += __ldcg(gsum + (size_t)j * 8 + i);
    }
#pragma unroll
    for (int i = 0; i < 7; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
    if (lane == 0) {
      out7[0] = v[0] * escale;
      for (int i = 1; i < 7; ++i) out7[i] = v[i] * pscale;
      counters[ng] = 0;
    }
  }
}

// P3a: z pencils line = by*ldx + kx: forward C2C; the in-band kz box goes to
// spec (cuFFT half-spectrum layout) and into the fixed-order energy/pressure
// reduction (warp shuffle -> block -> per-block partials -> last block).
// IK (small pencils only): the same CTA then builds the ik (or potential)
// spectra of its pencils from the transformed values still in shared memory
// and runs their inverse z transforms (what k_z_ik does), saving a launch and
// the spectrum's round trip through memory.
template <typename real, int N, bool IK = false>
__global__ void __launch_bounds__(threads_yz<real>(N), ESP_YZ_MINB)
k_z_reduce(const typename Cx<real>::t* __restrict__ in, typename Cx<real>::t* __restrict__ spec,
           const typename Cx<real>::t* __restrict__ tw, FusedArgs fa, long long nlines,
           double* __restrict__ partials, double* __restrict__ gsum,
           int* __restrict__ counters, double* __restrict__ out7,
           typename Cx<real>::t* __restrict__ ik = nullptr) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N), LP = pitch(N), NT = threads_yz<real>(N);
  constexpr int ZS = NT / L, nld = N / ZS;
  static_assert(NT % L == 0 && N % ZS == 0, "CTA shape");
  extern __shared__ __align__(16) unsigned char sm[];
  C* X = reinterpret_cast<C*>(sm);
  const int ldx = fa.ldx, nbx = fa.nbx, nby = fa.nby, nbz = fa.nbz;
  const long long zstride = (long long)fa.npy * ldx;
  const int l = threadIdx.x % L;
  const long long line = (long long)blockIdx.x * L + l;
  const bool valid = line < nlines;
  int by = 0, mx = 0, my = 0;
  bool live = false;
  auto pencil = [&]() {   // (by, kx) of this thread's line
    const int byl = valid ? (int)(line / ldx) : 0;
    mx = valid ? (int)(line - (long long)byl * ldx) : 0;
    by = fa.by0 + byl;
    live = valid && mx < nbx;
    my = band_mode(by, nby, fa.M[1]);
  };
  // Mode tables: A, B and k_c = (K_c,x[mx] + K_c,y[my]) + K_c,z[mz] (the
  // order of mesh.py:242).  Masked modes have A = B = 0 and add exact zeros.
  // Small pencils (short latency chains, few CTAs) issue every table load
  // before the transform so that they overlap the input loads; large ones
  // load A, B, K_z after it (register budget).
  constexpr bool PF = nld <= 6;
  constexpr int NP = PF ? nld : 1;
  double pA[NP], pB[NP], pk[3][NP], kxy[3];
  if constexpr (PF) {
    pencil();
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double* K = fa.axis_k + c * fa.Msum;
      kxy[c] = live ? __dadd_rn(__ldg(K + fa.koff[0] + mx), __ldg(K + fa.koff[1] + my)) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < NP; ++it) {
      const int bz = threadIdx.x / L + it * ZS;
      pA[it] = pB[it] = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) pk[c][it] = 0.0;
      if (live && bz < nbz) {
        const long long be = ((long long)bz * nby + by) * nbx + mx;
        const int mz = band_mode(bz, nbz, N);
        pA[it] = __ldg(fa.modeA + be);
        pB[it] = __ldg(fa.modeB + be);
#pragma unroll
        for (int c = 0; c < 3; ++c) pk[c][it] = __ldg(fa.axis_k + c * fa.Msum + fa.koff[2] + mz);
      }
    }
  }
  {
    C v[nld];
#pragma unroll
    for (int it = 0; it < nld; ++it) {
      const int z = threadIdx.x / L + it * ZS;
      if (valid) v[it] = __ldcs(in + (long long)z * zstride + line);
      else v[it].x = v[it].y = real(0);
    }
#pragma unroll
    for (int it = 0; it < nld; ++it) X[l * LP + pidx(threadIdx.x / L + it * ZS)] = v[it];
  }
  __syncthreads();
  fft_lines<N, L, NT, -1, false>(X, tw);
  if constexpr (!PF) pencil();
  double acc[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) acc[i] = 0.0;
  if (live) {
    const double wx = (mx == 0 || 2 * mx == fa.M[0]) ? 1.0 : 2.0;
    if constexpr (PF) {
#pragma unroll
      for (int it = 0; it < NP; ++it) {
        const int bz = threadIdx.x / L + it * ZS;
        if (bz >= nbz) continue;
        const int mz = band_mode(bz, nbz, N);
        const C Xv = X[l * LP + pidx(mz)];
        spec[((long long)mz * fa.M[1] + my) * fa.Hx + mx] = Xv;
        const double A = pA[it], B = pB[it];
        if (A == 0.0) continue;
        const double xr = (double)Xv.x, xi = (double)Xv.y;
        const double w = wx * (xr * xr + xi * xi);
        const double kx = __dadd_rn(kxy[0], pk[0][it]), ky = __dadd_rn(kxy[1], pk[1][it]),
                     kz = __dadd_rn(kxy[2], pk[2][it]);
        const double wa = w * A, t = w * B;
        acc[0] += wa;
        acc[1] += t * kx * kx + wa;
        acc[2] += t * kx * ky;
        acc[3] += t * kx * kz;
        acc[4] += t * ky * ky + wa;
        acc[5] += t * ky * kz;
        acc[6] += t * kz * kz + wa;
      }
    } else {
      const double* Kz[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double* K = fa.axis_k + c * fa.Msum;
        kxy[c] = __dadd_rn(__ldg(K + fa.koff[0] + mx), __ldg(K + fa.koff[1] + my));
        Kz[c] = K + fa.koff[2];
      }
      for (int bz = threadIdx.x / L; bz < nbz; bz += ZS) {
        const int mz = band_mode(bz, nbz, N);
        const C Xv = X[l * LP + pidx(mz)];
        spec[((long long)mz * fa.M[1] + my) * fa.Hx + mx] = Xv;
        const long long be = ((long long)bz * nby + by) * nbx + mx;
        const double A = __ldg(fa.modeA + be);
        if (A == 0.0) continue;
        const double B = __ldg(fa.modeB + be);
        const double xr = (double)Xv.x, xi = (double)Xv.y;
        const double w = wx * (xr * xr + xi * xi);
        const double kx = __dadd_rn(kxy[0], __ldg(Kz[0] + mz)),
                     ky = __dadd_rn(kxy[1], __ldg(Kz[1] + mz)),
                     kz = __dadd_rn(kxy[2], __ldg(Kz[2] + mz));
        const double wa = w * A, t = w * B;
        acc[0] += wa;
        acc[1] += t * kx * kx + wa;
        acc[2] += t * kx * ky;
        acc[3] += t * kx * kz;
        acc[4] += t * ky * ky + wa;
        acc[5] += t * ky * kz;
        acc[6] += t * kz * kz + wa;
      }
    }
  }
  if constexpr (IK && PF) {
    // ik pencils: T = i k_c A X h3/G (or A X h3/G, potential) on the in-band
    // modes, zero elsewhere; inverse z transform; store as k_z_ik does
    C* T = X + L * LP;
    const int ncomp = fa.potential ? 1 : 3;
    for (int c = 0; c < ncomp; ++c) {
#pragma unroll
      for (int it = 0; it < nld; ++it) {
        C z;
        z.x = z.y = real(0);
        T[l * LP + pidx(threadIdx.x / L + it * ZS)] = z;
      }
      __syncthreads();
      if (live) {
#pragma unroll
        for (int it = 0; it < NP; ++it) {
          const int bz = threadIdx.x / L + it * ZS;
          if (bz >= nbz) continue;
          const int mz = band_mode(bz, nbz, N);
          const C Xv = X[l * LP + pidx(mz)];
          C v;
          if (fa.potential) {
            const double cf = pA[it] * fa.ik_scale;
            v.x = (real)(cf * (double)Xv.x);
            v.y = (real)(cf * (double)Xv.y);
          } else {
            const double kc = c == 0 ? __dadd_rn(kxy[0], pk[0][it])
                                     : (c == 1 ? __dadd_rn(kxy[1], pk[1][it])
                                               : __dadd_rn(kxy[2], pk[2][it]));
            const double cf = pA[it] * fa.ik_scale * kc;
            v.x = (real)(-cf * (double)Xv.y);
            v.y = (real)(cf * (double)Xv.x);
          }
          T[l * LP + pidx(mz)] = v;
        }
      }
      __syncthreads();
      fft_lines<N, L, NT, +1, false>(T, tw);
      if (valid) {
        C* dst = ik + (long long)c * N * zstride + line;
#pragma unroll
        for (int it = 0; it < nld; ++it) {
          const int z = threadIdx.x / L + it * ZS;
          __stcs(dst + (long long)z * zstride, T[l * LP + pidx(z)]);
        }
      }
      __syncthreads();
    }
  }
  constexpr int NW = (NT + 31) / 32;
  __shared__ double red[NW][7];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 7; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 7; ++i) red[warp][i] = acc[i];
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][threadIdx.x];
    partials[(size_t)blockIdx.x * 8 + threadIdx.x] = s;
  }
  tree_finish(partials, gsum, counters, out7, fa.escale, fa.pscale);
}

// P3b: ik pencils, one force component per blockIdx.y: i k_c A X h3/G on the
// retained modes (zero elsewhere, mesh.py:333-341), inverse C2C along z ->
// ik[c][z][by][kx].  X is the box spectrum P3a wrote.
template <typename real, int N>
__global__ void __launch_bounds__(threads_yz<real>(N), ESP_YZ_MINB)
k_z_ik(const typename Cx<real>::t* __restrict__ spec, typename Cx<real>::t* __restrict__ ik,
       const typename Cx<real>::t* __restrict__ tw, FusedArgs fa, long long nlines,
       SlabMap smap) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N), LP = pitch(N), NT = threads_yz<real>(N);
  constexpr int ZS = NT / L, nld = N / ZS;
  extern __shared__ __align__(16) unsigned char sm[];
  C* T = reinterpret_cast<C*>(sm);
  const int comp = blockIdx.y;
  const int ldx = fa.ldx, nbx = fa.nbx, nby = fa.nby, nbz = fa.nbz;
  const long long zstride = (long long)fa.npy * ldx;
  const int l = threadIdx.x % L;
  const long long line = (long long)blockIdx.x * L + l;
  const bool valid = line < nlines;
  const int byl = valid ? (int)(line / ldx) : 0;
  const int mx = valid ? (int)(line - (long long)byl * ldx) : 0;
  const int by = fa.by0 + byl;
  const bool live = valid && mx < nbx;
  const int my = band_mode(by, nby, fa.M[1]);
  const double* K = fa.axis_k + comp * fa.Msum;
  const double kxy = live ? __dadd_rn(K[fa.koff[0] + mx], K[fa.koff[1] + my]) : 0.0;
  {
    C v[nld];
#pragma unroll
    for (int it = 0; it < nld; ++it) {
      const int mz = threadIdx.x / L + it * ZS;
      v[it].x = v[it].y = real(0);
      const int bz = band_index(mz, nbz, N);
      if (live && bz >= 0) {
        const double A = __ldg(fa.modeA + ((long long)bz * nby + by) * nbx + mx);
        const C Xv = __ldg(spec + ((long long)mz * fa.M[1] + my) * fa.Hx + mx);
        if (fa.potential) {   // analytic forces: A X h3/G (mesh.py:344-346)
          const double cf = A * fa.ik_scale;
          v[it].x = (real)(cf * (double)Xv.x);
          v[it].y = (real)(cf * (double)Xv.y);
        } else {              // ik forces: i k_d A X h3/G
          const double cf = A * fa.ik_scale * __dadd_rn(kxy, __ldg(K + fa.koff[2] + mz));
          v[it].x = (real)(-cf * (double)Xv.y);
          v[it].y = (real)(cf * (double)Xv.x);
        }
      }
    }
#pragma unroll
    for (int it = 0; it < nld; ++it) T[l * LP + pidx(threadIdx.x / L + it * ZS)] = v[it];
  }
  __syncthreads();
  fft_lines<N, L, NT, +1, false>(T, tw);
  if (!valid) return;
  if (smap.R == 0) {
    C* dst = ik + (long long)comp * N * zstride + line;
#pragma unroll
    for (int it = 0; it < nld; ++it) {
      const int z = threadIdx.x / L + it * ZS;
      __stcs(dst + (long long)z * zstride, T[l * LP + pidx(z)]);
    }
  } else {   // transpose back into the plane owner's buffer: [3][nz_r][nby][ldx]
#pragma unroll 4
    for (int it = 0; it < nld; ++it) {
      const int z = threadIdx.x / L + it * ZS;
      const int r = slab_owner(smap.z_start, smap.R, z);
      const int nz_r = smap.z_start[r + 1] - smap.z_start[r];
      C* dst = reinterpret_cast<C*>(smap.peers[r]);
      dst[(((long long)comp * nz_r + (z - smap.z_start[r])) * nby + by) * ldx + mx] =
          T[l * LP + pidx(z)];
    }
  }
}

// P4: y lines (c, z, kx): inverse C2C from the nby in-band ky rows (zero
// elsewhere).  in[(cz*nby + by)*ldx + kx] -> out[(cz*N + y)*ldx + kx].
template <typename real, int N>
__global__ void __launch_bounds__(threads_yz<real>(N), ESP_YZ_MINB)
k_y_inv(const typename Cx<real>::t* __restrict__ in, typename Cx<real>::t* __restrict__ out,
        const typename Cx<real>::t* __restrict__ tw, long long nlines, int ldx, int nby) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N), LP = pitch(N), NT = threads_yz<real>(N);
  constexpr int YS = NT / L, nld = N / YS;
  static_assert(NT % L == 0 && N % YS == 0, "CTA shape");
  extern __shared__ __align__(16) unsigned char sm[];
  C* buf = reinterpret_cast<C*>(sm);
  const int l = threadIdx.x % L;
  const long long line = (long long)blockIdx.x * L + l;
  const bool valid = line < nlines;
  const long long cz = valid ? line / ldx : 0, kx = valid ? line - cz * ldx : 0;
  const C* src = in + cz * (long long)nby * ldx + kx;
  C v[nld];
#pragma unroll
  for (int it = 0; it < nld; ++it) {
    const int y = threadIdx.x / L + it * YS;
    const int by = band_index(y, nby, N);
    if (valid && by >= 0) v[it] = __ldcs(src + (long long)by * ldx);
    else v[it].x = v[it].y = real(0);
  }
#pragma unroll
  for (int it = 0; it < nld; ++it) buf[l * LP + pidx(threadIdx.x / L + it * YS)] = v[it];
  __syncthreads();
  fft_lines<N, L, NT, +1, false>(buf, tw);
  if (!valid) return;
  C* dst = out + cz * (long long)N * ldx + kx;
#pragma unroll
  for (int it = 0; it < nld; ++it) {
    const int y = threadIdx.x / L + it * YS;
    dst[(long long)y * ldx] = buf[l * LP + pidx(y)];
  }
}

// P5: x rows, complex -> real, two rows per transform; columns kx < nbx
// (zero-padded to the half spectrum; kx = 0 and Nyquist taken as real, as a
// C2R transform does).  Each in-band column is read once and placed at k and
// N - k (conjugate-symmetric extension).
// Ghost-padded field rows (esp_gather_tma.cu): row `ra` = (c*Mz + z)*My + y
// of the fields lands at up to 4 padded rows (its y and z periodic images);
// the CTA precomputes their base offsets once, so each element store is one
// add (plus its x image near the row ends).
__host__ __device__ constexpr int pad_rows_smem(int PP) { return 2 * PP; }

struct PadRows {
  long long base[4];
  int n;
};

__device__ __forceinline__ PadRows pad_rows(const FieldPad& f, int ra) {
  const int My = f.M[1], Mz = f.M[2];
  const int c = ra / (My * Mz);
  const int rem = ra - c * My * Mz;
  const int z = rem / My, y = rem - z * My;
  int ys[2], zs[2], ny = 0, nz = 0;
  ys[ny++] = y + f.S[1];
  if (y + f.S[1] + My < f.E[1]) ys[ny++] = y + f.S[1] + My;
  else if (y + f.S[1] - My >= 0) ys[ny++] = y + f.S[1] - My;
  zs[nz++] = z + f.S[2];
  if (z + f.S[2] + Mz < f.E[2]) zs[nz++] = z + f.S[2] + Mz;
  else if (z + f.S[2] - Mz >= 0) zs[nz++] = z + f.S[2] - Mz;
  PadRows r;
  r.n = 0;
  for (int a = 0; a < nz; ++a)
    for (int b = 0; b < ny; ++b)
      r.base[r.n++] = (long long)c * f.cstride + ((long long)zs[a] * f.E[1] + ys[b]) * f.E[0] +
                      f.S[0];
  return r;
}

template <typename real>
__device__ __forceinline__ void store_padded(const FieldPad& f, const PadRows& r,
                                             real* __restrict__ fld, int x, real v) {
  const int Mx = f.M[0];
  const int xi = x + f.S[0] + Mx < f.E[0] ? Mx : (x + f.S[0] - Mx >= 0 ? -Mx : 0);
  __stcs(fld + r.base[0] + x, v);
  if (xi) __stcs(fld + r.base[0] + x + xi, v);
  if (r.n > 1) {                          // y / z ghost rows (a few rows per plane)
    for (int k = 1; k < r.n; ++k) {
      __stcs(fld + r.base[k] + x, v);
      if (xi) __stcs(fld + r.base[k] + x + xi, v);
    }
  }
}

template <typename real, int N>
__global__ void __launch_bounds__(kThreadsX, ESP_X_MINB)
k_x_c2r(const typename Cx<real>::t* __restrict__ in, real* __restrict__ fld,
        const typename Cx<real>::t* __restrict__ tw, long long nrows, int ldx, int nbx,
        FieldPad pad) {
  using C = typename Cx<real>::t;
  constexpr int PP = pairs_x(N), LP = pitch(N), NT = kThreadsX;
  constexpr int half = N / 2, NH = half + 1;
  __shared__ C buf[PP * LP];
  const long long r0 = 2LL * blockIdx.x * PP;
  // in-band columns: thread k < nbx loads column k of every row of the CTA
  // (all loads first), places Z_k = A + i B and its mirror Z_{N-k}; the
  // out-of-band entries nbx .. N - nbx of each line are zero-filled
  if (nbx <= NT) {
    C va[PP], vb[PP];
    const int k = threadIdx.x;
    if (k < nbx) {
#pragma unroll
      for (int l = 0; l < PP; ++l) {
        const long long ra = r0 + 2 * l;
        va[l].x = va[l].y = vb[l].x = vb[l].y = real(0);
        if (ra < nrows) va[l] = __ldcs(in + ra * ldx + k);
        if (ra + 1 < nrows) vb[l] = __ldcs(in + (ra + 1) * ldx + k);
      }
    }
    for (int e = threadIdx.x; e < PP * (N + 1 - 2 * nbx); e += NT) {
      const int l = e / (N + 1 - 2 * nbx), i = nbx + (e - l * (N + 1 - 2 * nbx));
      C z;
      z.x = z.y = real(0);
      buf[l * LP + pidx(i)] = z;
    }
    if (k < nbx) {
#pragma unroll
      for (int l = 0; l < PP; ++l) {
        C A = va[l], B = vb[l];
        if (k == 0 || k == half) {
          A.y = real(0);
          B.y = real(0);
        }
        C z;   // Z_k = A + i B
        z.x = A.x - B.y;
        z.y = A.y + B.x;
        buf[l * LP + pidx(k)] = z;
        if (k != 0 && k != half) {   // Z_{N-k} = conj A + i conj B
          z.x = A.x + B.y;
          z.y = B.x - A.y;
          buf[l * LP + pidx(N - k)] = z;
        }
      }
    }
  } else {
  constexpr int nhl = (PP * NH + NT - 1) / NT;
  C va[nhl], vb[nhl];
#pragma unroll
  for (int it = 0; it < nhl; ++it) {
    const int e = threadIdx.x + it * NT;
    const int l = e / NH, k = e - l * NH;
    const long long ra = r0 + 2 * l;
    va[it].x = va[it].y = vb[it].x = vb[it].y = real(0);
    if (e < PP * NH && k < nbx) {
      if (ra < nrows) va[it] = __ldcs(in + ra * ldx + k);
      if (ra + 1 < nrows) vb[it] = __ldcs(in + (ra + 1) * ldx + k);
    }
  }
#pragma unroll
  for (int it = 0; it < nhl; ++it) {
    const int e = threadIdx.x + it * NT;
    if (e < PP * NH) {
      const int l = e / NH, k = e - l * NH;
      C A = va[it], B = vb[it];
      if (k == 0 || k == half) {
        A.y = real(0);
        B.y = real(0);
      }
      C z;   // Z_k = A + i B
      z.x = A.x - B.y;
      z.y = A.y + B.x;
      buf[l * LP + pidx(k)] = z;
      if (k != 0 && k != half) {   // Z_{N-k} = conj A + i conj B
        z.x = A.x + B.y;
        z.y = B.x - A.y;
        buf[l * LP + pidx(N - k)] = z;
      }
    }
  }
  }
  __shared__ PadRows s_rows[pad_rows_smem(PP)];
  if (pad.enabled && threadIdx.x < 2 * PP && r0 + threadIdx.x < nrows)
    s_rows[threadIdx.x] = pad_rows(pad, (int)(r0 + threadIdx.x));
  __syncthreads();
  fft_ip<N, 1, PP, NT, +1>(buf, tw);
  constexpr int nld = (PP * N + NT - 1) / NT;
  if constexpr (N % NT == 0) {
    // a thread's elements are its N / NT columns of every row pair: the x
    // ghost image of each column is looked up once, the row bases come from
    // shared memory, and a row's y / z ghost copies (a few rows per plane)
    // take the general store (config 4: the store phase was half of this
    // kernel's instructions)
    constexpr int XC = N / NT;
    if (pad.enabled) {
      int xi[XC];
#pragma unroll
      for (int k = 0; k < XC; ++k) {
        const int x = threadIdx.x + k * NT;
        xi[k] = x + pad.S[0] + N < pad.E[0] ? N : (x + pad.S[0] - N >= 0 ? -N : 0);
      }
#pragma unroll
      for (int l = 0; l < PP; ++l) {
        const bool okA = r0 + 2 * l < nrows, okB = r0 + 2 * l + 1 < nrows;
        const PadRows& rA = s_rows[2 * l];
        const PadRows& rB = s_rows[2 * l + 1];
        real* rowA = fld + (okA ? rA.base[0] : 0);
        real* rowB = fld + (okB ? rB.base[0] : 0);
        const int nA = okA ? rA.n : 0, nB = okB ? rB.n : 0;
#pragma unroll
        for (int k = 0; k < XC; ++k) {
          const int x = threadIdx.x + k * NT;
          const C z = buf[l * LP + pidx(x)];
          if (okA) {
            __stcs(rowA + x, z.x);
            if (xi[k]) __stcs(rowA + x + xi[k], z.x);
          }
          if (okB) {
            __stcs(rowB + x, z.y);
            if (xi[k]) __stcs(rowB + x + xi[k], z.y);
          }
          if (nA > 1 || nB > 1) {   // y / z ghost copies of these rows
            for (int m = 1; m < nA; ++m) {
              __stcs(fld + rA.base[m] + x, z.x);
              if (xi[k]) __stcs(fld + rA.base[m] + x + xi[k], z.x);
            }
            for (int m = 1; m < nB; ++m) {
              __stcs(fld + rB.base[m] + x, z.y);
              if (xi[k]) __stcs(fld + rB.base[m] + x + xi[k], z.y);
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int l = 0; l < PP; ++l) {
        const long long ra = r0 + 2 * l;
#pragma unroll
        for (int k = 0; k < XC; ++k) {
          const int x = threadIdx.x + k * NT;
          const C z = buf[l * LP + pidx(x)];
          if (ra < nrows) __stcs(fld + ra * N + x, z.x);
          if (ra + 1 < nrows) __stcs(fld + (ra + 1) * N + x, z.y);
        }
      }
    }
  } else {
#pragma unroll 4
    for (int it = 0; it < nld; ++it) {
      const int e = threadIdx.x + it * NT;
      if ((PP * N) % NT == 0 || e < PP * N) {
        const int l = e / N, i = e - l * N;
        const long long ra = r0 + 2 * l;
        const C z = buf[l * LP + pidx(i)];
        if (pad.enabled) {
          if (ra < nrows) store_padded(pad, s_rows[2 * l], fld, i, z.x);
          if (ra + 1 < nrows) store_padded(pad, s_rows[2 * l + 1], fld, i, z.y);
        } else {
          if (ra < nrows) __stcs(fld + ra * N + i, z.x);
          if (ra + 1 < nrows) __stcs(fld + (ra + 1) * N + i, z.y);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Small square planes (Mx == My <= 64): the x and y passes of one z plane in
// ONE CTA (the whole plane fits in shared memory), forward and inverse.  Two
// passes and two global round trips fewer on the latency-bound small grids.

// P1+P2: plane z -> out[(z*nby + by)*ldx + kx] (kx >= nbx written as zero).
template <typename real, int N>
__global__ void __launch_bounds__(256)
k_xy_fwd(const real* __restrict__ grid, typename Cx<real>::t* __restrict__ out,
         const typename Cx<real>::t* __restrict__ tw, int ldx, int nbx, int nby) {
  using C = typename Cx<real>::t;
  constexpr int LP = pitch(N), NH = N / 2 + 1, NP = N / 2, NT = 256;
  extern __shared__ __align__(16) unsigned char sm[];
  C* A = reinterpret_cast<C*>(sm);          // NP row pairs x N (x along the line)
  C* B = A + NP * LP;                       // NH kx columns x N (y along the line)
  const real* g = grid + (long long)blockIdx.x * N * N;
  for (int e = threadIdx.x; e < NP * N; e += NT) {
    const int pr = e / N, x = e - pr * N;
    C z;
    z.x = __ldcs(g + (2 * pr) * N + x);
    z.y = __ldcs(g + (2 * pr + 1) * N + x);
    A[pr * LP + pidx(x)] = z;
  }
  __syncthreads();
  fft_ip<N, 1, NP, NT, -1>(A, tw);
  for (int e = threadIdx.x; e < NP * NH; e += NT) {
    const int pr = e / NH, k = e - pr * NH;
    C a, b;
    a.x = a.y = b.x = b.y = real(0);
    if (k < nbx) {
      const C zk = A[pr * LP + pidx(k)], zm = A[pr * LP + pidx((N - k) % N)];
      a.x = real(0.5) * (zk.x + zm.x);
      a.y = real(0.5) * (zk.y - zm.y);
      b.x = real(0.5) * (zk.y + zm.y);
      b.y = real(-0.5) * (zk.x - zm.x);
    }
    B[k * LP + pidx(2 * pr)] = a;
    B[k * LP + pidx(2 * pr + 1)] = b;
  }
  __syncthreads();
  fft_ip<N, 1, NH, NT, -1>(B, tw);
  C* dst = out + (long long)blockIdx.x * nby * ldx;
  for (int e = threadIdx.x; e < nby * ldx; e += NT) {
    const int by = e / ldx, kx = e - by * ldx;
    C v;
    v.x = v.y = real(0);
    if (kx < nbx) v = B[kx * LP + pidx(band_mode(by, nby, N))];
    dst[e] = v;
  }
}

// P4+P5: plane cz = comp*Mz + z: in[(cz*nby + by)*ldx + kx] -> real rows of
// field comp.
template <typename real, int N>
__global__ void __launch_bounds__(256)
k_yx_inv(const typename Cx<real>::t* __restrict__ in, real* __restrict__ fld,
         const typename Cx<real>::t* __restrict__ tw, int ldx, int nbx, int nby) {
  using C = typename Cx<real>::t;
  constexpr int LP = pitch(N), NH = N / 2 + 1, NP = N / 2, NT = 256, half = N / 2;
  extern __shared__ __align__(16) unsigned char sm[];
  C* A = reinterpret_cast<C*>(sm);
  C* B = A + NP * LP;
  const C* src = in + (long long)blockIdx.x * nby * ldx;
  for (int e = threadIdx.x; e < NH * N; e += NT) {   // B[kx][y], zero outside the band
    const int k = e / N, y = e - k * N;
    const int by = band_index(y, nby, N);
    C v;
    v.x = v.y = real(0);
    if (k < nbx && by >= 0) v = src[by * ldx + k];
    B[k * LP + pidx(y)] = v;
  }
  __syncthreads();
  fft_ip<N, 1, NH, NT, +1>(B, tw);
  for (int e = threadIdx.x; e < NP * N; e += NT) {   // Z = A + i B rows, Hermitian extension
    const int pr = e / N, k = e - pr * N;
    const int kk = k <= half ? k : N - k;
    C a = B[kk * LP + pidx(2 * pr)], b = B[kk * LP + pidx(2 * pr + 1)];
    if (kk == 0 || kk == half) {
      a.y = real(0);
      b.y = real(0);
    }
    if (k > half) {
      a.y = -a.y;
      b.y = -b.y;
    }
    C z;
    z.x = a.x - b.y;
    z.y = a.y + b.x;
    A[pr * LP + pidx(k)] = z;
  }
  __syncthreads();
  fft_ip<N, 1, NP, NT, +1>(A, tw);
  real* f = fld + (long long)blockIdx.x * N * N;
  for (int e = threadIdx.x; e < NP * N; e += NT) {
    const int pr = e / N, x = e - pr * N;
    const C z = A[pr * LP + pidx(x)];
    __stcs(f + (2 * pr) * N + x, z.x);
    __stcs(f + (2 * pr + 1) * N + x, z.y);
  }
}

// ---------------------------------------------------------------------------
// Host side

static bool supported(int n) {
  switch (n) {
#define ESP_CASE(v) case v:
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
    return true;
    default:
      return false;
  }
}

// Per-stage twiddles in the kernels' order: for each stage with span Ns > 1
// and radix R, entries [(t-1)*Ns + k] = e^{-2 pi i t k / (Ns R)}.
static std::vector<double2> twiddles(int n) {
  std::vector<double2> h;
  int Ns = 1;
  while (Ns < n) {
    const int R = pick_radix(n / Ns);
    if (Ns > 1)
      for (int t = 1; t < R; ++t)
        for (int k = 0; k < Ns; ++k) {
          const double a = -2.0 * 3.14159265358979323846 * (double)(t * k) / (double)(Ns * R);
          h.push_back(make_double2(std::cos(a), std::sin(a)));
        }
    Ns *= R;
  }
  if (h.empty()) h.push_back(make_double2(1.0, 0.0));
  return h;
}

template <typename real, int N>
static cudaError_t launch_x_r2c(const esp_plan* p, const void* grid, void* out, const void* tw,
                                int ldx, int nz, cudaStream_t s) {
  using C = typename Cx<real>::t;
  constexpr int PP = pairs_x(N);
  const long long nrows = (long long)p->M[1] * nz;
  const long long nblk = (nrows + 2 * PP - 1) / (2 * PP);
  k_x_r2c<real, N><<<(unsigned)nblk, kThreadsX, 0, s>>>(
      reinterpret_cast<const real*>(grid), reinterpret_cast<C*>(out),
      reinterpret_cast<const C*>(tw), nrows, ldx, p->nbx);
  return cudaGetLastError();
}

template <typename real, int N>
static cudaError_t launch_x_comb_r2c(const esp_plan* p, void* out, const void* tw, int ldx,
                                     int nz, cudaStream_t s) {
  using C = typename Cx<real>::t;
  constexpr int PP = pairs_x(N);
  const long long nrows = (long long)p->M[1] * nz;
  const long long nblk = (nrows + 2 * PP - 1) / (2 * PP);
  k_x_comb_r2c<real, N><<<(unsigned)nblk, kThreadsX, 0, s>>>(
      make_geom(p), combine_tabs(p), reinterpret_cast<const real*>(p->d_scratch),
      reinterpret_cast<C*>(out), reinterpret_cast<const C*>(tw), nrows, ldx, p->nbx);
  return cudaGetLastError();
}

// Bulk-staged variant for the long rows (N a multiple of 64, >= 192): the
// scratch rows plus the FFT line in dynamic shared memory.  With My even the
// planes under one z tile and the planes under two run as two launches (4 and
// 8 staged rows per pair: seven and four CTAs per SM); otherwise one launch
// stages 8 rows for every pair.
template <typename real, int N>
static cudaError_t launch_x_bulk_r2c(const esp_plan* p, void* out, const void* tw, int ldx,
                                     int nz, cudaStream_t s, bool* taken) {
  using C = typename Cx<real>::t;
  *taken = false;
  if constexpr (N % 64 == 0 && N >= 192) {
    static const bool off = std::getenv("ESP_NO_XBULK") != nullptr;   // A/B diagnostics
    static const bool one_class = std::getenv("ESP_XBULK_ONE") != nullptr;
    const Geom g = make_geom(p);
    const size_t row = (size_t)g.ntx * kPad * sizeof(real);
    const size_t smem8 = ((8 * row + 15) & ~size_t(15)) + sizeof(C) * pitch(N);
    const size_t smem4 = ((4 * row + 15) & ~size_t(15)) + sizeof(C) * pitch(N);
    if (off || smem8 > 56 * 1024 || p->comb_max[0] > 3 || p->comb_max[1] > 3 ||
        p->comb_max[2] > 2)
      return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_x_bulk_r2c<real, N, 2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_x_bulk_r2c<real, N, 1>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4);
    if (e != cudaSuccess) return e;
    const long long nrows = (long long)p->M[1] * nz;
    if (!one_class && p->M[1] % 2 == 0 && nz == p->M[2] && p->d_zlist && p->n_z_single > 0) {
      const long long ppp = p->M[1] / 2;
      const long long n1 = p->n_z_single * ppp, n2 = (p->M[2] - p->n_z_single) * ppp;
      k_x_bulk_r2c<real, N, 1><<<(unsigned)n1, threads_xb(N), smem4, s>>>(
          g, combine_tabs(p), reinterpret_cast<const real*>(p->d_scratch),
          reinterpret_cast<C*>(out), reinterpret_cast<const C*>(tw), nrows, ldx, p->nbx,
          p->d_zlist);
      if (n2 > 0) const_cast<esp_plan*>(p)->launches++;   // the caller counts one
      if (n2 > 0)
        k_x_bulk_r2c<real, N, 2><<<(unsigned)n2, threads_xb(N), smem8, s>>>(
            g, combine_tabs(p), reinterpret_cast<const real*>(p->d_scratch),
            reinterpret_cast<C*>(out), reinterpret_cast<const C*>(tw), nrows, ldx, p->nbx,
            p->d_zlist + p->n_z_single);
    } else {
      k_x_bulk_r2c<real, N, 2><<<(unsigned)((nrows + 1) / 2), threads_xb(N), smem8, s>>>(
          g, combine_tabs(p), reinterpret_cast<const real*>(p->d_scratch),
          reinterpret_cast<C*>(out), reinterpret_cast<const C*>(tw), nrows, ldx, p->nbx, nullptr);
    }
    *taken = true;
    return cudaGetLastError();
  }
  return cudaSuccess;
}

template <typename real, int N>
static cudaError_t launch_y_fwd(const esp_plan* p, const void* in, void* out, const void* tw,
                                int ldx, int nz, const SlabMap& smap, cudaStream_t s) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N);
  const long long nlines = (long long)nz * ldx;
  const size_t smem = sizeof(C) * L * pitch(N);
  cudaError_t e = cudaFuncSetAttribute(k_y_fwd<real, N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_y_fwd<real, N><<<(unsigned)((nlines + L - 1) / L), threads_yz<real>(N), smem, s>>>(
      reinterpret_cast<const C*>(in), reinterpret_cast<C*>(out), reinterpret_cast<const C*>(tw),
      nlines, ldx, p->nby, smap);
  return cudaGetLastError();
}

// Small pencils (the table prefetch branch of k_z_reduce): the ik spectra and
// their inverse z transforms can ride in the same kernel.
template <typename real, int N>
constexpr bool z_fusable() {
  return N / (threads_yz<real>(N) / lines_yz<real>(N)) <= 6;
}

template <typename real, int N>
static cudaError_t launch_z_reduce(const esp_plan* p, const void* in, const void* tw,
                                   const FusedArgs& fa, double* partials, long long nblk_cap,
                                   double* out7, cudaStream_t s, void* ik = nullptr) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N);
  const long long nlines = (long long)fa.npy * fa.ldx;
  const long long nblk = (nlines + L - 1) / L;
  if (nblk > nblk_cap) return cudaErrorInvalidConfiguration;
  int* counters = reinterpret_cast<int*>(partials + (nblk_cap + (nblk_cap + 31) / 32) * 8);
  if constexpr (z_fusable<real, N>()) {
    if (ik) {
      const size_t smem = 2 * sizeof(C) * L * pitch(N);
      cudaError_t e = cudaFuncSetAttribute(k_z_reduce<real, N, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      k_z_reduce<real, N, true><<<(unsigned)nblk, threads_yz<real>(N), smem, s>>>(
          reinterpret_cast<const C*>(in), reinterpret_cast<C*>(p->d_spec),
          reinterpret_cast<const C*>(tw), fa, nlines, partials, partials + nblk_cap * 8,
          counters, out7, reinterpret_cast<C*>(ik));
      return cudaGetLastError();
    }
  }
  const size_t smem = sizeof(C) * L * pitch(N);
  cudaError_t e = cudaFuncSetAttribute(k_z_reduce<real, N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_z_reduce<real, N><<<(unsigned)nblk, threads_yz<real>(N), smem, s>>>(
      reinterpret_cast<const C*>(in), reinterpret_cast<C*>(p->d_spec),
      reinterpret_cast<const C*>(tw), fa, nlines, partials, partials + nblk_cap * 8,
      counters, out7);
  return cudaGetLastError();
}

template <typename real, int N>
static cudaError_t launch_z_ik(const esp_plan* p, void* ik, const void* tw, const FusedArgs& fa,
                               const SlabMap& smap, cudaStream_t s) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N);
  const size_t smem = sizeof(C) * L * pitch(N);
  cudaError_t e = cudaFuncSetAttribute(k_z_ik<real, N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long nlines = (long long)fa.npy * fa.ldx;
  const dim3 grid((unsigned)((nlines + L - 1) / L), fa.potential ? 1 : 3);
  k_z_ik<real, N><<<grid, threads_yz<real>(N), smem, s>>>(
      reinterpret_cast<const C*>(p->d_spec), reinterpret_cast<C*>(ik),
      reinterpret_cast<const C*>(tw), fa, nlines, smap);
  return cudaGetLastError();
}

template <typename real, int N>
static cudaError_t launch_y_inv(const esp_plan* p, const void* in, void* out, const void* tw,
                                int ldx, int nz, cudaStream_t s, int ncomp = 3) {
  using C = typename Cx<real>::t;
  constexpr int L = lines_yz<real>(N);
  const long long nlines = (long long)ncomp * nz * ldx;
  const size_t smem = sizeof(C) * L * pitch(N);
  cudaError_t e = cudaFuncSetAttribute(k_y_inv<real, N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_y_inv<real, N><<<(unsigned)((nlines + L - 1) / L), threads_yz<real>(N), smem, s>>>(
      reinterpret_cast<const C*>(in), reinterpret_cast<C*>(out), reinterpret_cast<const C*>(tw),
      nlines, ldx, p->nby);
  return cudaGetLastError();
}

template <typename real, int N>
static cudaError_t launch_x_c2r(const esp_plan* p, const void* in, void* fld, const void* tw,
                                int ldx, int nz, cudaStream_t s, int ncomp = 3,
                                FieldPad pad = FieldPad{}) {
  using C = typename Cx<real>::t;
  constexpr int PP = pairs_x(N);
  const long long nrows = (long long)ncomp * p->M[1] * nz;
  const long long nblk = (nrows + 2 * PP - 1) / (2 * PP);
  k_x_c2r<real, N><<<(unsigned)nblk, kThreadsX, 0, s>>>(
      reinterpret_cast<const C*>(in), reinterpret_cast<real*>(fld),
      reinterpret_cast<const C*>(tw), nrows, ldx, p->nbx, pad);
  return cudaGetLastError();
}

template <typename real, int N>
static size_t plane_smem() {
  using C = typename Cx<real>::t;
  return sizeof(C) * (size_t)(N / 2 + N / 2 + 1) * pitch(N);
}

template <typename real, int N>
static cudaError_t launch_xy_fwd(const esp_plan* p, void* out, const void* tw, int ldx,
                                 cudaStream_t s) {
  using C = typename Cx<real>::t;
  const size_t smem = plane_smem<real, N>();
  cudaError_t e = cudaFuncSetAttribute(k_xy_fwd<real, N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_xy_fwd<real, N><<<(unsigned)p->M[2], 256, smem, s>>>(
      reinterpret_cast<const real*>(p->d_grid), reinterpret_cast<C*>(out),
      reinterpret_cast<const C*>(tw), ldx, p->nbx, p->nby);
  return cudaGetLastError();
}

template <typename real, int N>
static cudaError_t launch_yx_inv(const esp_plan* p, const void* in, const void* tw, int ldx,
                                 cudaStream_t s, int ncomp = 3) {
  using C = typename Cx<real>::t;
  const size_t smem = plane_smem<real, N>();
  cudaError_t e = cudaFuncSetAttribute(k_yx_inv<real, N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_yx_inv<real, N><<<(unsigned)(ncomp * p->M[2]), 256, smem, s>>>(
      reinterpret_cast<const C*>(in), reinterpret_cast<real*>(p->d_fields),
      reinterpret_cast<const C*>(tw), ldx, p->nbx, p->nby);
  return cudaGetLastError();
}

}  // namespace fft

struct FusedFft {
  void* tw[3];   // per-axis twiddles in the plan's precision
  void* bufA;   // x-pass output [Mz][My][ldx]
  void* bufB;   // y-pass output [Mz][nby][ldx]
  void* bufC;   // ik pencils    [3][Mz][nby][ldx]
  void* bufD;   // y-inverse     [3][Mz][My][ldx]
  int ldx, nbx, nby, nbz;
  bool fp64;
};

}  // namespace esp

using esp::FusedFft;

void esp_fused_fft_destroy(void* h) {
  auto* f = reinterpret_cast<FusedFft*>(h);
  if (!f) return;
  for (int d = 0; d < 3; ++d)
    if (f->tw[d]) cudaFree(f->tw[d]);
  if (f->bufA) cudaFree(f->bufA);
  if (f->bufB) cudaFree(f->bufB);
  if (f->bufC) cudaFree(f->bufC);
  if (f->bufD) cudaFree(f->bufD);
  delete f;
}

bool esp_fused_fft_matches(const void* h, const esp_plan* p) {
  const auto* f = reinterpret_cast<const FusedFft*>(h);
  return f && f->nbx == p->nbx && f->nby == p->nby && f->nbz == p->nbz &&
         f->fp64 == (p->precision == ESP_FP64);
}

// Build the fused transform for the plan's grid and current box; nullptr if a
// grid length is not one of ESP_FFT_SIZES (the plan then uses cuFFT).
void* esp_fused_fft_create(esp_plan* p) {
  for (int d = 0; d < 3; ++d)
    if (!esp::fft::supported(p->M[d])) return nullptr;
  auto* f = new FusedFft;
  std::memset(f, 0, sizeof(FusedFft));
  for (int d = 0; d < 3; ++d) {
    const std::vector<double2> h = esp::fft::twiddles(p->M[d]);
    std::vector<float2> hf(h.size());
    for (size_t i = 0; i < h.size(); ++i) hf[i] = make_float2((float)h[i].x, (float)h[i].y);
    const bool dp = p->precision == ESP_FP64;
    const size_t bytes = (dp ? sizeof(double2) : sizeof(float2)) * h.size();
    const void* src = dp ? (const void*)h.data() : (const void*)hf.data();
    if (cudaMalloc(&f->tw[d], bytes) != cudaSuccess ||
        cudaMemcpy(f->tw[d], src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
      esp_fused_fft_destroy(f);
      return nullptr;
    }
  }
  const size_t cs = p->precision == ESP_FP64 ? sizeof(double2) : sizeof(float2);
  f->nbx = p->nbx;
  f->nby = p->nby;
  f->nbz = p->nbz;
  f->fp64 = p->precision == ESP_FP64;
  f->ldx = (p->nbx + 7) / 8 * 8;
  const long long My = p->M[1], Mz = p->M[2], ldx = f->ldx;
  if (cudaMalloc(&f->bufA, cs * Mz * My * ldx) != cudaSuccess ||
      cudaMalloc(&f->bufB, cs * Mz * p->nby * ldx) != cudaSuccess ||
      cudaMalloc(&f->bufC, cs * 3 * Mz * p->nby * ldx) != cudaSuccess ||
      cudaMalloc(&f->bufD, cs * 3 * Mz * My * ldx) != cudaSuccess) {
    cudaGetLastError();
    esp_fused_fft_destroy(f);
    return nullptr;
  }
  return f;
}

namespace esp {

// Upper bound on the blocks of the fused reduction (the plan sizes its
// partials | group sums | counters buffer from it, see tree_finish).
int fused_reduce_blocks(const esp_plan* p) {
  const int ldx = (p->nbx + 7) / 8 * 8;
  const int L = p->precision == ESP_FP64 ? fft::lines_yz<double>(p->M[2])
                                         : fft::lines_yz<float>(p->M[2]);
  return (int)(((long long)p->nby * ldx + L - 1) / L);
}

// ESP_FFT_DEBUG=1: synchronize after every pass and name the failing one.
static cudaError_t debug_check(cudaStream_t s, const char* what) {
  static const bool on = std::getenv("ESP_FFT_DEBUG") != nullptr;
  if (!on) return cudaSuccess;
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) std::fprintf(stderr, "esp_fft: %s failed: %s\n", what, cudaGetErrorString(e));
  return e;
}

// small square planes: x and y in one kernel per plane
static bool fused_plane(const esp_plan* p) {
  static const bool no_plane = std::getenv("ESP_FFT_NO_PLANE") != nullptr;   // A/B diagnostics
  return !no_plane && p->M[0] == p->M[1] && (p->M[0] == 32 || p->M[0] == 48 || p->M[0] == 64);
}

bool fused_x_combines(const esp_plan* p) {
  // A/B diagnostics and the bitwise test; read per call so a test can switch it
  const bool off = std::getenv("ESP_NO_XCOMBINE") != nullptr;
  return p->fused && !off && !fused_plane(p) && p->Mu[2] == p->M[2] && p->zshift == 0;
}

template <typename real>
static cudaError_t fused_run(esp_plan* p, FusedFft* f, int want_ik, double* d_out7,
                             cudaStream_t s) {
  using namespace fft;
  cudaError_t e = cudaErrorInvalidValue;
  const int ldx = f->ldx;
  SlabMap one;   // single-GPU layout
  std::memset(&one, 0, sizeof(one));
  const bool plane = fused_plane(p);
  if (plane) {
    switch (p->M[0]) {
      case 32: e = launch_xy_fwd<real, 32>(p, f->bufB, f->tw[0], ldx, s); break;
      case 48: e = launch_xy_fwd<real, 48>(p, f->bufB, f->tw[0], ldx, s); break;
      case 64: e = launch_xy_fwd<real, 64>(p, f->bufB, f->tw[0], ldx, s); break;
    }
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "fft_xy");
    if ((e = debug_check(s, "fft_xy")) != cudaSuccess) return e;
  } else {
    if (p->grid_in_scratch) {
      // the spread left its tile blocks uncombined: sum them in the x pass
      bool taken = false;
      switch (p->M[0]) {
#define ESP_CASE(v)                                                                      \
  case v:                                                                                \
    e = launch_x_bulk_r2c<real, v>(p, f->bufA, f->tw[0], ldx, p->M[2], s, &taken);       \
    if (e == cudaSuccess && !taken)                                                      \
      e = launch_x_comb_r2c<real, v>(p, f->bufA, f->tw[0], ldx, p->M[2], s);             \
    break;
        ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
      }
    } else {
      switch (p->M[0]) {
#define ESP_CASE(v) \
  case v: e = launch_x_r2c<real, v>(p, p->d_grid, f->bufA, f->tw[0], ldx, p->M[2], s); break;
        ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
      }
    }
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "fft_x");
    if ((e = debug_check(s, "fft_x")) != cudaSuccess) return e;
    e = cudaErrorInvalidValue;
    switch (p->M[1]) {
#define ESP_CASE(v) \
  case v: e = launch_y_fwd<real, v>(p, f->bufA, f->bufB, f->tw[1], ldx, p->M[2], one, s); break;
      ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
    }
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "fft_y");
    if ((e = debug_check(s, "fft_y")) != cudaSuccess) return e;
  }
  FusedArgs fa{};
  for (int d = 0; d < 3; ++d) {
    fa.M[d] = p->M[d];
    fa.koff[d] = p->koff[d];
  }
  fa.nbx = p->nbx;
  fa.nby = p->nby;
  fa.nbz = p->nbz;
  fa.ldx = ldx;
  fa.Hx = p->Hx;
  fa.Msum = (long long)p->M[0] + p->M[1] + p->M[2];
  fa.axis_k = p->d_axis_k;
  fa.modeA = p->d_modeA;
  fa.modeB = p->d_modeB;
  fa.ik_scale = p->h3 / (double)p->G;
  const double h3sq = p->h3 * p->h3;
  fa.escale = h3sq / (2.0 * p->volume);
  fa.pscale = h3sq / (2.0 * p->volume * p->volume);
  fa.by0 = 0;
  fa.npy = p->nby;
  fa.potential = want_ik == 2 ? 1 : 0;
  const int ncomp = want_ik == 2 ? 1 : 3;
  // small pencils: the ik spectra and inverse z transforms run inside the
  // z-reduce kernel (ESP_FFT_NO_ZFUSE=1 keeps them separate)
  static const bool no_zfuse = std::getenv("ESP_FFT_NO_ZFUSE") != nullptr;
  bool zfused = false;
  if (want_ik && !no_zfuse) {
    switch (p->M[2]) {
#define ESP_CASE(v) \
  case v: zfused = z_fusable<real, v>(); break;
      ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
    }
  }
  e = cudaErrorInvalidValue;
  switch (p->M[2]) {
#define ESP_CASE(v)                                                                       \
  case v:                                                                                 \
    e = launch_z_reduce<real, v>(p, f->bufB, f->tw[2], fa, p->d_partials_fft,            \
                                 p->n_red_blocks_fft, d_out7, s,                          \
                                 zfused ? f->bufC : nullptr);                             \
    break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  if (e != cudaSuccess) return e;
  p->launches++;
  prof_mark(p, s, "fft_z_scale_reduce");
  if ((e = debug_check(s, "fft_z_scale_reduce")) != cudaSuccess) return e;
  if (!want_ik) return cudaSuccess;
  if (!zfused) {
    e = cudaErrorInvalidValue;
    switch (p->M[2]) {
#define ESP_CASE(v) \
  case v: e = launch_z_ik<real, v>(p, f->bufC, f->tw[2], fa, one, s); break;
      ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
    }
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "ifft_z_ik");
  }
  if ((e = debug_check(s, "ifft_z_ik")) != cudaSuccess) return e;
  if (plane) {
    e = cudaErrorInvalidValue;
    switch (p->M[0]) {
      case 32: e = launch_yx_inv<real, 32>(p, f->bufC, f->tw[0], ldx, s, ncomp); break;
      case 48: e = launch_yx_inv<real, 48>(p, f->bufC, f->tw[0], ldx, s, ncomp); break;
      case 64: e = launch_yx_inv<real, 64>(p, f->bufC, f->tw[0], ldx, s, ncomp); break;
    }
    if (e != cudaSuccess) return e;
    p->launches++;
    prof_mark(p, s, "ifft_yx");
    return debug_check(s, "ifft_yx");
  }
  e = cudaErrorInvalidValue;
  switch (p->M[1]) {
#define ESP_CASE(v) \
  case v: e = launch_y_inv<real, v>(p, f->bufC, f->bufD, f->tw[1], ldx, p->M[2], s, ncomp); break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  if (e != cudaSuccess) return e;
  p->launches++;
  prof_mark(p, s, "ifft_y");
  if ((e = debug_check(s, "ifft_y")) != cudaSuccess) return e;
  // ik fields of a TMA-gather plan go straight into the ghost-padded layout
  // (the fp64 potential of an analytic step too, when its binning wrote
  // derivative records: the TMA gradient gather reads both)
  const bool padded = p->d_fpad != nullptr &&
                      (ncomp == 3 || (p->precision == ESP_FP64 && p->drec_ready &&
                                      p->records_ready));
  p->fpad_written = padded ? 1 : 0;
  void* fdst = padded ? p->d_fpad : p->d_fields;
  const FieldPad pad = padded ? p->fpad : FieldPad{};
  e = cudaErrorInvalidValue;
  switch (p->M[0]) {
#define ESP_CASE(v) \
  case v: e = launch_x_c2r<real, v>(p, f->bufD, fdst, f->tw[0], ldx, p->M[2], s, ncomp, pad); \
    break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  if (e != cudaSuccess) return e;
  p->launches++;
  prof_mark(p, s, "ifft_x");
  if ((e = debug_check(s, "ifft_x")) != cudaSuccess) return e;
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Distributed (z-slab) steps on a full-grid plan's fused transforms.

static void slab_map(const esp_slab_desc* d, const int* by_start, int z0, void* const* peers,
                     fft::SlabMap& m) {
  std::memset(&m, 0, sizeof(m));
  m.R = d->nranks;
  m.z0 = z0;
  for (int r = 0; r <= d->nranks; ++r) {
    m.by_start[r] = by_start[r];
    m.z_start[r] = d->z_start[r];
  }
  for (int r = 0; r < d->nranks; ++r) m.peers[r] = peers[r];
}

void slab_by_split(int nby, int R, int* by_start) {
  by_start[0] = 0;
  for (int r = 0; r < R; ++r) by_start[r + 1] = by_start[r] + nby / R + (r < nby % R ? 1 : 0);
}

template <typename real>
static cudaError_t slab_forward_t(esp_plan* p, const esp_slab_desc* d, const void* own,
                                  cudaStream_t s) {
  using namespace fft;
  auto* f = reinterpret_cast<FusedFft*>(p->fused);
  const int r = d->rank, z0 = d->z_start[r], nz = d->z_start[r + 1] - z0;
  int by_start[kMaxRanks + 1];
  slab_by_split(p->nby, d->nranks, by_start);
  SlabMap m;
  slab_map(d, by_start, z0, d->fwd_peers, m);
  cudaError_t e = cudaErrorInvalidValue;
  switch (p->M[0]) {
#define ESP_CASE(v) \
  case v: e = launch_x_r2c<real, v>(p, own, f->bufA, f->tw[0], f->ldx, nz, s); break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  if (e != cudaSuccess) return e;
  e = cudaErrorInvalidValue;
  switch (p->M[1]) {
#define ESP_CASE(v) \
  case v: e = launch_y_fwd<real, v>(p, f->bufA, nullptr, f->tw[1], f->ldx, nz, m, s); break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  p->launches += 2;
  return e;
}

template <typename real>
static cudaError_t slab_reduce_t(esp_plan* p, const esp_slab_desc* d, const void* recv,
                                 int want_ik, double* d_out7, cudaStream_t s) {
  using namespace fft;
  auto* f = reinterpret_cast<FusedFft*>(p->fused);
  int by_start[kMaxRanks + 1];
  slab_by_split(p->nby, d->nranks, by_start);
  FusedArgs fa{};
  for (int k = 0; k < 3; ++k) {
    fa.M[k] = p->M[k];
    fa.koff[k] = p->koff[k];
  }
  fa.nbx = p->nbx;
  fa.nby = p->nby;
  fa.nbz = p->nbz;
  fa.ldx = f->ldx;
  fa.Hx = p->Hx;
  fa.Msum = (long long)p->M[0] + p->M[1] + p->M[2];
  fa.axis_k = p->d_axis_k;
  fa.modeA = p->d_modeA;
  fa.modeB = p->d_modeB;
  fa.ik_scale = p->h3 / (double)p->G;
  const double h3sq = p->h3 * p->h3;
  fa.escale = h3sq / (2.0 * p->volume);
  fa.pscale = h3sq / (2.0 * p->volume * p->volume);
  fa.by0 = by_start[d->rank];
  fa.npy = by_start[d->rank + 1] - by_start[d->rank];
  cudaError_t e = cudaErrorInvalidValue;
  if (fa.npy == 0) {   // no ky rows on this rank: zero partial sums
    e = cudaMemsetAsync(d_out7, 0, 7 * sizeof(double), s);
  } else {
    switch (p->M[2]) {
#define ESP_CASE(v)                                                                        \
  case v:                                                                                  \
    e = launch_z_reduce<real, v>(p, recv, f->tw[2], fa, p->d_partials_fft,                \
                                 p->n_red_blocks_fft, d_out7, s);                          \
    break;
      ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
    }
  }
  if (e != cudaSuccess || !want_ik || fa.npy == 0) return e;
  SlabMap m;
  slab_map(d, by_start, 0, d->back_peers, m);
  e = cudaErrorInvalidValue;
  switch (p->M[2]) {
#define ESP_CASE(v) \
  case v: e = launch_z_ik<real, v>(p, nullptr, f->tw[2], fa, m, s); break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  p->launches += 2;
  return e;
}

template <typename real>
static cudaError_t slab_inverse_t(esp_plan* p, const esp_slab_desc* d, const void* recv,
                                  void* fields, cudaStream_t s) {
  using namespace fft;
  auto* f = reinterpret_cast<FusedFft*>(p->fused);
  const int r = d->rank, nz = d->z_start[r + 1] - d->z_start[r];
  cudaError_t e = cudaErrorInvalidValue;
  switch (p->M[1]) {
#define ESP_CASE(v) \
  case v: e = launch_y_inv<real, v>(p, recv, f->bufD, f->tw[1], f->ldx, nz, s); break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  if (e != cudaSuccess) return e;
  e = cudaErrorInvalidValue;
  switch (p->M[0]) {
#define ESP_CASE(v) \
  case v: e = launch_x_c2r<real, v>(p, f->bufD, fields, f->tw[0], f->ldx, nz, s); break;
    ESP_FFT_SIZES(ESP_CASE)
#undef ESP_CASE
  }
  p->launches += 2;
  return e;
}

cudaError_t slab_forward(esp_plan* p, const esp_slab_desc* d, const void* own, cudaStream_t s) {
  return p->precision == ESP_FP64 ? slab_forward_t<double>(p, d, own, s)
                                  : slab_forward_t<float>(p, d, own, s);
}
cudaError_t slab_reduce(esp_plan* p, const esp_slab_desc* d, const void* recv, int want_ik,
                        double* d_out7, cudaStream_t s) {
  return p->precision == ESP_FP64 ? slab_reduce_t<double>(p, d, recv, want_ik, d_out7, s)
                                  : slab_reduce_t<float>(p, d, recv, want_ik, d_out7, s);
}
cudaError_t slab_inverse(esp_plan* p, const esp_slab_desc* d, const void* recv, void* fields,
                         cudaStream_t s) {
  return p->precision == ESP_FP64 ? slab_inverse_t<double>(p, d, recv, fields, s)
                                  : slab_inverse_t<float>(p, d, recv, fields, s);
}
int fused_ldx(const esp_plan* p) {
  return p->fused ? reinterpret_cast<const FusedFft*>(p->fused)->ldx : 0;
}

cudaError_t launch_fused_fft(esp_plan* p, int want_ik, double* d_out7, cudaStream_t s) {
  auto* f = reinterpret_cast<FusedFft*>(p->fused);
  return p->precision == ESP_FP64 ? fused_run<double>(p, f, want_ik, d_out7, s)
                                  : fused_run<float>(p, f, want_ik, d_out7, s);
}

}  // namespace esp
