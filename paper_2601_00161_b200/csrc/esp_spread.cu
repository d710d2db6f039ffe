// esp_spread.cu — PSWF charge spreading (mesh.py:204-210) as a tile kernel
// plus a deterministic halo combine.
//
// Design:
//  * CTA = one anchor tile of TX x TY columns x TZS planes (TX = TY = 17 - P),
//    whose stencils cover a padded block of 16 x 16 columns x PZS = TZS+P-1
//    planes.  Its particles are a contiguous, z-anchor-sorted range of the
//    binned arrays (esp_bin.cu).
//  * Threads own padded (x, y) columns and keep a P-deep sliding window of z
//    accumulators for each in registers.  Particles are visited in z-anchor
//    order; when the anchor advances the window slides and the finished
//    plane is stored (plain store, exclusive owner).
//      k_spread_warp (P <= 8, production): 2 or 4 warps per tile, a thread
//        owns a strip of 4 (or 2) columns along y; every charge is one visit
//        of each warp whose rows it touches.
//      k_spread_tiles (tiny grids, P > 8): 4 warps of 8 x 8 column blocks,
//        2 columns per lane, per-warp ballot-compacted particle lists.
//  * 1D weights come from the per-particle records written by the binning
//    pass (unrolled Horner on the reference's degree-18 piecewise table,
//    pswf.py:238-293) and are staged in shared memory as zero-padded rows;
//    q is folded into the x weights.
//  * The padded blocks go to a scratch buffer laid out [tz][pz][ty][py][tx][px]
//    (scr_index): one padded row of all tiles along x is contiguous, so the
//    combine's loads for a grid row stream (config 4 combine 0.82 -> 0.70 ms
//    against whole blocks stored one after another).  k_combine sums, for
//    every grid point, the contributions of the (at most 8) covering tiles in
//    a fixed order read from precomputed per-axis tables.  No atomics:
//    results are bitwise reproducible.  esp_evaluate on the fused transforms
//    skips k_combine: its forward x pass sums the same blocks in the same
//    order (esp_fft.cu: k_x_bulk_r2c / k_x_comb_r2c).
#include <cstdlib>

#include "esp_internal.cuh"

#ifndef ESP_SPREAD_U8
#define ESP_SPREAD_U8 2   // charges unrolled in the 8-rows-per-thread layout (diagnostic: 1.98 ms against 2.19 at 1)
#endif
namespace esp {

// Per-particle staging record (reals): x weights and y weights each stored
// in a zero-padded row of RL = P + 16 entries (weight s at offset 8 + s), so a
// lane reads its column's weight at (cx - xl + 8) with no clamp or predicate;
// then the P z weights.  The x row carries q.
template <int P>
struct SpreadRec {
  static constexpr int RL = P + 16;
  static constexpr int kX = 0, kY = RL, kZ = 2 * RL;
  static constexpr int kLen = ((2 * RL + P) + 1) & ~1;   // keep 16B alignment
};

// Particles staged per spread pass: 128 on small grids (few, dense tiles),
// 64 on large grids (halves the CTA's shared memory: more CTAs per SM).

template <typename real, int P>
struct SpreadLayout {
  static size_t bytes(int kSChunk) {
    size_t b = sizeof(real) * (size_t)kSChunk * SpreadRec<P>::kLen;
    b += sizeof(int) * (size_t)kSChunk * (3 + 1 + 8);   // anchors, packed, 4 warp lists x2
    b += sizeof(int) * 8;                               // list lengths
    return b;
  }
};

template <typename real, int P>
__global__ void __launch_bounds__(kSpreadThreads)
k_spread_tiles(Geom g, const int* __restrict__ offsets, const real* __restrict__ wrec,
               const int* __restrict__ PK, const double* __restrict__ Q,
               real* __restrict__ scratch, int kSChunk) {
  using Rec = SpreadRec<P>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tile = blockIdx.x;
  const int tz = tile % g.ntzs;
  const int txy = tile / g.ntzs;
  const int tx = txy % g.ntx, ty = txy / g.ntx;
  const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZS;
  const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZS);
  const long long p0 = offsets[key0], p1 = offsets[key1];
  const ScrLayout SL = scr_layout(g);
  real* blk = scratch + scr_index(g, SL, tx, ty, tz, 0, 0, 0);
  if (p0 == p1) {  // empty tile: a zero block keeps k_combine branch-free
    for (int i = threadIdx.x; i < g.PZS * kPad * kPad; i += blockDim.x)
      blk[(i >> 8) * SL.plane + ((i >> 4) & 15) * SL.row + (i & 15)] = real(0);
    return;
  }

  size_t off = 0;
  real* s_rec = reinterpret_cast<real*>(smem_raw + off);
  off += sizeof(real) * (size_t)kSChunk * Rec::kLen;
  int* s_anc = reinterpret_cast<int*>(smem_raw + off);   // [3][kSChunk]
  int* s_pk = s_anc + 3 * kSChunk;                       // packed x | y<<8 | z<<16
  int* s_list = s_pk + kSChunk;                          // [4][kSChunk]
  int* s_lpk = s_list + 4 * kSChunk;                     // packed anchors, list order
  int* s_len = s_lpk + 4 * kSChunk;

  // Warp w owns the 8x8 column block (wx0.., wy0..); lane owns (cx, cy) and
  // (cx, cy + 4).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 8;
  const int cx = wx0 + (lane & 7), cy = wy0 + (lane >> 3);
  real* outA = blk + cy * SL.row + cx;
  real* outB = outA + 4 * SL.row;
  const size_t plane = (size_t)SL.plane;

  real winA[P], winB[P];
#pragma unroll
  for (int s = 0; s < P; ++s) {
    winA[s] = real(0);
    winB[s] = real(0);
  }
  int zc = 0;

  for (long long c0 = p0; c0 < p1; c0 += kSChunk) {
    const int n = (int)min((long long)kSChunk, p1 - c0);
    __syncthreads();
    // (1) padded weight rows from the per-particle records (esp_bin.cu),
    //     one (particle, dim) per thread; q folded into the x row
    constexpr int RS = rec_stride(P);
    for (int item = threadIdx.x; item < 3 * n; item += blockDim.x) {
      const int d = item / n, pl = item - d * n;
      const real* src = wrec + (c0 + pl) * (3 * RS) + d * RS;
      real w[P];
#pragma unroll
      for (int t = 0; t < P; ++t) w[t] = src[t];
      real* rec = s_rec + (size_t)pl * Rec::kLen;
      if (d < 2) {
        const real qf = d == 0 ? (real)Q[c0 + pl] : real(1);
        real* row = rec + (d == 0 ? Rec::kX : Rec::kY);
#pragma unroll
        for (int t = 0; t < 8; ++t) row[t] = real(0);
#pragma unroll
        for (int t = 0; t < P; ++t) row[8 + t] = w[t] * qf;
#pragma unroll
        for (int t = 8 + P; t < Rec::RL; ++t) row[t] = real(0);
      } else {
#pragma unroll
        for (int t = 0; t < P; ++t) rec[Rec::kZ + t] = w[t];
        const int pk = PK[c0 + pl];
        s_pk[pl] = pk;
        s_anc[pl] = pk & 0xff;
        s_anc[kSChunk + pl] = (pk >> 8) & 0xff;
      }
    }
    __syncthreads();
    // (2) per-warp ordered lists of overlapping particles
    {
      int cnt = 0;
      for (int base = 0; base < n; base += 32) {
        const int pl = base + lane;
        bool hit = false;
        if (pl < n) {
          const int xl = s_anc[pl], yl = s_anc[kSChunk + pl];
          hit = xl < wx0 + 8 && xl + P > wx0 && yl < wy0 + 8 && yl + P > wy0;
        }
        const unsigned bits = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int at = warp * kSChunk + cnt + __popc(bits & ((1u << lane) - 1u));
          s_list[at] = pl;
          s_lpk[at] = s_pk[pl];
        }
        cnt += __popc(bits);
      }
      if (lane == 0) s_len[warp] = cnt;
    }
    __syncthreads();
    const int cnt = s_len[warp];
    const int* list = s_list + warp * kSChunk;
    const int* lpk = s_lpk + warp * kSChunk;
    const int ofx = cx + 8, ofy = cy + 8;
    // Particles arrive in z-anchor order.  The loop is software-pipelined
    // with two register sets (A/B ping-pong, no copies): the shared-memory
    // loads of particle t+1 are in flight while particle t's FMAs issue.
    // The window slides (register rotation + plane store) only when the
    // z anchor advances.
    struct Ld {
      real wx, wa, wb;
      real wz[P];
      int zl;
    };
    // loads only: nothing here consumes a pending shared-memory load, so the
    // in-order warp goes on to the previous particle's FMAs while they land
    auto load = [&](int tt, Ld& L) {
      const int pl = list[tt];
      const int pk = lpk[tt];
      const real* rec = s_rec + (size_t)pl * Rec::kLen;
      const int xl = pk & 0xff, yl = (pk >> 8) & 0xff;
      L.wx = rec[Rec::kX + ofx - xl];
      L.wa = rec[Rec::kY + ofy - yl];
      L.wb = rec[Rec::kY + ofy + 4 - yl];
#pragma unroll
      for (int s = 0; s < P; ++s) L.wz[s] = rec[Rec::kZ + s];
      L.zl = (pk >> 16) - tz * g.TZS;
    };
    auto proc = [&](const Ld& L) {
      const real a = L.wx * L.wa, b = L.wx * L.wb;
      while (zc < L.zl) {  // slide: plane zc is final for these columns
        outA[(size_t)zc * plane] = winA[0];
        outB[(size_t)zc * plane] = winB[0];
#pragma unroll
        for (int s = 0; s < P - 1; ++s) {
          winA[s] = winA[s + 1];
          winB[s] = winB[s + 1];
        }
        winA[P - 1] = real(0);
        winB[P - 1] = real(0);
        ++zc;
      }
#pragma unroll
      for (int s = 0; s < P; ++s) {
        winA[s] = fma(a, L.wz[s], winA[s]);
        winB[s] = fma(b, L.wz[s], winB[s]);
      }
    };
    Ld LA, LB;
    int t = 0;
    if (cnt > 0) load(0, LA);
    while (t < cnt) {
      if (t + 1 < cnt) load(t + 1, LB);
      proc(LA);
      if (++t >= cnt) break;
      if (t + 1 < cnt) load(t + 1, LA);
      proc(LB);
      ++t;
    }
  }
  while (zc < g.PZS) {
    outA[(size_t)zc * plane] = winA[0];
    outB[(size_t)zc * plane] = winB[0];
#pragma unroll
    for (int s = 0; s < P - 1; ++s) {
      winA[s] = winA[s + 1];
      winB[s] = winB[s + 1];
    }
    winA[P - 1] = real(0);
    winB[P - 1] = real(0);
    ++zc;
  }
}

// ---------------------------------------------------------------------------
// k_spread_warp (P <= 8, the production path): CTA = one tile, two warps.
// Thread (x = t & 15, q = t >> 4) owns the 4 padded columns (x, 4q..4q+3)
// and keeps a P-deep sliding z window for each (4 x P accumulators in
// registers); warp w covers rows 8w..8w+7.  A charge is one visit of each
// warp its stencil rows touch (a warp-uniform test, no lists): 4 products
// wx * wy[r] and 4 x P independent FMAs per thread (columns the stencil
// misses add exact zeros), so the instruction stream is dominated by FMAs.
// Raw weight records are double-buffered in shared memory with cp.async; the
// x/y weights are re-laid as zero-padded rows (weight s at OFF + s), so each
// thread's weights are immediate-offset loads from one base.  Column owners
// write each finished plane once: no atomics, bitwise reproducible.
template <int P>
struct WarpRow {
  static constexpr int OFF = 16 - P;   // cx - xl + OFF >= 0 for every anchor of the tile
  static constexpr int RL = 32 - P;    // covers cx - xl + OFF <= 31 - P
};
// ROWS = 4: 64 threads per tile (large grids); ROWS = 2: 128 threads per
// tile, for grids with few tiles (more warps in flight per SM).
__host__ __device__ constexpr int spread_warp_threads(int rows) { return 16 * (16 / rows); }

template <typename real, int P, int ROWS>
__global__ void __launch_bounds__(spread_warp_threads(ROWS))
k_spread_warp(Geom g, const int* __restrict__ offsets, const real* __restrict__ wrec,
              const int* __restrict__ PK, const double* __restrict__ Q,
              real* __restrict__ scratch) {
  static_assert(P <= 8, "warp spread: at most 8 stencil rows");
  constexpr int NT = spread_warp_threads(ROWS);
  constexpr int C = 32;                       // charges per staged chunk
  constexpr int RS = rec_stride(P), KREC = 3 * RS;
  constexpr int OFF = WarpRow<P>::OFF, RL = WarpRow<P>::RL;
  constexpr int kChargeUnroll = ROWS == 8 ? ESP_SPREAD_U8 : 4;
  __shared__ __align__(16) real s_raw[2][C * KREC];
  __shared__ __align__(16) real s_row[C][2 * RL];
  __shared__ int s_pk[2][C];
  __shared__ __align__(16) double s_q[2][C];

  const int tile = blockIdx.x;
  const int tz = tile % g.ntzs;
  const int txy = tile / g.ntzs;
  const long long key0 = (long long)txy * g.M[2] + (long long)tz * g.TZS;
  const long long key1 = (long long)txy * g.M[2] + min(g.M[2], (tz + 1) * g.TZS);
  const long long p0 = offsets[key0], p1 = offsets[key1];
  const int tid = threadIdx.x;
  const ScrLayout SL = scr_layout(g);
  real* blk = scratch + scr_index(g, SL, txy % g.ntx, txy / g.ntx, tz, 0, 0, 0);
  if (p0 == p1) {  // empty tile: a zero block keeps k_combine branch-free
    for (int i = tid; i < g.PZS * kPad * kPad; i += NT)
      blk[(i >> 8) * SL.plane + ((i >> 4) & 15) * SL.row + (i & 15)] = real(0);
    return;
  }
  // zero padding of the x/y rows is written once; chunks overwrite only the
  // P weight slots
  for (int i = tid; i < C * 2 * RL; i += NT) (&s_row[0][0])[i] = real(0);

  auto fetch = [&](long long c0, int b) {
    const int n = (int)min((long long)C, p1 - c0);
    const int pieces = n * KREC * (int)sizeof(real) / 16;
    const char* src = reinterpret_cast<const char*>(wrec + c0 * KREC);
    for (int i = tid; i < pieces; i += NT) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(
          reinterpret_cast<char*>(&s_raw[b][0]) + 16 * i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + 16 * i));
    }
    if (NT < 64) {   // one warp: both small arrays from every lane
      if (tid < n) {
        const unsigned dpk = (unsigned)__cvta_generic_to_shared(&s_pk[b][tid]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dpk), "l"(PK + c0 + tid));
        const unsigned dq = (unsigned)__cvta_generic_to_shared(&s_q[b][tid]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dq), "l"(Q + c0 + tid));
      }
    } else if (tid < n) {
      const unsigned dpk = (unsigned)__cvta_generic_to_shared(&s_pk[b][tid]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dpk), "l"(PK + c0 + tid));
    } else if (tid >= 32 && tid < 64 && tid - 32 < n) {
      const unsigned dq = (unsigned)__cvta_generic_to_shared(&s_q[b][tid - 32]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dq),
                   "l"(Q + c0 + tid - 32));
    }
    asm volatile("cp.async.commit_group;");
  };

  // warp w covers rows [w * 2 ROWS, (w + 1) * 2 ROWS)
  const int cx = tid & 15, ry0 = (tid >> 4) * ROWS, wy0 = (tid >> 5) * 2 * ROWS;
  real* out = blk + ry0 * SL.row + cx;
  const size_t plane = (size_t)SL.plane;
  const long long rowst = SL.row;
  real win[ROWS][P];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int s2 = 0; s2 < P; ++s2) win[r][s2] = real(0);
  int zc = 0;
  auto slide_to = [&](int zl) {   // planes < zl are final for these columns
    while (zc < zl) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) out[(size_t)zc * plane + r * rowst] = win[r][0];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
#pragma unroll
        for (int s2 = 0; s2 < P - 1; ++s2) win[r][s2] = win[r][s2 + 1];
        win[r][P - 1] = real(0);
      }
      ++zc;
    }
  };

  int b = 0;
  fetch(p0, 0);
  for (long long c0 = p0; c0 < p1; c0 += C, b ^= 1) {
    const int n = (int)min((long long)C, p1 - c0);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // padded x (q folded) and y rows of this chunk
    for (int i = tid; i < n * 2 * P; i += NT) {
      const int t = i / (2 * P), e = i - t * (2 * P);
      const int d = e / P, sidx = e - d * P;
      real v = s_raw[b][t * KREC + d * RS + sidx];
      if (d == 0) v = (real)((double)v * s_q[b][t]);
      s_row[t][d * RL + OFF + sidx] = v;
    }
    __syncthreads();
    if (c0 + C < p1) fetch(c0 + C, b ^ 1);   // next chunk lands during this one
    // 4 charges unrolled: their record loads overlap the previous FMAs
    // (config 1 spread 47 -> 42.5 us, config 4 2.06 -> 1.86 ms; 8 is slower)
#pragma unroll kChargeUnroll
    for (int t = 0; t < n; ++t) {
      const int pk = s_pk[b][t];
      const int xl = pk & 0xff, yl = (pk >> 8) & 0xff;
      if (yl >= wy0 + 2 * ROWS || yl + P <= wy0) continue;   // warp-uniform: rows untouched
      slide_to((pk >> 16) - tz * g.TZS);
      const real wx = s_row[t][cx - xl + OFF];
      const real* ry = &s_row[t][RL + ry0 - yl + OFF];
      const real* rz = &s_raw[b][t * KREC + 2 * RS];
      real wz[P];
#pragma unroll
      for (int s2 = 0; s2 < P; ++s2) wz[s2] = rz[s2];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const real a = wx * ry[r];
#pragma unroll
        for (int s2 = 0; s2 < P; ++s2) win[r][s2] = fma(a, wz[s2], win[r][s2]);
      }
    }
    __syncthreads();   // s_row / s_raw[b] are rewritten by the next chunks
  }
  slide_to(g.PZS);
}

template <typename real>
__global__ void __launch_bounds__(1024)
k_combine(Geom g, CombineTabs ct, const real* __restrict__ scratch, real* __restrict__ grid) {
  const long long G = (long long)g.M[0] * g.M[1] * g.M[2];
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= G) return;
  const int x = (int)(gid % g.M[0]);
  const int y = (int)((gid / g.M[0]) % g.M[1]);
  const int z = (int)(gid / ((long long)g.M[0] * g.M[1]));
  grid[gid] = (real)combine_at(g, ct, scratch, x, y, z);
}

CombineTabs combine_tabs(const esp_plan* p) {
  CombineTabs ct;
  for (int d = 0; d < 3; ++d) {
    ct.ent[d] = p->d_comb_ent + kCombW * p->comb_off[d];
    ct.cnt[d] = p->d_comb_cnt + p->comb_off[d];
  }
  return ct;
}

bool spread_uses_warp(const esp_plan* p) {
  static const bool legacy = std::getenv("ESP_SPREAD_LEGACY") != nullptr;   // A/B diagnostics
  // k_spread_warp needs enough tiles to fill the SMs; tiny grids keep the
  // 4-warp column-block kernel
  return p->P <= 8 && !legacy && p->n_tiles_s * 2 >= 148 * 4;
}

// Measured and rejected (config 4, spread kernel ms): evaluating the weights
// inside k_spread_warp from u instead of reading the binning pass's records —
// 2.97 with the per-chunk prologue on the accumulating threads, 2.86-3.6 with
// 32/64/96 producer threads filling a double-buffered stage behind named
// barriers (fewer accumulating warps per SM) — against 1.85 + 0.56 for the
// separate coalesced records pass.
template <typename real, int P>
static cudaError_t spread_p(esp_plan* p, cudaStream_t s, bool with_combine) {
  Geom g = make_geom(p);
  // both spread kernels read the per-particle weight records
  const cudaError_t er = ensure_records(p, s);
  if (er != cudaSuccess) return er;
  if (P <= 8 && spread_uses_warp(p)) {
    constexpr int PW = P <= 8 ? P : 8;
    static const int rows_env = std::getenv("ESP_SPREAD_ROWS") ? std::atoi(std::getenv("ESP_SPREAD_ROWS")) : 0;
    if (rows_env == 1) {
      k_spread_warp<real, PW, 1><<<(unsigned)p->n_tiles_s, spread_warp_threads(1), 0, s>>>(
          g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec), p->d_pk, p->d_q,
          reinterpret_cast<real*>(p->d_scratch));
    } else if (rows_env == 8) {
      k_spread_warp<real, PW, 8><<<(unsigned)p->n_tiles_s, spread_warp_threads(8), 0, s>>>(
          g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec), p->d_pk, p->d_q,
          reinterpret_cast<real*>(p->d_scratch));
    } else if (rows_env == 4 || (rows_env == 0 && p->n_tiles_s * 2 >= 148 * 12)) {
      k_spread_warp<real, PW, 4><<<(unsigned)p->n_tiles_s, spread_warp_threads(4), 0, s>>>(
          g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec), p->d_pk, p->d_q,
          reinterpret_cast<real*>(p->d_scratch));
    } else {
      k_spread_warp<real, PW, 2><<<(unsigned)p->n_tiles_s, spread_warp_threads(2), 0, s>>>(
          g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec), p->d_pk, p->d_q,
          reinterpret_cast<real*>(p->d_scratch));
    }
  } else {
    const int chunk = p->M[2] <= 128 ? 128 : 64;
    const size_t smem = SpreadLayout<real, P>::bytes(chunk);
    // the opt-in is per device: set it on every call (host-only, capture-safe)
    cudaError_t e = cudaFuncSetAttribute(k_spread_tiles<real, P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_spread_tiles<real, P><<<(unsigned)p->n_tiles_s, kSpreadThreads, smem, s>>>(
        g, p->d_offsets, reinterpret_cast<const real*>(p->d_wrec), p->d_pk, p->d_q,
        reinterpret_cast<real*>(p->d_scratch), chunk);
  }
  p->launches++;
  prof_mark(p, s, "spread");
  if (!with_combine) return cudaGetLastError();
  const CombineTabs ct = combine_tabs(p);
  // 128-thread blocks: config 4 combine 0.88 -> 0.82 ms against 256 (ESP_COMBINE_B sweeps)
  static const int B = [] {
    const char* e = std::getenv("ESP_COMBINE_B");
    const int v = e ? std::atoi(e) : 0;
    return v >= 32 && v <= 1024 && v % 32 == 0 ? v : 128;
  }();
  // Measured and rejected (config 4, row-contiguous scratch, combine ms):
  // 2 / 4 points per thread with every load issued before the sums 0.83 /
  // 0.95 against 0.70; a column-stationary CTA (32 x 8 columns x 16 planes,
  // per-column table lookups hoisted) 0.93 (block layout); fusing the combine
  // into the spread's CTAs (the CTA completing a brick's count sums it from
  // L2) 6.9 ms for spread + combine: latency-bound tails hold the FMA slots.
  k_combine<real><<<(unsigned)((p->G + B - 1) / B), B, 0, s>>>(
      g, ct, reinterpret_cast<const real*>(p->d_scratch), reinterpret_cast<real*>(p->d_grid));
  p->launches++;
  prof_mark(p, s, "combine");
  return cudaGetLastError();
}

template <typename real>
static cudaError_t spread_r(esp_plan* p, cudaStream_t s, bool with_combine) {
  switch (p->P) {
    case 2: return spread_p<real, 2>(p, s, with_combine);
    case 3: return spread_p<real, 3>(p, s, with_combine);
    case 4: return spread_p<real, 4>(p, s, with_combine);
    case 5: return spread_p<real, 5>(p, s, with_combine);
    case 6: return spread_p<real, 6>(p, s, with_combine);
    case 7: return spread_p<real, 7>(p, s, with_combine);
    case 8: return spread_p<real, 8>(p, s, with_combine);
    case 9: return spread_p<real, 9>(p, s, with_combine);
    case 10: return spread_p<real, 10>(p, s, with_combine);
    case 11: return spread_p<real, 11>(p, s, with_combine);
    case 12: return spread_p<real, 12>(p, s, with_combine);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_spread(esp_plan* p, cudaStream_t s, bool with_combine) {
  return p->precision == ESP_FP64 ? spread_r<double>(p, s, with_combine)
                                  : spread_r<float>(p, s, with_combine);
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
