// esp_spectral.cu — mode workspace setup and the fused deconvolution-scaling
// + energy/pressure reduction pass of the cuFFT path (grids without fused
// transforms, the stage-level API, analytic forces and local pressure; the
// fused-transform path does the same sums inside k_z_reduce, esp_fft.cu).
//
// Reference: ModeWorkspace (mesh.py:229-282), long_range_energy
// (mesh.py:285-292), long_range_pressure (mesh.py:295-312) and the spectrum
// scaling of long_range_forces (mesh.py:333-341).
//
// The plan keeps only the in-band box of the half spectrum (|m_d| <= band_d,
// m_x >= 0): mask, Fhat*What^-2 (A) and (dterm - 2 Fhat/k^2)*What^-2 (B) are
// precomputed there once per cell.  One pass over the box then produces
//   E      = h3^2/(2V)   * sum_w A |X|^2
//   P_ab   = h3^2/(2V^2) * sum_w (B k_a k_b + delta_ab A) |X|^2
// (w = 1 on the m_x = 0 and Nyquist planes, 2 elsewhere: Hermitian pairs of
// the full-spectrum sum) and, for the force path, the three ik spectra
// i k_d A X h3/G.  The reduction is a fixed tree (warp shuffle -> block ->
// per-block partials -> one final block), so it is deterministic.
#include "esp_internal.cuh"

namespace esp {

struct ModeArgs {
  int M[3];
  long long Hx;
  int nbx, nby, nbz;
  long long nbox;
  long long Msum;
  long long koff[3];
  const double* axis_k;
  const double* axis_w;
  const int* box_iy;
  const int* box_iz;
};

__device__ __forceinline__ double kcomp(const ModeArgs& a, int comp, int mx, int my,
                                        int mz) {
  const double* K = a.axis_k + comp * a.Msum;
  return __dadd_rn(__dadd_rn(K[a.koff[0] + mx], K[a.koff[1] + my]), K[a.koff[2] + mz]);
}

__global__ void k_mode_setup(ModeArgs a, double kmax, double r_c, double c_split,
                             double pref, const double* __restrict__ leg, int n_leg,
                             const double* __restrict__ legd, int n_legd,
                             double what_zero, double* __restrict__ modeA,
                             double* __restrict__ modeB, int* __restrict__ err,
                             unsigned long long* __restrict__ n_modes) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= a.nbox) return;
  const int bx = (int)(e % a.nbx);
  const int by = (int)((e / a.nbx) % a.nby);
  const int bz = (int)(e / ((long long)a.nbx * a.nby));
  const int mx = bx, my = a.box_iy[by], mz = a.box_iz[bz];
  const double kx = kcomp(a, 0, mx, my, mz);
  const double ky = kcomp(a, 1, mx, my, mz);
  const double kz = kcomp(a, 2, mx, my, mz);
  const double k2 = __dadd_rn(__dadd_rn(__dmul_rn(kx, kx), __dmul_rn(ky, ky)),
                              __dmul_rn(kz, kz));
  const double kmag = __dsqrt_rn(k2);
  if (!(kmag <= kmax && k2 > 0.0)) {
    modeA[e] = 0.0;
    modeB[e] = 0.0;
    return;
  }
  const double* W = a.axis_w;
  const double what = __dmul_rn(__dmul_rn(W[a.koff[0] + mx], W[a.koff[1] + my]),
                                W[a.koff[2] + mz]);
  if (fabs(what) < 1e-13 * fabs(what_zero)) atomicExch(err, 1);
  const double winv2 = __ddiv_rn(1.0, __dmul_rn(what, what));
  double x = __ddiv_rn(__dmul_rn(kmag, r_c), c_split);
  x = fmin(fmax(x, 0.0), 1.0);
  const double psi = legval(x, leg, n_leg);
  const double dpsi = legval(x, legd, n_legd);
  const double fhat = __ddiv_rn(__dmul_rn(pref, psi), k2);
  const double dterm = __ddiv_rn(__dmul_rn(__dmul_rn(pref, x), dpsi), __dmul_rn(k2, k2));
  const double A = __dmul_rn(fhat, winv2);
  modeA[e] = A;
  modeB[e] = dterm * winv2 - 2.0 * A / k2;
  const int wt = (mx == 0 || 2 * mx == a.M[0]) ? 1 : 2;
  atomicAdd(n_modes, (unsigned long long)wt);
}

template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* out) {
  __shared__ double red[32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp][i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) s += red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
}

template <typename real>
__global__ void __launch_bounds__(kRedThreads)
k_scale_reduce(ModeArgs a, const typename Cplx<real>::type* __restrict__ spec,
               const double* __restrict__ modeA, const double* __restrict__ modeB,
               double ik_scale, double lp_scale, int write_ik,
               typename Cplx<real>::type* __restrict__ ik,
               long long H, double* __restrict__ partials, int* __restrict__ done,
               double escale, double pscale, double* __restrict__ out7) {
  using C = typename Cplx<real>::type;
  double acc[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) acc[i] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < a.nbox;
       e += stride) {
    const double A = modeA[e];
    if (A == 0.0) continue;  // outside the mask (ik spectra pre-zeroed)
    const double B = modeB[e];
    const int bx = (int)(e % a.nbx);
    const int by = (int)((e / a.nbx) % a.nby);
    const int bz = (int)(e / ((long long)a.nbx * a.nby));
    const int mx = bx, my = a.box_iy[by], mz = a.box_iz[bz];
    const long long sidx = ((long long)mz * a.M[1] + my) * a.Hx + mx;
    const C X = spec[sidx];
    const double xr = (double)X.x, xi = (double)X.y;
    const double amp2 = xr * xr + xi * xi;
    const double w = ((mx == 0 || 2 * mx == a.M[0]) ? 1.0 : 2.0) * amp2;
    const double kx = kcomp(a, 0, mx, my, mz);
    const double ky = kcomp(a, 1, mx, my, mz);
    const double kz = kcomp(a, 2, mx, my, mz);
    const double wa = w * A, t = w * B;
    acc[0] += wa;
    acc[1] += t * kx * kx + wa;
    acc[2] += t * kx * ky;
    acc[3] += t * kx * kz;
    acc[4] += t * ky * ky + wa;
    acc[5] += t * ky * kz;
    acc[6] += t * kz * kz + wa;
    if (write_ik == 1) {            // ik forces: i k_d A X h3/G
      const double c = A * ik_scale;
      const double cr = c * xr, ci = c * xi;
      C o;
      o.x = (real)(-kx * ci); o.y = (real)(kx * cr); ik[sidx] = o;
      o.x = (real)(-ky * ci); o.y = (real)(ky * cr); ik[H + sidx] = o;
      o.x = (real)(-kz * ci); o.y = (real)(kz * cr); ik[2 * H + sidx] = o;
    } else if (write_ik == 2) {     // analytic forces: A X h3/G (mesh.py:344-346)
      const double c = A * ik_scale;
      C o;
      o.x = (real)(c * xr); o.y = (real)(c * xi); ik[sidx] = o;
    } else if (write_ik >= 3) {     // local pressure: -(B k_a k_b + d_ab A) X h3/(2 V G)
      const double ka[3] = {kx, ky, kz};
      const int bs[2][3] = {{0, 1, 2}, {1, 2, 2}};   // (xx,xy,xz) | (yy,yz,zz)
      const int as[2][3] = {{0, 0, 0}, {1, 1, 2}};
      const int m = write_ik - 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int aa = as[m][c], bb = bs[m][c];
        const double kern = B * ka[aa] * ka[bb] + (aa == bb ? A : 0.0);
        const double f = -kern * lp_scale;
        C o;
        o.x = (real)(f * xr);
        o.y = (real)(f * xi);
        ik[(long long)c * H + sidx] = o;
      }
    }
  }
  block_reduce_store<7>(acc, partials + (size_t)blockIdx.x * 8);
  // Last block to finish sums the per-block partials in a fixed order (same
  // tree as a separate final kernel would use): deterministic, one launch.
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) v[i] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int i = 0; i < 7; ++i) v[i] += __ldcg(partials + (size_t)b * 8 + i);
  }
  __shared__ double res[8];
  __syncthreads();   // block_reduce_store's scratch is reused
  block_reduce_store<7>(v, res);
  __syncthreads();
  if (threadIdx.x == 0) {
    out7[0] = res[0] * escale;
    for (int i = 1; i < 7; ++i) out7[i] = res[i] * pscale;
    *done = 0;       // re-arm for the next launch (graph replays)
  }
}


static ModeArgs mode_args(const esp_plan* p) {
  ModeArgs a;
  for (int d = 0; d < 3; ++d) {
    a.M[d] = p->M[d];
    a.koff[d] = p->koff[d];
  }
  a.Hx = p->Hx;
  a.nbx = p->nbx;
  a.nby = p->nby;
  a.nbz = p->nbz;
  a.nbox = p->nbox;
  a.Msum = (long long)p->M[0] + p->M[1] + p->M[2];
  a.axis_k = p->d_axis_k;
  a.axis_w = p->d_axis_w;
  a.box_iy = p->d_box_iy;
  a.box_iz = p->d_box_iz;
  return a;
}

cudaError_t launch_mode_setup(esp_plan* p, double what_zero, cudaStream_t s) {
  ModeArgs a = mode_args(p);
  const double pref = 2.0 * 3.141592653589793 * p->split_lambda0 / p->split_C0;
  unsigned long long* d_nm = reinterpret_cast<unsigned long long*>(p->d_err + 2);
  cudaError_t e = cudaMemsetAsync(p->d_err, 0, 4 * sizeof(int), s);
  if (e != cudaSuccess) return e;
  const int B = 256;
  k_mode_setup<<<(unsigned)((p->nbox + B - 1) / B), B, 0, s>>>(
      a, p->kmax, p->r_c, p->split_c, pref, p->d_leg, p->n_leg, p->d_legd, p->n_legd,
      what_zero, p->d_modeA, p->d_modeB, p->d_err, d_nm);
  return cudaGetLastError();
}

cudaError_t launch_scale_reduce(esp_plan* p, double* d_out7, int write_ik,
                                cudaStream_t s) {
  ModeArgs a = mode_args(p);
  const double G = (double)p->G;
  const double lp_scale = p->h3 / (2.0 * p->volume * G);
  cudaError_t e;
  const size_t cbytes = p->precision == ESP_FP64 ? sizeof(double2) : sizeof(float2);
  if (write_ik && !p->ik_zeroed) {
    const size_t nspec = write_ik == 2 ? 1 : 3;
    e = cudaMemsetAsync(p->d_ikspec, 0, nspec * (size_t)p->H * cbytes, s);
    if (e != cudaSuccess) return e;
    prof_mark(p, s, "ik_memset");
  }
  if (write_ik) p->ik_zeroed = 0;
  const double h3sq = p->h3 * p->h3;
  const double escale = h3sq / (2.0 * p->volume);
  const double pscale = h3sq / (2.0 * p->volume * p->volume);
  int* done = p->d_err + 1;
  if (p->precision == ESP_FP64) {
    k_scale_reduce<double><<<p->n_red_blocks, kRedThreads, 0, s>>>(
        a, reinterpret_cast<const double2*>(p->d_spec), p->d_modeA, p->d_modeB,
        p->h3 / G, lp_scale, write_ik, reinterpret_cast<double2*>(p->d_ikspec), p->H,
        p->d_partials, done, escale, pscale, d_out7);
  } else {
    k_scale_reduce<float><<<p->n_red_blocks, kRedThreads, 0, s>>>(
        a, reinterpret_cast<const float2*>(p->d_spec), p->d_modeA, p->d_modeB,
        p->h3 / G, lp_scale, write_ik, reinterpret_cast<float2*>(p->d_ikspec), p->H,
        p->d_partials, done, escale, pscale, d_out7);
  }
  p->launches++;
  prof_mark(p, s, "scale_reduce");
  return cudaGetLastError();
}

}  // namespace esp

namespace esp {

// FP64 pipe probe: independent DFMA chains, no memory traffic in the loop.
__global__ void k_probe_fp64(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
  double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double r = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (r == 1234.5678) out[0] = r;  // keep the chains alive
}

}  // namespace esp

extern "C" int esp_probe_fp64(double* tflops, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return ESP_ERR_OOM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  esp::k_probe_fp64<<<blocks, threads, 0, s>>>(d, 64, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(e0, s);
  esp::k_probe_fp64<<<blocks, threads, 0, s>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8.0 * 16.0 * iters * (double)blocks * threads;
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    esp::set_error(cudaGetErrorString(err));
    return ESP_ERR_CUDA;
  }
  return ESP_OK;
}
