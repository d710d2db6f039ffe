// esp_api.cu — plan lifetime, cuFFT plans and the C ABI (include/esp_b200.h).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "esp_internal.cuh"

namespace esp {

size_t scan_temp_bytes(long long n_items);
size_t sort_temp_bytes(long long cap, long long n_keys);

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

Geom make_geom(const esp_plan* p) {
  Geom g;
  for (int d = 0; d < 3; ++d) {
    g.M[d] = p->M[d];
    g.Mu[d] = p->Mu[d];
    g.spacing[d] = p->spacing[d];
  }
  g.zshift = p->zshift;
  for (int i = 0; i < 9; ++i) g.hinv[i] = p->hinv[i];
  g.P = p->P;
  g.lo = p->lo;
  g.odd = p->odd;
  g.ortho = p->ortho;
  g.TX = p->TX;
  g.TY = p->TY;
  g.TZ = p->TZ;
  g.PZ = p->PZ;
  g.ntx = p->ntx;
  g.nty = p->nty;
  g.ntz = p->ntz;
  g.TZS = p->TZS;
  g.PZS = p->PZS;
  g.ntzs = p->ntzs;
  g.n_keys = p->n_keys;
  return g;
}

}  // namespace esp

using esp::set_error;

#define ESP_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                #call);                                                        \
      return e_ == cudaErrorMemoryAllocation ? ESP_ERR_OOM : ESP_ERR_CUDA;     \
    }                                                                          \
  } while (0)

#define ESP_CUFFT(call)                                                        \
  do {                                                                         \
    cufftResult r_ = (call);                                                   \
    if (r_ != CUFFT_SUCCESS) {                                                 \
      set_error(std::string("cuFFT error ") + std::to_string((int)r_) + " at " + \
                #call);                                                        \
      return ESP_ERR_CUFFT;                                                    \
    }                                                                          \
  } while (0)

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
}

static void free_all(esp_plan* p) {
  void* ptrs[] = {p->d_tab,     p->d_dtab,     p->d_breaks,  p->d_tabf,    p->d_dtabf,
                  p->d_leg,     p->d_legd,     p->d_key,     p->d_slot,    p->d_counts,
                  p->d_offsets, p->d_bkey,     p->d_u,       p->d_q,       p->d_idx,
                  p->d_u_tmp,   p->d_q_tmp,    p->d_idx_tmp, p->d_cub,     p->d_scratch,
                  p->d_grid,    p->d_spec,     p->d_ikspec,  p->d_fields,  p->d_axis_k,
                  p->d_axis_w,  p->d_box_iy,   p->d_box_iz,  p->d_modeA,   p->d_modeB,
                  p->d_partials, p->d_err,       p->d_comb_ent, p->d_comb_cnt,
                  p->d_wrec,     p->d_pk,       p->d_drec,    p->d_err_out7,
                  p->d_sort_tmp, p->d_partials_fft, p->d_fpad,   p->d_zlist};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  esp_fused_fft_destroy(p->fused);
  p->fused = nullptr;
  if (p->have_fwd) cufftDestroy(p->fwd);
  if (p->have_inv3) cufftDestroy(p->inv3);
  if (p->have_inv1) cufftDestroy(p->inv1);
  if (p->profiling)
    for (int i = 0; i < 48; ++i) cudaEventDestroy(p->ev[i]);
  if (p->have_side) {
    cudaEventDestroy(p->ev_fork);
    cudaEventDestroy(p->ev_join);
    for (int i = 0; i < 8; ++i) cudaEventDestroy(p->ev_chunk[i]);
    cudaStreamDestroy(p->side);
  }
  delete p->h_fast;
  p->h_fast = nullptr;
  delete p->h_fast_d;
  p->h_fast_d = nullptr;
}

extern "C" {

const char* esp_last_error(void) { return esp::g_last_error.c_str(); }

int esp_version(void) { return 100; }

int esp_set_charges_event(esp_plan* p, void* event) {
  if (!p) {
    set_error("null plan");
    return ESP_ERR_PARAM;
  }
  p->q_ready = (cudaEvent_t)event;
  return ESP_OK;
}

int esp_set_host_forces(esp_plan* p, double* host_forces, int32_t nchunks) {
  if (!p || nchunks < 0 || nchunks > 8 || (nchunks > 0 && !host_forces)) {
    set_error("esp_set_host_forces: null plan, or chunks outside [0, 8] without a buffer");
    return ESP_ERR_PARAM;
  }
  p->host_forces = nchunks ? host_forces : nullptr;
  p->host_chunks = nchunks;
  return ESP_OK;
}

int esp_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) {
    set_error("bad host allocation arguments");
    return ESP_ERR_PARAM;
  }
  *out = nullptr;
  ESP_CUDA(cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 1), cudaHostAllocDefault));
  return ESP_OK;
}

int esp_host_free(void* p) {
  if (p) ESP_CUDA(cudaFreeHost(p));
  return ESP_OK;
}

int esp_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) {
    set_error("bad copy arguments");
    return ESP_ERR_PARAM;
  }
  if (bytes == 0) return ESP_OK;
  ESP_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return ESP_OK;
}

int esp_plan_create(const esp_plan_desc* d, esp_plan** out) {
  if (!d || !out) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  *out = nullptr;
  if (d->P < 2 || d->P > 12) {
    set_error("spreading order P must be in [2, 12] on the B200 path");
    return ESP_ERR_PLANNING;
  }
  for (int k = 0; k < 3; ++k) {
    if (d->M[k] < 2 || d->M[k] <= d->P) {
      set_error("grid count must exceed the stencil width P");
      return ESP_ERR_PLANNING;
    }
  }
  if (d->M[0] % 2) {
    set_error("M_x must be even (half-spectrum layout)");
    return ESP_ERR_PLANNING;
  }
  if (d->n_pieces < 1 || d->n_pieces > esp::kMaxPieces || d->degree + 1 > esp::kMaxCoef ||
      d->degree < 0) {
    set_error("window table shape unsupported");
    return ESP_ERR_PLANNING;
  }
  if (d->precision != ESP_FP64 && d->precision != ESP_FP32) {
    set_error("unknown precision");
    return ESP_ERR_PARAM;
  }
  esp_plan* p = new esp_plan;
  std::memset(p, 0, sizeof(esp_plan));
  p->need_records = 0;   // radix binning: records-free gather + coalesced records pass
  for (int k = 0; k < 3; ++k) p->M[k] = p->Mu[k] = d->M[k];
  if (d->slab_mz_global > 0) {
    // z-slab plan: local planes [0, M[2]) hold global planes zshift + i
    // (owned planes plus P-1 ghost planes); no periodic wrap inside the slab.
    p->Mu[2] = d->slab_mz_global;
    p->zshift = d->slab_z0 - ((d->P - 1) / 2);
  }
  p->G = (long long)d->M[0] * d->M[1] * d->M[2];
  p->Hx = d->M[0] / 2 + 1;
  p->H = p->Hx * d->M[1] * d->M[2];
  p->P = d->P;
  p->lo = -((d->P - 1) / 2);
  p->odd = d->P % 2;
  p->precision = d->precision;
  p->deterministic = d->deterministic ? 1 : 0;
  p->cap = std::max<long long>(d->max_particles, 1);
  p->n_pieces = d->n_pieces;
  p->ncoef = d->degree + 1;
  p->kmax = d->kmax;
  p->r_c = d->r_c;
  p->split_c = d->split_c;
  p->split_lambda0 = d->split_lambda0;
  p->split_C0 = d->split_C0;
  p->n_leg = d->n_legendre;
  p->n_legd = d->n_legendre_deriv;
  // tiles
  p->TX = d->tile[0] > 0 ? d->tile[0] : esp::kPad - d->P + 1;
  p->TY = d->tile[1] > 0 ? d->tile[1] : esp::kPad - d->P + 1;
  if (p->TX + d->P - 1 != esp::kPad || p->TY + d->P - 1 != esp::kPad) {
    set_error("tile x/y extent must be 17 - P");
    delete p;
    return ESP_ERR_PARAM;
  }
  int tz = d->tile[2] > 0 ? d->tile[2] : 8;
  p->TZ = std::min(tz, d->M[2]);
  p->PZ = p->TZ + d->P - 1;
  p->ntx = (d->M[0] + p->TX - 1) / p->TX;
  p->nty = (d->M[1] + p->TY - 1) / p->TY;
  p->ntz = (d->M[2] + p->TZ - 1) / p->TZ;
  p->n_tiles = (long long)p->ntx * p->nty * p->ntz;
  // spread tiles share the x-y decomposition (and so the binning keys) but run
  // deeper in z on large grids: the scratch halo shrinks from (TZ+P-1)/TZ.
  // small grids: shallow spread tiles (more tiles in flight; the extra
  // scratch halo is L2-resident)
  p->TZS = std::min(d->M[2] <= 128 ? 4 : std::max(p->TZ, 32), d->M[2]);
  // grids with tiles to spare go 64 planes deep: fewer planes lie under two
  // z tiles, so the combining x pass stages less (config 4: step 8.28 ->
  // 8.24 ms; 96 and 128 planes lose it again in the spread's tail)
  if (d->M[2] >= 256 && (long long)p->ntx * p->nty * (d->M[2] / 64) >= 148 * 8 * 4)
    p->TZS = std::min(std::max(p->TZ, 64), d->M[2]);
  if (const char* env = getenv("ESP_TILE_ZS")) {   // diagnostic override (tuning sweeps)
    const int v = atoi(env);
    if (v > 0) p->TZS = std::min(v, d->M[2]);
  }
  p->PZS = p->TZS + d->P - 1;
  p->ntzs = (d->M[2] + p->TZS - 1) / p->TZS;
  p->n_tiles_s = (long long)p->ntx * p->nty * p->ntzs;
  p->n_keys = (long long)p->ntx * p->nty * d->M[2];

  const size_t real_sz = p->precision == ESP_FP64 ? sizeof(double) : sizeof(float);
  const size_t nt = (size_t)p->n_pieces * p->ncoef;
  cudaError_t e = cudaSuccess;
#define TRY(x)                                                      \
  do {                                                              \
    e = (x);                                                        \
    if (e != cudaSuccess) {                                         \
      set_error(std::string("plan allocation failed: ") +           \
                cudaGetErrorString(e) + " at " #x);                 \
      free_all(p);                                                  \
      delete p;                                                     \
      return e == cudaErrorMemoryAllocation ? ESP_ERR_OOM : ESP_ERR_CUDA; \
    }                                                               \
  } while (0)
  TRY(dalloc(&p->d_tab, nt));
  TRY(dalloc(&p->d_dtab, nt));
  TRY(dalloc(&p->d_tabf, nt));
  TRY(dalloc(&p->d_dtabf, nt));
  TRY(dalloc(&p->d_breaks, (size_t)p->n_pieces + 1));
  TRY(dalloc(&p->d_leg, (size_t)std::max(p->n_leg, 1)));
  TRY(dalloc(&p->d_legd, (size_t)std::max(p->n_legd, 1)));
  TRY(cudaMemcpy(p->d_tab, d->h_window_coef, sizeof(double) * nt, cudaMemcpyHostToDevice));
  TRY(cudaMemcpy(p->d_dtab, d->h_window_deriv_coef ? d->h_window_deriv_coef : d->h_window_coef,
                 sizeof(double) * nt, cudaMemcpyHostToDevice));
  {
    std::vector<float> tf(nt), dtf(nt);
    for (size_t i = 0; i < nt; ++i) {
      tf[i] = (float)d->h_window_coef[i];
      dtf[i] = (float)(d->h_window_deriv_coef ? d->h_window_deriv_coef[i] : 0.0);
    }
    TRY(cudaMemcpy(p->d_tabf, tf.data(), sizeof(float) * nt, cudaMemcpyHostToDevice));
    TRY(cudaMemcpy(p->d_dtabf, dtf.data(), sizeof(float) * nt, cudaMemcpyHostToDevice));
  }
  TRY(cudaMemcpy(p->d_breaks, d->h_window_breaks, sizeof(double) * (p->n_pieces + 1),
                 cudaMemcpyHostToDevice));
  if (p->n_leg > 0)
    TRY(cudaMemcpy(p->d_leg, d->h_legendre, sizeof(double) * p->n_leg, cudaMemcpyHostToDevice));
  if (p->n_legd > 0)
    TRY(cudaMemcpy(p->d_legd, d->h_legendre_deriv, sizeof(double) * p->n_legd,
                   cudaMemcpyHostToDevice));
  const size_t cap = (size_t)p->cap;
  TRY(dalloc(&p->d_key, cap));
  TRY(dalloc(&p->d_slot, cap));
  TRY(dalloc(&p->d_bkey, cap));
  TRY(dalloc(&p->d_counts, (size_t)p->n_keys + 1));
  TRY(dalloc(&p->d_offsets, (size_t)p->n_keys + 1));
  TRY(dalloc(&p->d_u, 3 * cap));
  TRY(dalloc(&p->d_q, cap));
  TRY(dalloc(&p->d_idx, cap));
  TRY(dalloc(&p->d_u_tmp, 3 * cap));
  TRY(dalloc(&p->d_q_tmp, cap));
  TRY(dalloc(&p->d_idx_tmp, cap));
  TRY(cudaMalloc(&p->d_wrec, real_sz * 3 * esp::rec_stride(p->P) * cap));
  TRY(cudaMalloc(&p->d_drec, real_sz * 3 * esp::rec_stride(p->P) * cap));
  TRY(dalloc(&p->d_pk, cap));
  p->cub_bytes = esp::scan_temp_bytes(p->n_keys + 1);
  TRY(cudaMalloc(&p->d_cub, std::max<size_t>(p->cub_bytes, 16)));
  p->sort_threshold = esp::kSortThreshold;
  if (const char* env = getenv("ESP_SORT_THRESHOLD")) p->sort_threshold = atoll(env);
  if (p->cap >= p->sort_threshold) {
    p->sort_bytes = esp::sort_temp_bytes(p->cap, p->n_keys);
    TRY(cudaMalloc(&p->d_sort_tmp, std::max<size_t>(p->sort_bytes, 16)));
  }
  TRY(cudaMalloc(&p->d_scratch,
                 real_sz * (size_t)p->n_tiles_s * p->PZS * esp::kPad * esp::kPad));
  TRY(cudaMalloc(&p->d_grid, real_sz * (size_t)p->G));
  TRY(cudaMemset(p->d_grid, 0, real_sz * (size_t)p->G));
  TRY(cudaMalloc(&p->d_spec, 2 * real_sz * (size_t)p->H));
  TRY(cudaMalloc(&p->d_ikspec, 3 * 2 * real_sz * (size_t)p->H));
  TRY(cudaMalloc(&p->d_fields, 3 * real_sz * (size_t)p->G));
  TRY(dalloc(&p->d_err, 4));
  TRY(cudaMemset(p->d_err, 0, 4 * sizeof(int)));
  TRY(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
  TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  for (int i = 0; i < 8; ++i)
    TRY(cudaEventCreateWithFlags(&p->ev_chunk[i], cudaEventDisableTiming));
  p->have_side = 1;
  TRY(dalloc(&p->d_err_out7, 8));
  // fast window table (kernel parameter) and deterministic-combine tables
  p->h_fast = new esp::FastTab;
  std::memset(p->h_fast, 0, sizeof(esp::FastTab));
  // fast table: P pieces, each exactly one grid spacing wide (stencil_weights
  // shares the in-piece offset between the P weights of an axis)
  bool unit_pieces = p->n_pieces == p->P;
  for (int i = 0; unit_pieces && i < p->n_pieces; ++i)
    unit_pieces = d->h_window_breaks[i + 1] - d->h_window_breaks[i] == 1.0;
  if (unit_pieces && p->ncoef == esp::kFastNC && p->P <= esp::kFastMaxP) {
    p->h_fast->enabled = 1;
    for (size_t i = 0; i < nt; ++i) {
      p->h_fast->c[i] = d->h_window_coef[i];
      p->h_fast->cf[i] = (float)d->h_window_coef[i];
    }
    for (int i = 0; i <= p->n_pieces; ++i) p->h_fast->brk[i] = d->h_window_breaks[i];
  }
  p->h_fast_d = new esp::FastTab;
  std::memset(p->h_fast_d, 0, sizeof(esp::FastTab));
  if (p->h_fast->enabled && d->h_window_deriv_coef) {
    p->h_fast_d->enabled = 1;
    for (size_t i = 0; i < nt; ++i) {
      p->h_fast_d->c[i] = d->h_window_deriv_coef[i];
      p->h_fast_d->cf[i] = (float)d->h_window_deriv_coef[i];
    }
    for (int i = 0; i <= p->n_pieces; ++i) p->h_fast_d->brk[i] = d->h_window_breaks[i];
  }
  {
    std::vector<int> ent_all, cnt_all;
    const int T[3] = {p->TX, p->TY, p->TZS};
    const int E[3] = {esp::kPad, esp::kPad, p->PZS};
    const int NT[3] = {p->ntx, p->nty, p->ntzs};
    long long off = 0;
    std::vector<int> zlist;
    for (int a = 0; a < 3; ++a) {
      std::vector<int> ent, cnt;
      esp::build_combine_axis(p->M[a], T[a], E[a], NT[a], p->lo, ent, cnt);
      for (int c : cnt) {
        if (c > esp::kCombW) {
          set_error("grid too small for the tile decomposition (combine width)");
          free_all(p);
          delete p;
          return ESP_ERR_PLANNING;
        }
      }
      p->comb_off[a] = off;
      p->comb_max[a] = 0;
      for (int c : cnt) p->comb_max[a] = std::max(p->comb_max[a], c);
      if (a == 2) {
        // z planes by the number of covering z tiles: one first, then more
        // (the bulk-staged x pass stages half as many scratch rows for the
        // first class and runs more CTAs per SM on it)
        zlist.clear();
        for (int z = 0; z < p->M[2]; ++z)
          if (cnt[z] == 1) zlist.push_back(z);
        p->n_z_single = (int)zlist.size();
        for (int z = 0; z < p->M[2]; ++z)
          if (cnt[z] != 1) zlist.push_back(z);
      }
      off += p->M[a];
      ent_all.insert(ent_all.end(), ent.begin(), ent.end());
      cnt_all.insert(cnt_all.end(), cnt.begin(), cnt.end());
    }
    TRY(dalloc(&p->d_comb_ent, ent_all.size()));
    TRY(dalloc(&p->d_comb_cnt, cnt_all.size()));
    TRY(dalloc(&p->d_zlist, zlist.size()));
    TRY(cudaMemcpy(p->d_zlist, zlist.data(), sizeof(int) * zlist.size(), cudaMemcpyHostToDevice));
    TRY(cudaMemcpy(p->d_comb_ent, ent_all.data(), sizeof(int) * ent_all.size(),
                   cudaMemcpyHostToDevice));
    TRY(cudaMemcpy(p->d_comb_cnt, cnt_all.data(), sizeof(int) * cnt_all.size(),
                   cudaMemcpyHostToDevice));
  }
#undef TRY
  // cuFFT plans: [z][y][x] row-major, x fastest.
  const cufftType fwd_t = p->precision == ESP_FP64 ? CUFFT_D2Z : CUFFT_R2C;
  const cufftType inv_t = p->precision == ESP_FP64 ? CUFFT_Z2D : CUFFT_C2R;
  int n3[3] = {d->M[2], d->M[1], d->M[0]};
  if (cufftPlan3d(&p->fwd, d->M[2], d->M[1], d->M[0], fwd_t) != CUFFT_SUCCESS) {
    set_error("cufftPlan3d (forward) failed");
    free_all(p);
    delete p;
    return ESP_ERR_CUFFT;
  }
  p->have_fwd = 1;
  if (cufftPlanMany(&p->inv3, 3, n3, nullptr, 1, (int)p->H, nullptr, 1, (int)p->G, inv_t,
                    3) != CUFFT_SUCCESS) {
    set_error("cufftPlanMany (inverse x3) failed");
    free_all(p);
    delete p;
    return ESP_ERR_CUFFT;
  }
  p->have_inv3 = 1;
  if (cufftPlan3d(&p->inv1, d->M[2], d->M[1], d->M[0], inv_t) != CUFFT_SUCCESS) {
    set_error("cufftPlan3d (inverse) failed");
    free_all(p);
    delete p;
    return ESP_ERR_CUFFT;
  }
  p->have_inv1 = 1;
  *out = p;
  return ESP_OK;
}

int esp_plan_destroy(esp_plan* p) {
  if (!p) return ESP_OK;
  cudaDeviceSynchronize();
  free_all(p);
  delete p;
  return ESP_OK;
}

int esp_plan_set_cell(esp_plan* p, const esp_cell_desc* c, void* stream) {
  if (!p || !c) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  p->ortho = c->orthorhombic ? 1 : 0;
  for (int i = 0; i < 9; ++i) {
    p->hinv[i] = c->hinv[i];
    p->hmat[i] = c->h[i];
  }
  for (int d = 0; d < 3; ++d) {
    p->spacing[d] = c->spacing[d];
    p->band[d] = c->band[d];
    p->grad_scale[d] = c->grad_scale[d];
  }
  p->volume = c->volume;
  p->h3 = c->volume_element;
  // in-band box of the half spectrum
  const int bx = std::max(0, std::min(c->band[0], p->M[0] / 2));
  p->nbx = bx + 1;
  std::vector<int> iy, iz;
  for (int ax = 1; ax <= 2; ++ax) {
    std::vector<int>& v = ax == 1 ? iy : iz;
    const int M = p->M[ax], b = std::max(0, c->band[ax]);
    for (int m = 0; m < M; ++m) {
      const int f = m < (M + 1) / 2 ? m : m - M;  // numpy fftfreq integer
      if (std::abs(f) <= b) v.push_back(m);
    }
  }
  p->nby = (int)iy.size();
  p->nbz = (int)iz.size();
  p->nbox = (long long)p->nbx * p->nby * p->nbz;
  const long long msum = (long long)p->M[0] + p->M[1] + p->M[2];
  p->koff[0] = 0;
  p->koff[1] = p->M[0];
  p->koff[2] = (long long)p->M[0] + p->M[1];
  if (p->d_axis_k) cudaFree(p->d_axis_k);
  if (p->d_axis_w) cudaFree(p->d_axis_w);
  if (p->d_box_iy) cudaFree(p->d_box_iy);
  if (p->d_box_iz) cudaFree(p->d_box_iz);
  if (p->d_modeA) cudaFree(p->d_modeA);
  if (p->d_modeB) cudaFree(p->d_modeB);
  if (p->d_partials) cudaFree(p->d_partials);
  p->d_axis_k = nullptr;
  p->d_axis_w = nullptr;
  p->d_box_iy = p->d_box_iz = nullptr;
  p->d_modeA = p->d_modeB = p->d_partials = nullptr;
  ESP_CUDA(dalloc(&p->d_axis_k, 3 * msum));
  ESP_CUDA(dalloc(&p->d_axis_w, msum));
  ESP_CUDA(dalloc(&p->d_box_iy, iy.size()));
  ESP_CUDA(dalloc(&p->d_box_iz, iz.size()));
  ESP_CUDA(dalloc(&p->d_modeA, (size_t)p->nbox));
  ESP_CUDA(dalloc(&p->d_modeB, (size_t)p->nbox));
  p->n_red_blocks = (int)std::max<long long>(
      1, std::min<long long>((p->nbox + esp::kRedThreads - 1) / esp::kRedThreads, 148 * 4));
  ESP_CUDA(dalloc(&p->d_partials, (size_t)p->n_red_blocks * 8));
  // band-pruned fused transforms for esp_evaluate (full-grid plans whose
  // lengths factor into 2s and 3s; ESP_FFT=cufft keeps the cuFFT path)
  // (a cell change that keeps the in-band box keeps the buffers: NPT loops
  // rebind the cell every step)
  {
    const char* env = std::getenv("ESP_FFT");
    const bool want = !(env && std::string(env) == "cufft");
    const bool keep = want && p->fused && esp_fused_fft_matches(p->fused, p);
    if (!keep) {
      esp_fused_fft_destroy(p->fused);
      p->fused = nullptr;
      if (p->d_partials_fft) cudaFree(p->d_partials_fft);
      p->d_partials_fft = nullptr;
    }
    if (!keep && want && p->Mu[2] == p->M[2] && p->zshift == 0) {
      p->fused = esp_fused_fft_create(p);
      // ghost-padded ik fields + tensor map for the TMA gather (grids whose
      // inverse x pass is k_x_c2r: not the small square plane kernels)
      const bool plane_grid = p->M[0] == p->M[1] &&
                              (p->M[0] == 32 || p->M[0] == 48 || p->M[0] == 64);
      if (p->fused && !p->d_fpad && !plane_grid && esp::tma_gather_eligible(p)) {
        p->fpad = esp::make_field_pad(p);
        const size_t fb = (p->precision == ESP_FP64 ? sizeof(double) : sizeof(float)) * 3 *
                          (size_t)p->fpad.cstride;
        ESP_CUDA(cudaMalloc(&p->d_fpad, fb));
        ESP_CUDA(cudaMemset(p->d_fpad, 0, fb));
        if (esp::make_field_tmap(p) != cudaSuccess) {   // no TMA: the cp.async gather
          cudaFree(p->d_fpad);
          p->d_fpad = nullptr;
        }
      }
      if (p->fused) {
        p->n_red_blocks_fft = esp::fused_reduce_blocks(p);
        const long long nb = p->n_red_blocks_fft, ng = (nb + 31) / 32;
        const size_t nd = (size_t)(nb + ng) * 8 + (size_t)(ng + 2) / 2 + 1;
        ESP_CUDA(dalloc(&p->d_partials_fft, nd));
        ESP_CUDA(cudaMemset(p->d_partials_fft, 0, nd * sizeof(double)));
      }
    }
  }
  std::vector<double> hk(3 * msum), hw(msum);
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d)
      std::memcpy(&hk[a * msum + p->koff[d]], c->h_axis_k[3 * a + d],
                  sizeof(double) * p->M[d]);
  for (int d = 0; d < 3; ++d)
    std::memcpy(&hw[p->koff[d]], c->h_axis_what[d], sizeof(double) * p->M[d]);
  ESP_CUDA(cudaMemcpyAsync(p->d_axis_k, hk.data(), sizeof(double) * hk.size(),
                           cudaMemcpyHostToDevice, s));
  ESP_CUDA(cudaMemcpyAsync(p->d_axis_w, hw.data(), sizeof(double) * hw.size(),
                           cudaMemcpyHostToDevice, s));
  ESP_CUDA(cudaMemcpyAsync(p->d_box_iy, iy.data(), sizeof(int) * iy.size(),
                           cudaMemcpyHostToDevice, s));
  ESP_CUDA(cudaMemcpyAsync(p->d_box_iz, iz.data(), sizeof(int) * iz.size(),
                           cudaMemcpyHostToDevice, s));
  ESP_CUDA(esp::launch_mode_setup(p, c->what_zero, s));
  int herr[4] = {0, 0, 0, 0};
  ESP_CUDA(cudaMemcpyAsync(herr, p->d_err, sizeof(herr), cudaMemcpyDeviceToHost, s));
  ESP_CUDA(cudaStreamSynchronize(s));
  unsigned long long nm = 0;
  std::memcpy(&nm, &herr[2], sizeof(nm));
  p->n_modes = (long long)nm;
  p->have_cell = 1;
  p->have_spec = 0;
  p->have_ik = 0;
  if (herr[0]) {
    set_error("window transform underflow on a retained mode; the plan does not "
              "cover the kernel band");
    return ESP_ERR_PLANNING;
  }
  return ESP_OK;
}

static int check_ready(esp_plan* p) {
  if (!p) {
    set_error("null plan");
    return ESP_ERR_PARAM;
  }
  if (!p->have_cell) {
    set_error("esp_plan_set_cell has not been called");
    return ESP_ERR_MESH;
  }
  return ESP_OK;
}

int esp_spread(esp_plan* p, const double* d_pos, const double* d_q, int64_t n, void* d_grid,
               void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (n < 0 || n > p->cap) {
    set_error("particle count exceeds the plan capacity");
    return ESP_ERR_CAPACITY;
  }
  cudaStream_t s = (cudaStream_t)stream;
  p->last_n = n;          // the bins below are for these n charges
  ESP_CUDA(esp::launch_bin(p, d_pos, d_q, n, s));
  ESP_CUDA(esp::launch_spread(p, s, !p->grid_in_scratch));
  if (d_grid) {
    const size_t real_sz = p->precision == ESP_FP64 ? sizeof(double) : sizeof(float);
    ESP_CUDA(cudaMemcpyAsync(d_grid, p->d_grid, real_sz * p->G, cudaMemcpyDeviceToDevice, s));
  }
  p->have_bins = 1;
  p->last_n = n;
  return ESP_OK;
}

int esp_forward(esp_plan* p, const void* d_grid, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t real_sz = p->precision == ESP_FP64 ? sizeof(double) : sizeof(float);
  if (d_grid)
    ESP_CUDA(cudaMemcpyAsync(p->d_grid, d_grid, real_sz * p->G, cudaMemcpyDeviceToDevice, s));
  ESP_CUFFT(cufftSetStream(p->fwd, s));
  if (p->precision == ESP_FP64) {
    ESP_CUFFT(cufftExecD2Z(p->fwd, (cufftDoubleReal*)p->d_grid,
                           (cufftDoubleComplex*)p->d_spec));
  } else {
    ESP_CUFFT(cufftExecR2C(p->fwd, (cufftReal*)p->d_grid, (cufftComplex*)p->d_spec));
  }
  esp::prof_mark(p, s, "fft_forward");
  p->fwd_count++;
  p->have_spec = 1;
  p->have_ik = 0;
  return ESP_OK;
}

int esp_set_spectrum(esp_plan* p, const void* d_spectrum, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  const size_t real_sz = p->precision == ESP_FP64 ? sizeof(double) : sizeof(float);
  ESP_CUDA(cudaMemcpyAsync(p->d_spec, d_spectrum, 2 * real_sz * p->H,
                           cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  p->have_spec = 1;
  p->have_ik = 0;
  return ESP_OK;
}

int esp_scale_reduce(esp_plan* p, double* d_out7, int32_t write_ik, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!p->have_spec) {
    set_error("scale/reduce needs a spectral density (call esp_forward first)");
    return ESP_ERR_MESH;
  }
  ESP_CUDA(esp::launch_scale_reduce(p, d_out7, write_ik, (cudaStream_t)stream));
  p->have_ik = write_ik ? 1 : 0;
  return ESP_OK;
}

int esp_forces_ik(esp_plan* p, double* d_forces, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!p->have_ik || !p->have_bins) {
    set_error("ik forces need esp_spread and esp_scale_reduce(write_ik=1) first");
    return ESP_ERR_MESH;
  }
  cudaStream_t s = (cudaStream_t)stream;
  ESP_CUFFT(cufftSetStream(p->inv3, s));
  if (p->precision == ESP_FP64) {
    ESP_CUFFT(cufftExecZ2D(p->inv3, (cufftDoubleComplex*)p->d_ikspec,
                           (cufftDoubleReal*)p->d_fields));
  } else {
    ESP_CUFFT(cufftExecC2R(p->inv3, (cufftComplex*)p->d_ikspec, (cufftReal*)p->d_fields));
  }
  esp::prof_mark(p, s, "fft_inverse_x3");
  p->fpad_written = 0;
  p->inv_count += 3;
  p->have_ik = 0;  // the C2R transform overwrites its input
  if (p->last_n > 0) ESP_CUDA(esp::launch_gather_ik(p, d_forces, s));
  return ESP_OK;
}

int esp_gather_fields(esp_plan* p, const void* d_fields, double* d_forces, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!p->have_bins) {
    set_error("esp_gather_fields needs a preceding esp_spread (particle bins)");
    return ESP_ERR_MESH;
  }
  if (p->last_n > 0)
    ESP_CUDA(esp::launch_gather_ik(p, d_forces, (cudaStream_t)stream, d_fields));
  return ESP_OK;
}

int esp_forces_analytic(esp_plan* p, double* d_forces, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!p->have_spec || !p->have_bins) {
    set_error("analytic forces need esp_spread and esp_forward first");
    return ESP_ERR_MESH;
  }
  if (p->P > 8) {
    set_error("analytic-differentiation gather supports P <= 8");
    return ESP_ERR_PLANNING;
  }
  cudaStream_t s = (cudaStream_t)stream;
  ESP_CUDA(esp::launch_scale_reduce(p, p->d_err_out7, 2, s));
  ESP_CUFFT(cufftSetStream(p->inv1, s));
  if (p->precision == ESP_FP64) {
    ESP_CUFFT(cufftExecZ2D(p->inv1, (cufftDoubleComplex*)p->d_ikspec,
                           (cufftDoubleReal*)p->d_fields));
  } else {
    ESP_CUFFT(cufftExecC2R(p->inv1, (cufftComplex*)p->d_ikspec, (cufftReal*)p->d_fields));
  }
  p->fpad_written = 0;
  esp::prof_mark(p, s, "fft_inverse_x1");
  p->inv_count += 1;
  p->have_ik = 0;
  if (p->last_n > 0) ESP_CUDA(esp::launch_gather_grad(p, d_forces, s));
  return ESP_OK;
}

int esp_local_pressure(esp_plan* p, double* d_tensors, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!p->have_spec || !p->have_bins) {
    set_error("local pressure needs esp_spread and esp_forward first");
    return ESP_ERR_MESH;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // (xx, xy, xz) -> tensor slots (0, 1, 2) + mirrors (-, 3, 6);
  // (yy, yz, zz) -> (4, 5, 8) + mirrors (-, 7, -)   (mesh.py:371-378)
  const esp::OutMap maps[2] = {{9, {0, 1, 2}, {-1, 3, 6}}, {9, {4, 5, 8}, {-1, 7, -1}}};
  for (int half = 0; half < 2; ++half) {
    ESP_CUDA(esp::launch_scale_reduce(p, p->d_err_out7, 3 + half, s));
    ESP_CUFFT(cufftSetStream(p->inv3, s));
    if (p->precision == ESP_FP64) {
      ESP_CUFFT(cufftExecZ2D(p->inv3, (cufftDoubleComplex*)p->d_ikspec,
                             (cufftDoubleReal*)p->d_fields));
    } else {
      ESP_CUFFT(cufftExecC2R(p->inv3, (cufftComplex*)p->d_ikspec, (cufftReal*)p->d_fields));
    }
    p->fpad_written = 0;
    p->inv_count += 3;
    if (p->last_n > 0) ESP_CUDA(esp::launch_gather_ik(p, d_tensors, s, nullptr, maps[half]));
  }
  p->have_ik = 0;
  return ESP_OK;
}

int esp_evaluate(esp_plan* p, const double* d_pos, const double* d_q, int64_t n,
                 int32_t flags, double* d_out7, double* d_forces, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  const int want_f = (flags & ESP_WANT_FORCES) != 0;
  const int analytic = (flags & ESP_FORCES_ANALYTIC) != 0;
  p->launches = 0;
  p->n_ev = 0;
  cudaStream_t s0 = (cudaStream_t)stream;
  esp::prof_mark(p, s0, "start");
  const int ikmode = want_f ? (analytic ? 2 : 1) : 0;
  if (p->fused && (!analytic || p->P <= 8)) {
    // spread -> fused band-pruned transforms (+ scale/reduce, the ik spectra
    // or, for analytic forces, the potential spectrum, and the inverse
    // transforms) -> gather
    p->want_drec = want_f && analytic;
    // analytic steps write weight and derivative records in one pass; other
    // steps bin with the records-free gather and a coalesced records pass
    p->need_records = 0;   // records (and derivative records) by the coalesced pass
    // the forward x pass sums the spread's tile blocks itself where it can
    // (no k_combine, d_grid not written by this step)
    p->grid_in_scratch = esp::fused_x_combines(p) ? 1 : 0;
    rc = esp_spread(p, d_pos, d_q, n, nullptr, stream);
    p->want_drec = 0;
    p->need_records = 0;
    if (rc) {
      p->grid_in_scratch = 0;
      return rc;
    }
    const cudaError_t fe = esp::launch_fused_fft(p, want_f ? (analytic ? 2 : 1) : 0, d_out7, s0);
    p->grid_in_scratch = 0;
    ESP_CUDA(fe);
    p->fwd_count++;
    p->have_spec = 1;   // in-band box of d_spec is current
    p->have_ik = 0;
    if (want_f) {
      p->inv_count += analytic ? 1 : 3;
      const int chunked = p->host_chunks > 1 && !analytic && p->fpad_written && !p->profiling &&
                          p->have_side && n >= 8 * p->host_chunks;
      if (chunked) {
        // host-buffer step: gather the charges in original-index ranges and
        // copy each range to the pinned host buffer on the side stream while
        // the next range is gathered
        // two ranges: the first larger — its copy overlaps the second gather,
        // the second range's copy is the exposed tail (config-4 e2e, first
        // range 45 / 50 / 55 / 60 / 65 / 70%: 15.00 / 14.82 / 14.62 / 14.45 /
        // 14.57 / 14.69 ms; ESP_HOST_SPLIT overrides)
        static const int split_pct = [] {
          const char* e = std::getenv("ESP_HOST_SPLIT");
          const int v = e ? std::atoi(e) : 0;
          return v >= 10 && v <= 90 ? v : 60;
        }();
        for (int c = 0; c < p->host_chunks; ++c) {
          int64_t lo = n * c / p->host_chunks, hi = n * (c + 1) / p->host_chunks;
          if (p->host_chunks == 2) {
            const int64_t mid = n * split_pct / 100;
            lo = c == 0 ? 0 : mid;
            hi = c == 0 ? mid : n;
          }
          ESP_CUDA(esp::launch_gather_tma(p, d_forces, s0, (int)lo, (int)hi));
          ESP_CUDA(cudaEventRecord(p->ev_chunk[c], s0));
          ESP_CUDA(cudaStreamWaitEvent(p->side, p->ev_chunk[c], 0));
          ESP_CUDA(cudaMemcpyAsync(p->host_forces + 3 * lo, d_forces + 3 * lo,
                                   3 * (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost,
                                   p->side));
        }
        ESP_CUDA(cudaEventRecord(p->ev_join, p->side));
        ESP_CUDA(cudaStreamWaitEvent(s0, p->ev_join, 0));
        return ESP_OK;
      }
      if (p->last_n > 0)
        ESP_CUDA(analytic ? (p->fpad_written ? esp::launch_gather_grad_tma(p, d_forces, s0)
                                             : esp::launch_gather_grad(p, d_forces, s0))
                 : p->fpad_written ? esp::launch_gather_tma(p, d_forces, s0)
                                   : esp::launch_gather_ik(p, d_forces, s0));
    }
    if (want_f && p->host_chunks > 0 && n > 0)
      ESP_CUDA(cudaMemcpyAsync(p->host_forces, d_forces, 3 * n * sizeof(double),
                               cudaMemcpyDeviceToHost, s0));
    return ESP_OK;
  }
  if (ikmode && !p->profiling) {
    // zero the force spectra on a side stream while binning/spreading run
    ESP_CUDA(cudaEventRecord(p->ev_fork, s0));
    ESP_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    const size_t cbytes = p->precision == ESP_FP64 ? sizeof(double2) : sizeof(float2);
    ESP_CUDA(cudaMemsetAsync(p->d_ikspec, 0, (ikmode == 2 ? 1 : 3) * (size_t)p->H * cbytes,
                             p->side));
    ESP_CUDA(cudaEventRecord(p->ev_join, p->side));
  }
  rc = esp_spread(p, d_pos, d_q, n, nullptr, stream);
  if (rc) return rc;
  rc = esp_forward(p, nullptr, stream);
  if (rc) return rc;
  if (ikmode && !p->profiling) {
    ESP_CUDA(cudaStreamWaitEvent(s0, p->ev_join, 0));
    p->ik_zeroed = 1;
  }
  rc = esp_scale_reduce(p, d_out7, want_f && !analytic, stream);
  if (rc) return rc;
  if (want_f) rc = analytic ? esp_forces_analytic(p, d_forces, stream)
                            : esp_forces_ik(p, d_forces, stream);
  if (!rc && want_f && p->host_chunks > 0 && n > 0)
    ESP_CUDA(cudaMemcpyAsync(p->host_forces, d_forces, 3 * n * sizeof(double),
                             cudaMemcpyDeviceToHost, s0));
  return rc;
}

int esp_counters(const esp_plan* p, int64_t* forward, int64_t* inverse) {
  if (!p) return ESP_ERR_PARAM;
  if (forward) *forward = p->fwd_count;
  if (inverse) *inverse = p->inv_count;
  return ESP_OK;
}

int esp_add_counters(esp_plan* p, int64_t forward, int64_t inverse) {
  if (!p) return ESP_ERR_PARAM;
  p->fwd_count += forward;
  p->inv_count += inverse;
  return ESP_OK;
}

int esp_reset_counters(esp_plan* p) {
  if (!p) return ESP_ERR_PARAM;
  p->fwd_count = 0;
  p->inv_count = 0;
  return ESP_OK;
}

int esp_set_profiling(esp_plan* p, int32_t on) {
  if (!p) return ESP_ERR_PARAM;
  if (on && !p->profiling) {
    for (int i = 0; i < 48; ++i) ESP_CUDA(cudaEventCreate(&p->ev[i]));
  }
  if (!on && p->profiling) {
    for (int i = 0; i < 48; ++i) cudaEventDestroy(p->ev[i]);
  }
  p->profiling = on ? 1 : 0;
  p->n_ev = 0;
  p->launches = 0;   // stage-level callers (slab plans) count launches from here
  return ESP_OK;
}

int esp_profile_read(esp_plan* p, char* names, int32_t names_len, double* ms, int32_t max_n) {
  if (!p || !p->profiling) return 0;
  int n = 0;
  std::string all;
  for (int i = 1; i < p->n_ev && n < max_n; ++i) {
    cudaError_t e = cudaEventSynchronize(p->ev[i]);
    if (e != cudaSuccess) {
      set_error(cudaGetErrorString(e));
      return -ESP_ERR_CUDA;
    }
    float t = 0.f;
    cudaEventElapsedTime(&t, p->ev[i - 1], p->ev[i]);
    ms[n++] = t;
    if (!all.empty()) all += ",";
    all += p->ev_name[i];
  }
  if (names && names_len > 0) {
    std::strncpy(names, all.c_str(), names_len - 1);
    names[names_len - 1] = 0;
  }
  return n;
}

void* esp_grid_ptr(esp_plan* p) { return p ? p->d_grid : nullptr; }
void* esp_spectrum_ptr(esp_plan* p) { return p ? p->d_spec : nullptr; }
void* esp_fields_ptr(esp_plan* p) {
  if (!p) return nullptr;
  return p->fpad_written ? p->d_fpad : p->d_fields;
}

int esp_fields_layout(const esp_plan* p, int64_t* layout5) {
  if (!p || !layout5) return ESP_ERR_PARAM;
  if (p->fpad_written) {
    const esp::FieldPad& f = p->fpad;
    layout5[0] = ((long long)f.S[2] * f.E[1] + f.S[1]) * f.E[0] + f.S[0];
    layout5[1] = f.E[0];
    layout5[2] = f.E[1];
    layout5[3] = f.E[2];
    layout5[4] = f.cstride;
  } else {
    layout5[0] = 0;
    layout5[1] = p->M[0];
    layout5[2] = p->M[1];
    layout5[3] = p->M[2];
    layout5[4] = p->G;
  }
  return ESP_OK;
}

int esp_fft_path(const esp_plan* p) { return p && p->fused ? 1 : 0; }

static int check_slab(esp_plan* p, const esp_slab_desc* d) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!d || d->nranks < 1 || d->nranks > 8 || d->rank < 0 || d->rank >= d->nranks) {
    set_error("slab descriptor: 1..8 ranks and 0 <= rank < nranks");
    return ESP_ERR_PARAM;
  }
  if (!p->fused) {
    set_error("slab transforms need the fused transform path (esp_fft_path() == 1)");
    return ESP_ERR_PLANNING;
  }
  if (d->z_start[0] != 0 || d->z_start[d->nranks] != p->M[2]) {
    set_error("slab z_start must run from 0 to Mz");
    return ESP_ERR_PARAM;
  }
  for (int r = 0; r < d->nranks; ++r)
    if (d->z_start[r + 1] <= d->z_start[r]) {
      set_error("slab z_start must be increasing");
      return ESP_ERR_PARAM;
    }
  return ESP_OK;
}

int esp_slab_layout(const esp_plan* p, int32_t nranks, int32_t* by_start, int64_t* info4) {
  if (!p || nranks < 1 || nranks > 8) {
    set_error("slab layout: 1..8 ranks");
    return ESP_ERR_PARAM;
  }
  if (!p->have_cell || !p->fused) {
    set_error("slab layout needs a cell and the fused transform path");
    return ESP_ERR_PLANNING;
  }
  int bs[9];
  esp::slab_by_split(p->nby, nranks, bs);
  if (by_start)
    for (int r = 0; r <= nranks; ++r) by_start[r] = bs[r];
  if (info4) {
    info4[0] = esp::fused_ldx(p);
    info4[1] = p->nby;
    info4[2] = p->nbx;
    info4[3] = p->precision == ESP_FP64 ? 16 : 8;
  }
  return ESP_OK;
}

int esp_slab_forward(esp_plan* p, const esp_slab_desc* d, const void* d_own, void* stream) {
  int rc = check_slab(p, d);
  if (rc) return rc;
  ESP_CUDA(esp::slab_forward(p, d, d_own, (cudaStream_t)stream));
  p->fwd_count++;
  return ESP_OK;
}

int esp_slab_reduce(esp_plan* p, const esp_slab_desc* d, const void* d_recv_fwd, int32_t want_ik,
                    double* d_out7, void* stream) {
  int rc = check_slab(p, d);
  if (rc) return rc;
  ESP_CUDA(esp::slab_reduce(p, d, d_recv_fwd, want_ik, d_out7, (cudaStream_t)stream));
  if (want_ik) p->inv_count += 3;
  return ESP_OK;
}

int esp_slab_inverse(esp_plan* p, const esp_slab_desc* d, const void* d_recv_back, void* d_fields,
                     void* stream) {
  int rc = check_slab(p, d);
  if (rc) return rc;
  ESP_CUDA(esp::slab_inverse(p, d, d_recv_back, d_fields, (cudaStream_t)stream));
  return ESP_OK;
}

int esp_grid_info(const esp_plan* p, int64_t* info) {
  if (!p || !info) return ESP_ERR_PARAM;
  info[0] = p->M[0];
  info[1] = p->M[1];
  info[2] = p->M[2];
  info[3] = p->Hx;
  info[4] = p->n_modes;
  info[5] = p->launches;
  info[6] = p->n_tiles;
  info[7] = p->precision;
  return ESP_OK;
}

int esp_binning_radix(const esp_plan* p, int64_t n, int32_t* radix) {
  if (!p || !radix) return ESP_ERR_PARAM;
  *radix = (n >= p->sort_threshold && p->d_sort_tmp) ? 1 : 0;
  return ESP_OK;
}

}  // extern "C"
