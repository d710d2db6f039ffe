/*
 * esp_b200.h — C ABI of the B200-native ESP k-space (long-range) path, plus
 * the near-field pair sum and the particle-file reader that complete a step.
 *
 * Drop-in replacement for the k-space pipeline of the reference package
 * `prolate_ewald` (arXiv 2601.00161), /root/reference/pkg/src/prolate_ewald:
 *
 *   esp_spread        <- mesh.spread_charges            (mesh.py:204-210)
 *   esp_forward       <- TransformProvider.forward x h3 (mesh.py:45-47, 221-226)
 *   esp_scale_reduce  <- long_range_energy + long_range_pressure
 *                                                     (mesh.py:285-312)
 *   esp_forces_ik     <- long_range_forces(mode="ik")   (mesh.py:315-342)
 *   esp_forces_analytic <- long_range_forces(mode="analytic") (mesh.py:343-349)
 *   esp_local_pressure  <- local_pressure               (mesh.py:353-379)
 *   esp_evaluate      <- CoulombSolver.evaluate far-field part
 *                                                     (evaluate.py:125-144)
 *   esp_plan_create / esp_plan_set_cell
 *                     <- plan_grid + ModeWorkspace      (mesh.py:81-142, 229-282)
 *   esp_counters      <- TransformProvider.forward_count / inverse_count
 *                                                     (mesh.py:33-55)
 *   esp_near_*        <- realspace.short_range / build_pair_table,
 *                        system.build_cell_list        (realspace.py:29-157,
 *                                                     system.py:144-222)
 *   esp_particles_*   <- cli.read_particles / write_particles (cli.py:57-112)
 *
 * Conventions
 *  - All pointers named d_* are DEVICE pointers; h_* are host pointers.
 *  - Positions: (N,3) row-major f64 (the reference's ParticleSystem.positions,
 *    already wrapped into the cell).  Charges: (N,) f64.
 *  - Forces: (N,3) row-major f64, in the caller's particle order.
 *  - out7: 7 f64 = [E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz] (far-field energy and the
 *    symmetric pressure tensor, prefactor 1, as mesh.py returns them).
 *  - Device grid layout is [z][y][x] (x contiguous): a relabelling of the
 *    reference's C-order [x][y][z]; values are identical.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*).
 *    Calls on one plan must not run concurrently.
 *  - Return value: ESP_OK or an error code; esp_last_error() gives the text.
 *    Error codes map onto the reference's exception classes
 *    (PlanningError mesh.py:25, MeshError mesh.py:29, ParameterError
 *    evaluate.py:247) in the Python wrapper.
 */
#ifndef ESP_B200_H
#define ESP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum esp_status {
  ESP_OK = 0,
  ESP_ERR_PLANNING = 1,   /* grid invariant / window / underflow (PlanningError) */
  ESP_ERR_MESH = 2,       /* wrong call order / unknown mode (MeshError) */
  ESP_ERR_PARAM = 3,      /* bad argument (ParameterError) */
  ESP_ERR_CUDA = 4,
  ESP_ERR_CUFFT = 5,
  ESP_ERR_OOM = 6,
  ESP_ERR_CAPACITY = 7,   /* N above the plan's particle capacity */
  ESP_ERR_INPUT = 8       /* malformed particle file (cli.InputError) */
};

enum esp_precision { ESP_FP64 = 0, ESP_FP32 = 1 };

/* Flags for esp_evaluate. */
enum esp_eval_flags {
  ESP_WANT_ENERGY_PRESSURE = 1,
  ESP_WANT_FORCES = 2,
  ESP_FORCES_ANALYTIC = 4
};

typedef struct esp_plan esp_plan;

/* Static plan description (grid counts, window, basis constants). */
typedef struct esp_plan_desc {
  int32_t M[3];            /* grid counts along lattice axes x, y, z        */
  int32_t P;               /* stencil width                                  */
  int32_t precision;       /* esp_precision                                  */
  int32_t deterministic;   /* 1: bitwise run-to-run reproducible ordering    */
  int64_t max_particles;   /* particle capacity of the plan's buffers       */
  /* Spreading window W(t) = psi_0(2t/P): piecewise monomial table
   * (pswf.py:238-293); coef[j*(degree+1)+m] = scipy PPoly c[m][j]
   * (highest power first), breaks[0..n_pieces].                            */
  int32_t n_pieces;
  int32_t degree;
  const double* h_window_coef;
  const double* h_window_deriv_coef;   /* derivative table (analytic mode)  */
  const double* h_window_breaks;
  /* Splitting basis psi_0^c as a Legendre series (pswf.py:41-84) and its
   * derivative series (numpy legder), for Fhat and dterm (mesh.py:269-275). */
  int32_t n_legendre;
  const double* h_legendre;
  int32_t n_legendre_deriv;
  const double* h_legendre_deriv;
  double split_c, split_lambda0, split_C0;
  double r_c;
  double kmax;             /* split_c / r_c (kernel.py:28-39)                */
  /* Tile shape override (0 = automatic).                                   */
  int32_t tile[3];
  /* z-slab plans (multi-GPU slab decomposition): 0 = whole
   * periodic grid.  Otherwise M[2] = owned planes + P - 1 ghost planes,
   * slab_mz_global = global Mz and slab_z0 = first owned global plane.      */
  int32_t slab_mz_global;
  int32_t slab_z0;
} esp_plan_desc;

/* Per-cell data (ModeWorkspace inputs; re-sent on NPT rebind with M pinned,
 * evaluate.py:99-112).  Arrays are host arrays of length M[d].             */
typedef struct esp_cell_desc {
  double h[9];             /* cell matrix, row-major, columns = cell vectors */
  double hinv[9];          /* inverse of h, row-major                        */
  int32_t orthorhombic;
  double spacing[3];       /* L_d / M_d (orthorhombic u = x / spacing)       */
  double volume;           /* det h                                          */
  double volume_element;   /* h_x h_y h_z (ortho) or V/G (triclinic)         */
  /* K[a*3+d][m]: Cartesian component a of k contributed by index m along
   * lattice axis d (mesh.py:242; 2 pi h^-T m for triclinic).               */
  const double* h_axis_k[9];
  /* Per-axis window transforms; What(m) = (w0[mx]*w1[my])*w2[mz]
   * (mesh.py:258-261).                                                     */
  const double* h_axis_what[3];
  double what_zero;        /* What(0) for the underflow guard (mesh.py:262)  */
  int32_t band[3];         /* max |m_d| that can lie inside |k| <= kmax      */
  double grad_scale[3];    /* 1/spacing_d for the analytic window gradient   */
} esp_cell_desc;

/* --- lifetime ----------------------------------------------------------- */
int esp_plan_create(const esp_plan_desc* desc, esp_plan** out);
int esp_plan_destroy(esp_plan* plan);
int esp_plan_set_cell(esp_plan* plan, const esp_cell_desc* cell, void* stream);
const char* esp_last_error(void);
int esp_version(void);
/* Stream-ordered copy (cudaMemcpyDefault: host <-> device by pointer), so a
 * host-buffer step captured in a CUDA graph moves its inputs and outputs as
 * copy-engine DMA at full PCIe rate (pinned host memory).                   */
int esp_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* Page-locked host buffers for the host-buffer step (cudaHostAlloc).  On the
 * measured B200 box, H2D copies from these run at ~52 GB/s against ~12 GB/s
 * from torch's pinned allocator (copy probe).          */
int esp_host_alloc(int64_t bytes, void** out);
/* The next esp_evaluate / esp_spread waits on `event` (a cudaEvent_t) before
 * its first kernel that reads the charges, so a charge copy on another
 * stream overlaps the position binning (host-buffer step).  One-shot.      */
int esp_set_charges_event(esp_plan* plan, void* event);
/* Every later force-computing esp_evaluate also copies its forces (N x 3
 * doubles, original order) to `host_forces` (page-locked).  With nchunks > 1
 * the fused ik step gathers the charges in nchunks original-index ranges and
 * copies each range on a side stream while the next is gathered; other paths
 * copy once after the gather.  The copy is stream-ordered: it has finished
 * when the esp_evaluate stream is synchronised.  nchunks = 0 turns it off;
 * at most 8.                                                                */
int esp_set_host_forces(esp_plan* plan, double* host_forces, int32_t nchunks);
int esp_host_free(void* p);

/* --- stages (reference-function granularity) ----------------------------- */
/* Bin + spread: writes the real charge grid (device layout [z][y][x]).
 * d_grid may be NULL to keep it only in the plan.                          */
int esp_spread(esp_plan* plan, const double* d_pos, const double* d_q,
               int64_t n, void* d_grid, void* stream);
/* Forward transform of the plan's grid -> plan spectrum (half spectrum along
 * x, [kz][ky][kx<=Mx/2], complex, NOT yet multiplied by h3).  If d_grid is
 * non-NULL it is copied into the plan first.  Counts one forward transform. */
int esp_forward(esp_plan* plan, const void* d_grid, void* stream);
/* Fused deconvolution scaling + energy/pressure reduction over the plan
 * spectrum; optionally writes the three ik-scaled spectra for the force
 * path in the same pass.  d_out7 is a device pointer (7 doubles).          */
int esp_scale_reduce(esp_plan* plan, double* d_out7, int32_t write_ik, void* stream);
/* Three inverse transforms of the ik spectra + force gather (requires a
 * preceding esp_spread on the same particles and esp_scale_reduce with
 * write_ik=1).  Counts three inverse transforms.                           */
int esp_forces_ik(esp_plan* plan, double* d_forces, void* stream);
/* Gather ik forces from caller-provided field grids [3][M2][M1][M0] (e.g. a
 * slab with ghost planes) for the particles of the last esp_spread.        */
int esp_gather_fields(esp_plan* plan, const void* d_fields, double* d_forces,
                      void* stream);
/* One inverse transform + window-gradient gather (orthorhombic only).      */
int esp_forces_analytic(esp_plan* plan, double* d_forces, void* stream);
/* Six inverse transforms + gathers -> per-particle tensors (N,3,3).        */
int esp_local_pressure(esp_plan* plan, double* d_tensors, void* stream);
/* Whole step: spread, 1 forward FFT, fused scale/reduce, and (flags) forces. */
int esp_evaluate(esp_plan* plan, const double* d_pos, const double* d_q,
                 int64_t n, int32_t flags, double* d_out7, double* d_forces,
                 void* stream);

/* --- introspection -------------------------------------------------------- */
int esp_counters(const esp_plan* plan, int64_t* forward, int64_t* inverse);
int esp_reset_counters(esp_plan* plan);
/* Add to the transform counters: a captured CUDA graph counts its transforms
 * when it is captured, not when it replays, so the graph owner adds the
 * captured step's counts at every replay (TransformProvider counters,
 * mesh.py:33-55).                                                           */
int esp_add_counters(esp_plan* plan, int64_t forward, int64_t inverse);
/* Device pointers into the plan (valid until destroy / next set_cell).     */
void* esp_grid_ptr(esp_plan* plan);       /* real grid, [z][y][x]: the grid of the
                                             last esp_spread (esp_evaluate on the
                                             fused transforms sums the spread's tile
                                             blocks inside its x pass and does not
                                             write this grid)                  */
void* esp_spectrum_ptr(esp_plan* plan);   /* complex half spectrum          */
void* esp_fields_ptr(esp_plan* plan);     /* 3 ik force fields (layout below) */
/* Layout of the fields behind esp_fields_ptr after the last force step:
 * {origin offset, row pitch, rows per plane, planes, component stride} in
 * elements; field c at (x, y, z) is ptr[origin + c*cstride + (z*rows + y)*pitch
 * + x].  The band-pruned ik path of fp64 plans writes ghost-padded fields
 * (periodic images around the grid, read by the TMA gather); other paths
 * write the dense [3][z][y][x] grid (origin 0, pitch Mx). */
int esp_fields_layout(const esp_plan* plan, int64_t* layout5);
int esp_grid_info(const esp_plan* plan, int64_t* info8);
/* 1 in *radix when a step over n charges bins with the device radix sort
 * (n >= the plan's sort threshold; ESP_SORT_THRESHOLD at plan creation
 * overrides the default 5e5), 0 for the counting sort.  Both binnings give
 * bitwise-identical results (replaces nothing: introspection for tests). */
int esp_binning_radix(const esp_plan* plan, int64_t n, int32_t* radix);
/* info8 = {Mx, My, Mz, Hx(=Mx/2+1), n_modes_retained(full spectrum),
 *          kernel_launches_last_step, n_tiles, precision}                   */
int esp_set_spectrum(esp_plan* plan, const void* d_spectrum, void* stream);
/* Transform path esp_evaluate uses: 1 = band-pruned fused transforms
 * (grid lengths in {32,48,64,96,128,192,256,384}, full-grid plans),
 * 0 = cuFFT.  ESP_FFT=cufft in the environment forces 0 at set_cell. */
int esp_fft_path(const esp_plan* plan);

/* --- particle files (cli.py:57-112) -----------------------
 * Native reader / writer of the reference's text format: header 'cell Lx Ly
 * Lz' or 'cell3' + h in column order, then 'x y z q m' lines; '#' comments.
 * Errors (ESP_ERR_INPUT) carry path:line[:column] as cli.InputError does.
 * h9 is row-major (columns = cell vectors).  Positions are returned as read
 * (the Python ParticleSystem wraps them, as the reference does).            */
typedef struct esp_particles esp_particles;
int esp_particles_read(const char* path, esp_particles** out);
int esp_particles_info(const esp_particles* p, int64_t* n, int32_t* triclinic, double* h9);
int esp_particles_copy(const esp_particles* p, double* h_pos, double* h_q, double* h_m);
int esp_particles_free(esp_particles* p);
int esp_particles_write(const char* path, int64_t n, const double* h9, int32_t triclinic,
                        const double* h_pos, const double* h_q, const double* h_m);

/* --- distributed z-slab transforms --------------------------- */
/* Rank `rank` of `nranks` (<= 8) slabs of a full-grid plan whose
 * esp_fft_path() is 1.  Planes are split by z_start (nranks+1 entries); the
 * in-band ky rows are split evenly (esp_slab_layout).  The forward and
 * backward transposes are fused into the transform kernels: they store
 * straight into the destination rank's receive buffer, so fwd_peers[r] /
 * back_peers[r] must be rank r's buffers mapped into this process (NVLink
 * peer memory; on one GPU, plain device buffers).  Between the stages the
 * caller orders the ranks (a stream-ordered barrier): forward ->
 * barrier -> reduce -> barrier -> inverse.  Replaces the rfft2 /
 * all_to_all / fft sequence of the slab orchestration. */
typedef struct {
  int32_t nranks, rank;
  int32_t z_start[9];
  void* fwd_peers[8];    /* rank r: [Mz][ny_r][ldx] complex (plan precision) */
  void* back_peers[8];   /* rank r: [3][nz_r][nby][ldx] complex              */
} esp_slab_desc;
/* by_start (nranks+1 entries) and info4 = {ldx, nby, nbx, complex bytes}.  */
int esp_slab_layout(const esp_plan* plan, int32_t nranks, int32_t* by_start, int64_t* info4);
/* own planes [nz][My][Mx] (real) -> x, y passes -> every rank's fwd buffer */
int esp_slab_forward(esp_plan* plan, const esp_slab_desc* d, const void* d_own, void* stream);
/* this rank's fwd buffer -> z pass, this rank's share of [E, P_ab] into
 * d_out7 (sum the ranks' out7 in rank order); want_ik: ik + inverse z ->
 * every rank's back buffer */
int esp_slab_reduce(esp_plan* plan, const esp_slab_desc* d, const void* d_recv_fwd,
                    int32_t want_ik, double* d_out7, void* stream);
/* this rank's back buffer -> inverse y, x -> the rank's three field slabs
 * [3][nz][My][Mx] (unghosted)                                             */
int esp_slab_inverse(esp_plan* plan, const esp_slab_desc* d, const void* d_recv_back,
                     void* d_fields, void* stream);

/* --- diagnostics (bench / roofline) ----------------------------------------- */
/* Record a CUDA event after every stage kernel of esp_evaluate.            */
int esp_set_profiling(esp_plan* plan, int32_t on);
/* Per-kernel durations (ms) of the last profiled esp_evaluate; names are
 * written comma-separated.  Returns the count (synchronises on the events). */
int esp_profile_read(esp_plan* plan, char* names, int32_t names_len, double* ms,
                     int32_t max_n);
/* Measured FP64 FMA throughput of this device (TFLOP/s), DFMA-chain probe. */
int esp_probe_fp64(double* tflops, void* stream);

/* --- near field (real-space pair sum) ---------------------
 *
 *   esp_near_evaluate        <- build_cell_list + short_range
 *                               (system.py:144-222, realspace.py:115-157)
 *   esp_near_evaluate_pairs  <- short_range with a caller NeighborList
 *                               (realspace.py:115-157, system.py:123-135)
 *   esp_near_desc tables     <- PairTable / build_pair_table (realspace.py:29-112)
 *                               or, use_table = 0, kernel.near_field / fn_weight
 *                               (kernel.py:41-97) from the Legendre series
 *
 * out7 = [E_near, P_xx, P_xy, P_xz, P_yy, P_yz, P_zz] (pressure = virial / V,
 * realspace.py:155-156); forces (N,3) in the caller's order (overwritten, or
 * added to with ESP_NEAR_ACCUMULATE); stats (device int64[4]) = {pair count
 * within r_c, first coincident pair (i << 32 | j) or -1, first pair with an
 * index outside [0, N) or -1, directed pair count}.  A coincident pair (r < 1e-12 r_c) is the
 * reference's SingularPairError (realspace.py:20-21, 134-137).            */
enum esp_near_flags { ESP_NEAR_ACCUMULATE = 1 };

typedef struct esp_near esp_near;

typedef struct esp_near_desc {
  double r_c;               /* cutoff (SplitKernel.r_c)                      */
  double reach;             /* cell-list reach, >= r_c (r_c + skin)          */
  int32_t use_table;        /* 1: PairTable values, 0: exact series          */
  /* PairTable (realspace.py:29-40): polynomial pieces on [0, r_in],
   * ascending powers; cubic splines on [r_in, r_c] as scipy PPoly: knots
   * (n_knots) and c[4][n_knots-1], highest power first.                     */
  double r_in;
  int32_t poly_order;
  const double* h_smooth_poly;
  const double* h_fn_poly;
  int32_t n_knots;
  const double* h_knots;
  const double* h_smooth_spline;
  const double* h_fn_spline;
  /* psi_0 Legendre series and its integral from 0 (pswf.py:123-160),
   * C0 = int_0^1 psi_0                                                      */
  int32_t n_legendre;
  const double* h_legendre;
  int32_t n_cumint;
  const double* h_cumint;
  double C0;
  int64_t max_particles;
  int32_t cell_div;         /* cells per reach along each axis (0 = 2)       */
} esp_near_desc;

int esp_near_create(const esp_near_desc* desc, esp_near** out);
int esp_near_destroy(esp_near* plan);
/* Grow the particle / pair-list capacity (allocates; call outside graphs). */
int esp_near_reserve(esp_near* plan, int64_t n_particles, int64_t n_pairs);
/* Bind a cell: h and h^-1 row-major (columns of h = cell vectors).  Checks
 * reach < half the minimum perpendicular width (system.py:137-141,
 * GeometryError) and builds the cell lattice and stencil.                  */
int esp_near_set_cell(esp_near* plan, const double* h_h, const double* h_hinv,
                      int32_t orthorhombic, double volume);
int esp_near_evaluate(esp_near* plan, const double* d_pos, const double* d_q, int64_t n,
                      int32_t flags, double* d_out7, double* d_forces, int64_t* d_stats,
                      void* stream);
/* Slab-local variant (multi-GPU near field): particles [0, n_owned) of the
 * input are this rank's, [n_owned, n) ghosts within reach of its slab from
 * other ranks.  Sums (out7, forces, directed count) cover the owned
 * particles' directed pairs only; forces has n_owned rows.                  */
int esp_near_evaluate_local(esp_near* plan, const double* d_pos, const double* d_q, int64_t n,
                            int64_t n_owned, int32_t flags, double* d_out7, double* d_forces,
                            int64_t* d_stats, void* stream);
/* Pairs (d_i[k], d_j[k]) as given (int64 device arrays), separation by
 * minimum_image.                                                           */
int esp_near_evaluate_pairs(esp_near* plan, const double* d_pos, const double* d_q,
                            int64_t n, const int64_t* d_i, const int64_t* d_j,
                            int64_t n_pairs, int32_t flags, double* d_out7,
                            double* d_forces, int64_t* d_stats, void* stream);
/* Pair enumeration (system.build_cell_list, system.py:144-222): every
 * unordered pair within reach under the minimum image, as i < j (original
 * indices) sorted by (i, j), into plan-owned buffers; *n_pairs = the count
 * (host).  Synchronises `stream`.  esp_near_copy_pairs then copies the list
 * into caller int64 device arrays of n_pairs entries each.                 */
int esp_near_build_pairs(esp_near* plan, const double* d_pos, int64_t n, int64_t* n_pairs,
                         void* stream);
int esp_near_copy_pairs(esp_near* plan, int64_t* d_i, int64_t* d_j, void* stream);
/* info8 = {nc_x, nc_y, nc_z, candidate rows, capacity, launches last call,
 *          cells per reach, use_table}                                      */
int esp_near_info(const esp_near* plan, int64_t* info8);

#ifdef __cplusplus
}
#endif
#endif /* ESP_B200_H */
