/*
 * seethrough_b200 -- C ABI of the B200-native EM light-field background
 * reconstruction (arXiv 2003.11076).
 *
 * The reference (`seethrough`, pure Python/numpy) has no native FFI; its
 * public entry points for this path are Python functions.  Each entry point
 * below is the native replacement a ctypes binding calls in place of the
 * reference function cited next to it (paths relative to
 * /root/reference/pkg/src/seethrough/).  See INTEGRATION.md for the binding.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers (caller-owned; the Python layer
 *     allocates them as torch CUDA tensors).  Calls are ordered on `stream`
 *     (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - Images are (K, H, W, 3) uint8, priors (K, H, W) float32, descriptors
 *     (K, H, W, 16) uint8, per-pixel maps are row-major H*W.
 *   - Return 0 on success, a negative ST_E* code on failure; the message is
 *     available from st_last_error() (thread-local).  Validation errors carry
 *     the reference's exact ValueError text.
 *   - No CPU fallback exists: every compute entry point launches sm_100a
 *     kernels and fails with ST_ECUDA when no device is usable.
 */
#ifndef SEETHROUGH_B200_H
#define SEETHROUGH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_MAX_VIEWS 12   /* solver.py:46 MAX_ENUMERATED_VIEWS */
#define ST_MAX_ITERS 1024 /* capacity of the per-iteration EMStats arrays; larger max_iters is
                             rejected with ST_EINVAL (solver.py:461 has no cap) */
#define ST_DESC_LEN 16    /* features.py:19 */
#define ST_DESC_MARGIN 3  /* features.py:20 */

enum {
  ST_OK = 0,
  ST_EINVAL = -1,  /* bad argument (ValueError in the reference) */
  ST_ECUDA = -2,   /* CUDA runtime / launch failure */
  ST_ENOMEM = -3,  /* workspace too small */
  ST_EAGAIN = -4,  /* row bands: redo the frame with a whole-frame surface raster */
};

/* solver.py:48-50 */
enum { ST_STATUS_VALID = 0, ST_STATUS_LOW_TEXTURE = 1, ST_STATUS_NO_STATIC_EVIDENCE = 2 };
/* refocus.py:19-21 */
enum { ST_PROV_FALLBACK = 0, ST_PROV_COPIED = 128, ST_PROV_REFOCUSED = 255 };

/* CameraRig warp tables (geometry.py:156-172, 200-202): the homogeneous warp
 * of reference pixel (u, v) at disparity d into view k is
 * h = A_k (u, v, 1) + d b_k, evaluated left to right in fp64. */
typedef struct {
  int32_t num_views;
  int32_t ref_index;
  int32_t width, height;                    /* frame size (every view) */
  double warp_a[ST_MAX_VIEWS][9];           /* row-major 3x3 */
  double warp_b[ST_MAX_VIEWS][3];
  int32_t view_w[ST_MAX_VIEWS];             /* rig intrinsics size, for the margin test */
  int32_t view_h[ST_MAX_VIEWS];             /* (solver.py:197-204 uses rig dims)        */
} st_rig;

/* SolverParams (solver.py:56-62) + PriorParams (prior.py:33-40). */
typedef struct {
  double beta;
  double threshold;
  int32_t max_iters;
  int32_t min_static_rays;
  double epsilon_prior;
  double sigma;
  double gamma;
  double d_max;
  double neighborhood_radius;
  int32_t forced_iters; /* >0: run exactly this many iterations (bench mode, non-reference) */
  int32_t timing;       /* 1: st_solve brackets its kernels with CUDA events (st_stats.kernel_ms) */
} st_params;

/* EMStats (solver.py:84-90) */
typedef struct {
  int32_t iterations_run;
  int32_t converged_after;           /* -1 == None */
  double mean_energy[ST_MAX_ITERS];
  double prev_energy[ST_MAX_ITERS];
  double changed_fraction[ST_MAX_ITERS];
  int64_t active_pixels;
  int64_t support_records;           /* diagnostic: (tile, value) records built */
  int64_t candidates_total;          /* sum over iterations/pixels of candidates in range */
  int64_t energy_evals;              /* sum of candidate energies actually evaluated */
  int64_t prev_evals;                /* previous-disparity energies computed (iterations >= 2) */
  int64_t msteps;                    /* pixel M-steps computed (incremental EM skips the rest) */
  int64_t esteps;                    /* pixel E-steps computed */
  /* with st_params.timing: summed CUDA-event durations per kernel family
   * [0] k_m_step, [1] k_e_step_at, [2] k_initial_masks, [3] the rest */
  double kernel_ms[4];
  int32_t kernel_launches[4];
  int64_t hopeless_msteps;           /* pixel M-steps with fewer static views than min_static_rays */
  int64_t energy_samples;            /* M-step descriptor samples: static in-margin rays of the real
                                        candidates evaluated (incl. previous-disparity energies) */
} st_stats;

const char* st_last_error(void);
int st_version(void);
int st_device_count(void);
/* sizeof the ABI structs as this library was compiled (binding checks, no GPU
 * needed): which = 0 st_rig, 1 st_params, 2 st_stats, 3 st_frame, 4 st_tri,
 * 5 st_cams, 6 st_frame_plan, 7 st_scene; -1 for an unknown id. */
int64_t st_struct_size(int32_t which);
/* Cumulative number of __global__ launches issued by this library (all
 * threads; CUB's internal launches inside st_support_build / st_solve count
 * as one per CUB call). */
int64_t st_launch_count(void);
/* The EM tail loop (iterations >= 3 of a one-device solve run as a CUDA
 * graph WHILE loop, cached per argument set; the environment variable
 * ST_NO_GRAPH selects the plain launch loop): which = 0 graphs built,
 * 1 graph launches, cumulative.  A graph launch counts its body's kernels
 * once in st_launch_count. */
int64_t st_tail_graph_count(int32_t which);
/* Diagnostics: which = 1 checks the kernels' exact small-integer division
 * (div_small) against __ddiv_rn on n random doubles x 12 divisors and
 * returns the number of bit mismatches (expected 0). */
int st_selftest(int32_t which, int64_t n, uint64_t seed, int64_t* mismatches, void* stream);

/* Diagnostics: measured FP64 (DFMA) throughput of this device in TFLOP/s
 * (8 independent FMA chains per thread, best of 5; synchronises). */
int st_fp64_peak(double* tflops, void* stream);

/* ---- L1 primitives ---------------------------------------------------- */

/* features.py:81-104 compute_descriptors (with rgb_to_gray :29-36 and
 * sobel_responses :39-58) for K views at once.  channels = 3 (RGB) or 1. */
int st_descriptors(const uint8_t* images, int32_t K, int32_t H, int32_t W, int32_t channels,
                   uint8_t* desc_out, uint8_t* gray_out /* nullable (K,H,W) */,
                   uint8_t* sobel_out /* nullable (K,H,W,2): biased gx, gy */, void* stream);

/* sampling.py:21-55 bilinear on an (h*w, c) float32 plane; out (n, c) f64. */
int st_bilinear(const float* plane, int32_t h, int32_t w, int32_t c, const double* u,
                const double* v, int64_t n, double* out, void* stream);

/* geometry.py:204-219 CameraRig.warp for view k; ok is uint8. */
int st_warp(const st_rig* rig, int32_t k, const double* u, const double* v, const double* d,
            int64_t n, double* pu, double* pv, uint8_t* ok, void* stream);

/* TriangulationPrior (prior.py:265-315) on the device, with the Qhull tables
 * scipy's Delaunay.find_simplex walks (scipy.spatial.Delaunay: neighbors,
 * transform, equations, paraboloid_scale/shift, min/max_bound). */
typedef struct {
  const double* points;       /* (n_pts,2) vertex coordinates (u, v) */
  const double* disparities;  /* (n_pts) */
  const int32_t* simplices;   /* (n_tri,3) */
  const double* planes;       /* (n_tri,3) d = a u + b v + c */
  const int32_t* neighbors;   /* (n_tri,3) Qhull neighbour opposite vertex k, -1 on the hull */
  const double* transform;    /* (n_tri,3,2) barycentric transforms */
  const double* equations;    /* (n_tri,4) lifted facet hyperplanes */
  int32_t n_pts, n_tri;
  double paraboloid_scale, paraboloid_shift;
  double min_bound[2], max_bound[2];
  double centroid[2];         /* points.mean(axis=0) as numpy computes it (prior.py:290) */
} st_tri;

/* The two per-triangle tables the reference computes on the host with
 * LAPACK, recomputed on the device with the same operation order:
 *  - planes (n_tri,3): np.linalg.solve([u v 1], d) of triangulate
 *    (prior.py:351-357) -- OpenBLAS dgesv = getf2 (left-looking, pivot
 *    scaling by the reciprocal, fused dot updates) + trsv (fused axpy,
 *    division by the diagonal);
 *  - transform (n_tri,3,2): scipy Delaunay.transform
 *    (_get_barycentric_transforms) -- getf2 + trsm on the identity
 *    (reciprocal diagonal); rows of NaN for flat triangles.
 * Pixel coordinates must be integers of magnitude < 2^24 (support points
 * and corner anchors are), which makes the scipy condition-number test
 * exact: flat <=> integer determinant 0.  *flags (device int32, or-ed):
 * 1 = some plane system hit an exact zero pivot (numpy raises
 * LinAlgError -> "zero-area triangle").  Reads points/disparities/simplices
 * of *tri, writes through planes_out / transform_out. */
int st_tri_tables(const st_tri* tri, double* planes_out, double* transform_out, int32_t* flags,
                  void* stream);

/* prior.py:276-310 TriangulationPrior.disparity_map -- the containing
 * triangle's plane at every pixel centre, choosing the triangle exactly as
 * scipy's find_simplex walk does for a raster-order batch -- then the
 * solver's clip to [1e-6, d_max] (solver.py:185-186) when clip_dmax > 0.
 * mu out (H*W) f64. */
int st_mu_raster(const st_tri* tri, int32_t W, int32_t H, double clip_dmax, double* mu_out,
                 void* workspace, int64_t workspace_bytes, void* stream);
int64_t st_mu_raster_workspace(int32_t W, int32_t H, int32_t n_tri);
/* st_mu_raster for rows [row0, row1) only (a row band's solved rows): the
 * Qhull walk replay runs over those rows plus 2 halo rows above, whose walks
 * seed the band's (a pixel with a single claiming triangle ends every
 * dependency chain).  *unsafe_out (device int, nullable) is set when the
 * chain entering the band starts at the window's first pixel, or when a
 * band pixel lies off the hull (the reference's nudged batch carries its
 * start across the whole frame): the band's mu is then not exact and the
 * caller rasters the whole frame instead. */
int st_mu_raster_rows(const st_tri* tri, int32_t W, int32_t H, double clip_dmax,
                      double* mu_out, void* workspace, int64_t workspace_bytes, int32_t row0,
                      int32_t row1, int32_t* unsafe_out, void* stream);

/* ---- solver pieces (DisparitySolver API, solver.py:162-432) ----------- */

/* Per-frame device context the solver entry points share. */
typedef struct {
  const uint8_t* images;   /* (K,H,W,3) */
  const float* priors;     /* (K,H,W)   */
  const uint8_t* desc;     /* (K,H,W,16) */
  const double* mu;        /* (H*W) clipped surface */
  /* support candidate groups built by st_support_build: for every 32x8
   * pixel tile, its distinct fp32 support disparities (ascending) with a
   * 32x8 bit mask of the tile pixels whose radius holds such a point */
  const uint32_t* sup_tile_start;  /* (n_tiles+1) first group of each tile */
  const float* sup_value;          /* (n_groups) fp32-rounded support disparity */
  const uint32_t* sup_mask;        /* (n_groups, 8) row bit masks */
  /* nullable: device flag from st_mu_raster_rows; nonzero = this shard's
   * row-window raster could not be made exact (st_solve_rows then returns
   * ST_EAGAIN on every shard and the caller rasters the whole frame) */
  const int32_t* mu_unsafe;
} st_frame;

/* Build per-tile support candidate lists (solver.py:286-321 semantics).
 * support_uv (n,2) f64 pixel coords, support_d (n) f64.  Writes into
 * workspace; fills the sup_* pointers of *frame.  With n_records non-NULL
 * the record count is read back (one host synchronisation) and returned;
 * with n_records NULL nothing waits on the device (the sort runs over the
 * workspace's record bound with padding keys). */
int st_support_build(const double* support_uv, const double* support_d, int32_t n,
                     int32_t W, int32_t H, const st_params* params, st_frame* frame,
                     void* workspace, int64_t workspace_bytes, int64_t* n_records,
                     void* stream);
int64_t st_support_workspace(int32_t n, int32_t W, int32_t H, double radius);
/* st_support_build for the tiles of rows [row0, row1) only (a row band's
 * solved rows): the other tiles get no candidate groups. */
int st_support_build_rows(const double* support_uv, const double* support_d, int32_t n,
                          int32_t W, int32_t H, const st_params* p, st_frame* frame,
                          void* workspace, int64_t workspace_bytes, int64_t* n_records,
                          int32_t row0, int32_t row1, void* stream);

/* ---- support harvest (prior.py:51-260) ----------------- */

/* The rig quantities collect_support reads (geometry.py:128-252), with the
 * pair warps precomputed on the host by the reference's own numpy
 * expressions (pair_warp_coefficients, geometry.py:221-240). */
typedef struct st_cams {
  int32_t num_views;
  int32_t ref_index;
  int32_t width, height;                  /* every view */
  int32_t nn[ST_MAX_VIEWS];               /* nearest_neighbor(k), geometry.py:191-196 */
  double fx[ST_MAX_VIEWS], fy[ST_MAX_VIEWS], cx[ST_MAX_VIEWS], cy[ST_MAX_VIEWS];
  double rot[ST_MAX_VIEWS][9];            /* extrinsics rotation, row-major */
  double trans[ST_MAX_VIEWS][3];
  double unit_baseline;
  double fw_a[ST_MAX_VIEWS][9], fw_b[ST_MAX_VIEWS][3];  /* warp k -> nn[k] */
  double bw_a[ST_MAX_VIEWS][9], bw_b[ST_MAX_VIEWS][3];  /* warp nn[k] -> k */
  double lr_scale[ST_MAX_VIEWS];          /* fx[k] / fx[nn[k]] (prior.py:132) */
} st_cams;

/* collect_support up to (not including) deduplicate: detection on the
 * stride grid (prior.py:51-66) gated by the eroded prior (:215-230, :248-250),
 * forward SAD scan + uniqueness ratio + left-right check against the nearest
 * neighbour (:69-138), and reprojection of other views' matches into the
 * reference (:146-180).  n_d = len(np.arange(0.5, d_max + 0.25, 0.5)) <= 512.
 * Writes the collected points in the reference's collection order (view,
 * then raster) to out_u/out_v/out_d/out_src (device, capacity
 * st_harvest_capacity) and their number to *out_count (device int64). */
int st_harvest(const uint8_t* desc, const float* priors, const st_cams* cams, double d_max,
               int32_t n_d, float threshold, int32_t stride, double min_texture,
               int32_t* out_u, int32_t* out_v, double* out_d, int32_t* out_src,
               int64_t* out_count, int64_t* counters, void* workspace, int64_t workspace_bytes,
               void* stream);
/* counters (nullable, device int64[2]): candidates scanned, reverse scans run
 * (each scan = n_d descriptor samples; the bench's roofline unit). */
int64_t st_harvest_capacity(int32_t K, int32_t W, int32_t H, int32_t stride);
int64_t st_harvest_workspace(int32_t K, int32_t W, int32_t H, int32_t stride);

/* deduplicate (prior.py:183-212) on the host: stable priority sort by
 * (src != ref, d, v, u), greedy acceptance (pixel free and no accepted
 * 8-neighbour more than 2 disparity units away), raster sort by (v, u, d).
 * Writes the accepted input indices to keep (capacity n), count to *n_keep. */
int st_support_dedup(const int32_t* u, const int32_t* v, const double* d, const int32_t* src,
                     int64_t n, int32_t ref_index, int32_t W, int32_t H, int64_t* keep,
                     int64_t* n_keep);

/* solver.py:421-432 initial_masks over pix (nullable = all H*W pixels). */
int st_initial_masks(const st_frame* f, const st_rig* rig, const st_params* p,
                     const int64_t* pix, int64_t n, uint32_t* static_out,
                     uint32_t* valid_out, void* stream);

/* solver.py:206-227 gather_rays: desc (n,K,16) f64, valid (n,K) u8, q (n,K) f64. */
int st_gather_rays(const st_frame* f, const st_rig* rig, const int64_t* pix,
                   const double* d, int64_t n, double* desc, uint8_t* valid, double* q,
                   void* stream);

/* solver.py:229-260 _energy: energy (n) f64 and real (n) u8. */
int st_energy(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* pix,
              const double* d, const uint32_t* bits, int64_t n, double* energy,
              uint8_t* real, void* stream);

/* solver.py:325-407 m_step over active pixels (sorted; nullable = all).
 * static_all is the full H*W mask map.  Outputs per active pixel. */
int st_m_step(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* active,
              int64_t n, const uint32_t* static_all, double* d_out, double* e_out,
              uint8_t* status_out, void* stream);

/* solver.py:409-419 e_step_at: mask reassignment at d (per listed pixel). */
int st_e_step_at(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* pix,
                 const double* d, int64_t n, uint32_t* static_out, uint32_t* valid_out,
                 void* stream);

/* solver.py:115-157 e_step on gathered rays: desc (n,K,16) f64,
 * valid (n,K) u8, q (n,K) f64 -> out (n) u32. */
int st_e_step(const double* desc, const uint8_t* valid, const double* q, int64_t n, int32_t K,
              const st_params* p, uint32_t* out, void* stream);

/* solver.py:93-107 masked_variance, batched: desc (n,K,16) f64, mask (n,K) u8 -> var (n). */
int st_masked_variance(const double* desc, const uint8_t* mask, int64_t n, int32_t K,
                       double* out, void* stream);

/* ---- the fused solve (solver.py:436-508) ------------------------------ */

/* st_solve for a dense single-device solve (dynamic_only = 0, no active
 * mask, no shard reduction, no timing) without any host synchronisation:
 * the convergence test of solver.py:483-485 and the EM statistics run on
 * the device, kernels of the iterations after convergence exit at once, and
 * the statistics land in *stats_dev (device or pinned-mapped memory) when
 * the stream reaches that point.  Same results as st_solve. */
int st_solve_async(const st_frame* frame, const st_rig* rig, const st_params* params,
                   float* values, uint8_t* status, uint32_t* static_bits, uint32_t* valid_bits,
                   st_stats* stats_dev, void* workspace, int64_t workspace_bytes, void* stream);
int64_t st_solve_workspace(int32_t W, int32_t H, int32_t K);

/* Full EM: initial masks, M/E alternation with the reference's global
 * convergence rule (or forced_iters), outputs values f32 / status u8 /
 * static u32 / valid u32 (H*W each).  dynamic_only selects active pixels
 * with ref prior < threshold (solver.py:449-452).  The optional reduce
 * callback all-reduces (sum, in place) `n` per-iteration values (energy sums
 * and integer counts, exact below 2^53) across row-band shards for the
 * global convergence rule and EMStats means; NULL on a single device. */
typedef int (*st_reduce_fn)(double* values, int32_t n, void* user);
int st_solve(const st_frame* f, const st_rig* rig, const st_params* p, int32_t dynamic_only,
             const uint8_t* active_mask /* nullable: explicit H*W active map */,
             float* values, uint8_t* status, uint32_t* static_bits, uint32_t* valid_bits,
             st_stats* stats, void* workspace, int64_t workspace_bytes,
             st_reduce_fn reduce, void* reduce_user, void* stream);

/* solver.py:466 `finite.mean()`: the mean of the finite values of x (n
 * float64, device) in numpy's own summation order (0.0 + pairwise_sum over
 * the compacted array, then / count; NaN when none is finite), into
 * out[0] (device).  The EM statistics of the single-device solves use the
 * same kernels. */
int st_numpy_mean(const double* x, int64_t n, double* out, void* workspace,
                  int64_t workspace_bytes, void* stream);
int64_t st_numpy_mean_workspace(int64_t n);

/* ---- row bands (BASELINE C3/C4) ------------------------ */

/* Per-iteration exchange of the row-band shards' statistics records
 * (solver.py:473-485's GLOBAL convergence rule, EMStats means): gather
 * every shard's record (st_band_record_bytes bytes, at rec_send) into
 * rec_recv (world records, rank order), stream-ordered on `stream` (e.g.
 * ncclAllGather; torch.distributed all_gather_into_tensor).  0 = success. */
typedef int (*st_exchange_fn)(void* stream, void* user);
int64_t st_band_record_bytes(void);

/* st_solve_async for one row band of a frame split across shards: pixels
 * of rows [ext0, ext1) are solved (the band [row0, row1) plus the halo rows
 * the median reads; halo pixels are pure per-pixel functions, so they equal
 * the neighbour's own), only rows [row0, row1) enter the statistics, and
 * after each iteration's statistics the record exchange + k_band_control
 * apply the reference's global stop rule on every shard (the host reads the
 * stop flag back once per iteration instead of enqueueing max_iters rounds
 * of exchanges).  Outputs are full-frame arrays of which rows [ext0, ext1)
 * are written.  dynamic_only: active = ref prior < threshold within the
 * rows (solver.py:449-452; one host read-back for the list size).  With
 * world == 1 and exchange == NULL this is the single-device solve of rows
 * [row0, row1) (the dynamic_only path of reconstruct_stream). */
int st_solve_rows(const st_frame* f, const st_rig* rig, const st_params* p,
                  int32_t dynamic_only, int32_t row0, int32_t row1, int32_t ext0, int32_t ext1,
                  float* values, uint8_t* status, uint32_t* static_bits, uint32_t* valid_bits,
                  st_stats* stats_dev, void* workspace, int64_t workspace_bytes,
                  st_exchange_fn exchange, void* user, int32_t world, void* rec_send,
                  void* rec_recv, void* stream);

/* features.py:81-104 for rows [row0, row1) of K RGB views only (row bands:
 * the images must hold rows [row0 - 3, row1 + 3) of the frame, clipped). */
int st_descriptors_rows(const uint8_t* images, int32_t K, int32_t H, int32_t W,
                        uint8_t* desc_out, int32_t row0, int32_t row1, void* stream);

/* st_synthesize restricted to a row band: the refocus of rows [ext0, ext1)
 * and the median rewrite of rows [row0, row1) (ext must cover row0 - r and
 * row1 + r, clipped to the frame). */
int st_synthesize_rows(const uint8_t* images, const st_rig* rig, const float* values,
                       const uint8_t* status, const uint32_t* static_bits,
                       int32_t min_static_rays, int32_t median_radius,
                       const uint8_t* copy_mask, uint8_t* image_out, uint8_t* prov_out,
                       uint8_t* n_rays_out, uint8_t* scratch, int32_t row0, int32_t row1,
                       int32_t ext0, int32_t ext1, void* stream);

/* ---- refocus (refocus.py:24-148) ------------------------------------- */

/* synthesize: Eq. 2 static-ray average + provenance + n_rays, then the
 * clipped median rewrite of every non-COPIED pixel.  copy_mask nullable. */
int st_synthesize(const uint8_t* images, const st_rig* rig, const float* values,
                  const uint8_t* status, const uint32_t* static_bits, int32_t min_static_rays,
                  int32_t median_radius, const uint8_t* copy_mask, uint8_t* image_out,
                  uint8_t* prov_out, uint8_t* n_rays_out, uint8_t* scratch /* H*W*3 */,
                  void* stream);

/* refocus.py:52-65 refocus_pixel / :24-49 gather_static_colors, batched
 * over listed pixels: rgb (n,3) u8, count (n), prov (n), totals (n,3) f64
 * (nullable). */
int st_refocus_pixels(const uint8_t* images, const st_rig* rig, const int64_t* pix,
                      const double* d, const uint32_t* bits, int64_t n, int32_t min_static_rays,
                      uint8_t* rgb, int32_t* count, uint8_t* prov, double* totals, void* stream);

/* pipeline.py:254-255 (dynamic_only): copy_mask = ref prior >= threshold,
 * compared in float32 like numpy; out (n) u8. */
int st_copy_mask(const float* ref_prior, int64_t n, double threshold, uint8_t* out,
                 void* stream);

/* refocus.py:68-106 median_filter on an (H,W,C) uint8 image. */
int st_median(const uint8_t* image, int32_t H, int32_t W, int32_t C, int32_t radius,
              uint8_t* out, void* stream);

/* ---- one frame, one call (the host runtime of reconstruct_stream) ------- */

/* Host gathers of the streaming runtime (one C call per frame; ctypes drops
 * the GIL for it): dst + dst_off[i] <- srcs[i], sizes[i] bytes -- host to
 * host (st_host_gather), host to device asynchronously on `stream`
 * (st_h2d_gather). */
int st_host_gather(void* dst, const void* const* srcs, const int64_t* dst_off,
                   const int64_t* sizes, int32_t n);
int st_h2d_gather(void* dst_dev, const void* const* srcs, const int64_t* dst_off,
                  const int64_t* sizes, int32_t n, void* stream);

/* L2 residency (experiments and the stream runtime): set aside `bytes` of L2
 * for persisting lines (clamped to the device maximum; 0 releases it), and
 * mark [base, base + bytes) persisting for the kernels of `stream`
 * (hit_ratio of its lines; bytes = 0 clears the window). */
int st_l2_set_aside(int64_t bytes);
/* Benchmark clock sampler: a native thread polls NVML every interval_us for
 * the SM clock and the clock-event (throttle) reason bits of the current
 * device; st_clocks_stop joins it and copies up to cap samples, returning
 * their number (< 0: not running). */
int st_clocks_start(int32_t interval_us);
int64_t st_clocks_stop(uint32_t* sm_mhz, uint32_t* max_mhz, uint64_t* reason_bits, int64_t cap);
int st_stream_l2_window(void* stream, void* base, int64_t bytes, float hit_ratio);

/* Everything a frame pipeline keeps across frames: the persistent device
 * buffers, workspaces, streams and (after st_frame_plan_init) its events. */
typedef struct st_frame_plan {
  st_frame frame;              /* images, priors, desc, mu; sup_* filled per frame */
  st_rig rig;
  st_params params;            /* dense async solve: forced_iters, no timing */
  int32_t median_radius;
  int32_t descriptors_ready;   /* 1: desc already computed on the main stream */
  float* values;
  uint8_t* status;
  uint32_t* static_bits;
  uint32_t* valid_bits;
  uint8_t* image;
  uint8_t* prov;
  uint8_t* n_rays;
  uint8_t* scratch;            /* H*W*3 */
  st_stats* stats_dev;
  void* mu_ws;
  int64_t mu_ws_bytes;
  void* sup_ws;
  int64_t sup_ws_bytes;
  void* solve_ws;
  int64_t solve_ws_bytes;
  void* main_stream;           /* cudaStream_t handles */
  void* side_stream;           /* mu raster */
  void* side2_stream;          /* descriptors + support groups */
  void* out_stream;            /* D2H of the artefacts (null = the default stream) */
  void* events[4];             /* owned, created by st_frame_plan_init */
} st_frame_plan;

int st_frame_plan_init(st_frame_plan* plan);
int st_frame_plan_destroy(st_frame_plan* plan);

/* One frame of pipeline.py:247-261 (solve + synthesize) with no host
 * synchronisation: the mu raster (side stream) and the descriptors + support
 * candidate groups (side2) start at `ready` (a cudaEvent_t; nullable = now
 * on the main stream), the dense asynchronous solve and the refocus run on
 * the main stream, and when host_block (pinned, nullable) is given the
 * artefacts -- values, status, static, valid, image, provenance, n_rays,
 * st_stats, each 256-byte aligned in that order -- are copied into it on the
 * out stream.  `done` (cudaEvent_t, nullable) is recorded after the copies
 * (or after the refocus). */
int st_frame_run(st_frame_plan* plan, const st_tri* tri, const double* support_uv,
                 const double* support_d, int32_t n_support, void* ready, void* host_block,
                 void* done);
int64_t st_frame_host_bytes(int32_t W, int32_t H);

/* ---- synthetic light fields on the device -------------
 * Replaces the reference renderer `render` (synth.py:244-309: _trace
 * :174-230, surface_color :59-82, value noise :25-56, billboard edges
 * :264-283, ground truth :287-290) and `corrupt_prior` (synth.py:334-346).
 * The host side (render.py) draws each surface's texture constants with
 * numpy exactly as surface_color does and passes them in st_surface. */
#define ST_MAX_SURFACES 8

typedef struct st_surface {
  int32_t is_occluder;      /* OccluderSpec (1) or PlaneSpec (0) */
  int32_t seed;             /* lattice-noise seed (low 32 bits used, synth.py:33) */
  int32_t has_x_min, has_x_max;
  double depth, base, amplitude, frequency;
  double x_min, x_max;      /* planes: px >= x_min, px < x_max */
  double half_w, half_h;    /* occluders: width / 2.0, height / 2.0 */
  double center_x, center_y;
  double c0[3];             /* 2.0 * np.pi * rate[i] */
  double ca[3], sa[3];      /* np.cos(ang[i]), np.sin(ang[i]) */
  double ph[3][3];          /* ph[i][c] */
  double nw[3];
} st_surface;

typedef struct st_scene {
  int32_t width, height;
  int32_t n_surfaces;       /* in trace order: occluders by depth, then planes by depth */
  int32_t pad_;
  double fx, fy, cx, cy;    /* SceneSpec.intrinsics() */
  st_surface surf[ST_MAX_SURFACES];
} st_scene;

/* One view: image (H, W, 3) u8 and occluder mask (H, W) u8 (cover >= 0.5),
 * with the 4-sample supersampling on the billboard edges of the n_rects
 * occluder rectangles (device array of (u0, u1, v0, v1), synth.py:236-241).
 * center = camera centre, rotation = the extrinsic rotation (row-major).
 * *fail (device) is set to 1 when a ray hits no surface (the reference's
 * ValueError). */
int st_render_view(const st_scene* scene, const double* center, const double* rotation,
                   const double* rects_dev, int32_t n_rects, uint8_t* image, uint8_t* mask,
                   int32_t* fail, void* stream);
/* The reference view's background (no occluders) and ground-truth
 * disparity float32(focal_baseline / depth) (synth.py:287-290). */
int st_render_background(const st_scene* scene, const double* center, const double* rotation,
                         double focal_baseline, uint8_t* image, float* disparity, int32_t* fail,
                         void* stream);
/* corrupt_prior(1 - mask, p_flip, blur_radius, seed) -> float32 (H, W):
 * pcg_state = numpy PCG64 {state_hi, state_lo, inc_hi, inc_lo} of
 * default_rng(seed) (the flips are its first H*W random() draws). */
int st_corrupt_prior(const uint8_t* mask, int32_t W, int32_t H, const uint64_t* pcg_state,
                     double p_flip, int32_t blur_radius, float* prior, void* workspace,
                     int64_t workspace_bytes, void* stream);
int64_t st_corrupt_prior_workspace(int32_t W, int32_t H);

#ifdef __cplusplus
}
#endif
#endif /* SEETHROUGH_B200_H */
