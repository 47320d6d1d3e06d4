/* gridshift_c.h — C-ABI of the B200-native GridShift engine (libgridshift_cuda.so).
 *
 * Drop-in boundary for the reference's engine API.  The reference exposes no FFI: its
 * boundary is the C++ library call
 *     gridshift::ClusterLabeling gridshift::run(const Dataset&, const EngineConfig&)
 * specified at /root/reference/SPEC.md:135-143 (types SPEC.md:107-114, errors
 * /root/reference/proj/include/gridshift/errors.hpp:9-72).  Each entry point below names the
 * SPEC operation it replaces.  Only C types cross this boundary; the C++ wrapper
 * (include/gridshift/gridshift.hpp) keeps the SPEC signature and rethrows status codes as the
 * errors.hpp exception types.  The engine runs on an sm_100a GPU; there is no CPU fallback
 * (a missing device is GS_E_NO_DEVICE, never a silent host path).
 *
 * Ownership: inputs are borrowed for the duration of the call; outputs go into caller buffers.
 * Threading: a gs_ctx is not thread-safe; distinct contexts may run concurrently
 * ("independent runs ... fully isolated state").
 */
#ifndef GRIDSHIFT_C_H_
#define GRIDSHIFT_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_MAX_DIM 12 /* SPEC.md:96 documented limit d <= 12 */

/* Status codes map 1:1 onto errors.hpp (see gridshift::throw_for_status). */
typedef enum {
  GS_OK = 0,
  GS_E_INVALID_INPUT = 1,      /* InvalidInputError: non-finite coordinate  */
  GS_E_INVALID_BANDWIDTH = 2,  /* InvalidBandwidthError: h <= 0 or non-finite     */
  GS_E_EMPTY_INPUT = 3,        /* EmptyInputError: n == 0                         */
  GS_E_INVALID_PARAMETER = 4,  /* InvalidParameterError: d, batch, max_iter, dtype out of range */
  GS_E_INTERNAL_INVARIANT = 5, /* InternalInvariantError: partition/merge invariant broken      */
  GS_E_KEY_RANGE = 6,          /* InvalidParameterError: key box exceeds the dense cell grid   */
  GS_E_CUDA = 7,               /* Error: CUDA runtime failure                                   */
  GS_E_OOM = 8,                /* Error: device allocation failed                               */
  GS_E_NCCL = 9,               /* Error: collective failure (multi-GPU driver)                  */
  GS_E_NO_DEVICE = 10,         /* Error: no sm_100 device visible                               */
  GS_E_TUNING_FAILED = 11,     /* TuningFailureError: no bandwidth gave a scorable clustering   */
  GS_E_UNDEFINED_SCORE = 12,   /* UndefinedScoreError: silhouette of < 2 clusters */
  GS_E_INVALID_WINDOW = 13,    /* InvalidWindowError: tracking window outside the frame         */
  GS_E_SELECTION = 14          /* SelectionError: selected cluster id does not exist            */
} gs_status;

/* GS_U8: 8-bit RGB pixels, 3 bytes per point, turned into features on the device exactly as
 * the segmentation front end does: d = 3 -> (r,g,b)/255; d = 5 -> (r,g,b)/255
 * followed by x = col/(W-1), y = row/(H-1) with the image width W in gs_input.reserved
 * (n = W*H, row-major).  Reads 3 B/pixel instead of 12-20 B of fp32 features. */
typedef enum { GS_F32 = 0, GS_F64 = 1, GS_U8 = 2 } gs_dtype;

/* A dataset: `batch` independent frames of n points each, d coordinates,
 * row-major [batch][n][d].  Frames are clustered independently.  With
 * on_device != 0, `points` is a device pointer on the context's device. */
typedef struct {
  const void* points;
  int64_t n;      /* points per frame, >= 1 */
  int32_t d;      /* 1 .. GS_MAX_DIM */
  int32_t dtype;  /* gs_dtype */
  int64_t batch;  /* frames, >= 1 */
  int32_t on_device;
  int32_t reserved;  /* GS_U8 with d = 5: the image width W; else 0 */
} gs_input;

#define GS_RECORD_HISTORY 0x1u  /* keep per-iteration (m, max displacement)   */
#define GS_DEVICE_OUTPUTS 0x2u  /* result.labels is a device pointer                          */
#define GS_TIME_PHASES 0x4u    /* record phase events: gs_stats ms_* (costs ~30 us per run)  */
#define GS_TIME_KERNEL 0x8u    /* record the binning kernel's events only: gs_stats ms_k_bin  */
#define GS_NO_PIPELINE 0x10u     /* host frames: one whole-batch copy, no frame-group pipeline  */
#define GS_DEBUG_GLOBAL_PATH 0x80000000u /* test hook: iterate on the multi-CTA path only */
#define GS_DEBUG_PIPELINE 0x40000000u   /* test hook: pipeline host frames in groups of 2 */
#define GS_DEBUG_SWEEP_FLOW 0x20000000u   /* test hook: global path sweeps use the dataflow sweep */
#define GS_DEBUG_SWEEP_LEVELS 0x10000000u /* test hook: level-synchronous cluster sweep only */
#define GS_DEBUG_SWEEP_SINGLE 0x08000000u /* test hook: the single-CTA sweep only */

/* EngineConfig. */
typedef struct {
  double h;          /* bandwidth = cell side, > 0 */
  int32_t max_iter;  /* >= 1; SPEC default 1000 */
  uint32_t flags;
} gs_config;

/* ClusterLabeling, per frame.  Caller-owned buffers:
 *   labels      batch*n cluster ids; id = lexicographic rank of the final cell
 *   k           batch entries: clusters per frame
 *   iterations  batch entries: completed shift iterations (do-while, >= 1)
 *   converged   batch entries: 0 = max_iter reached (warning, not an error) */
typedef struct {
  int32_t* labels;
  int64_t* k;
  int32_t* iterations;
  int32_t* converged;
} gs_result;

typedef struct gs_ctx gs_ctx;

/* Host-only argument validation with the same codes gs_run returns (no device needed). */
gs_status gs_validate(const gs_input* in, const gs_config* cfg);

/* Create an engine context on `device`; cuda_stream is a cudaStream_t (NULL = own stream). */
gs_status gs_create(int device, void* cuda_stream, gs_ctx** out);
void gs_destroy(gs_ctx* ctx);

/* engine.run over every frame of `in`.  Synchronous w.r.t. the caller:
 * on return the result buffers are filled.  Host-resident batches of several frames larger
 * than 64 MB are pipelined by frame groups (unless GS_NO_PIPELINE): the copy of group g+1
 * overlaps the clustering of group g and the label write-back of group g-1; results are
 * identical (frames are independent).  After such a run gs_render serves only
 * the frames of the last group. */
gs_status gs_run(gs_ctx* ctx, const gs_input* in, const gs_config* cfg, gs_result* out);

/* Cluster centroids of `frame` from the last gs_run: k x d fp64 in cluster-id order. */
gs_status gs_get_centroids(gs_ctx* ctx, int64_t frame, double* out, int64_t cap_k);

/* History of `frame` from the last gs_run (needs GS_RECORD_HISTORY): m_t = active cells
 * entering iteration t, maxdisp_t = max Euclidean sweep displacement.  Writes min(cap, iters). */
gs_status gs_get_history(gs_ctx* ctx, int64_t frame, int64_t* m_t, double* maxdisp_t,
                         int32_t cap);

/* Per-run counters of the last gs_run.  The ms_* times are CUDA events on the ctx stream and
 * are only recorded with GS_TIME_PHASES (ms_k_bin also with GS_TIME_KERNEL); else 0. */
typedef struct {
  double ms_total;       /* first kernel to last kernel (device-resident input/outputs)   */
  double ms_bin;         /* bounds + binning + compaction (n-scale)                        */
  double ms_iterate;     /* the iteration phase (all iterations)                           */
  double ms_label;       /* label propagation (n-scale)                                    */
  double ms_h2d;         /* host->device copy of the points (0 when on_device)             */
  double ms_d2h;         /* device->host copy of the labels (0 with GS_DEVICE_OUTPUTS)     */
  int64_t cells_swept;   /* sum over frames and iterations of active cells (Σ m_t)         */
  int64_t m0;            /* initial active cells (all frames)                              */
  int64_t k_total;       /* final cells (all frames)                                       */
  int64_t kernel_launches;
  int32_t max_iterations;/* max over frames                                                */
  int32_t fixed_shift;   /* F of the fixed-point cell sums                                 */
  int64_t dense_cells;   /* size of the dense cell grid (all frames)                       */
  double ms_k_bin;       /* the binning kernel K2 alone                                     */
  double ms_k_label;     /* the label kernel K7 alone                                       */
  int64_t lib_calls;     /* library (CUB) device calls, not counted in kernel_launches      */
  int64_t sweep_modes[3];/* K8 iterations by sweep mode: fixed-stride lists / scanned lists /
                            inline lookups */
  int64_t resident_cycles[8]; /* K8 SM cycles per phase with GS_PROF set (lists, sweep, rehome,
                                 sort, merge, converged, first sweep, load), summed over frames */
  int32_t slot_bytes;     /* bytes per point of the point -> cell map (2: frames of <= 65536 cells) */
  int32_t predicted_box;  /* 1: binned against the previous run's key box (no bounds pass)   */
} gs_stats;
gs_status gs_get_stats(gs_ctx* ctx, gs_stats* out);

const char* gs_last_error(const gs_ctx* ctx); /* valid until the next call on ctx */
const char* gs_status_string(gs_status s);

/* Segmentation render (fused K7 epilogue) for `frame` of the last gs_run:
 * every pixel replaced by its segment's mean colour, the centroid's first three components
 * times 255 rounded half-up, clamped to 0..255.  out: n*3 bytes, host memory
 * or (on_device) device memory. */
gs_status gs_render(gs_ctx* ctx, int64_t frame, uint8_t* out, int32_t on_device);

/* ---- multi-GPU: one point cloud split over R ranks ----
 * Each rank calls, on its own contiguous shard of the cloud (batch = 1):
 *  1. gs_shard_keybounds: the shard's per-dim cell-key range floor(min/h) .. floor(max/h);
 *     the caller all-reduces them (min of klo, max of khi) and the point counts (sum);
 *  2. gs_shard_bin: bins the shard into partial cells of the global key box (dense linear
 *     keys, counts and raw fixed-point sums -- integers, so partials merge exactly); the
 *     caller all-gathers every rank's partial cells.  Returns GS_E_INVALID_PARAMETER with
 *     *m_out = the needed count when cap is too small;
 *  3. gs_shard_run: merges all partial cells (any order) into the global initial cells --
 *     bit-identical to a single-GPU build_active_grid over the whole cloud -- runs the
 *     iteration and labels this rank's shard.  Every rank computes the same clusters;
 *     gs_get_centroids / gs_get_history then work as after gs_run.
 * The calls must be made in order on the same ctx (the shard's point-to-cell map is kept from
 * 2 to 3).  Replaces the whole-cloud engine.run of SPEC.md:135-143 for one dataset. */
gs_status gs_shard_keybounds(gs_ctx* ctx, const gs_input* shard, double h, int64_t* klo,
                             int64_t* khi);
gs_status gs_shard_bin(gs_ctx* ctx, const gs_input* shard, double h, int64_t n_global,
                       const int64_t* klo, const int64_t* khi, int64_t cap, int64_t* m_out,
                       uint32_t* keys, uint32_t* counts, int64_t* sums);
gs_status gs_shard_run(gs_ctx* ctx, int64_t m_all, const uint32_t* keys, const uint32_t* counts,
                       const int64_t* sums, int64_t n_shard, const gs_config* cfg,
                       gs_result* out);

/* ---- multi-GPU drivers: one host thread drives R ranks, each an engine
 * context on its own device (devices may repeat: loopback ranks share a GPU).
 *  gs_dist_run_frames: independent frames in contiguous blocks per rank (one host thread per
 *    rank), no exchange -- replaces engine.run over a frame batch.
 *  gs_dist_run_slabs: ONE cloud (batch 1, host memory, d <= 6) split into R contiguous point
 *    shards; cells owned by dim-0 slabs of the global key box; per iteration the first key
 *    layer of each slab goes to the rank below (old centroids), the sweep runs slab after slab
 *    with the lower neighbour's swept last layer (the in-place lex sweep of SPEC.md:117-125
 *    across slabs), cells whose new key leaves the slab migrate to its owner and every owner
 *    folds its members in old global lex order (Eq. 3), has_converged sees the neighbours'
 *    new boundary layers.  Labels, centroids, iterations and history are bit-identical to one
 *    GPU clustering the whole cloud (gs_run).  Data moves are device-to-device peer copies.
 * Results: out as gs_run's (labels of all points); centroids / history by gs_dist_get_*. */
typedef struct gs_dist gs_dist;
gs_status gs_dist_create(int ndev, const int* devices, gs_dist** out);
void gs_dist_destroy(gs_dist* D);
const char* gs_dist_last_error(const gs_dist* D);
gs_status gs_dist_run_frames(gs_dist* D, const gs_input* in, const gs_config* cfg, gs_result* out);
gs_status gs_dist_run_slabs(gs_dist* D, const gs_input* in, const gs_config* cfg, gs_result* out);
gs_status gs_dist_get_centroids(gs_dist* D, int64_t frame, double* out, int64_t cap_k);
gs_status gs_dist_get_history(gs_dist* D, int64_t* m_t, double* maxdisp_t, int32_t cap);

/* ---- bandwidth sweep (reference module `metrics`) ----
 * gs_tune_bandwidth replaces tune_bandwidth(X, clusterer, h_grid) with the
 * GridShift engine as the clusterer and silhouette_subsampled as the score:
 * per grid value one engine.run on the GPU, then the silhouette of a seeded subsample of
 * min(n, cap) points.  Entries with < 2 clusters in the sample are recorded with valid = 0
 * and skipped; best_h = argmax score, ties -> smallest h; no valid entry ->
 * GS_E_TUNING_FAILED.  Grid values must lie in (0, 1] (GS_E_INVALID_BANDWIDTH), X is one
 * dataset (batch 1) of fp32/fp64 features, normalised to [0,1] by the caller.
 * Subsample and summation order are pinned (oracle/gs_oracle.cpp S1-S3): results equal the
 * CPU oracle's bit for bit.  A gs_tuner runs up to `max_concurrent` entries at once, each on
 * its own engine context and stream (entries may evaluate concurrently). */
typedef struct {
  double h;
  double score;       /* subsample silhouette; 0 when !valid                      */
  int64_t k;          /* clusters of the whole dataset                            */
  int32_t iterations;
  int32_t converged;
  int32_t valid;      /* 0: fewer than 2 clusters in the sample (undefined entry) */
  int32_t reserved;
} gs_sweep_entry;

typedef struct gs_tuner gs_tuner;
gs_status gs_tuner_create(int device, int32_t max_concurrent, gs_tuner** out);
void gs_tuner_destroy(gs_tuner* t);
const char* gs_tuner_last_error(const gs_tuner* t);
gs_status gs_tune_bandwidth(gs_tuner* t, const gs_input* X, const double* h_grid, int32_t nh,
                            int32_t max_iter, int64_t cap, uint64_t seed, gs_sweep_entry* out,
                            double* best_h);
/* silhouette_subsampled(X, labels, cap, seed): labels n int32 (host, or
 * device with labels_on_device); < 2 clusters in the sample -> GS_E_UNDEFINED_SCORE. */
gs_status gs_silhouette_subsampled(gs_tuner* t, const gs_input* X, const int32_t* labels,
                                   int32_t labels_on_device, int64_t cap, uint64_t seed,
                                   double* score);

/* ---- tracker (reference module `tracker`, Algorithm 2) ----
 * init_tracker -> gs_track_init: engine.run on the (r,g,b)/255 colours of the
 * window's pixels of frame0 (H x W x 3 u8, row-major), selection of the top_k largest clusters
 * (or n_ids explicit ids), reference bin B = colour cells of the selected pixels.
 * track_sequence -> gs_track_sequence: track_frame on each
 * of T frames in order, continuing the tracker's state across calls; out[t] = emitted window,
 * lost[t] = 1 when the target was not found in any inner iteration, inner[t] = iterations.
 * Window, colour-cell and inner-loop semantics are pinned (oracle/gs_oracle.cpp T1-T5); the
 * results equal the CPU oracle's bit for bit.  The whole sequence runs in one kernel launch. */
typedef struct {
  double ox, oy;  /* centre (x = column, y = row), pixels */
  double l, w;    /* length (x extent) and width (y extent), pixels, > 0 */
} gs_window;

typedef struct {
  double h;                /* colour bandwidth, > 0 (and >= ~1/72: the cell bitmap is on chip) */
  double f;                /* increment factor >= 1 (search region W(o, l/f, w/f)); SPEC default 1 */
  double eta;              /* centre tolerance in pixels, > 0; SPEC default 1 */
  int32_t max_inner_iters; /* SPEC default 20 */
  int32_t engine_max_iter; /* engine.run max_iterations for init (SPEC default 1000) */
  int32_t top_k;           /* selection: k largest clusters (SPEC default 1) when n_ids == 0 */
  int32_t n_ids;
  const int32_t* ids;      /* explicit cluster ids (n_ids > 0) */
} gs_tracker_config;

typedef struct gs_tracker gs_tracker;
gs_status gs_tracker_create(int device, gs_tracker** out);
void gs_tracker_destroy(gs_tracker* t);
const char* gs_tracker_last_error(const gs_tracker* t);
gs_status gs_track_init(gs_tracker* t, const uint8_t* frame0, int32_t H, int32_t W,
                        int32_t on_device, const gs_window* win, const gs_tracker_config* cfg,
                        int64_t* k_out);
gs_status gs_track_sequence(gs_tracker* t, const uint8_t* frames, int64_t T, int32_t on_device,
                            gs_window* out, int32_t* lost, int32_t* inner);

/* ---- MS++ baseline (reference module `baselines`, mspp_run SPEC.md:197-203)
 * Per-point grid mean shift with parallel (Jacobi, Eq. 6) updates: every iteration re-grids the
 * current positions and moves every point to the count-weighted mean of its cell's
 * 1-neighbourhood centroids computed from the previous state; stop when the max displacement
 * < tol (SPEC default 1e-6*h) or after max_iter (SPEC default 300); clusters = points sharing a
 * final cell, ids by lexicographic key.  Pins M1-M5 (oracle/gs_oracle.cpp): results equal the
 * oracle's bit for bit.  One dataset (batch 1) of fp32/fp64 features, d <= 6, whose first grid
 * fits one CTA's shared memory (2,048 cells at d = 3).  out->k/iterations/converged get one
 * entry; disp_hist (nullable, max_iter entries) the per-iteration displacement;
 * gs_get_centroids(ctx, 0, ...) the final centroids. */
gs_status gs_mspp_run(gs_ctx* ctx, const gs_input* in, double h, double tol, int32_t max_iter,
                      gs_result* out, double* disp_hist);

/* ---- test hooks (parity harness; not needed by callers) ---- */

/* build_active_grid only on one frame: m0 cells in lex order.
 * keys m0*d int64, counts m0, centroids m0*d, slot n (cell rank of each point). */
gs_status gs_debug_build(gs_ctx* ctx, const gs_input* in, double h, int64_t cap_m,
                         int64_t* m_out, int64_t* keys, int64_t* counts, double* centroids,
                         int64_t* slot);

/* One iterate_once on an injected lex-sorted state; outputs mirror
 * oracle gso_iterate_once: new state, post-sweep centroids, parent ranks, flags. */
gs_status gs_debug_iterate_once(gs_ctx* ctx, int32_t d, double h, int64_t m,
                                const int64_t* keys, const int64_t* counts,
                                const double* centroids, int64_t* m_out, int64_t* keys_out,
                                int64_t* counts_out, double* centroids_out, double* swept_out,
                                int64_t* parent_out, int32_t* changed_out,
                                int32_t* converged_out, double* maxdisp_out);

/* One iteration of K8 (the CTA-resident engine) on an injected lex-sorted state of <= its
 * capacity: the cells after iterate_once (keys, counts, centroids in id order), parent_out[i] =
 * the new cell of injected cell i, stop_out = converged-or-unchanged (the do-while exit of
 * SPEC.md:141), maxdisp_out = the sweep's max displacement.  Mirrors oracle gso_iterate_once. */
gs_status gs_debug_resident_once(gs_ctx* ctx, int32_t d, double h, int64_t m, const int64_t* keys,
                                 const int64_t* counts, const double* centroids, int64_t* m_out,
                                 int64_t* keys_out, int64_t* counts_out, double* centroids_out,
                                 int64_t* parent_out, int32_t* stop_out, double* maxdisp_out);

/* The fixed-point exponent F used for the binning sums of a frame of n points at bandwidth h. */
int32_t gs_fixed_shift(int64_t n, double h);

#ifdef __cplusplus
}
#endif

#endif /* GRIDSHIFT_C_H_ */
