/*
 * sqv.h — C ABI of the B200 superquadric voxelizer (libsqv.so).
 *
 * The reference (SuperQuadricOcc, arXiv 2511.17361) has no native code and no
 * FFI: its voxelization path exists as the Python operations specified in
 * /root/reference/SPEC.md:345-373 (voxelize / voxelize_bruteforce / finalize)
 * and SPEC.md:494-512 (voxel_iou / miou), over the primitive math of
 * /root/reference/pkg/src/sqocc/core.py:237-282 (to_local, inside_outside,
 * density).  Each entry point below is the native body of one of those
 * operations; the Python layer (paper_2511_17361_b200.voxelize / .metrics)
 * binds them with ctypes exactly as a maintainer would bind them into the
 * reference package.
 *
 * Conventions
 *   - Plain C types only.  Every array argument is a DEVICE pointer unless the
 *     name ends in _host.  `stream` is a cudaStream_t passed as void*.
 *   - Primitive inputs are FP64 structure-of-arrays, frame-major:
 *       mu[F][N][3] scale[F][N][3] rot[F][N][4] (w,x,y,z) opacity[F][N]
 *       eps[F][N][2] (eps1, eps2) logits[F][N][C]
 *     i.e. the fields of SuperQuadric (core.py:134-141) for F frames of N
 *     primitives.  n_valid[F] (nullable) marks ragged frames: primitives
 *     i >= n_valid[f] are ignored.
 *   - Voxel arrays are x-fastest: index = x + nx*(y + ny*z),
 *     frame-major; v_c is [F][V][C] with the class index fastest.
 *   - Return value: SQV_OK (0) or a negative SQV_ERR_* code; a message is
 *     available from sqv_last_error() (thread-local).
 *   - The library never allocates device memory and keeps no global mutable
 *     state besides the thread-local error string, a launch counter, the
 *     opt-in stage profiler (sqv_profile_*) and the optional work-counter
 *     pointer (sqv_stats_attach) — instrumentation, process-wide.
 *     Scratch comes from the caller's workspace pointer.
 *   - Results are deterministic: identical inputs give bit-identical outputs
 *      regardless of batch composition or GPU count.
 */
#ifndef SQV_H_
#define SQV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SQV_ABI_VERSION 1

/* Binning tile (voxels).  The bins (tile -> ascending primitive ids) are part
 * of the bit-exact contract with the CPU oracle, so the tile shape is ABI. */
#define SQV_TILE_X 8
#define SQV_TILE_Y 8
#define SQV_TILE_Z 16

/* Largest class count the device evaluator is instantiated for. */
#define SQV_MAX_CLASSES 32

/* Status codes */
#define SQV_OK 0
#define SQV_ERR_ARG (-1)          /* invalid argument (dims, res, tau, ...) */
#define SQV_ERR_CUDA (-2)         /* a CUDA runtime call failed */
#define SQV_ERR_WORKSPACE (-3)    /* workspace too small: see *ws_needed */
#define SQV_ERR_INVALID_PRIM (-4) /* a primitive failed validation (core.py:147-159) */
#define SQV_ERR_UNSUPPORTED (-5)  /* e.g. more classes than SQV_MAX_CLASSES */
#define SQV_ERR_CAPACITY (-6)     /* caller-provided bins buffer too small */

/* Per-primitive validation failure bits (first failing primitive reported).
 * Same checks, same order as SuperQuadric.__post_init__ (core.py:143-165)
 * and quat_normalize (core.py:30-35). */
#define SQV_BAD_MU_SCALE_FINITE 1   /* "mu/scale must be finite" */
#define SQV_BAD_SCALE_POSITIVE 2    /* "scale components must be strictly positive" */
#define SQV_BAD_LOGITS_FINITE 4     /* "logits must be finite" */
#define SQV_BAD_OPACITY 8           /* "opacity must lie in [0, 1]" */
#define SQV_BAD_QUAT 16             /* "cannot normalize near-zero quaternion" */
#define SQV_BAD_EPS 32              /* eps not finite (core.py:160-165 would propagate NaN) */

/* VoxelGridSpec. */
typedef struct sqv_grid {
  double origin[3];
  int32_t dims[3];
  double resolution;
} sqv_grid;

/* VoxelizeConfig plus the window constants of the
 * design ledger. */
typedef struct sqv_cfg {
  double tau;                  /* occupancy threshold, default 0.01 */
  int32_t neighborhood_radius; /* base window radius in voxels, default 5 */
  int32_t truncate;            /* 1: Chebyshev window (voxelize); 0: whole grid (voxelize_bruteforce) */
  int32_t semantic_mode;       /* 0: logit-sum (default), 1: prob-sum (softmax first) */
  int32_t free_label;          /* u8 code written for free voxels (0..255, outside [0, C)) */
  double window_extent;        /* max K of the scaled family, default 2.5 */
  int32_t precision;           /* 1: strict (default) — coordinate logs on the FMA pipe for
                                  primitives with 2/eps1 > 4, densities within 1e-5 relative
                                  down to 1e-3*tau; 0: fast — all logs on the SFU (~5% faster,
                                  3e-5 relative down to 1e-3*tau) */
} sqv_cfg;

/* Primitive batch (device pointers, FP64). */
typedef struct sqv_prims {
  const double* mu;
  const double* scale;
  const double* rot;
  const double* opacity;
  const double* eps;
  const double* logits;
  const int32_t* n_valid; /* nullable */
  int32_t n_frames;
  int32_t n_prims;
  int32_t n_classes;
} sqv_prims;

/* Outputs (device).  labels is required; v_o and v_c may be NULL, in which
 * case the dense grids are only formed on chip (finalize is fused). */
typedef struct sqv_outputs {
  uint8_t* labels; /* [F][V] */
  float* v_o;      /* [F][V]    nullable */
  float* v_c;      /* [F][V][C] nullable */
} sqv_outputs;

/* Optional export of the binning (for parity tests and sqocc tooling). */
typedef struct sqv_bins {
  int32_t* windows;  /* [F][N][6] lo_x,lo_y,lo_z,hi_x,hi_y,hi_z (empty: lo > hi); nullable */
  int32_t* tile_off; /* [F*T + 1] exclusive offsets into prim_ids; nullable */
  int32_t* prim_ids; /* [capacity] frame-local primitive index, ascending per tile; nullable */
  int64_t capacity;  /* elements available in prim_ids */
  int64_t n_entries; /* out: number of (tile, primitive) entries */
  int64_t n_pairs;   /* out: algorithmic (primitive, in-window voxel) pairs, sigma > 0 */
} sqv_bins;

/* ---- library info ---- */
int sqv_abi_version(void);
const char* sqv_last_error(void);
/* Number of kernels this library has launched in this process. */
int64_t sqv_launch_count(void);

/* Tiles per frame for a grid. */
int64_t sqv_tiles_per_frame(const sqv_grid* grid);

/* Workspace bytes for a batch with `n_entries` bin entries (pass 0 for the
 * fixed part only; sqv_voxelize reports the exact need via *ws_needed). */
size_t sqv_workspace_bytes(int32_t n_frames, int32_t n_prims, int32_t n_classes,
                           const sqv_grid* grid, int64_t n_entries);

/*
 * voxelize / voxelize_bruteforce (cfg.truncate = 0),
 * with finalize fused into the evaluator epilogue.
 * Pipeline on `stream`: prep -> tile-count scan -> [one 8-byte D2H read of
 * the entry count + validation word] -> emit -> radix sort -> tile scan ->
 * evaluate+finalize.  Returns SQV_ERR_WORKSPACE (with *ws_needed) if the
 * workspace is too small, SQV_ERR_INVALID_PRIM (with *bad_prim = f*N+i and
 * *bad_bits) if a primitive fails validation.  bins may be NULL.
 */
int sqv_voxelize(const sqv_prims* prims, const sqv_grid* grid, const sqv_cfg* cfg,
                 const sqv_outputs* out, sqv_bins* bins,
                 void* workspace, size_t ws_bytes, size_t* ws_needed,
                 int64_t* bad_prim, int32_t* bad_bits, void* stream);

/* finalize: labels from dense grids; tau sweeps without re-scatter. */
int sqv_finalize(const float* v_o, const float* v_c, int64_t n_voxels, int32_t n_classes,
                 double tau, int32_t free_label, uint8_t* labels, void* stream);

/*
 * Confusion counts for voxel_iou / miou: cm[(C+1)*(C+1)]
 * int64, row = gt class, column = predicted class, index C = free.  Labels
 * equal to free_label map to index C; any other label >= C also maps to C.
 * cm is ACCUMULATED into (zero it first).
 */
int sqv_confusion(const uint8_t* pred, const uint8_t* gt, int64_t n_voxels, int32_t n_classes,
                  int32_t free_label, int64_t* cm, void* stream);

/*
 * Point-wise density (core.py:276-282) and inside-outside F (core.py:254-273)
 * of primitive j (FP64 SoA, 1 frame of n_prims) at world points
 * points[n_points][3] for each (prim, point) pair listed in pair_prim[]:
 * F[k] and density[k] for point k evaluated against primitive pair_prim[k].
 */
int sqv_density(const sqv_prims* prims, const double* points, const int32_t* pair_prim,
                int64_t n_points, float* F, float* density, void* stream);

/*
 * ray_iou.  pred/gt: [n_frames][V] u8 label grids
 * (x-fastest; labels >= n_classes are free), host-side thresholds[n_thr]
 * (metres, 1..16), device origins/dirs [n_rays][3] FP64 (unit dirs).  Per
 * (frame, ray): first occupied voxel of pred and of gt along origin + t*dir
 * by a 3D DDA; hit distance = t at which the ray enters that voxel (0 if the
 * origin lies in it).  counts[n_thr][3] int64 (TP, FP, FN) are ACCUMULATED:
 * TP when both hit with equal classes and |d_pred - d_gt| <= thr; a pred hit
 * without a matching gt hit is an FP, a gt hit without a matching pred hit an
 * FN.  hits (nullable) receives per-ray [n_frames][n_rays] distances (-1 = no
 * hit) and classes (-1 = no hit).  Zero rays -> SQV_ERR_ARG ("zero rays").
 */
typedef struct sqv_ray_hits {
  double* d_pred;
  int32_t* c_pred;
  double* d_gt;
  int32_t* c_gt;
} sqv_ray_hits;
int sqv_ray_iou(const uint8_t* pred, const uint8_t* gt, int32_t n_frames, const sqv_grid* grid,
                int32_t n_classes, const double* origins, const double* dirs, int64_t n_rays,
                const double* thresholds, int32_t n_thr, int64_t* counts, sqv_ray_hits* hits,
                void* stream);

/*
 * Device-side seeded scene generation (gen_scene): frames
 * first_frame .. first_frame+n_frames-1 of the Philox4x32-10 stream `seed`,
 * written as the FP64 SoA inputs of sqv_voxelize (device pointers, frame
 * major): mu ~ U(grid bounds), scale ~ U[smin, smax], rot = normalised
 * N(0,1)^4, opacity ~ U[0,1], eps ~ U[emin, 2], logits ~ N(0,1).  A frame's
 * primitives depend only on (seed, frame index, primitive index).
 */
int sqv_gen_frames(uint64_t seed, int64_t first_frame, int32_t n_frames, int32_t n_prims,
                   int32_t n_classes, const sqv_grid* grid, double smin, double smax,
                   double emin, double* mu, double* scale, double* rot, double* opacity,
                   double* eps, double* logits, void* stream);

/* ---- instrumentation (bench / profiling; not part of the reference API) ----
 * When enabled, sqv_voxelize records CUDA events around its device stages on
 * the caller's stream and accumulates their durations:
 *   ms[0] prep + count scan, ms[1] emit + radix sort + tile scan,
 *   ms[2] block masks + evaluate + finalize, ms[3] sum of the three,
 *   ms[4] evaluate + finalize alone (the hot kernel).
 * sqv_profile_read synchronises the pending events; reset != 0 zeroes. */
#define SQV_NSTAGES 5
int sqv_profile_enable(int on);
int sqv_profile_read(double* ms, int64_t* calls, int reset);

/* Evaluator work counters: while attached, every sqv_voxelize call adds to
 * counters[0] the MUFU (SFU) operations its evaluators issue (thread level)
 * and to counters[1] the (primitive, voxel) pairs they evaluate (whole warp
 * blocks of 128 voxels, so culled-in but window-dead voxels count).  The
 * caller owns the int64[2] device buffer; NULL detaches.  One atomic pair per
 * warp and staged chunk; for benchmarks, not part of the reference API. */
int sqv_stats_attach(int64_t* counters);

/* Microbenchmarks of the pipes that bound the evaluator (roofline
 * denominators measured on the running GPU): which = 0 -> MUFU (SFU) ex2/lg2
 * ops/s, 1 -> FP32 FFMA lanes/s.  *ops_per_s receives the achieved rate. */
int sqv_microbench(int which, double* ops_per_s, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SQV_H_ */
