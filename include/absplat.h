/* absplat.h -- C ABI of the B200 abstract-rendering library (libabsplat.so).
 *
 * Computes, for a Gaussian-splat scene and a box of camera poses / scene parameters, lower
 * and upper bound images lo <= hi that contain every concrete render GaussianSplat(Sc, C, u)
 * (Alg. 1) for every scene Sc and camera C in the box (abstract rendering
 * problem; Theorem 1).  The method is AbstractSplat
 * (PAPER.md:539-558): Alg. 1 lifted to affine forms, MatrixInv (Alg. 4) at
 * line 8 and BlendInd (Alg. 3) at line 11, evaluated per image tile and
 * Gaussian batch, with the readings listed in DESIGN.md §2.
 *
 * Conventions (all functions):
 *   - return an as_status; on error nothing is written to caller outputs and
 *     as_last_error(ctx) describes the failure;
 *   - no C++ types or exceptions cross the ABI; all pointers are plain host or device
 *     pointers as documented per argument; inputs are copied (the library owns its copies),
 *     outputs are caller-owned;
 *   - work is enqueued on the context's CUDA stream (as_create); one context per host thread.
 */
#ifndef ABSPLAT_H
#define ABSPLAT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ABSPLAT_VERSION 1
#define AS_MAX_VARS 9 /* 3 translation + 3 Euler + up to 3 group-shift variables */

typedef struct as_ctx as_ctx; /* opaque; owns all device state */

typedef enum {
  AS_OK = 0,
  AS_E_ARG = 1,     /* invalid argument (sizes, ranges, NULL pointers, bad flags) */
  AS_E_SCENE = 2,   /* scene data invalid (non-finite, chol diagonal <= 0, o or c outside [0,1]) */
  AS_E_NUMERIC = 3, /* reserved: numerical failure that has no sound fallback */
  AS_E_CUDA = 4,    /* a CUDA runtime call failed */
  AS_E_OOM = 5,     /* device allocation failed */
  AS_E_STATE = 6,   /* call order violated (e.g. render before as_load_scene) */
  AS_E_COMM = 7     /* NCCL unavailable or a collective failed (multi-GPU contexts) */
} as_status;

/* Camera.  Extrinsics as XYZ Euler angles of the camera->world
 * rotation, R_c2w = Rz(euler[2]) Ry(euler[1]) Rx(euler[0]) (Table 3 caption PAPER.md:624,
 * reading G9), camera centre t in world; the camera looks along +z_cam; the world->camera
 * rotation of Alg. 1 line 2 is R = R_c2w^T.  Pixel (x, y) has centre (x + 0.5, y + 0.5). */
typedef struct {
  double fx, fy, cx, cy;
  int32_t W, H;
  double euler[3];
  double t[3];
} as_camera;

/* Pose box B_{eps_t, eps_R}(C0): translation offset in
 * [t_off - eps_t, t_off + eps_t] per axis (world axes, or the nominal camera axes when
 * t_frame == 1), Euler offset in [R_off - eps_R, R_off + eps_R].  A zero half-width means the
 * axis is not perturbed.  parts[k] >= 1 splits axis k into that many equal sub-intervals
 * (input-set partitioning); parts > 1 on an unperturbed axis is AS_E_ARG.
 * Axis order: tx, ty, tz, e0, e1, e2. */
typedef struct {
  double eps_t[3];
  double eps_R[3];
  double t_off[3];
  double R_off[3];
  int32_t t_frame;
  int32_t parts[6];
} as_pose_box;

/* Scene-parameter box.  All pointers are HOST pointers; data is copied.
 *   n_groups 0..3 shared mean-shift groups: Gaussian i with group_of[i] = g >= 0 has its mean
 *   moved by s * dir[g] with s in [shift_lo[g], shift_hi[g]] (one shared variable per group);
 *   col_lo/col_hi [N][3] (or NULL): colour intervals; op_lo/op_hi [N] (or NULL): opacity
 *   intervals.  Intervals must satisfy 0 <= lo <= hi <= 1. */
typedef struct {
  int32_t n_groups;
  const int32_t* group_of; /* [N] or NULL if n_groups == 0 */
  const double* dir;       /* [n_groups][3] */
  const double* shift_lo;  /* [n_groups] */
  const double* shift_hi;  /* [n_groups] */
  int32_t parts[3];        /* partitions per group variable */
  const float* col_lo;
  const float* col_hi;
  const float* op_lo;
  const float* op_hi;
  /* [N][3] or NULL (NEXT-2): per-Gaussian private mean offsets in world units, independent
   * across Gaussians: Gaussian i's mean is mean[i] + delta with delta_b in
   * [priv_lo[i][b], priv_hi[i][b]].  They add three private variables to every Gaussian's
   * forms (n = shared + 3 <= 9); depth comparisons treat them as independent. */
  const float* priv_lo;
  const float* priv_hi;
} as_scene_box;

/* Counters and per-phase device times of the last render (times in ms, CUDA events). */
typedef struct {
  int64_t pairs;           /* sum over (sub-box, tile) of |L_T| (tile-level Gaussian lists) */
  int64_t active_pairs;    /* (pixel, Gaussian) pairs not culled at the pixel */
  int64_t uncertain_pairs; /* unordered depth pairs with Ind = '?' */
  int64_t fails;           /* MatrixInv FAIL Gaussians (summed over sub-boxes) */
  int64_t straddles;       /* Gaussians whose depth straddles d_min */
  int64_t dropped;         /* Gaussians entirely behind d_min (or with o_hi <= tau) */
  int64_t order_violations;/* pairs contradicting the (kappa, index) order (must be 0) */
  int64_t launches;        /* kernel launches issued (own kernels + CUB calls) */
  int32_t kmax;            /* max |L_T| */
  int32_t n_sub;           /* number of sub-boxes */
  int32_t n_vars;          /* number of box variables n */
  int32_t n_tiles;         /* tiles rendered by this context */
  double ms_pose, ms_setup, ms_bin, ms_pairs, ms_tile, ms_total;
  double tile_kernel_ms;   /* sum of k_tile durations */
  size_t device_bytes;     /* bytes currently held by the context */
  int32_t n_items;         /* (tile, chunk) work items (max over sub-boxes) */
  int32_t grid;            /* persistent CTAs of the tile kernel (last sub-box) */
  int32_t ring_len;        /* exception ring length R allocated (last sub-box; 1 = none) */
  int32_t max_window;      /* longest exception window, positions (max over sub-boxes) */
  double ms_gather;        /* multi-GPU: the collective (all-gather of bound tiles or
                              all-reduce min/max of sub-box unions) and the untile */
  int32_t world;           /* ranks of the context's communicator (1 = single GPU) */
  int32_t n_owned;         /* tiles this rank rendered (tile sharding), else n_tiles */
  size_t peak_bytes;       /* device bytes held by the context at its largest */
  int32_t host_syncs;      /* blocking device-to-host reads inside the render pipeline: 0 when
                              it ran sync-free (sizes remembered from an earlier render of the
                              same tile / batch / box dimension, checked once at the end) */
  int32_t resized;         /* 1: the sync-free attempt outgrew the remembered sizes and the
                              render was repeated reading each size back (result unaffected) */
  int32_t graph_replay;    /* 1: the sync-free pipeline ran as one replay of the CUDA graph
                              captured from an identical earlier render (same sizes, tile, batch,
                              outputs; no state-changing call in between) */
  double ms_sort;          /* radix sorts of the binning (kappa order, pairs by tile), inside ms_bin */
  double ms_merge;         /* front-to-back composition of split tiles and its write of lo / hi
                              (the union over sub-boxes is fused into these writes: min / max) */
  double kmean;            /* mean |L_T| over non-empty (sub-box, tile) lists */
} as_stats;

/* Flags */
#define AS_PTR_DEVICE 1 /* pointer arguments are device pointers */
#define AS_ASYNC 2      /* return without synchronising the stream (device outputs only) */

/* Create a context on CUDA device `device`, enqueueing on `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream). */
as_status as_create(as_ctx** out, int32_t device, void* cuda_stream);
as_status as_destroy(as_ctx* ctx);
const char* as_last_error(const as_ctx* ctx); /* owned by ctx; valid until the next call */
int32_t as_version(void);

/* Load the scene (Gaussians <uw, Mw, o, c>): mean [N][3], chol [N][6]
 * (lower-triangular Cholesky factor Mw of Cov = Mw Mw^T, packed m00 m10 m11 m20 m21 m22),
 * opacity [N] in [0,1], color [N][3] in [0,1]; float32.  Host pointers unless AS_PTR_DEVICE.
 * Validated: finite, chol diagonal > 0, o and c in [0,1] (AS_E_SCENE otherwise).
 * Clears any scene box. */
as_status as_load_scene(as_ctx* ctx, int64_t N, const float* mean, const float* chol,
                        const float* opacity, const float* color, int32_t flags);
as_status as_set_camera(as_ctx* ctx, const as_camera* cam);
as_status as_set_pose_box(as_ctx* ctx, const as_pose_box* box);
/* Optional scene box (NULL clears).  Must be called after as_load_scene (uses N).  Host
 * arrays, copied; validated on the device (group ids in [-1, n_groups), colour / opacity
 * intervals inside [0,1] with lo <= hi, private-mean intervals finite with lo <= hi): on a bad
 * entry the scene box is cleared and AS_E_ARG (group id) or AS_E_SCENE is returned. */
as_status as_set_scene_box(as_ctx* ctx, const as_scene_box* sbox);

/* Abstract render of the whole image.  tile = TS in {8, 16, 32}; batch = BS, the number of
 * Gaussians staged in shared memory per step (1..256).  TS and BS are performance knobs
 * only (reading O1): the bounds do not depend on them.  lo/hi: caller-owned float32
 * [H][W][3], host pointers unless AS_PTR_DEVICE.  Returns once lo/hi are written unless
 * AS_ASYNC (device outputs only).  stats may be NULL.
 * Single-GPU interval renders after the first of a (tile, batch, box dimension) shape run
 * sync-free: no blocking host read inside the pipeline, buffer sizes remembered from an
 * earlier render and checked once at the end (a render that outgrows them is repeated
 * reading each size back: stats->resized); once such a render allocated nothing, the next
 * identical call is captured into a CUDA graph and later ones replay it (stats->graph_replay)
 * until any as_set_* / as_load_* call.  Results are bit-identical either way. */
as_status as_render_bounds(as_ctx* ctx, int32_t tile, int32_t batch, float* lo, float* hi,
                           int32_t flags, as_stats* stats);

/* ---- sub-box ranges (SURVEY.md §8(e) second sharding axis) ----
 * The abstract image is the elementwise union (lo = min, hi = max) over the P sub-boxes of
 * the partitioned input box (step 22).  as_render_subboxes renders the union
 * over sub-boxes [sub_begin, sub_end) only (0 <= sub_begin <= sub_end <= P; sub-box s is the
 * multi-index over the partitioned axes, tx fastest, as in as_pose_box.parts); an empty
 * range writes the union's identities lo = 1, hi = 0.  Disjoint ranges rendered on different
 * ranks therefore combine with an all-reduce MIN / MAX into the full image, bit for bit.
 * Arguments otherwise as as_render_bounds.  as_subbox_count returns P for the current box. */
as_status as_render_subboxes(as_ctx* ctx, int32_t tile, int32_t batch, int32_t sub_begin,
                             int32_t sub_end, float* lo, float* hi, int32_t flags,
                             as_stats* stats);
as_status as_subbox_count(as_ctx* ctx, int32_t* n_sub);

/* ---- explicit partitions and adaptive refinement (PAPER.md:470 (2):
 * "iteratively divide the input range until the assertion [rho < 1] is satisfied") ----
 * as_set_subboxes replaces the uniform grid of as_pose_box.parts by n explicit sub-boxes:
 * bounds [n][9][2] = (lo, hi) per box axis (tx, ty, tz, e0, e1, e2 in as_pose_box units, then
 * the group shifts 0..2), each inside the box (AS_E_ARG otherwise; an axis the box does not
 * perturb must be given as its fixed value).  Host pointer, copied.  n = 0 restores the
 * uniform grid; as_set_pose_box also clears the list.  Sub-box s of the list is sub-box s of
 * as_render_subboxes.
 * as_subbox_fails writes, for every sub-box of the current partition, the number of
 * (non-dropped) Gaussians whose MatrixInv fails there (det <= 0 or rho >= 1: a in [0, o_hi]),
 * running only the per-Gaussian setup; fails is host int64[n >= number of sub-boxes].  The
 * Python driver `paper_2503_00308_b200.refine` bisects failing sub-boxes with these counts. */
as_status as_set_subboxes(as_ctx* ctx, int32_t n, const double* bounds);
/* Adaptive MatrixInv order (PAPER.md:470 (3): "increase k until Eps falls below the given
 * tolerance"): with k_tol > 0 every Gaussian uses the smallest k >= 8 whose remainder
 * Eps = |X0|_F rho^(k+1) / (1 - rho) is <= k_tol, at most k_max (8..64); k_tol <= 0 restores the
 * fixed k = 8.  Applies to subsequent renders. */
as_status as_set_matrixinv(as_ctx* ctx, double k_tol, int32_t k_max);
/* MatrixInv conic bounds: backward = 0 (default) concretises the
 * forward forms of Xp = X0 + X0 sum_i P^i (reading G3); backward = 1 bounds each conic entry
 * by back-substitution (CROWN-style) through P^i = P^{i-1} E with the same
 * McCormick planes down to E = I - X X0, the intermediate P^i bounds back-substituted too
 * (reading O17); tighter (Example 1: 0.7588 -> 0.6875 at k = 8; the paper prints 0.70).
 * With back-substitution the adaptive order is limited to k_max <= 32. */
as_status as_set_inverse_mode(as_ctx* ctx, int32_t backward);
as_status as_subbox_fails(as_ctx* ctx, int32_t n, int64_t* fails);

/* ---- blend mode ----
 * mode 0 (default): the interval blend (reading O7).  mode 1: additionally BlendInd is
 * evaluated with linear relations along the sorted fold (a = o Exp(-s/2) with Table 2's
 * tangent / chord kept linear in the box variables, T as an affine form through McCormick
 * products, Alg. 3): a position without uncertain depth partners contributes
 * Mul(T, a) c, one with uncertain partners (Table 2's Ind "?") its interval-blend term
 * [T_lo a_lo c_lo, T_hi a_hi c_hi] (reading O20); the result is intersected with the interval
 * bounds, per sub-box, before the union.  Boxes with up to 9 variables; full-image renders
 * (as_render_bounds / as_render_subboxes, and the sub-box sharding axis); AS_E_ARG for tile
 * sharding. */
as_status as_set_blend(as_ctx* ctx, int32_t mode);

/* ---- work split (performance knob, like tile and batch) ----
 * A tile's sorted Gaussian list is cut into chunks of `target` positions that the tile kernel
 * processes independently and composes front to back; target = 0 (default)
 * picks it from the list lengths and the grid (about six chunks per CTA), any other value
 * >= 1 fixes it (clamped to at least the batch size).  The bounds do not depend on it beyond
 * fp32 rounding of the composition. */
as_status as_set_chunk_target(as_ctx* ctx, int32_t target);

/* ---- tile sharding over ranks (PAPER.md:602-603 tiles; north_star: tiles across GPUs) ----
 * Every rank holds the full scene and runs the per-Gaussian setup; image tiles are
 * assigned to ranks by a deterministic longest-processing-time rule over per-tile Gaussian
 * counts (identical on every rank), so each rank renders only its own tiles and the bound
 * images are assembled with one gather.
 *
 * as_render_shard: renders the tiles owned by `rank` of `world` into the compact tile-major
 * buffers lo_tm/hi_tm [max_tiles][tile*tile][3] (device pointers unless flags lack
 * AS_PTR_DEVICE) and writes their tile ids (ascending) to owned[] (host, int32[max_tiles])
 * and their number to *n_owned.  max_tiles (identical on every rank) caps the tiles per rank
 * and must be >= ceil(n_tiles / world), n_tiles = ceil(W/tile)*ceil(H/tile). */
as_status as_render_shard(as_ctx* ctx, int32_t tile, int32_t batch, int32_t rank, int32_t world,
                          float* lo_tm, float* hi_tm, int32_t max_tiles, int32_t* owned,
                          int32_t* n_owned, int32_t flags, as_stats* stats);
/* Assemble gathered tile-major buffers of `world` ranks ([world][max_tiles][tile*tile][3]
 * floats, with owned ids [world][max_tiles] and counts n_owned[world], host int32 arrays)
 * into row-major images lo/hi [H][W][3].  Pointer space per AS_PTR_DEVICE (tm and images
 * alike); with host pointers ctx may be NULL (pure host index arithmetic).  Every tile must be
 * owned exactly once (AS_E_ARG otherwise). */
as_status as_untile(as_ctx* ctx, int32_t W, int32_t H, int32_t tile, int32_t world,
                    int32_t max_tiles, const int32_t* owned, const int32_t* n_owned,
                    const float* lo_tm, const float* hi_tm, float* lo, float* hi, int32_t flags);
/* The deterministic owner map used by as_render_shard for the current scene / camera /
 * box (host int32 [n_tiles]); costs optional (host int64 [n_tiles], per-tile pair counts
 * summed over sub-boxes).  Runs the setup and counting passes. */
as_status as_tile_owners(as_ctx* ctx, int32_t tile, int32_t world, int32_t max_tiles,
                         int32_t* owner, int64_t* costs);
/* Pure host function: longest-processing-time assignment of n_tiles tiles with the given
 * costs to `world` ranks, at most `cap` tiles per rank (cap >= ceil(n_tiles / world)).
 * Tiles in descending cost (ties: lower id first) go to the least-loaded rank with room
 * (ties: lower rank).  owner: int32 [n_tiles]. */
as_status as_lpt_assign(int32_t n_tiles, const int64_t* costs, int32_t world, int32_t cap,
                        int32_t* owner);

/* ---- multi-GPU: one process (or host thread) per GPU, one NCCL communicator per context
 * (north_star (3): image tiles across GPUs with ONE gather of the bound images; SURVEY.md
 * §8(b), §8(e)).  NCCL is resolved at run time (libnccl.so.2, the copy the process already
 * loaded if any); AS_E_COMM when it is unavailable or a call fails.
 *   as_nccl_id: writes a fresh NCCL unique id (128 bytes) into id; call on one rank and pass
 *     the bytes to every rank by any out-of-band channel.
 *   as_comm_init: joins rank `rank` of `world` (1 <= world <= 128) on the context's device
 *     (collective: every rank calls it with the same id).  A context joined with world > 1
 *     renders in parallel: as_render_bounds / as_render_subboxes split the work over the
 *     ranks, run ONE collective on the context stream and write the complete lo / hi on
 *     every rank.  Axis (as_set_shard_axis): 1 = image tiles -- every rank runs the
 *     per-Gaussian setup and a per-tile cost count, the deterministic device LPT owner map
 *     (identical on every rank, that of as_lpt_assign with cap = ceil(n_tiles/world) +
 *     max(1, ceil(n_tiles/world)/4)) picks this rank's tiles, they are rendered into a compact
 *     tile-major buffer, one ncclAllGather of the bound tiles and an on-device untile follow;
 *     2 = sub-boxes -- rank r renders the union over its contiguous balanced range of the
 *     sub-boxes (as_render_subboxes semantics) and one ncclAllReduce MIN on lo / MAX on hi
 *     completes the union (step 22); 0 (default) = sub-boxes when there are at
 *     least `world` sub-boxes, else tiles.  With world == 1 an explicit axis still runs the
 *     collective path (single-rank communicator), which tests it on one GPU.
 *   The result is bitwise identical to the single-GPU render for both axes. */
as_status as_nccl_id(uint8_t id[128]);
as_status as_comm_init(as_ctx* ctx, int32_t rank, int32_t world, const uint8_t id[128]);
as_status as_set_shard_axis(as_ctx* ctx, int32_t axis);

/* ---- device scratch allocator ----
 * All device memory the context holds (scene copy, per-Gaussian records, pair lists, sort
 * buffers, exception metadata, the tile kernel's ring and partial sums) comes from
 * alloc(user, bytes, stream) and goes back through free(user, ptr, bytes, stream), where
 * stream is the context stream (cudaStream_t).  Buffers are grow-only and reused across
 * renders; a buffer is returned to the allocator that produced it.  alloc returning NULL is
 * AS_E_OOM.  alloc == NULL and free == NULL restore the default (cudaMalloc / cudaFree).
 * Buffers allocated before the call stay with their allocator until they grow or the
 * context is destroyed.  The Python binding binds this to torch's caching allocator. */
typedef void* (*as_alloc_fn)(void* user, size_t bytes, void* stream);
typedef void (*as_free_fn)(void* user, void* ptr, size_t bytes, void* stream);
as_status as_set_allocator(as_ctx* ctx, as_alloc_fn alloc, as_free_fn free_fn, void* user);

/* ---- rare-path evidence (tests) ----
 * enable = 1 makes subsequent renders count how often the tile kernel takes each slow path of
 * the depth-exception machinery (rows a7/a9: Alg. 3 P:377-389 with uncertain Ind pairs,
 * Table 2); 0 switches counting off; -1 leaves the setting.  out (host uint64
 * [AS_DBG_N], may be NULL) receives the counts of the last render (zeros if counting was off):
 *   0 upper-transmittance window re-multiplied from the 128-bit E_F mask (many operands or an
 *     unsafe division), 1 division by the E_F factors refused (product below 1e-20 or running
 *     product below 1e-25, reading H3), 2 window longer than 128 positions (global exception
 *     lists), 3 such a window re-multiplied instead of divided, 4 finalisation with more than
 *     60 E_G operands or a long list, 5 finalisation record beyond the 48 staged per batch,
 *     6 finalisation through global E_G lists (window > 128), 7 T_hi window with more than 32
 *     operands.  Counting costs atomics on those paths only. */
#define AS_DBG_N 8
as_status as_debug_counters(as_ctx* ctx, int32_t enable, uint64_t* out);

/* Concrete render (Alg. 1 + BlendSort, reading G6/G8) at one point of the box: xi[n] in
 * [-1,1]^n are the box variables of the FULL box in order (perturbed axes tx,ty,tz,e0,e1,e2,
 * then group shifts), with the scene's nominal colours and opacities.  img: [H][W][3]
 * float32, host unless AS_PTR_DEVICE.  Used by soundness tests on large scenes. */
as_status as_render_concrete(as_ctx* ctx, const double* xi, float* img, int32_t flags);

#ifdef __cplusplus
}
#endif
#endif
