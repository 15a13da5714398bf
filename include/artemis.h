/*
 * libartemis — B200 (sm_100a) kernels for the ARTEMIS warp -> octree
 * rebuild -> render hot path, behind a plain C ABI.
 *
 * The reference's native boundary is the flat-array `kernels` module that
 * animvox/backend.py:19-31 binds (compiled: animvox/_core.pyx, pure:
 * animvox/_pure.py). Every entry point below replaces one of those
 * functions, or one of the numpy stages the reference runs around them
 * (rigging.warp_voxels, rigging.resolve_collisions, volume.build_octree,
 * geometry.rays_for_camera); the citation is on each declaration.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless a parameter says "host".
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and returns an artemis_status for argument errors
 *    detectable without synchronising. Data-dependent results (counts,
 *    duplicate detection) are written to device memory the caller reads.
 *  - Layouts are the reference's: Morton codes u64 with x in the lowest
 *    interleave slot, 21 bits per axis; tree arrays int32 with leaves encoded
 *    as ~leaf; FLUT column h*C + c, density last (split here into an fp32
 *    coefficient block and an fp64 density column).
 *  - No torch types appear here. The Python layer (paper_2202_05628_b200)
 *    uses torch only to own device memory and streams.
 */
#ifndef ARTEMIS_H
#define ARTEMIS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *artemis_stream;

typedef enum {
    ARTEMIS_OK = 0,
    ARTEMIS_ERR_ARG = 1,        /* null pointer / bad size / unsupported option */
    ARTEMIS_ERR_RANGE = 2,      /* grid coordinate outside [0, 2^21) (_core.pyx:81-82) */
    ARTEMIS_ERR_EMPTY = 3,      /* empty leaf set (_core.pyx:196-197) */
    ARTEMIS_ERR_DUPLICATE = 4,  /* duplicate Morton code (volume.py:244-247) */
    ARTEMIS_ERR_OOM = 5,
    ARTEMIS_ERR_CUDA = 6,       /* launch failure; see artemis_last_cuda_error */
    ARTEMIS_ERR_WORKSPACE = 7,  /* workspace smaller than *_workspace_bytes */
    ARTEMIS_ERR_NODEVICE = 8,   /* no sm_100 device visible */
    /* .nvo asset container (assetio.py:86-136): TruncatedAssetError, ... */
    ARTEMIS_ASSET_TRUNCATED_HEADER = 20,
    ARTEMIS_ASSET_BAD_MAGIC = 21,       /* MagicMismatchError */
    ARTEMIS_ASSET_BAD_VERSION = 22,     /* AssetFormatError */
    ARTEMIS_ASSET_ZERO_COUNT = 23,      /* CountMismatchError */
    ARTEMIS_ASSET_TRUNCATED_LEAVES = 24,
    ARTEMIS_ASSET_TRUNCATED_FLUT = 25,
    ARTEMIS_ASSET_RIG_OFFSET = 26,      /* CountMismatchError */
    ARTEMIS_ASSET_TRUNCATED_RIG = 27,
    ARTEMIS_ASSET_TRAILING = 28         /* CountMismatchError */
} artemis_status;

const char *artemis_version(void);
const char *artemis_status_string(int status);
const char *artemis_last_cuda_error(void);
/* 1 when a CUDA device of compute capability 10.x is visible. */
int artemis_device_ok(void);

/* ---- Morton codes ------------------------------------------------------
 * replaces animvox/_core.pyx:79-92 morton_encode, :95-105 morton_decode.
 * coords: (n, 3) int64 row-major. `range_flag` (device int32, may be NULL)
 * is set to 1 when any coordinate is outside [0, 2^21) (the caller raises
 * ValueError, as _core.pyx:81-82 does). */
int artemis_morton_encode(const int64_t *coords, int64_t n, uint64_t *codes,
                          int32_t *range_flag, artemis_stream stream);
int artemis_morton_decode(const uint64_t *codes, int64_t n, int64_t *coords,
                          artemis_stream stream);

/* ---- Stable radix sort (onesweep, decoupled look-back) --------------------
 * replaces animvox/_core.pyx:111-167 sort_order (stable LSD, 8-bit digits,
 * ceil(key_bits/8) passes). Sorts (key, value) pairs ascending by the low
 * `key_bits` bits of the key; equal keys keep input order. `vals_in` NULL
 * means values 0..n-1, i.e. the permutation sort_order returns.
 * n < 2^30. Workspace is caller-allocated device memory. */
size_t artemis_sort_workspace_bytes(int64_t n, int key_bits, int key_bytes);
int artemis_sort_pairs_u64(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                           uint32_t *vals_out, int64_t n, int key_bits, void *workspace,
                           size_t workspace_bytes, artemis_stream stream);
int artemis_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                           uint32_t *vals_out, int64_t n, int key_bits, void *workspace,
                           size_t workspace_bytes, artemis_stream stream);

/* ---- Karras radix tree ------------------------------------------------
 * replaces animvox/_core.pyx:193-246 build_tree (node numbering, ~leaf child
 * links and octant boxes identical). codes: strictly sorted u64, n >= 1.
 * left/right: (n-1) int32, box_min/box_size: (n-1, 3) int32. The root is 0
 * (n > 1) or ~0 (n == 1), as in the reference. `dup_flag` (device int32,
 * may be NULL; the caller initialises it to INT32_MAX) receives the
 * smallest i with codes[i] == codes[i+1] (volume.py:244-247's check). */
int artemis_build_tree(const uint64_t *codes, int64_t n, int32_t *left, int32_t *right,
                       int32_t *box_min, int32_t *box_size, int32_t *dup_flag,
                       artemis_stream stream);

/* ---- Traversal structure ------------------------------------------------
 * The render kernels walk a packed copy of the tree: one 32-byte record per
 * internal node holding both children's boxes (so a visit is one sector),
 * plus a super-root record at index max(n-1, 0) whose left child is the
 * root, and one 32-byte record per leaf {x, y, z, flut row, density,
 * rotation index}. Built from the reference arrays (API path) or directly
 * by artemis_frame_run (device pipeline). sigma/rot_index are indexed by
 * FLUT row and may be NULL for trees that are only traversed (not shaded).
 * nodes: n x 64 bytes (two-level records), leaves: n x 32 bytes. */
int artemis_pack_tree(const uint64_t *codes, const uint32_t *flut_idx, int64_t n, int32_t root,
                      const int32_t *left, const int32_t *right, const int32_t *box_min,
                      const int32_t *box_size, const double *sigma, const int32_t *rot_index,
                      void *nodes, void *leaves, artemis_stream stream);

/* FLUT (n, width) row-major -> fp32 coefficients (n, width-1) + fp64
 * density (n). Replaces the FLUT.data gather layout of _core.pyx:536-551. */
int artemis_flut_split_f64(const double *flut, int64_t n, int width, float *coef,
                           double *sigma, artemis_stream stream);
int artemis_flut_split_f32(const float *flut, int64_t n, int width, float *coef,
                           double *sigma, artemis_stream stream);

/* Occupancy brick map of a leaf set: dense table of 8^3-cell bricks over
 * brick coordinates [org, org + dims), 128-byte records (512-bit mask,
 * per-word prefix counts, first leaf), and the leaf AABB. With it the render
 * kernels enumerate a ray's hit leaves by an exact cell walk (bricks.cuh
 * explains why that equals the reference's DFS order). */
typedef struct {
    int32_t *table;
    void *recs;
    int32_t *aabb;              /* [6] leaf cells: lo xyz inclusive, hi xyz exclusive */
    int32_t org[3], dims[3];
} artemis_brickmap;

size_t artemis_brickmap_bytes(int64_t n_leaves, const int32_t *dims /* host [3] */);
/* codes: sorted unique u64 (n); org/dims host [3] brick-coordinate box that
 * covers every leaf; storage >= artemis_brickmap_bytes. Fills *out (host). */
int artemis_brickmap_build(const uint64_t *codes, int64_t n, const int32_t *org,
                           const int32_t *dims, void *storage, size_t storage_bytes,
                           artemis_brickmap *out, artemis_stream stream);

typedef struct {
    const void *nodes;          /* artemis_pack_tree output: internal records */
    const void *leaves;         /* artemis_pack_tree output: leaf records */
    int64_t n_leaves;           /* host value; ignored when n_leaves_dev != NULL */
    const int32_t *n_leaves_dev;/* device count (device pipeline), may be NULL */
    double coord_max;           /* bound on every box coordinate (the grid
                                   resolution); 0 = 2^21. Only tunes the fp32
                                   filter; results never depend on it. */
    const artemis_brickmap *bricks; /* host pointer; non-NULL selects the exact
                                   cell walk instead of the tree DFS (same
                                   results) */
} artemis_tree_view;

typedef struct {
    const float *coef;          /* (N, H*C) fp32, column h*C + c */
    const double *sigma;        /* (N) fp64 density */
    const int32_t *rot_index;   /* (N) per FLUT row rotation index */
    const double *rot_inv;      /* (J, 3, 3) fp64 */
    int degree;                 /* SH degree 0..4 */
    int channels;               /* C >= 1 */
    int coef_stride;            /* floats per coef row (FLUT width - 1); 0 = H*C */
} artemis_shading;

typedef struct {
    const double *origins_g;    /* (R, 3) grid-space origins */
    const double *dirs_g;       /* (R, 3) grid-space directions */
    const double *dirs_w;       /* (R, 3) unit world directions (SH input) */
    int64_t n_rays;
    double t_min, t_max;
    int32_t fast_div;           /* 1: the caller vouches that every origins_g
                                   component is 0 or of magnitude in [2^-300, 2^300]
                                   and every dirs_g component 0 or in
                                   [2^-600, 2^300]; the cell walk then divides by
                                   a corrected reciprocal (same bits, faster).
                                   0: __ddiv_rn. */
} artemis_rays;

/* Pinhole camera, evaluated per pixel exactly as rays_for_camera
 * (geometry.py:242-263) + _grid_rays (render.py:181-185) do on the host. */
typedef struct {
    double R[9];                /* camera-to-world rotation, row-major */
    double origin[3];           /* camera centre, world */
    double fx, fy, cx, cy;
    int32_t width, height;
    double lo[3], cell[3];      /* grid bounds min and cell size */
    int32_t tile_start, tile_stride; /* frame pipeline: render only the 8x4 pixel
                                   tiles t with t % tile_stride == tile_start
                                   (multi-GPU tile sharding); other pixels get
                                   F = 0, alpha = 0, depth = +inf. 0/0 or 0/1 =
                                   every tile. */
} artemis_camera;

/* replaces animvox/_core.pyx:473-559 render_rays. F: (R, C) fp32,
 * alpha/depth: (R) fp64 (depth +inf when no voxel passed sigma_dep). */
int artemis_render_rays(const artemis_tree_view *tree, const artemis_shading *shade,
                        const artemis_rays *rays, double lambda_th, double sigma_dep,
                        int early_stop, float *F, double *alpha, double *depth,
                        artemis_stream stream);

/* replaces the count pass of animvox/_core.pyx:586-596 (forward_fit) and
 * traverse_ray :358-389: hits per ray. counts: (R) int64. */
int artemis_count_hits(const artemis_tree_view *tree, const artemis_rays *rays, int64_t *counts,
                       artemis_stream stream);

/* replaces the fill pass of animvox/_core.pyx:597-655 forward_fit: CSR
 * trace at `offsets` (R+1, exclusive scan of counts) plus F/alpha without
 * early stop. hit_idx int64, hit_t0/t1 fp64. */
int artemis_forward_fit(const artemis_tree_view *tree, const artemis_shading *shade,
                        const artemis_rays *rays, const int64_t *offsets, int64_t *hit_idx,
                        double *hit_t0, double *hit_t1, float *F, double *alpha,
                        artemis_stream stream);

/* ---- Training gradients ----------------------------------------------
 * replaces animvox/_core.pyx:661-755 backward_rays (fit.py:108-146
 * backward_batch). The CSR trace of artemis_forward_fit / forward_fit
 * (offsets (R+1) int64, hit_idx/t0/t1 (M)), unit world directions (R,3),
 * rot tables, the FLUT (n_flut, width) and dL/dF (R,C), dL/dalpha (R) in
 * the same real type (real_bytes 4 = float, 8 = double, as the reference's
 * fused real_t) -> grad (n_flut, width) of that type, zero for untouched
 * rows. Accumulation is deterministic (each grad entry summed in ascending
 * ray order, the reference's deterministic schedule) for either value of
 * `deterministic`. Workspace: artemis_backward_workspace_bytes. */
size_t artemis_backward_workspace_bytes(int64_t n_hits, int64_t n_flut);
int artemis_backward_rays(const int64_t *offsets, int64_t n_rays, const int64_t *hit_idx,
                          const double *hit_t0, const double *hit_t1, int64_t n_hits,
                          const double *dirs_w, const int32_t *rot_index, const double *rot_inv,
                          const void *flut, int64_t n_flut, int width, const void *dldf,
                          const void *dlda, int real_bytes, int degree, int channels,
                          int deterministic, void *grad, void *workspace,
                          size_t workspace_bytes, artemis_stream stream);

/* ---- Training iteration bookkeeping (fit.py:474-501, :308-330) ---------
 * artemis_l1_grads: dL/dF = sign(F - gt_F) / R, dL/dalpha = sign(alpha -
 * gt_alpha) / R (F fp32 from artemis_forward_fit, the rest fp64), the
 * per-ray loss term sum_c |dF| + |dalpha| into loss_rays and their ordered
 * sum into *loss_sum (device). artemis_mark_touched: touched[row] = 1 for
 * every hit (backward_batch's bitmap). artemis_vrt_grads: the collision
 * pair term, grad[w] += s, grad[l] -= s with s = sign(data[w] - data[l]) *
 * scale, applied per row in np.add.at's order; marks the rows touched.
 * artemis_sparse_adam: SparseAdam.step on touched rows (bias1/bias2 =
 * 1 - beta^t from the host), then the density clamp of those rows. */
int artemis_l1_grads(const float *F, const double *alpha, const double *gt_F,
                     const double *gt_alpha, int64_t n_rays, int channels, double *dldf,
                     double *dlda, double *loss_rays, double *loss_sum, artemis_stream stream);
int artemis_mark_touched(const int64_t *hit_idx, int64_t n_hits, uint8_t *touched,
                         artemis_stream stream);
size_t artemis_vrt_workspace_bytes(int64_t n_pairs, int64_t n_rows);
int artemis_vrt_grads(const double *data, int64_t n_rows, int width, const int64_t *pairs,
                      int64_t n_pairs, double scale, double *grad, uint8_t *touched,
                      void *workspace, size_t workspace_bytes, artemis_stream stream);
int artemis_sparse_adam(double *params, double *m, double *v, const double *grad,
                        const uint8_t *touched, int64_t n_rows, int width, double lr,
                        double beta1, double beta2, double eps, double bias1, double bias2,
                        artemis_stream stream);

/* Device ray generation (parity helper for rays_for_camera + _grid_rays).
 * og/dg/dw: (W*H, 3) fp64, row-major pixels. */
int artemis_camera_rays(const artemis_camera *cam /* host */, double *og, double *dg,
                        double *dw, artemis_stream stream);

/* ---- Warp and collision resolve --------------------------------------
 * replaces animvox/rigging.py:327-371 (warp_voxels numerics). cells (N,3)
 * int32 canonical; joint_idx (N,K) int32 (-1 = unused slot); weights (N,K)
 * fp64; joint_aff (J,12) fp64 = rows 0..2 of the per-joint delta matrices.
 * lo and cell are HOST pointers to 3 doubles (Bounds.lo, Bounds.cell_size).
 * Outputs (any may be NULL): positions (N,3) fp64, cells_out (N,3) int32
 * (-1 when out of bounds), in_bounds (N) uint8, rotation_joint (N) int32. */
int artemis_warp(const int32_t *cells, int64_t n, int slots, const int32_t *joint_idx,
                 const double *weights, const double *joint_aff, int n_joints,
                 const double *lo, const double *cell, int resolution, double *positions,
                 int32_t *cells_out, uint8_t *in_bounds, int32_t *rotation_joint,
                 artemis_stream stream);

/* replaces animvox/rigging.py:433-459 (resolve_collisions). Input: the
 * in-bounds canonical indices' Morton codes sorted STABLY (so equal codes
 * list canonical indices ascending), n_sorted entries, and the fp64
 * density per canonical index. Output: live codes (unique, ascending),
 * winners (highest density, lowest index on ties) and, when pairs != NULL,
 * the (winner, loser) rows in the reference's (-sigma, index) order.
 * n_live_out (device int32). Workspace: artemis_resolve_workspace_bytes. */
size_t artemis_resolve_workspace_bytes(int64_t n_sorted);
int artemis_resolve_u64(const uint64_t *sorted_codes, const uint32_t *sorted_idx,
                        int64_t n_sorted, const int32_t *n_sorted_dev, const double *sigma,
                        uint64_t *live_codes, uint32_t *winners, int64_t *pairs,
                        int32_t *n_live_out, void *workspace, size_t workspace_bytes,
                        artemis_stream stream);

/* ---- Device-resident frame pipeline ------------------------------------
 * One posed frame end to end on the device (render.timed_render_frame,
 * render.py:284-319): warp -> stable sort of the warped keys -> resolve ->
 * Karras build -> tile-ordered render with in-kernel ray generation. The
 * handle owns every intermediate buffer; the asset buffers stay owned by
 * the caller and must outlive the handle. */
typedef struct artemis_frame_s *artemis_frame;

typedef struct {
    int64_t n_voxels;
    int32_t resolution;         /* power of two <= 2^21 */
    int32_t slots;              /* K skin-weight slots */
    int32_t max_joints;
    int32_t degree, channels;
    double lo[3], hi[3];
    const int32_t *cells;       /* (N,3) int32 canonical cells */
    const int32_t *joint_idx;   /* (N,K) int32 */
    const double *weights;      /* (N,K) fp64 */
    const float *coef;          /* (N, H*C) fp32 */
    const double *sigma;        /* (N) fp64 */
} artemis_asset;

int artemis_frame_create(const artemis_asset *asset, artemis_frame *out);
int artemis_frame_destroy(artemis_frame frame);

/* Per-frame inputs are HOST pointers: joint_aff (J,12) fp64 (rows 0..2 of
 * the per-joint delta matrices, rigging.py:343-345), rot_inv (J,3,3) fp64
 * (rigging.py:347) and the camera. They are staged in pinned host memory (a
 * ring of 4 blocks) and copied asynchronously into a device parameter block
 * ahead of the frame, so a captured graph replays unchanged for any pose and
 * camera of the same image size. Up to 4 graphs are cached per handle
 * (keyed by image size, flags and output pointers), so callers may rotate
 * output buffers to overlap a frame's D2H read with the next frame. joint_aff == NULL renders the
 * canonical cells (identity warp, render.py:162-167).
 * flags: bit0 early stop, bit1 capture/replay a CUDA graph (needs a
 * non-default stream); bit2 is accepted for compatibility (the reference
 * tree arrays left/right/box_min/box_size are rebuilt every frame); bit3
 * (ARTEMIS_FRAME_MAPS64) writes alpha/depth as double with exact fp64 entry
 * distances, as artemis_render_rays does (the reference's FrameBuffers
 * precision), instead of float; bit4 (ARTEMIS_FRAME_REUSE_TREE) renders
 * another view of the tree the previous run built (multi-view / stereo:
 * one warp + rebuild per pose), skipping warp, sort, resolve and build --
 * the pose tables passed must be the ones that tree was built with.
 * F (W*H, C) fp32, alpha/depth (W*H) float or double, row-major pixels. */
#define ARTEMIS_FRAME_EARLY_STOP 1
#define ARTEMIS_FRAME_GRAPH 2
#define ARTEMIS_FRAME_MAPS64 8
#define ARTEMIS_FRAME_REUSE_TREE 16
int artemis_frame_run(artemis_frame frame, const double *joint_aff, const double *rot_inv,
                      int n_joints, const artemis_camera *cam, double lambda_th,
                      double sigma_dep, int flags, float *F, void *alpha, void *depth,
                      artemis_stream stream);

/* (no reference counterpart: multi-GPU assembly) Tile-sharded frames
 * (camera tile_stride > 1) of this handle write their
 * pixels straight into F / alpha / depth -- the destination rank's
 * full-frame buffers mapped into this process (CUDA IPC, peer access over
 * NVLink), or this rank's own on the destination -- instead of the local
 * outputs (left untouched). The destination initialises them (F 0, alpha 0,
 * depth +inf) before any rank renders; each rank writes exactly its own
 * tiles, so the assembled frame needs no gather. alpha/depth are float, or
 * double with ARTEMIS_FRAME_MAPS64. F == NULL restores the local outputs.
 * n_pixels / maps64 describe the peer maps: a sharded artemis_frame_run whose
 * image size or map type differs returns ARTEMIS_ERR_ARG (no stores past the
 * end of another rank's buffers). */
int artemis_frame_set_output_peer(artemis_frame frame, float *F, void *alpha, void *depth,
                                  int64_t n_pixels, int maps64);

/* (no reference counterpart: scheduling only) Render order of the 8x4 ray
 * tiles for one image size: `order` (HOST,
 * ceil(w/8)*ceil(h/4) int32) must be a permutation of the tile indices
 * (row-major tile numbering); ARTEMIS_ERR_ARG otherwise. Without it the
 * pipeline renders centre-out while the asset's FLUT coefficients fit in
 * 16x L2, row-major beyond (ARTEMIS_TILE_ORDER=rowmajor|centre forces one).
 * The order never changes the maps: every ray is rendered independently. */
int artemis_frame_set_tile_order(artemis_frame frame, int width, int height,
                                 const int32_t *order);

/* replaces one animvox/render.py:154-178 posed_octree followed by one
 * render_view (render.py:322-363) per camera. One pose, several views
 * (configs[1] views, configs[4] stereo eyes): warp + rebuild once, then ONE render launch over all n_views (<= 8) cameras of
 * the same image size, their 8x4 tiles interleaved in the ray queue so the
 * views' rays over the same leaves are in flight together and share the
 * FLUT rows in L2. Outputs per view: F[v], alpha[v], depth[v] (as
 * artemis_frame_run). Unsharded cameras only. Flags as artemis_frame_run. */
int artemis_frame_run_views(artemis_frame frame, const double *joint_aff, const double *rot_inv,
                            int n_joints, const artemis_camera *cams, int n_views,
                            double lambda_th, double sigma_dep, int flags, float *const *F,
                            void *const *alpha, void *const *depth, artemis_stream stream);

/* Read back the last frame's counts (synchronises the stream). */
int artemis_frame_counts(artemis_frame frame, int64_t *n_in_bounds, int64_t *n_live,
                         artemis_stream stream);

/* Device pointers to the last frame's rebuilt tree (reference layout) and
 * the per-canonical-voxel rotation index, for parity checks. Codes are
 * 4-byte when 3*log2(resolution)+1 <= 32 (sentinel bit included), else 8. */
typedef struct {
    const void *codes;          /* (n_live) Morton codes, code_bytes each */
    int32_t code_bytes;
    const uint32_t *flut_idx;   /* (n_live) */
    const int32_t *left, *right, *box_min, *box_size; /* (n_live-1[,3]) */
    const int32_t *rotation_joint; /* (N) */
    const int32_t *n_live_dev;
    const int32_t *n_in_dev;
} artemis_frame_tree;
int artemis_frame_get_tree(artemis_frame frame, artemis_frame_tree *out);

/* Stage timing for eager (non-graph) runs: after artemis_frame_profile(f, 1)
 * every eager artemis_frame_run records CUDA events between its stages;
 * artemis_frame_stage_ms writes 5 floats (ms): warp, sort, resolve, build,
 * render of the last such run (synchronises on its last event). */
int artemis_frame_profile(artemis_frame frame, int enable);
int artemis_frame_stage_ms(artemis_frame frame, float *ms);

/* ---- Device-resident asset ingestion ------
 * The .nvo container of animvox/assetio.py:49-202 (54-byte header, leaf
 * table of {u64 Morton code, u32 FLUT row}, f32 FLUT block, optional rig).
 * artemis_asset_probe (host) validates the header and the leaf/FLUT extents
 * in load_asset's order (assetio.py:88-104) and fills the info;
 * artemis_asset_decode_leaves (device) decodes the leaf table -- copied to
 * the device as it lies in the file -- into cells[row] (count, 3) int32
 * (assetio.py:118-122), setting *bad_flag (device) when the rows are not a
 * permutation (assetio.py:115-117); workspace >= 4 * count bytes. The f32
 * FLUT block goes to artemis_flut_split_f32 unchanged.
 * artemis_asset_decode_rig (host) decodes the rig block (assetio.py:158-202):
 * called first with parents == NULL it validates and sizes (n_joints, k_max,
 * name_bytes); called again with rig->k_max set and arrays of those sizes --
 * parents (J), bind (J, 7) {qw, qx, qy, qz, tx, ty, tz}, names (name_bytes)
 * with name_offsets (J + 1), joint_idx (count, k_max) int32 (-1 pad),
 * weights (count, k_max) fp64 (0 pad) -- it fills them. Also checks the rig
 * offset and trailing bytes (assetio.py:124-131). */
typedef struct {
    uint32_t version, resolution;
    int64_t count;
    int32_t degree, channels, width;
    double lo[3], hi[3];
    int64_t rig_offset, leaf_offset, flut_offset, flut_end;
} artemis_asset_info;

typedef struct {
    int32_t n_joints, k_max;
    int64_t name_bytes, end;
} artemis_asset_rig;

int artemis_asset_probe(const uint8_t *data /* host */, size_t size, artemis_asset_info *info);
int artemis_asset_decode_leaves(const uint8_t *leaf_table, int64_t count, int32_t *cells,
                                void *workspace, size_t workspace_bytes, int32_t *bad_flag,
                                artemis_stream stream);
int artemis_asset_decode_rig(const uint8_t *data /* host */, size_t size,
                             const artemis_asset_info *info, artemis_asset_rig *rig,
                             int32_t *parents, double *bind, char *names, int32_t *name_offsets,
                             int32_t *joint_idx, double *weights);

/* ---- Post-render frame-buffer step --------
 * On a device-resident frame: F (n_pix, C) fp32, alpha/depth (n_pix) float
 * (maps64 = 0) or double (maps64 = 1). Outputs fp64 (or uint8), row-major
 * pixels; fp64 arithmetic in the reference's order (bit-equal to numpy on
 * the same inputs).
 * over_background: out = F + (1 - alpha) * color[c]   (render.py:98-104)
 * composite: depth <= bg_depth ? F + (1 - alpha) * bg : bg (render.py:366-382)
 * straight_rgba (C = 3): (clip(F / alpha, 0, 1) where alpha > 0 else 0,
 *   alpha) as (n_pix, 4) fp64                      (assetio.py:265-275)
 * rgba8 (C = 3): straight_rgba quantised as save_png / encode_png do,
 *   clip(round_half_even(v * 255), 0, 255) -> (n_pix, 4) uint8
 *                                                    (assetio.py:209-245) */
int artemis_over_background(const float *F, const void *alpha, int maps64, int64_t n_pix,
                            int channels, const double *color, double *out,
                            artemis_stream stream);
int artemis_composite(const float *F, const void *alpha, const void *depth, int maps64,
                      int64_t n_pix, int channels, const double *bg_color,
                      const double *bg_depth, double *out, artemis_stream stream);
int artemis_straight_rgba(const float *F, const void *alpha, int maps64, int64_t n_pix,
                          double *rgba, artemis_stream stream);
int artemis_rgba8(const float *F, const void *alpha, int maps64, int64_t n_pix, uint8_t *rgba8,
                  artemis_stream stream);

/* ---- Sparse frame read-out (end-to-end host delivery) -----------------
 * artemis_frame_compact (device, async): the pixels of a frame with
 * alpha > 0 or finite depth, in pixel order, as records of C + 3 32-bit
 * words {pixel index, F[0..C), alpha, depth} (fp32), into `records`
 * (capacity n_pix records) and the record count into *count (device int64);
 * workspace >= artemis_compact_workspace_bytes(n_pix).
 * artemis_host_expand (host, synchronous): rebuild the dense fp32 maps from
 * `count` records: the `prev_count` pixels listed in prev_pixels (the
 * buffer's previous frame) are reset to F = 0, alpha = 0, depth = +inf,
 * then the records are written; the new pixel list goes to pixels_out.
 * `threads` host threads. The dense maps equal the frame's own bit for bit. */
size_t artemis_compact_workspace_bytes(int64_t n_pix);
int artemis_frame_compact(const float *F, const void *alpha, const void *depth, int maps64,
                          int64_t n_pix, int channels, void *records, int64_t *count,
                          void *workspace, size_t workspace_bytes, artemis_stream stream);
int artemis_host_expand(const void *records /* host */, int64_t count, int channels,
                        const uint32_t *prev_pixels, int64_t prev_count, float *F, float *alpha,
                        float *depth, uint32_t *pixels_out, int threads);

/* artemis_frame_bbox (device, async): bounding box of the covered pixels
 * (alpha > 0 or finite depth) as int32 {x0, y0, x1, y1}, inclusive, into
 * device memory; empty frame -> x1 = y1 = -1.
 * artemis_copy_rect_d2h: copy the rectangle of rows [y0, y0 + rows) and
 * bytes [x_bytes, x_bytes + width_bytes) of a row-major device image with
 * row pitch row_pitch bytes into the same place of a (pinned) host image of
 * the same layout, on the copy engine (cudaMemcpy2DAsync). With the union
 * of two consecutive frames' boxes this refreshes a persistent dense host
 * frame exactly: outside the union both frames are (0, 0, +inf). */
int artemis_frame_bbox(const void *alpha, const void *depth, int maps64, int width, int height,
                       int32_t *box, artemis_stream stream);
int artemis_copy_rect_d2h(void *dst_host, const void *src_dev, size_t row_pitch, size_t x_bytes,
                          size_t width_bytes, int64_t y0, int64_t rows, artemis_stream stream);
/* The same for several views of one size (multi-view / stereo frames):
 * artemis_views_bbox writes every view's box (device n_views x 4; alpha and
 * depth are HOST arrays of n_views device pointers); artemis_views_copy_union_d2h
 * refreshes n_views dense host frames from those boxes (host n_views x 4)
 * united with each host buffer's previous box (prev, host, updated), dev/host
 * being n_views x 3 pointer arrays {F, alpha, depth}; *bytes = bytes moved. */
int artemis_views_bbox(const void *const *alpha, const void *const *depth, int n_views,
                       int maps64, int width, int height, int32_t *boxes, artemis_stream stream);
int artemis_views_copy_union_d2h(int n_views, const int32_t *boxes, int32_t *prev,
                                 const void *const *dev, void *const *host, int width,
                                 int height, int channels, int maps64, int64_t *bytes,
                                 artemis_stream stream);

/* ---- Multi-GPU tile shards ----------------------
 * With tile sharding (artemis_camera tile_start/tile_stride) each rank packs
 * the pixels of its 8x4 tiles into one contiguous shard -- tile-major, 32
 * pixels per tile in tile-row order, (C + 2) floats per pixel: F[0..C),
 * alpha, depth -- so a single gather moves only rendered pixels; the root
 * unpacks every rank's shard into the full image. Replaces nothing in the
 * reference (its render is single-process, render.py:322-363); the
 * assembled image equals a single-GPU render bit for bit. */
int64_t artemis_tiles_shard_floats(int width, int height, int channels, int tile_start,
                                   int tile_stride);
int artemis_tiles_pack(const float *F, const float *alpha, const float *depth, int width,
                       int height, int channels, int tile_start, int tile_stride, float *packed,
                       artemis_stream stream);
int artemis_tiles_unpack(const float *packed, int width, int height, int channels,
                         int tile_start, int tile_stride, float *F, float *alpha, float *depth,
                         artemis_stream stream);

/* artemis_host_checksum (host, synchronous): 128-bit content digest of a
 * HOST buffer (every byte; 64 KB blocks over up to `threads` host threads,
 * combined in block order so the digest is thread-count independent) into
 * out[2]. No reference counterpart: the reference re-reads its numpy
 * arguments on every kernels.* call (_core.pyx:473-559, 562-655); the
 * kernel-contract shim keys its device copies of the FLUT and tree by this
 * digest so repeated calls (render.py:209-231 integrate_ray, fit.py:474-480)
 * skip the upload while an in-place edit still takes effect. */
int artemis_host_checksum(const void *data /* host */, size_t bytes, int threads,
                          uint64_t *out /* host, 2 words */);

/* Test hook (no reference counterpart): cap the persistent render grid at
 * max_blocks CTAs (0 = automatic). The maps must not depend on it -- the
 * race/determinism tests vary it to change the ray-to-warp schedule. */
int artemis_debug_set_render_blocks(int max_blocks);

/* Test hook (no reference counterpart): force the render launches' "FLUT is
 * L2-resident" decision (-1 = automatic by FLUT size vs L2, 0 = not resident:
 * L2 row prefetch and the phase-C member-count ranking, 1 = resident: no
 * prefetch, row groups split into items of <= 2 members). The maps must not
 * depend on it. */
int artemis_debug_set_flut_l2_resident(int mode);

/* artemis_host_pose_tables (host, synchronous): forward kinematics of a
 * wrapped pose and the per-joint delta tables the warp kernel and the
 * renderer need -- replaces the numpy body of rigging.py:228-247
 * (forward_kinematics) and :343-347 (posed * canonical^-1 per joint), with
 * the same doubles (the reference's numpy operation order, including the
 * FMA chains of the ddot / dgemv kernels numpy dispatches its norm and
 * 3x3 @ 3 products to). parents (J) parents-first, -1 = root; bind_q (J,4)
 * bind_t (J,3) the bind locals; euler (J,3) wrapped XYZ Euler angles;
 * global_q (4) global_t (3) the pose's global transform; canon_q (J,4)
 * canon_t (J,3) the canonical (zero-pose) globals. Out: delta_mats (J,4,4),
 * delta_quats (J,4), rot_inv (J,3,3). ARTEMIS_ERR_ARG for J outside
 * [1, 256], a parent out of order or a zero quaternion on the way. */
int artemis_host_pose_tables(int n_joints, const int32_t *parents, const double *bind_q,
                             const double *bind_t, const double *euler, const double *global_q,
                             const double *global_t, const double *canon_q,
                             const double *canon_t, double *delta_mats, double *delta_quats,
                             double *rot_inv);

/* artemis_host_widen_f32 (host, synchronous): dst[r][c] = (double)src[r][c]
 * for a rows x cols block (row pitches in elements) on up to `threads` host
 * threads -- the fp32 -> fp64 step of the per-frame API's FrameBuffers
 * (the reference's features are float64, render.py:359-363). */
int artemis_host_widen_f32(const float *src /* host */, int64_t rows, int64_t cols,
                           int64_t src_pitch, double *dst /* host */, int64_t dst_pitch,
                           int threads);

/* Test hook (no reference counterpart): n samples of the cell walk's
 * reciprocal-corrected division against __ddiv_rn; the number of results
 * that differ in any bit goes to *mismatches_host (must be 0). */
int artemis_debug_division_selftest(int64_t n, uint64_t seed,
                                    unsigned long long *mismatches_host,
                                    double *failed_host /* host, 48 doubles: first 16
                                                           failures (regime, n, d); may be NULL */);

/* Synchronous device -> host copy (parity helpers). */
int artemis_copy_to_host(void *dst_host, const void *src_dev, size_t bytes, artemis_stream stream);

/* Number of kernel launches one artemis_frame_run enqueues (bench). */
int artemis_frame_launches(artemis_frame frame);

#ifdef __cplusplus
}
#endif
#endif /* ARTEMIS_H */
