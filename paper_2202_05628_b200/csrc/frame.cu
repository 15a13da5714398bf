// Device-resident frame pipeline: warp -> stable sort -> resolve -> Karras
// build -> render, enqueued as one stream-ordered sequence and (optionally)
// captured once into a CUDA graph that every later frame replays.
//
// Replaces one call of animvox/render.py:284-319 (timed_render_frame):
//   warp_voxels          rigging.py:327-397    -> lbs_warp_kernel (keys, rotation joint)
//   resolve_collisions   rigging.py:419-459    -> onesweep sort + resolve kernels
//   build_octree         volume.py:212-261     -> build_tree_kernel (+ packed nodes)
//   render_view          render.py:322-363     -> render_kernel, camera rays in-kernel
// The in-bounds and live counts never leave the device: every kernel after
// the warp sizes its grid for the worst case and reads the count.
// Per-frame inputs (joint deltas, inverse rotations, cameras, tile-order
// flag) are copied into a device parameter block before the graph launch,
// so the graph itself is pose- and camera-independent. A side stream clears
// the outputs and builds the occupancy brick map while the main stream runs
// the rebuild; several views of one pose render in one launch
// (artemis_frame_run_views).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "bricks.cuh"
#include "common.cuh"
#include "render_common.cuh"
#include "tree.cuh"

namespace artemis {

int warp_pipeline(const int32_t *cells, int64_t n, int slots, const int32_t *jidx,
                  const double *w, const double *aff, int n_joints, const double lo[3],
                  const double cell[3], int res, int key_bytes, void *keys, uint32_t *vals,
                  int32_t *rot_joint, int32_t *n_in, uint64_t sentinel, int identity,
                  uint32_t *bmask, uint32_t *bocc, cudaStream_t st);
int counting_rebuild(const uint32_t *keys, int64_t n, uint32_t sentinel, const double *sigma,
                     uint32_t *bocc, uint32_t *bmask, int64_t n_words, uint32_t *wtmp,
                     BrickRec *recs, int32_t *table, const int dims[3], int32_t *aabb,
                     uint32_t *live_codes, unsigned long long *wmax,
                     int32_t *n_live, int32_t *n_recs, cudaStream_t st, int *launches);
int counting_prepare(int32_t *counters, int n_counters, int32_t *table, const int dims[3],
                     int32_t *aabb, cudaStream_t st);
int counting_finish(const int32_t *n_live, int64_t n_cap, unsigned long long *wmax,
                    uint32_t *winners, const uint32_t *codes, uint4 *leaves, const double *sigma,
                    const int32_t *rot_index, cudaStream_t st);
int render_camera(const artemis_tree_view *tree, const artemis_shading *shade,
                  const artemis_camera *cam_dev, int width, int height, int sharded,
                  double lambda_th, double sigma_dep, int early_stop, int maps64, float *F,
                  void *A, void *D, unsigned long long *queue, const int32_t *tile_order,
                  const int32_t *order_on, void *const *peer_out, int n_views,
                  float *const *Fv, void *const *Av, void *const *Dv, int64_t flut_rows,
                  int outputs_ready, int fast_div, const int32_t *view_shift, cudaStream_t st);
int render_clear_outputs(float *F, void *A, void *D, int64_t n, int channels, int sharded,
                         int maps64, cudaStream_t st);

// per-view outputs of a multi-view frame (artemis_frame_run_views)
struct ViewOut {
    int n = 1;
    float *F[kMaxViews] = {};
    void *A[kMaxViews] = {};
    void *D[kMaxViews] = {};
};

constexpr int kMaxFrameJoints = 256;

struct FrameParams {
    artemis_camera cam[kMaxViews];  // the frame's views (one unless artemis_frame_run_views)
    int32_t order_on;  // render the ray tiles in the size's centre-out order (else row-major)
    int32_t pad;
    // per view: x shift (in 8-pixel tiles) of the view's tile order, so the
    // views of one launch render the same part of the character at the same
    // time (stereo eyes: the disparity of the grid centre) -- rows shared in L2
    int32_t view_shift[kMaxViews];
    double aff[kMaxFrameJoints * 12];
    double rot_inv[kMaxFrameJoints * 9];
};

}  // namespace artemis

using namespace artemis;

struct artemis_frame_s {
    artemis_asset asset;
    int64_t n;
    int key_bytes, key_bits;
    uint64_t sentinel;
    double lo[3], cell[3];
    void *keys = nullptr, *keys_sorted = nullptr, *live_codes = nullptr;
    uint32_t *vals = nullptr, *vals_sorted = nullptr, *winners = nullptr;
    int32_t *rot_joint = nullptr, *counters = nullptr;
    int32_t *left = nullptr, *right = nullptr, *bmin = nullptr, *bsize = nullptr;
    WideNode *nodes = nullptr;
    uint4 *leaves = nullptr;
    // occupancy brick map (exact cell walk)
    int32_t *btable = nullptr, *bmeta = nullptr;
    BrickRec *brecs = nullptr;
    int bdims[3] = {1, 1, 1};
    artemis_brickmap bmap{};
    // counting rebuild (rebuild.cu) for grids <= 1024^3: dense per-brick cell
    // masks + brick bitmap (both kept zero between frames), per-word counts,
    // per-live-cell density keys
    int counting = 0;
    int karras_tail = 0;  // counting: Karras tree arrays built beside the render (ARTEMIS_KARRAS_TAIL)
    uint32_t *bmask = nullptr, *bocc = nullptr, *wtmp = nullptr;
    int64_t n_words = 0;
    // per live slot: 128-bit max of (density key, ~index), kept reset between frames
    unsigned long long *wkey = nullptr;
    void *sort_ws = nullptr, *resolve_ws = nullptr;
    size_t sort_ws_bytes = 0, resolve_ws_bytes = 0;
    FrameParams *params = nullptr;
    // pinned host staging for the per-frame inputs (a ring, so a frame's
    // H2D copy never races the host filling the next frame's block)
    static constexpr int kStaging = 4;
    FrameParams *staging = nullptr;
    cudaEvent_t staged[kStaging] = {nullptr, nullptr, nullptr, nullptr};
    int stage_next = 0;
    // captured graphs and the launch shape each was captured for: a few are
    // kept so callers can rotate output buffers (double-buffered D2H)
    // without re-capturing
    struct GraphSlot {
        cudaGraphExec_t exec = nullptr;
        int w = 0, h = 0, flags = 0, identity = -1, nj = 0, sharded = 0, fast_div = -1;
        const void *F = nullptr, *A = nullptr, *D = nullptr;
        cudaStream_t stream = nullptr;
        double lambda = 0, sigma_dep = 0;
        ViewOut views;
        unsigned long long used = 0;
    };
    static constexpr int kGraphSlots = 4;
    GraphSlot graphs[kGraphSlots];
    // render order of the 8x4 tiles per image size (see order_slot); a few
    // sizes cached, like the graphs
    struct OrderSlot {
        int w = 0, h = 0;
        int32_t *dev = nullptr;
        int mode = 0;  // 0 row-major, 1 the order in dev (centre-out or set_tile_order)
        unsigned long long used = 0;
    };
    OrderSlot orders[kGraphSlots];

    unsigned long long graph_clock = 0;
    int launches = 0;
    // stage profiling (eager runs only): events before warp, sort, resolve,
    // build, render and after render
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    // FLUT coefficients within 16x L2: centre-out tile order, several views
    // per render launch (order_slot, enqueue_frame); row-major and one launch
    // per view beyond
    int small_flut = 1;
    // second stream of the frame (output clearing, brick map) and its
    // fork / mid / join events
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_mid = nullptr, ev_join = nullptr, ev_tail = nullptr;
    // tile-sharded frames written straight into another rank's full-frame
    // F / alpha / depth (peer memory over NVLink): artemis_frame_set_output_peer
    void *peer_out[3] = {nullptr, nullptr, nullptr};
    int64_t peer_pixels = 0;  // size of the peer maps (pixels) and their alpha/depth type
    int peer_maps64 = 0;
    int fast_div = 0;  // this run's cameras are in div_fast's operand ranges
    int profile = 0;
};

namespace {

template <typename T>
int dev_alloc(T **p, size_t bytes) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), bytes ? bytes : 1);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return ARTEMIS_ERR_OOM;
    }
    return ARTEMIS_OK;
}

// The occupancy brick map, on the side stream once the live codes exist.
int bricks_on_side(artemis_frame f, cudaStream_t st) {
    ARTEMIS_TRY(cudaEventRecord(f->ev_mid, st));
    ARTEMIS_TRY(cudaStreamWaitEvent(f->side, f->ev_mid, 0));
    const int org[3] = {0, 0, 0};
    int rc = f->key_bytes == 4
                 ? build_bricks<uint32_t>((const uint32_t *)f->live_codes, 0, f->counters + 1,
                                          f->n, org, f->bdims, f->btable, f->brecs, f->bmeta,
                                          f->bmeta + 1, f->side)
                 : build_bricks<u64>((const u64 *)f->live_codes, 0, f->counters + 1, f->n, org,
                                     f->bdims, f->btable, f->brecs, f->bmeta, f->bmeta + 1,
                                     f->side);
    if (rc) return rc;
    ARTEMIS_TRY(cudaEventRecord(f->ev_join, f->side));
    return ARTEMIS_OK;
}

// NVTX ranges around the stages a frame enqueues (warp, sort, resolve,
// build, render): host-side ranges, so in eager runs they bracket each
// stage's launches on an nsys/ncu timeline; a graph replay shows one range
// per capture. No-ops without a tool attached.
struct NvtxStages {
    bool open = false;
    void next(int k) {
        static const char *names[5] = {"artemis warp", "artemis sort", "artemis resolve",
                                       "artemis build", "artemis render"};
        close();
        if (k < 5) {
            nvtxRangePushA(names[k]);
            open = true;
        }
    }
    void close() {
        if (open) nvtxRangePop();
        open = false;
    }
    ~NvtxStages() { close(); }
};

int enqueue_frame(artemis_frame f, int identity, int n_joints, int width, int height,
                  int sharded, double lambda_th, double sigma_dep, int flags, float *F, void *A,
                  void *D, const int32_t *order, const ViewOut &vo, cudaStream_t st) {
    const artemis_asset &as = f->asset;
    int rc;
    int launches = 0;
    bool tail_join = false;  // the Karras build runs beside the render (karras_tail)
    const bool prof = f->profile && !(flags & 2);
    NvtxStages nvtx;
    auto mark = [&](int k) {
        if (prof) cudaEventRecord(f->ev[k], st);
        nvtx.next(k);
    };
    mark(0);
    if (flags & 16) {  // ARTEMIS_FRAME_REUSE_TREE: another view of the last posed tree
        ARTEMIS_TRY(cudaMemsetAsync(f->counters + 2, 0, 2 * sizeof(int32_t), st));
        for (int k = 1; k <= 4; ++k) mark(k);
        artemis_tree_view tv{f->nodes, f->leaves, 0, f->counters + 1, (double)as.resolution,
                             &f->bmap};
        artemis_shading sh{as.coef, as.sigma, f->rot_joint, f->params->rot_inv, as.degree,
                           as.channels, 0};
        rc = render_camera(&tv, &sh, f->params->cam, width, height, sharded, lambda_th,
                           sigma_dep, flags & 1, (flags & 8) ? 1 : 0, F, A, D,
                           reinterpret_cast<unsigned long long *>(f->counters + 2), order,
                           &f->params->order_on, sharded ? f->peer_out : nullptr, vo.n, vo.F, vo.A,
                           vo.D, f->n, 0, f->fast_div, f->params->view_shift, st);
        mark(5);
        f->launches = 1;
        return rc;
    }
    // counters: [0] in-bounds, [1] live leaves, [2..3] render ray queue (u64);
    // reset with the brick table and AABB in one kernel (counting) below
    if (!f->counting) ARTEMIS_TRY(cudaMemsetAsync(f->counters, 0, 4 * sizeof(int32_t), st));
    // side stream: the outputs are cleared while the rebuild runs, and the
    // brick map is built beside the Karras tree (both only read the live
    // codes); joined before the render
    ARTEMIS_TRY(cudaEventRecord(f->ev_fork, st));
    ARTEMIS_TRY(cudaStreamWaitEvent(f->side, f->ev_fork, 0));
    {
        const int64_t px = (int64_t)width * height;
        const bool peer = sharded && f->peer_out[0];
        for (int v = 0; v < vo.n && !peer; ++v) {
            rc = render_clear_outputs(vo.n > 1 ? vo.F[v] : F, vo.n > 1 ? vo.A[v] : A,
                                      vo.n > 1 ? vo.D[v] : D, px, as.channels,
                                      vo.n > 1 ? 0 : sharded, (flags & 8) ? 1 : 0, f->side);
            if (rc) return rc;
        }
    }
    if (f->counting) {
        rc = counting_prepare(f->counters, 4, f->btable, f->bdims, f->bmeta + 1, st);
        if (rc) return rc;
        launches += 1;  // frame_prepare_kernel
    }
    rc = warp_pipeline(as.cells, f->n, as.slots, as.joint_idx, as.weights, f->params->aff,
                       identity ? 1 : n_joints, f->lo, f->cell, as.resolution, f->key_bytes,
                       f->keys, f->vals, f->rot_joint, f->counters, f->sentinel, identity,
                       f->counting ? f->bmask : nullptr, f->counting ? f->bocc : nullptr, st);
    if (rc) return rc;
    launches += 1;
    mark(1);
    if (f->counting) {
        // counting rebuild: Morton order and collision winners without a
        // sort (rebuild.cu), the brick map in the same passes
        rc = counting_rebuild((const uint32_t *)f->keys, f->n, (uint32_t)f->sentinel, as.sigma,
                              f->bocc, f->bmask, f->n_words, f->wtmp, f->brecs, f->btable,
                              f->bdims, f->bmeta + 1, (uint32_t *)f->live_codes,
                              f->wkey, f->counters + 1, f->bmeta, st, &launches);
        if (rc) return rc;
        mark(2);
        if (f->karras_tail) {
            // the leaf records come out of the finish pass, so the render
            // needs nothing from the Karras build: the tree arrays (the
            // rebuild stage's reference-layout output, volume.build_octree)
            // are built on the side stream after the output clears, launched
            // behind the render (which carries the higher launch priority) --
            // their blocks fill the SMs the render's tail releases; the frame
            // joins them after the render
            rc = counting_finish(f->counters + 1, f->n, f->wkey, f->winners,
                                 (const uint32_t *)f->live_codes, f->leaves, as.sigma,
                                 f->rot_joint, st);
            if (rc) return rc;
            mark(3);
            ARTEMIS_TRY(cudaEventRecord(f->ev_join, f->side));  // the clears
            ARTEMIS_TRY(cudaStreamWaitEvent(st, f->ev_join, 0));
            ARTEMIS_TRY(cudaEventRecord(f->ev_mid, st));
            ARTEMIS_TRY(cudaStreamWaitEvent(f->side, f->ev_mid, 0));
            rc = launch_build_tree<uint32_t>((const uint32_t *)f->live_codes, 0, f->counters + 1,
                                             f->n, f->left, f->right, f->bmin, f->bsize, nullptr,
                                             nullptr, nullptr, nullptr, nullptr, nullptr,
                                             f->side);
            if (rc) return rc;
            ARTEMIS_TRY(cudaEventRecord(f->ev_tail, f->side));
            tail_join = true;
        } else {
            rc = counting_finish(f->counters + 1, f->n, f->wkey, f->winners, nullptr, nullptr, nullptr,
                                 nullptr, st);
            if (rc) return rc;
            mark(3);
            rc = launch_build_tree<uint32_t>((const uint32_t *)f->live_codes, 0, f->counters + 1,
                                             f->n, f->left, f->right, f->bmin, f->bsize, nullptr,
                                             f->leaves, f->winners, as.sigma, f->rot_joint,
                                             nullptr, st);
            if (rc) return rc;
            // the side stream only cleared the outputs: join it before the render
            ARTEMIS_TRY(cudaEventRecord(f->ev_join, f->side));
            ARTEMIS_TRY(cudaStreamWaitEvent(st, f->ev_join, 0));
        }
        launches += 2;  // finish, the Karras build (count/scan/emit/slot counted above)
    } else {
    // the Karras tree arrays (reference layout) are rebuilt every frame: they
    // are the rebuild stage's output (volume.build_octree) even though the
    // renderer walks the brick map
    const bool write_ref = true;
    (void)flags;
    if (f->key_bytes == 4) {
        rc = sort_pairs<uint32_t>((const uint32_t *)f->keys, f->vals, (uint32_t *)f->keys_sorted,
                                  f->vals_sorted, f->n, f->key_bits, f->sort_ws, f->sort_ws_bytes,
                                  st);
        if (rc) return rc;
        mark(2);
        rc = resolve<uint32_t>((const uint32_t *)f->keys_sorted, f->vals_sorted, f->n,
                               f->counters, as.sigma, (uint32_t *)f->live_codes, f->winners,
                               nullptr, f->counters + 1, f->resolve_ws, f->resolve_ws_bytes, st);
        if (rc) return rc;
        mark(3);
        rc = bricks_on_side(f, st);
        if (rc) return rc;
        rc = launch_build_tree<uint32_t>((const uint32_t *)f->live_codes, 0, f->counters + 1,
                                         f->n, write_ref ? f->left : nullptr, f->right, f->bmin,
                                         f->bsize, nullptr, f->leaves, f->winners, as.sigma,
                                         f->rot_joint, nullptr, st);
    } else {
        rc = sort_pairs<u64>((const u64 *)f->keys, f->vals, (u64 *)f->keys_sorted, f->vals_sorted,
                             f->n, f->key_bits, f->sort_ws, f->sort_ws_bytes, st);
        if (rc) return rc;
        mark(2);
        rc = resolve<u64>((const u64 *)f->keys_sorted, f->vals_sorted, f->n, f->counters,
                          as.sigma, (u64 *)f->live_codes, f->winners, nullptr, f->counters + 1,
                          f->resolve_ws, f->resolve_ws_bytes, st);
        if (rc) return rc;
        mark(3);
        rc = bricks_on_side(f, st);
        if (rc) return rc;
        rc = launch_build_tree<u64>((const u64 *)f->live_codes, 0, f->counters + 1, f->n,
                                    write_ref ? f->left : nullptr, f->right, f->bmin, f->bsize,
                                    nullptr, f->leaves, f->winners, as.sigma, f->rot_joint,
                                    nullptr, st);
    }
    if (rc) return rc;
    ARTEMIS_TRY(cudaStreamWaitEvent(st, f->ev_join, 0));
    launches += 2;  // the brick passes (side stream)
    const int passes = f->key_bits <= 0 ? 1 : (f->key_bits + 7) / 8;
    launches += 2 + passes + 3 + 1;  // + 2 brick passes counted above
    }
    mark(4);
    artemis_tree_view tv{f->nodes, f->leaves, 0, f->counters + 1, (double)as.resolution, &f->bmap};
    artemis_shading sh{as.coef, as.sigma, f->rot_joint, f->params->rot_inv, as.degree,
                       as.channels, 0};
    // ahead of the Karras build on the side stream, if it runs there
    PriorityScope prio(tail_join && !getenv("ARTEMIS_NO_RENDER_PRIO"));
    // big FLUT: views rendered together thrash L2 (configs[4] stereo, unaligned:
    // 8.86 vs 8.27 ms) -- except a stereo pair aligned by disparity (8.14 ms)
    if (vo.n > 2 && !f->small_flut) {
        // big FLUT: the views' rows would not stay in L2 together (configs[4]
        // stereo: one launch 10.4 ms vs 9.6 ms for two), so one launch per view
        for (int v = 0; v < vo.n && !rc; ++v) {
            if (v) ARTEMIS_TRY(cudaMemsetAsync(f->counters + 2, 0, 2 * sizeof(int32_t), st));
            rc = render_camera(&tv, &sh, f->params->cam + v, width, height, 0, lambda_th,
                               sigma_dep, flags & 1, (flags & 8) ? 1 : 0, vo.F[v], vo.A[v],
                               vo.D[v], reinterpret_cast<unsigned long long *>(f->counters + 2),
                               order, &f->params->order_on, nullptr, 1, nullptr, nullptr, nullptr,
                               f->n, 1, f->fast_div, nullptr, st);
        }
        launches += vo.n - 1;
    } else {
        rc = render_camera(&tv, &sh, f->params->cam, width, height, sharded, lambda_th, sigma_dep,
                           flags & 1, (flags & 8) ? 1 : 0, F, A, D,
                           reinterpret_cast<unsigned long long *>(f->counters + 2), order,
                           &f->params->order_on, sharded ? f->peer_out : nullptr, vo.n, vo.F, vo.A,
                           vo.D, f->n, 1, f->fast_div, f->params->view_shift, st);
    }
    if (tail_join) ARTEMIS_TRY(cudaStreamWaitEvent(st, f->ev_tail, 0));
    mark(5);
    launches += 1;
    f->launches = launches;
    return rc;
}

}  // namespace

namespace {
bool same_views(const ViewOut &a, const ViewOut &b) {
    if (a.n != b.n) return false;
    for (int v = 0; v < a.n && a.n > 1; ++v)
        if (a.F[v] != b.F[v] || a.A[v] != b.A[v] || a.D[v] != b.D[v]) return false;
    return true;
}

// Render order of an image's 8x4 ray tiles: row-major, or centre-out (by
// distance of the tile centre from the image centre, ties row-major), which
// starts a framed character's expensive middle first so the cheap border
// fills the tail. Measured (same box, graph replay, L2 flushed): centre-out
// takes configs[2]/[3] 1.78 -> 1.72 ms and configs[1] 2.25 -> 2.19 ms, but
// configs[4] -- a 4.6 GB FLUT over 2.3 M-pixel eyes, whose in-flight rows
// already overflow L2 (DRAM reads 2x the rows touched) -- 9.5 -> 10.9 ms:
// a ring-shaped front of in-flight tiles re-reads more rows than a band.
// So centre-out is used while the FLUT coefficients fit in 16x L2 (1.1 GB
// at configs[2], 4.6 GB at configs[4]; ARTEMIS_TILE_ORDER=rowmajor|centre
// overrides, artemis_frame_set_tile_order installs any permutation).
// Per-frame trials of both orders were tried and rejected: frame-to-frame
// and view-to-view variation swamps a 3 % difference. Any order gives the
// same maps bit for bit: each ray is independent and its own sums keep hit
// order. Cached per image size next to the graphs that capture it; the
// choice travels in the parameter block, so one graph serves both.
artemis_frame_s::OrderSlot *order_slot(artemis_frame f, int w, int h, int *rc) {
    *rc = ARTEMIS_OK;
    artemis_frame_s::OrderSlot *slot = nullptr, *victim = &f->orders[0];
    for (auto &o : f->orders) {
        if (o.dev && o.w == w && o.h == h) {
            slot = &o;
            break;
        }
        if (!o.dev || (victim->dev && o.used < victim->used)) victim = &o;
    }
    if (!slot) {
        slot = victim;
        if (slot->dev) {  // graphs captured for that size read the old buffer
            for (auto &g : f->graphs)
                if (g.exec && g.w == slot->w && g.h == slot->h) {
                    cudaGraphExecDestroy(g.exec);
                    g.exec = nullptr;
                }
            cudaFree(slot->dev);
            slot->dev = nullptr;
        }
        const int tx = (w + 7) / 8, ty = (h + 3) / 4;
        const int64_t n = (int64_t)tx * ty;
        std::vector<int32_t> idx((size_t)n);
        std::vector<double> key((size_t)n);
        std::iota(idx.begin(), idx.end(), 0);
        for (int64_t t = 0; t < n; ++t) {
            const double dx = (double)(t % tx) * 8.0 + 4.0 - 0.5 * w;
            const double dy = (double)(t / tx) * 4.0 + 2.0 - 0.5 * h;
            key[(size_t)t] = dx * dx + dy * dy;
        }
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int32_t a, int32_t b) { return key[(size_t)a] < key[(size_t)b]; });
        *rc = dev_alloc(&slot->dev, (size_t)n * sizeof(int32_t));
        if (*rc) return nullptr;
        if (cudaMemcpy(slot->dev, idx.data(), (size_t)n * sizeof(int32_t),
                       cudaMemcpyHostToDevice) != cudaSuccess) {
            *rc = ARTEMIS_ERR_CUDA;
            return nullptr;
        }
        slot->w = w;
        slot->h = h;
        slot->mode = f->small_flut ? 1 : 0;
        const char *e = getenv("ARTEMIS_TILE_ORDER");  // "rowmajor" / "centre" force one
        if (e && !strcmp(e, "rowmajor")) slot->mode = 0;
        if (e && !strcmp(e, "centre")) slot->mode = 1;
    }
    slot->used = ++f->graph_clock;
    return slot;
}
}  // namespace

// Tile-sharded frames of this handle write their pixels into (F, alpha,
// depth) -- another rank's full-frame buffers mapped into this process
// (CUDA IPC; peer access over NVLink) or this rank's own -- instead of the
// local outputs, which then stay untouched. The owner initialises the maps
// (F 0, alpha 0, depth +inf) before any rank renders; every rank writes only
// its own tiles, so the assembled frame needs no gather. NULLs restore the
// local outputs. Captured graphs are dropped (they bake the pointers).
extern "C" int artemis_frame_set_output_peer(artemis_frame f, float *F, void *alpha, void *depth,
                                             int64_t n_pixels, int maps64) {
    if (!f || (F && (!alpha || !depth || n_pixels < 1))) return ARTEMIS_ERR_ARG;
    for (auto &g : f->graphs)
        if (g.exec) {
            cudaGraphExecDestroy(g.exec);
            g.exec = nullptr;
        }
    f->peer_out[0] = F;
    f->peer_out[1] = F ? alpha : nullptr;
    f->peer_out[2] = F ? depth : nullptr;
    f->peer_pixels = F ? n_pixels : 0;
    f->peer_maps64 = F ? (maps64 ? 1 : 0) : 0;
    return ARTEMIS_OK;
}

// Install a caller-supplied render order (a permutation of the w x h image's
// 8x4 tiles, host array) for that image size; graphs captured for the size
// are dropped.
extern "C" int artemis_frame_set_tile_order(artemis_frame f, int w, int h, const int32_t *order) {
    if (!f || w < 1 || h < 1 || !order) return ARTEMIS_ERR_ARG;
    int rc = ARTEMIS_OK;
    artemis_frame_s::OrderSlot *slot = order_slot(f, w, h, &rc);
    if (!slot) return rc;
    const int32_t *dev = slot->dev;
    slot->mode = 1;
    const int64_t n = (int64_t)((w + 7) / 8) * ((h + 3) / 4);
    std::vector<char> seen((size_t)n, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (order[i] < 0 || order[i] >= n || seen[(size_t)order[i]]) return ARTEMIS_ERR_ARG;
        seen[(size_t)order[i]] = 1;
    }
    for (auto &g : f->graphs)
        if (g.exec && g.w == w && g.h == h) {
            cudaGraphExecDestroy(g.exec);
            g.exec = nullptr;
        }
    ARTEMIS_TRY(cudaMemcpy(const_cast<int32_t *>(dev), order, (size_t)n * sizeof(int32_t),
                           cudaMemcpyHostToDevice));
    return ARTEMIS_OK;
}

extern "C" int artemis_frame_create(const artemis_asset *a, artemis_frame *out) {
    if (!a || !out || a->n_voxels < 1 || a->n_voxels >= (int64_t(1) << 30) || a->slots < 1 ||
        a->max_joints < 1 || a->max_joints > kMaxFrameJoints || a->degree < 0 || a->degree > 4 ||
        a->channels < 1 || a->resolution < 1 || (a->resolution & (a->resolution - 1)) ||
        a->resolution > (1 << 21) || !a->cells || !a->joint_idx || !a->weights || !a->coef ||
        !a->sigma)
        return ARTEMIS_ERR_ARG;
    artemis_frame f = new artemis_frame_s();
    f->asset = *a;
    f->n = a->n_voxels;
    int levels = 0;
    while ((1 << levels) < a->resolution) ++levels;
    f->key_bits = 3 * levels + 1;  // one extra bit for the out-of-bounds sentinel
    f->key_bytes = f->key_bits <= 32 ? 4 : 8;
    f->sentinel = uint64_t(1) << (3 * levels);
    for (int k = 0; k < 3; ++k) {
        f->lo[k] = a->lo[k];
        f->cell[k] = (a->hi[k] - a->lo[k]) / a->resolution;  // Bounds.cell_size (volume.py:45-46)
    }
    const int64_t n = f->n;
    int rc = ARTEMIS_OK;
    {
        int l2 = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        const double flut = (double)n * (a->degree + 1) * (a->degree + 1) * a->channels * 4.0;
        f->small_flut = flut <= 16.0 * (l2 > 0 ? l2 : (126 << 20));
    }
    rc = rc ? rc : dev_alloc(&f->keys, n * f->key_bytes);
    rc = rc ? rc : dev_alloc(&f->keys_sorted, n * f->key_bytes);
    rc = rc ? rc : dev_alloc(&f->live_codes, n * f->key_bytes);
    rc = rc ? rc : dev_alloc(&f->vals, n * 4);
    rc = rc ? rc : dev_alloc(&f->vals_sorted, n * 4);
    rc = rc ? rc : dev_alloc(&f->winners, n * 4);
    rc = rc ? rc : dev_alloc(&f->rot_joint, n * 4);
    if (!rc) {
        cudaError_t e = cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_mid, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_join, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_tail, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            set_cuda_error(e);
            rc = ARTEMIS_ERR_CUDA;
        }
    }
    rc = rc ? rc : dev_alloc(&f->counters, 64);
    if (!rc && cudaMemset(f->counters, 0, 64) != cudaSuccess) rc = ARTEMIS_ERR_CUDA;
    rc = rc ? rc : dev_alloc(&f->left, n * 4);
    rc = rc ? rc : dev_alloc(&f->right, n * 4);
    rc = rc ? rc : dev_alloc(&f->bmin, n * 12);
    rc = rc ? rc : dev_alloc(&f->bsize, n * 12);
    rc = rc ? rc : dev_alloc(&f->nodes, (n + 1) * sizeof(WideNode));
    rc = rc ? rc : dev_alloc(&f->leaves, 2 * (n + 1) * sizeof(uint4));
    for (int k = 0; k < 3; ++k) f->bdims[k] = (a->resolution + 7) / 8;
    rc = rc ? rc : dev_alloc(&f->btable, (size_t)f->bdims[0] * f->bdims[1] * f->bdims[2] * 4);
    rc = rc ? rc : dev_alloc(&f->brecs, (size_t)(n + 1) * sizeof(BrickRec));
    rc = rc ? rc : dev_alloc(&f->bmeta, 64);
    {   // counting rebuild for 32-bit keys (grids <= 1024^3); ARTEMIS_COUNTING=0
        // selects the onesweep sort + resolve path instead (A/B, tests)
        const char *env = getenv("ARTEMIS_COUNTING");
        f->counting = f->key_bytes == 4 && a->resolution <= 1024 && !(env && env[0] == '0');
        const char *kt = getenv("ARTEMIS_KARRAS_TAIL");
        f->karras_tail = f->counting && !(kt && kt[0] == '0');
    }
    if (!rc && f->counting) {
        const int64_t bricks = (int64_t)f->bdims[0] * f->bdims[1] * f->bdims[2];
        f->n_words = (bricks + 31) / 32;
        rc = rc ? rc : dev_alloc(&f->bmask, (size_t)f->n_words * 32 * 16 * 4);
        rc = rc ? rc : dev_alloc(&f->bocc, (size_t)f->n_words * 4);
        rc = rc ? rc : dev_alloc(&f->wtmp, (size_t)f->n_words * (8 + 32 * 4 + 8));
        rc = rc ? rc : dev_alloc(&f->wkey, (size_t)n * 16);
        if (!rc && (cudaMemset(f->bmask, 0, (size_t)f->n_words * 32 * 16 * 4) != cudaSuccess ||
                    cudaMemset(f->bocc, 0, (size_t)f->n_words * 4) != cudaSuccess ||
                    cudaMemset(f->wkey, 0, (size_t)n * 16) != cudaSuccess))
            rc = ARTEMIS_ERR_CUDA;
    }
    if (!rc) {
        f->bmap.table = f->btable;
        f->bmap.recs = f->brecs;
        f->bmap.aabb = f->bmeta + 1;
        for (int k = 0; k < 3; ++k) {
            f->bmap.org[k] = 0;
            f->bmap.dims[k] = f->bdims[k];
        }
    }
    f->sort_ws_bytes = sort_workspace_bytes(n, f->key_bits, f->key_bytes);
    f->resolve_ws_bytes = resolve_workspace_bytes(n);
    rc = rc ? rc : dev_alloc(&f->sort_ws, f->sort_ws_bytes);
    rc = rc ? rc : dev_alloc(&f->resolve_ws, f->resolve_ws_bytes);
    rc = rc ? rc : dev_alloc(&f->params, sizeof(FrameParams));
    if (!rc) {
        cudaError_t e = cudaMallocHost(reinterpret_cast<void **>(&f->staging),
                                       sizeof(FrameParams) * artemis_frame_s::kStaging);
        for (int k = 0; e == cudaSuccess && k < artemis_frame_s::kStaging; ++k)
            e = cudaEventCreateWithFlags(&f->staged[k], cudaEventDisableTiming);
        if (e != cudaSuccess) {
            set_cuda_error(e);
            rc = ARTEMIS_ERR_OOM;
        }
    }
    if (rc) {
        artemis_frame_destroy(f);
        return rc;
    }
    *out = f;
    return ARTEMIS_OK;
}

extern "C" int artemis_frame_destroy(artemis_frame f) {
    if (!f) return ARTEMIS_OK;
    for (auto &g : f->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (cudaEvent_t e : f->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : f->staged)
        if (e) cudaEventDestroy(e);
    if (f->staging) cudaFreeHost(f->staging);
    for (auto &o : f->orders)
        if (o.dev) cudaFree(o.dev);
    for (cudaEvent_t e : {f->ev_fork, f->ev_mid, f->ev_join, f->ev_tail})
        if (e) cudaEventDestroy(e);
    if (f->side) cudaStreamDestroy(f->side);

    void *bufs[] = {f->keys, f->keys_sorted, f->live_codes, f->vals, f->vals_sorted, f->winners,
                    f->rot_joint, f->counters, f->left, f->right, f->bmin, f->bsize, f->nodes,
                    f->leaves, f->btable, f->brecs, f->bmeta,
                    f->sort_ws, f->resolve_ws, f->params, f->bmask, f->bocc, f->wtmp, f->wkey};
    for (void *b : bufs)
        if (b) cudaFree(b);
    delete f;
    return ARTEMIS_OK;
}

static int run_frame_launch(artemis_frame f, int identity, int n_joints, const artemis_camera *cam,
                            int sharded, double lambda_th, double sigma_dep, int flags, float *F,
                            void *alpha, void *depth, const int32_t *order, const ViewOut &vo,
                            cudaStream_t st);

// One posed frame: warp + rebuild once, then one render launch over the
// views cam[0 .. vo.n) (the outputs of view v in vo, or F/alpha/depth for a
// single view).
// Whether every plane crossing and camera-ray division of frames seen
// through this camera stays inside div_fast's exact range (bricks.cuh):
// positive focal lengths in [2^-20, 2^60], principal point, rotation entries
// and grid-space origin each 0 or of magnitude in [2^-300, 2^300] (rotation
// entries at most 2), cell sizes in [2^-60, 2^60]. Then (u + 0.5) - cx is 0
// or >= 2^-353, every ray-direction component is 0 or >= 2^-427 with the
// norm >= 1, |k - og| is 0 or in [2^-353, 2^301] for the grid planes k
// (|k| <= 2^22), grid directions are 0 or in [2^-487, 2^60]: all quotients,
// products and residuals normal. Otherwise the launch takes __ddiv_rn (same
// bits, slower).
// Tile-order shifts that align the views of one multi-view launch: view v's
// tiles are taken shifted by the x offset (in tiles) between the grid
// centre's projection in view v and in view 0. Only the order changes (every
// pixel still rendered once, bit-identical maps).
static void align_views(const artemis_frame_s *f, const artemis_camera *cam, int n,
                        int32_t *shift) {
    double c[3];
    for (int a = 0; a < 3; ++a) c[a] = f->lo[a] + 0.5 * f->cell[a] * f->asset.resolution;
    double x0 = 0.0;
    for (int v = 0; v < kMaxViews; ++v) shift[v] = 0;
    for (int v = 0; v < n; ++v) {
        const artemis_camera &k = cam[v];
        double p[3];
        for (int a = 0; a < 3; ++a)  // camera coordinates: R^T (c - origin)
            p[a] = k.R[a] * (c[0] - k.origin[0]) + k.R[3 + a] * (c[1] - k.origin[1]) +
                   k.R[6 + a] * (c[2] - k.origin[2]);
        if (!(p[2] > 0.0)) return;  // centre behind a camera: no alignment
        const double x = k.fx * p[0] / p[2] + k.cx;
        if (v == 0)
            x0 = x;
        else
            shift[v] = (int32_t)lround((x - x0) / 8.0);
    }
}

static bool in_range_or_zero(double x, double lo, double hi) {
    const double a = fabs(x);
    return x == 0.0 || (a >= lo && a <= hi);
}

static bool camera_fast_div_ok(const artemis_camera &c) {
    const char *env = getenv("ARTEMIS_FAST_DIV");  // "0": always __ddiv_rn (A/B, tests)
    if (env && env[0] == '0') return false;
    if (!(c.fx >= 0x1p-20 && c.fx <= 0x1p60 && c.fy >= 0x1p-20 && c.fy <= 0x1p60)) return false;
    if (!in_range_or_zero(c.cx, 0x1p-300, 0x1p300) || !in_range_or_zero(c.cy, 0x1p-300, 0x1p300))
        return false;
    for (int i = 0; i < 9; ++i)
        if (!in_range_or_zero(c.R[i], 0x1p-300, 2.0)) return false;
    for (int a = 0; a < 3; ++a) {
        if (!(c.cell[a] >= 0x1p-60 && c.cell[a] <= 0x1p60)) return false;
        const double og = (c.origin[a] - c.lo[a]) / c.cell[a];  // = the device's __ddiv_rn value
        if (!in_range_or_zero(og, 0x1p-300, 0x1p300)) return false;
    }
    return true;
}

static int frame_run_impl(artemis_frame f, const double *joint_aff, const double *rot_inv,
                          int n_joints, const artemis_camera *cam, double lambda_th,
                          double sigma_dep, int flags, float *F, void *alpha, void *depth,
                          const ViewOut &vo, artemis_stream stream) {
    if (!f || !cam || !F || !alpha || !depth || cam->width < 1 || cam->height < 1 || vo.n < 1 ||
        vo.n > kMaxViews)
        return ARTEMIS_ERR_ARG;
    for (int v = 1; v < vo.n; ++v)
        if (cam[v].width != cam->width || cam[v].height != cam->height || cam[v].tile_stride > 1)
            return ARTEMIS_ERR_ARG;
    if (vo.n > 1 && cam->tile_stride > 1) return ARTEMIS_ERR_ARG;
    const int identity = joint_aff == nullptr;
    if (!identity && (!rot_inv || n_joints < 1 || n_joints > f->asset.max_joints))
        return ARTEMIS_ERR_ARG;
    cudaStream_t st = S(stream);
    // parameter block: camera + joint tables, staged in pinned host memory and
    // copied host -> device ahead of the graph on the frame's stream
    const int sidx = f->stage_next;
    f->stage_next = (sidx + 1) % artemis_frame_s::kStaging;
    FrameParams *hp = f->staging + sidx;
    ARTEMIS_TRY(cudaEventSynchronize(f->staged[sidx]));  // its last copy has completed
    for (int v = 0; v < vo.n; ++v) hp->cam[v] = cam[v];
    const int nj = identity ? 1 : n_joints;
    if (identity) {
        static const double eye[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        memcpy(hp->rot_inv, eye, sizeof(eye));
    } else {
        memcpy(hp->aff, joint_aff, sizeof(double) * 12 * n_joints);
        memcpy(hp->rot_inv, rot_inv, sizeof(double) * 9 * n_joints);
    }
    const int sharded = cam->tile_stride > 1;
    if (sharded && f->peer_out[0] &&
        ((int64_t)cam->width * cam->height != f->peer_pixels ||
         ((flags & 8) ? 1 : 0) != f->peer_maps64))
        return ARTEMIS_ERR_ARG;  // the peer maps are another image size / map type
    const int32_t *order = nullptr;
    hp->order_on = 0;
    if (!sharded) {
        int rc = ARTEMIS_OK;
        artemis_frame_s::OrderSlot *oslot = order_slot(f, cam->width, cam->height, &rc);
        if (!oslot) return rc;
        order = oslot->dev;
        hp->order_on = oslot->mode;
    }
    align_views(f, cam, vo.n, hp->view_shift);
    // one host -> device copy of the block's used prefix (cameras, order
    // switch, view shifts, joint tables up to the last used rotation)
    const size_t used = offsetof(FrameParams, rot_inv) + sizeof(double) * 9 * nj;
    ARTEMIS_TRY(cudaMemcpyAsync(f->params, hp, used, cudaMemcpyHostToDevice, st));
    ARTEMIS_TRY(cudaEventRecord(f->staged[sidx], st));  // the staging block may be reused after this
    f->fast_div = 1;
    for (int v = 0; v < vo.n; ++v)
        if (!camera_fast_div_ok(cam[v])) f->fast_div = 0;
    return run_frame_launch(f, identity, n_joints, cam, sharded, lambda_th, sigma_dep, flags, F,
                            alpha, depth, order, vo, st);
}

extern "C" int artemis_frame_run(artemis_frame f, const double *joint_aff, const double *rot_inv,
                                 int n_joints, const artemis_camera *cam, double lambda_th,
                                 double sigma_dep, int flags, float *F, void *alpha,
                                 void *depth, artemis_stream stream) {
    ViewOut vo;
    return frame_run_impl(f, joint_aff, rot_inv, n_joints, cam, lambda_th, sigma_dep, flags, F,
                          alpha, depth, vo, stream);
}

extern "C" int artemis_frame_run_views(artemis_frame f, const double *joint_aff,
                                       const double *rot_inv, int n_joints,
                                       const artemis_camera *cams, int n_views, double lambda_th,
                                       double sigma_dep, int flags, float *const *F,
                                       void *const *alpha, void *const *depth,
                                       artemis_stream stream) {
    if (n_views < 1 || n_views > kMaxViews || !F || !alpha || !depth) return ARTEMIS_ERR_ARG;
    ViewOut vo;
    vo.n = n_views;
    for (int v = 0; v < n_views; ++v) {
        if (!F[v] || !alpha[v] || !depth[v]) return ARTEMIS_ERR_ARG;
        vo.F[v] = F[v];
        vo.A[v] = alpha[v];
        vo.D[v] = depth[v];
    }
    return frame_run_impl(f, joint_aff, rot_inv, n_joints, cams, lambda_th, sigma_dep, flags,
                          F[0], alpha[0], depth[0], vo, stream);
}

// Eager enqueue or graph capture / replay of one frame (artemis_frame_run).
static int run_frame_launch(artemis_frame f, int identity, int n_joints, const artemis_camera *cam,
                            int sharded, double lambda_th, double sigma_dep, int flags, float *F,
                            void *alpha, void *depth, const int32_t *order, const ViewOut &vo,
                            cudaStream_t st) {
    const int use_graph = (flags & 2) && st != nullptr;
    if (!use_graph)
        return enqueue_frame(f, identity, n_joints, cam->width, cam->height, sharded, lambda_th,
                             sigma_dep, flags, F, alpha, depth, order, vo, st);
    artemis_frame_s::GraphSlot *slot = nullptr, *victim = &f->graphs[0];
    for (auto &g : f->graphs) {
        if (g.exec && g.w == cam->width && g.h == cam->height && g.flags == flags &&
            g.identity == identity && g.nj == n_joints && g.F == F && g.A == alpha &&
            g.D == depth && g.stream == st && g.lambda == lambda_th &&
            g.sigma_dep == sigma_dep && g.sharded == sharded && g.fast_div == f->fast_div &&
            same_views(g.views, vo)) {
            slot = &g;
            break;
        }
        if (!g.exec || (victim->exec && g.used < victim->used)) victim = &g;
    }
    if (!slot) {
        slot = victim;
        if (slot->exec) {
            cudaGraphExecDestroy(slot->exec);
            slot->exec = nullptr;
        }
        ARTEMIS_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_frame(f, identity, n_joints, cam->width, cam->height, sharded,
                               lambda_th, sigma_dep, flags, F, alpha, depth, order, vo, st);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(st, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) {
            set_cuda_error(e);
            return ARTEMIS_ERR_CUDA;
        }
        e = cudaGraphInstantiate(&slot->exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            set_cuda_error(e);
            slot->exec = nullptr;
            return ARTEMIS_ERR_CUDA;
        }
        slot->w = cam->width;
        slot->h = cam->height;
        slot->flags = flags;
        slot->identity = identity;
        slot->nj = n_joints;
        slot->F = F;
        slot->A = alpha;
        slot->D = depth;
        slot->stream = st;
        slot->lambda = lambda_th;
        slot->sigma_dep = sigma_dep;
        slot->sharded = sharded;
        slot->fast_div = f->fast_div;
        slot->views = vo;
    }
    slot->used = ++f->graph_clock;
    ARTEMIS_TRY(cudaGraphLaunch(slot->exec, st));
    return ARTEMIS_OK;
}

extern "C" int artemis_frame_counts(artemis_frame f, int64_t *n_in, int64_t *n_live,
                                    artemis_stream stream) {
    if (!f) return ARTEMIS_ERR_ARG;
    int32_t h[2] = {0, 0};
    ARTEMIS_TRY(cudaMemcpyAsync(h, f->counters, sizeof(h), cudaMemcpyDeviceToHost, S(stream)));
    ARTEMIS_TRY(cudaStreamSynchronize(S(stream)));
    if (n_in) *n_in = h[0];
    if (n_live) *n_live = h[1];
    return ARTEMIS_OK;
}

extern "C" int artemis_frame_get_tree(artemis_frame f, artemis_frame_tree *out) {
    if (!f || !out) return ARTEMIS_ERR_ARG;
    out->codes = f->live_codes;
    out->code_bytes = f->key_bytes;
    out->flut_idx = f->winners;
    out->left = f->left;
    out->right = f->right;
    out->box_min = f->bmin;
    out->box_size = f->bsize;
    out->rotation_joint = f->rot_joint;
    out->n_live_dev = f->counters + 1;
    out->n_in_dev = f->counters;
    return ARTEMIS_OK;
}

extern "C" int artemis_frame_launches(artemis_frame f) { return f ? f->launches : 0; }

extern "C" int artemis_frame_profile(artemis_frame f, int enable) {
    if (!f) return ARTEMIS_ERR_ARG;
    if (enable && !f->ev[0])
        for (auto &e : f->ev) ARTEMIS_TRY(cudaEventCreate(&e));
    f->profile = enable ? 1 : 0;
    return ARTEMIS_OK;
}

extern "C" int artemis_frame_stage_ms(artemis_frame f, float *ms) {
    if (!f || !ms || !f->ev[0]) return ARTEMIS_ERR_ARG;
    ARTEMIS_TRY(cudaEventSynchronize(f->ev[5]));
    for (int k = 0; k < 5; ++k) ARTEMIS_TRY(cudaEventElapsedTime(ms + k, f->ev[k], f->ev[k + 1]));
    return ARTEMIS_OK;
}
