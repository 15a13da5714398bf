// Per-ray traversal, SH shading and front-to-back compositing.
//
// Replaces animvox/_core.pyx:252-389 (slab / node_hit / _traverse /
// traverse_ray), :473-559 (render_rays) and :562-655 (forward_fit).
//
// Exactness: the traversal decisions and the emitted (leaf, t0, t1) are
// bit-identical to the reference: the slab test is evaluated in fp64 with
// true IEEE division, in x, y, z order, with the reference's comparisons,
// and children are visited in its DFS order (nearer entry first, left on
// ties). The transmittance chain (sigma, delta, exp, alpha, T, accumulated
// alpha, depth and the early-stop test) runs in fp64 per ray as in the
// reference; only the SH basis and the feature accumulation run in fp32
// (tolerance 1e-4 max / 1e-5 mean, BASELINE.json north_star).
//
// Work mapping (B200): one warp owns 32 rays -- an 8x4 pixel tile when
// rays come from a camera -- and each lane walks its own ray with a local
// stack. After every traversal step the lanes that produced a visible hit
// are shaded cooperatively: a group of GS = pow2(C) lanes takes one hit,
// lane c of the group owns channel c, so the FLUT row is read as H fully
// coalesced GS-float segments (9 x 128 B at C = 32) instead of one thread
// streaming 1156 B. Per-ray feature sums live in shared memory.
//
// Packed nodes (tree.cu) give both children's boxes in one 32-byte
// record, so an internal-node visit is a single sector load.
#include <math.h>
#include <stdlib.h>
#include <math_constants.h>

#include <type_traits>

#include "bricks.cuh"
#include "common.cuh"
#include "render_common.cuh"
#include "tree.cuh"

namespace artemis {

#ifndef ARTEMIS_SMEM_STACK
#define ARTEMIS_SMEM_STACK 28
#endif
#ifndef ARTEMIS_QCAP
#define ARTEMIS_QCAP 5
#endif
#ifndef ARTEMIS_QTHRESH
#define ARTEMIS_QTHRESH 48
#endif
#ifndef ARTEMIS_MIN_BLOCKS
#define ARTEMIS_MIN_BLOCKS 4
#endif
#ifndef ARTEMIS_DEDUP
#define ARTEMIS_DEDUP 1
#endif
#ifndef ARTEMIS_ROW_PREFETCH
#define ARTEMIS_ROW_PREFETCH 1  // 0 none, 1 every 128-B line of a queued row, 2 first line, 3 into L1,
                                // 4 one bulk (cp.async.bulk.prefetch.L2) per row
#endif
namespace {
constexpr int kRenderWarps = 4;
constexpr int kRenderThreads = 32 * kRenderWarps;
constexpr int kSmemStack = ARTEMIS_SMEM_STACK;  // per-thread stack entries in shared memory
constexpr int kStack = 100;  // <= 3 entries per two-level visit x 32 visits (64-bit keys) + slack
constexpr int kStackBytes = kSmemStack * kRenderThreads * 4;
// the exact cell walk keeps no DFS stack: its shared memory goes to L1
constexpr int stack_bytes(bool dda) { return dda ? 0 : kStackBytes; }
constexpr int kQCap = ARTEMIS_QCAP;  // leaves queued per lane per round
constexpr int kQThresh = ARTEMIS_QTHRESH;  // warp-wide queued leaves that end a traversal phase
constexpr int kMaxSteps = 64;        // traversal steps per phase at most
// per queued leaf: leaf id / FLUT row (4) + exp(-sigma*delta) (8) + (a, dir) (16) + entry
// distance t0 (fp32 in the frame pipeline, whose depth buffer is fp32; fp64 otherwise)
constexpr int queue_bytes(bool fp32_t0) {
    return kQCap * kRenderThreads * (4 + 8 + 16 + (fp32_t0 ? 4 : 8));
}
constexpr int kEnd = (int)0x80000000;  // empty-stack marker (never a node or ~leaf)
}  // namespace




#ifndef ARTEMIS_STREAM_OUT
#define ARTEMIS_STREAM_OUT 0  // 1: output maps stored evict-first (st.global.cs)
#endif
#ifndef ARTEMIS_SMEM_MASK
#define ARTEMIS_SMEM_MASK 0  // 1: the walk's brick mask cached in shared memory per lane
#endif
#ifndef ARTEMIS_A_CHECK
#define ARTEMIS_A_CHECK 1  // phase A: steps between checks of the warp's queued total
#endif
#ifndef ARTEMIS_FAST_CAMRAY
#define ARTEMIS_FAST_CAMRAY 1  // camera rays with reciprocal-corrected divisions
#endif
#ifndef ARTEMIS_CULL
#define ARTEMIS_CULL 0  // 1: fp32 AABB cull of camera rays (measured slower: DESIGN.md)
#endif
#ifndef ARTEMIS_FLAT_SHADE
#define ARTEMIS_FLAT_SHADE 0  // 1: shade a flat member list per level (see phase C)
#endif
#ifndef ARTEMIS_SPLIT_M
#define ARTEMIS_SPLIT_M 2  // phase C, L2-resident FLUT: row groups as items of <= M members (0: off)
#endif
#ifndef ARTEMIS_SPLIT_ALL
#define ARTEMIS_SPLIT_ALL 0  // 1: split whatever the FLUT size (experiment)
#endif
#ifndef ARTEMIS_SORT_ITEMS
#define ARTEMIS_SORT_ITEMS 1  // phase C: row groups in passes by member count (2: also L2-resident FLUTs)
#endif
#ifndef ARTEMIS_ROW_HINT
#define ARTEMIS_ROW_HINT 0  // 1: FLUT row loads carry an L2 evict_last policy
#endif

// Output stores: with ARTEMIS_STREAM_OUT the maps bypass L2 residency
// (streaming, evict-first) so they do not push FLUT rows out of L2.
template <typename T>
__device__ __forceinline__ void st_out(T *p, T v) {
    if (ARTEMIS_STREAM_OUT)
        __stcs(p, v);
    else
        *p = v;
}

__device__ __forceinline__ uint64_t row_policy() {
    uint64_t pol = 0;
#if ARTEMIS_ROW_HINT
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}

// One 16-byte slice of a FLUT row (read-only path; optionally evict_last in L2).
__device__ __forceinline__ float4 ld_row(const float4 *p, uint64_t pol) {
#if ARTEMIS_ROW_HINT
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}

// Conservative fp32 cull of a camera ray against the leaf-cell AABB grown by
// one cell on every side. fp32 rounding moves the ray by far less than a
// cell over the grid (|error| <~ 1e-6 x (|o| + |d t|) cells), so "misses the
// grown box in fp32" implies "misses the box exactly": such a pixel has no
// hit (alpha 0, depth +inf, F 0) and the exact fp64 ray is never built. A
// nearly axis-parallel fp32 direction is not culled (left to the exact path).
__device__ __forceinline__ bool ray_misses_aabb(const artemis_camera &c, int u, int v,
                                                const int32_t *aabb) {
    const float c0 = ((float)u + 0.5f - (float)c.cx) / (float)c.fx;
    const float c1 = ((float)v + 0.5f - (float)c.cy) / (float)c.fy;
    float t0 = 0.0f, t1 = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float d = ((float)c.R[3 * a] * c0 + (float)c.R[3 * a + 1] * c1 + (float)c.R[3 * a + 2]) /
                        (float)c.cell[a];
        const float o = (float)((c.origin[a] - c.lo[a]) / c.cell[a]);
        const float lo = (float)(__ldg(aabb + a) - 1), hi = (float)(__ldg(aabb + 3 + a) + 1);
        if (fabsf(d) < 1e-4f) return false;  // nearly parallel: exact path decides
        float ta = (lo - o) / d, tb = (hi - o) / d;
        if (ta > tb) {
            const float s = ta;
            ta = tb;
            tb = s;
        }
        t0 = fmaxf(t0, ta);
        t1 = fminf(t1, tb);
    }
    return t0 > t1;
}

// A camera pixel without hits: alpha 0 and depth +inf (F stays cleared).
__device__ __forceinline__ void write_empty_pixel(const RenderArgs &p, int64_t ray, int rv) {
    if (p.n_views > 1) {
        if (p.A64) {
            static_cast<double *>(p.Av[rv])[ray] = 0.0;
            static_cast<double *>(p.Dv[rv])[ray] = CUDART_INF;
        } else {
            static_cast<float *>(p.Av[rv])[ray] = 0.0f;
            static_cast<float *>(p.Dv[rv])[ray] = CUDART_INF_F;
        }
        return;
    }
    if (p.A64) p.A64[ray] = 0.0;
    if (p.A32) p.A32[ray] = 0.0f;
    if (p.D64) p.D64[ray] = CUDART_INF;
    if (p.D32) p.D32[ray] = CUDART_INF_F;
}

// Ray/box overlap of the child box packed in (w0, w1, w2) within
// [t_min, t_max]; exact port of the slab test (_core.pyx:252-285).
__device__ __forceinline__ bool clip_exact(uint32_t w0, uint32_t w1, uint32_t w2,
                                           const double o[3], const double d[3], double t_min,
                                           double t_max, double &t0o, double &t1o) {
    const uint32_t w[3] = {w0, w1, w2};
    double t0 = t_min, t1 = t_max;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int lo_i = (int)(w[a] & kCoordMask);
        const double lo = (double)lo_i;
        const double hi = (double)(lo_i + (1 << ((w[a] >> 21) & 31u)));
        if (d[a] == 0.0) {
            if (o[a] < lo || o[a] >= hi) return false;
        } else {
            double ta = __ddiv_rn(__dadd_rn(lo, -o[a]), d[a]);
            double tb = __ddiv_rn(__dadd_rn(hi, -o[a]), d[a]);
            if (ta > tb) {
                double s = ta;
                ta = tb;
                tb = s;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
            if (t0 >= t1) return false;
        }
    }
    t0o = t0;
    t1o = t1;
    return true;
}

#ifdef ARTEMIS_PHASE_CLOCKS
// per-phase SM cycles summed over warps: refill, A, B1, B2, C, retire, tail
__device__ unsigned long long g_phase_clocks[8];
__device__ unsigned long long g_fallbacks;
__device__ unsigned long long g_tests;
// shading reuse: visible entries, same-level row groups, unique rows per
// warp round (all levels), rounds
__device__ unsigned long long g_shade_stats[4];
extern "C" int artemis_debug_phase_clocks(unsigned long long *out, int reset) {
    cudaMemcpyFromSymbol(out + 13, g_shade_stats, sizeof(unsigned long long) * 4);
    cudaMemcpyFromSymbol(out, g_phase_clocks, sizeof(unsigned long long) * 7);
    cudaMemcpyFromSymbol(out + 7, g_fallbacks, sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 8, g_tests, sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 9, g_walk_stats, sizeof(unsigned long long) * 4);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_phase_clocks, z, sizeof(z));
        cudaMemcpyToSymbol(g_fallbacks, z, sizeof(unsigned long long));
        cudaMemcpyToSymbol(g_tests, z, sizeof(unsigned long long));
        cudaMemcpyToSymbol(g_walk_stats, z, sizeof(unsigned long long) * 4);
        cudaMemcpyToSymbol(g_shade_stats, z, sizeof(unsigned long long) * 4);
    }
    return 0;
}
#endif

// Per-ray constants of the fp32 filtered box test.
struct RayF {
    float o_inv[3], inv[3];  // o * (1/d) and 1/d in fp32 (axes with d != 0)
    float cmax;              // max |o/d| over the axes: the cancellation scale
    float tmin_up, tmin_dn, tmax_up, tmax_dn;
    bool exact_only;         // some d == 0: every test takes the exact path
};

__device__ __forceinline__ float int_to_float_exact(uint32_t v) {
    // v < 2^23: place v in the mantissa of 2^23 and subtract (exact, 2 ops)
    return __int_as_float(0x4B000000 | v) - 8388608.0f;
}

// Filtered hit test. Each plane distance t = (p - o)/d is evaluated in fp32
// as fma(p, 1/d, -o/d); with 1/d and o/d rounded to fp32 its error is below
// 2^-23 (|o/d| + |t|) <= 2^-23 (cmax + |t|), so t0 < t1 is decided from the
// fp32 entry maximum e and exit minimum x only when their gap exceeds
// 2^-20 (cmax + |e| + |x|) -- 4x the combined bound -- and otherwise by the
// exact fp64 slab test. The answer always equals clip_exact's; only its
// cost differs.
__device__ __forceinline__ bool hit_filtered(uint32_t w0, uint32_t w1, uint32_t w2,
                                             const RayF &rf, const double o[3],
                                             const double d[3], double t_min, double t_max) {
#ifdef ARTEMIS_PHASE_CLOCKS
    atomicAdd(&g_tests, 1ull);
#endif
    if (!rf.exact_only) {
        const uint32_t w[3] = {w0, w1, w2};
        float e = -INFINITY, x = INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint32_t lo_i = w[a] & kCoordMask;
            const float lo = int_to_float_exact(lo_i);
            const float hi = int_to_float_exact(lo_i + (1u << ((w[a] >> 21) & 31u)));
            const float ta = fmaf(lo, rf.inv[a], -rf.o_inv[a]);
            const float tb = fmaf(hi, rf.inv[a], -rf.o_inv[a]);
            e = fmaxf(e, fminf(ta, tb));
            x = fminf(x, fmaxf(ta, tb));
        }
        const float m = 9.5367431640625e-07f * (rf.cmax + fabsf(e) + fabsf(x));  // 2^-20
        if (e + m < x && e + m < rf.tmax_dn && rf.tmin_up + m < x) return true;
        if (e > x + m || e > rf.tmax_up + m || rf.tmin_dn > x + m) return false;
    }
#ifdef ARTEMIS_PHASE_CLOCKS
    atomicAdd(&g_fallbacks, 1ull);
#endif
    double e0, e1;
    return clip_exact(w0, w1, w2, o, d, t_min, t_max, e0, e1);
}

// Persistent warps pull rays from a global queue (ids in 8x4 pixel-tile order
// in camera mode) and refill idle lanes as rays finish. Each round runs
// three warp-uniform phases instead of one divergent per-ray loop:
//  A. traversal: every lane takes one DFS step per iteration (expand one
//     node, or queue one leaf) until the warp has kQThresh leaves queued.
//     A queued leaf is already known to be hit: near children are tested
//     when their parent is expanded, far children before they are pushed.
//  B. integration: the queued leaves are processed cooperatively (exact
//     fp64 slab interval, density, exp(-sigma delta), canonical direction);
//     then each lane runs the cheap sequential part of the reference's
//     per-ray loop over its own leaves in order -- transmittance, alpha,
//     depth, early stop (_core.pyx:534-556). Leaves queued past an early
//     stop are dropped.
//  C. shading: lane groups of C/4 lanes read one FLUT row as float4
//     segments per visible leaf, slot by slot so each ray's features
//     accumulate in ray order.
// The DFS stack lives in shared memory (a column per thread). Child order
// uses the split axis: the children's octants are separated by the plane of
// the node's highest differing Morton bit, so when both are hit the one on
// the ray's side of that plane has the smaller entry distance -- the order
// the reference's `lt0 <= rt0` comparison yields (_core.pyx:345). Internal
// tests use the fp32 filter; emitted leaves get exact fp64 intervals.
// kRays: 0 = explicit ray arrays (fp64 maps), 1 = in-kernel camera rays with
// fp32 alpha/depth maps (frame pipeline), 2 = camera rays with fp64 maps,
// 3 / 4 = as 1 / 2 over several views in one launch (run_views)
template <int kDeg, int kMode, int kRays, bool kVec, bool kDDA, bool kFast>
__global__ void __launch_bounds__(kRenderThreads, ARTEMIS_MIN_BLOCKS) render_kernel(RenderArgs p) {
    griddep_wait();  // launched as a dependent of the frame's last rebuild kernel
    constexpr bool kCamera = kRays != 0;
    constexpr bool kMulti = kRays >= 3;  // several views per launch (run_views)
    constexpr int H = (kDeg + 1) * (kDeg + 1);
    extern __shared__ __align__(16) unsigned char s_raw[];
    int *s_stack = reinterpret_cast<int *>(s_raw);
    __shared__ CamRecip s_camr[kCamera ? kMaxViews : 1];
    if (kCamera && kFast) {
        for (int v = threadIdx.x; v < (kMulti ? p.n_views : 1); v += blockDim.x)
            s_camr[v] = camera_recip(p.cam[v]);
        __syncthreads();
    }
    using T0 = typename std::conditional<kRays == 1 || kRays == 3, float, double>::type;
    constexpr int kQueueBytes = queue_bytes(kRays == 1 || kRays == 3);
    constexpr int kStackB = stack_bytes(kDDA);
    unsigned char *qbase = s_raw + kStackB;
    uint32_t *q_id = reinterpret_cast<uint32_t *>(qbase);                            // leaf, then row
    double *q_em = reinterpret_cast<double *>(qbase + kQCap * kRenderThreads * 4);
    float4 *q_val = reinterpret_cast<float4 *>(qbase + kQCap * kRenderThreads * 12);  // a, dir
    T0 *q_t0 = reinterpret_cast<T0 *>(qbase + kQCap * kRenderThreads * 28);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = p.channels;
    const int cp = kVec ? C : (C | 1);
    const uint64_t l2pol = row_policy();
    using FeatT = float;  // per-ray feature sums
    FeatT *feat = reinterpret_cast<FeatT *>(s_raw + kStackB + kQueueBytes) +
                  (size_t)warp * 32 * cp;
    // per-warp work list (lane | level << 5) used to hand queued leaves to
    // lanes, then (shading) the row groups' leaders; their member masks follow
    uint16_t *wl = reinterpret_cast<uint16_t *>(
                       s_raw + kStackB + kQueueBytes +
                       (kMode == kCount ? 0 : (size_t)kRenderWarps * 32 * cp * sizeof(FeatT))) +
                   warp * 32 * kQCap;
    uint32_t *wm = reinterpret_cast<uint32_t *>(
                       reinterpret_cast<uint16_t *>(
                           s_raw + kStackB + kQueueBytes +
                           (kMode == kCount ? 0 : (size_t)kRenderWarps * 32 * cp * sizeof(FeatT))) +
                       kRenderWarps * 32 * kQCap) +
                   warp * 32 * kQCap;
    // world directions of the lanes' rays (read by phase B1 for any lane's
    // queued leaves): shared memory instead of three registers pairs
    double *s_dw = reinterpret_cast<double *>(wm - warp * 32 * kQCap + kRenderWarps * 32 * kQCap);
    if (kMode != kCount)
        for (int i = lane; i < 32 * cp; i += 32) feat[i] = FeatT(0);
    const int64_t n_leaves = p.n_leaves_dev ? (int64_t)*p.n_leaves_dev : p.n_leaves;
    const int super_root = (int)(n_leaves > 1 ? n_leaves - 1 : 0);
    int tstart = 0, tstride = 1;
    if (kCamera && p.cam->tile_stride > 1) {
        tstart = p.cam->tile_start;
        tstride = p.cam->tile_stride;
    }
    const int64_t n_tiles = (int64_t)p.tiles_x * p.tiles_y;
    const int32_t *order =
        kCamera && p.tile_order && (!p.order_on || __ldg(p.order_on)) ? p.tile_order : nullptr;
    // camera mode: the tiles of all views interleave in the ray queue (tile t
    // of view 0, of view 1, ..., then tile t + 1), so the views' rays over
    // the same leaves are in flight together and share their FLUT rows in L2
    const int nv = kMulti ? p.n_views : 1;
    const int64_t n_ids = kCamera ? (tstart < n_tiles ? (n_tiles - tstart + tstride - 1) / tstride : 0) * 32 * nv
                                  : p.n_rays;
    const unsigned lt = lanemask_lt();
    const int wbase = warp * 32;  // this warp's column block in the queue arrays
#ifdef ARTEMIS_PHASE_CLOCKS
    unsigned long long ph_acc[7] = {0, 0, 0, 0, 0, 0, 0};
    long long ph_t = clock64();
    int ph_cur = 0;
#define ARTEMIS_PHASE(k)                          \
    do {                                          \
        const long long _t = clock64();           \
        ph_acc[ph_cur] += (unsigned long long)(_t - ph_t); \
        ph_t = _t;                                \
        ph_cur = (k) < 6 ? (k) : 6;               \
    } while (0)
#else
#define ARTEMIS_PHASE(k) \
    do {                 \
    } while (0)
#endif

    // per-lane ray state
    int64_t ray = -1;
    bool walking = false;  // DFS not exhausted
    double og[3], dg[3];
    double rg[3] = {0.0, 0.0, 0.0};  // correctly rounded 1/dg (ARTEMIS_RCP_CROSSING)
    RayF rf;
    // exact cell walk state (kDDA): current cell, step signs, exact entry /
    // exit crossing per axis, the leaf AABB exit, the cached brick
    int cc[3] = {0, 0, 0}, cs[3] = {0, 0, 0};
    // cell entry = max over the axes' slab entry crossings; it is the crossing
    // of the last step (steps are time-ordered, a synced slab's entry is never
    // later than the sync time), so one scalar replaces the per-axis entries
    double t_in = -CUDART_INF, cX[3] = {0, 0, 0};
    double t_end = 0.0;
    int cb[3] = {0, 0, 0}, cbid = -1;
    double cTb[3] = {0, 0, 0};
    // transmittance chain (T, accumulated alpha, depth): touched once per
    // round (phase B2) and at retirement, so it lives in shared memory
    double *s_tad = s_dw + 3 * kRenderThreads + 3 * tid;
    // the current brick's 512-bit occupancy mask per lane (cell walk), word-
    // major so a warp's lanes read distinct banks: one L2 round trip per
    // brick entered instead of one per cell step
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(s_dw + 6 * kRenderThreads);
    auto load_mask = [&]() {
#if ARTEMIS_SMEM_MASK
        const uint4 *src = reinterpret_cast<const uint4 *>(p.bm.recs[cbid].mask);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 v = __ldg(src + q4);
            s_mask[(4 * q4) * kRenderThreads + tid] = v.x;
            s_mask[(4 * q4 + 1) * kRenderThreads + tid] = v.y;
            s_mask[(4 * q4 + 2) * kRenderThreads + tid] = v.z;
            s_mask[(4 * q4 + 3) * kRenderThreads + tid] = v.w;
        }
#endif
    };
    (void)s_mask;
    int64_t hits = 0, trace_base = 0;
    int rv = 0;  // camera mode: view of this lane's ray
    int cur = kEnd, top = 0, nq = 0;
    int ovf[kStack - kSmemStack];
    bool queue_open = true;

    auto push = [&](int v) {
        ARTEMIS_DCHECK(top < kStack);
        if (top < kSmemStack)
            s_stack[top * kRenderThreads + tid] = v;
        else
            ovf[top - kSmemStack] = v;
        ++top;
    };
    auto pop = [&]() -> int {
        if (top == 0) return kEnd;
        --top;
        return top < kSmemStack ? s_stack[top * kRenderThreads + tid] : ovf[top - kSmemStack];
    };
    auto enqueue = [&](int leaf) {
        ARTEMIS_DCHECK(nq < kQCap && leaf >= 0 && leaf < n_leaves);
        q_id[nq * kRenderThreads + tid] = (uint32_t)leaf;
        ++nq;
        prefetch_l2(p.leaves + 2 * (size_t)leaf);  // its record is read in phase B1
    };
    // the cell walk knows the exact interval already: t0, and t1 - t0 (or t1
    // for the CSR trace)
    auto enqueue_hit = [&](uint32_t leaf, double t0, double t1) {
        ARTEMIS_DCHECK(nq < kQCap && (int64_t)leaf < n_leaves);
        const int qi = nq * kRenderThreads + tid;
        q_id[qi] = leaf;
        q_t0[qi] = (T0)t0;
        q_em[qi] = kMode == kTrace ? t1 : t1 - t0;
        ++nq;
        prefetch_l2(p.leaves + 2 * (size_t)leaf);
    };
    // ---- exact two-level walk (bricks.cuh): brick-level state (brick
    // index, exact crossing of its exit plane per axis) is always valid; the
    // cell-level state (cell, exact entry/exit crossing per axis) is valid
    // while inside an occupied brick. Empty bricks cost one crossing each;
    // entering an occupied brick re-derives the other axes' cells there.
    auto brick_exit = [&](int a) {  // exact crossing of the current brick's exit plane on axis a
        return cs[a] != 0 ? crossing<kFast>(cs[a] > 0 ? (cb[a] + 1) * 8 : cb[a] * 8, og[a], dg[a], rg[a])
                          : CUDART_INF;
    };
    auto enter_brick = [&](unsigned advanced, double tn) {
        double m = -CUDART_INF;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (cs[a] == 0) continue;
            if (advanced & (1u << a)) {
                const int cn = cs[a] > 0 ? cb[a] * 8 : cb[a] * 8 + 7;
                cc[a] = cn;
                m = fmax(m, tn);
                cX[a] = crossing<kFast>(cs[a] > 0 ? cn + 1 : cn, og[a], dg[a], rg[a]);
            } else {
                double E;
                sync_axis<kFast>(og[a], dg[a], rg[a], tn, cb[a] * 8, cb[a] * 8 + 7, cc[a], E, cX[a]);
                m = fmax(m, E);
            }
        }
        t_in = m;
    };
    auto walk_step = [&]() {
        if (cbid < 0) {  // empty brick: one brick step
            ARTEMIS_STAT(2);
            const double tn = fmin(cTb[0], fmin(cTb[1], cTb[2]));
            if (!(tn < p.t_max) || !(tn < t_end)) {
                walking = false;
                return;
            }
            unsigned adv = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (cTb[a] == tn) {
                    adv |= 1u << a;
                    cb[a] += cs[a];
                    cTb[a] = brick_exit(a);
                }
            cbid = brick_lookup(p.bm, cb[0], cb[1], cb[2]);
            if (cbid >= 0) {
                load_mask();
                enter_brick(adv, tn);
            }
            return;
        }
        ARTEMIS_STAT(1);
        // next cell: every axis whose exit crossing is the minimum steps
        const double tn = fmin(cX[0], fmin(cX[1], cX[2]));
        const double t0 = fmax(p.t_min, t_in);
        const double t1 = fmin(p.t_max, tn);
        const uint32_t m = spread3_small(cc[0] & 7) | (spread3_small(cc[1] & 7) << 1) |
                           (spread3_small(cc[2] & 7) << 2);
        const BrickRec &R = p.bm.recs[cbid];
#if ARTEMIS_SMEM_MASK
        const uint32_t word = s_mask[(m >> 5) * kRenderThreads + tid];  // cached at brick entry
#else
        const uint32_t word = __ldg(&R.mask[m >> 5]);
#endif
        if (((word >> (m & 31u)) & 1u) && t1 > t0) {
            const uint32_t leaf = __ldg(&R.first) + (uint32_t)__ldg(&R.prefix[m >> 5]) +
                                  (uint32_t)__popc(word & ((1u << (m & 31u)) - 1u));
            enqueue_hit(leaf, t0, t1);
        }
        if (!(tn < p.t_max) || !(tn < t_end)) {
            walking = false;
            return;
        }
        t_in = tn;
        unsigned pend = (cX[0] == tn ? 1u : 0u) | (cX[1] == tn ? 2u : 0u) | (cX[2] == tn ? 4u : 0u);
        bool new_brick = false;
        while (pend) {
            const int k = __ffs(pend) - 1;
            pend &= pend - 1;
            const int sk = k == 0 ? cs[0] : k == 1 ? cs[1] : cs[2];
            const int ck = (k == 0 ? cc[0] : k == 1 ? cc[1] : cc[2]) + sk;
            const double ok = k == 0 ? og[0] : k == 1 ? og[1] : og[2];
            const double dk = k == 0 ? dg[0] : k == 1 ? dg[1] : dg[2];
            const double rk = k == 0 ? rg[0] : k == 1 ? rg[1] : rg[2];
            const double xn = crossing<kFast>(sk > 0 ? ck + 1 : ck, ok, dk, rk);
            const bool bchg = (ck >> 3) != (k == 0 ? cb[0] : k == 1 ? cb[1] : cb[2]);
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (a == k) {
                    cc[a] = ck;
                    cX[a] = xn;
                    if (bchg) {  // the cell exit just crossed was this brick's exit plane
                        cb[a] = ck >> 3;
                        cTb[a] = brick_exit(a);
                    }
                }
            new_brick |= bchg;
        }
        if (new_brick) {
            cbid = brick_lookup(p.bm, cb[0], cb[1], cb[2]);
            if (cbid >= 0) load_mask();
        }
    };
    auto step = [&]() {
        if constexpr (kDDA) {
            walk_step();
            return;
        }
        if (cur == kEnd) {
            walking = false;
            return;
        }
        if (cur < 0) {  // a leaf, hit-tested before it was pushed
            enqueue(~cur);
            cur = pop();
            return;
        }
        const uint4 *rec = reinterpret_cast<const uint4 *>(p.nodes + cur);
        const uint4 s0 = __ldg(rec), s1 = __ldg(rec + 1), s2 = __ldg(rec + 2), s3 = __ldg(rec + 3);
        const bool h0 = hit_filtered(s0.x, s0.y, s0.z, rf, og, dg, p.t_min, p.t_max);
        const bool h1 = !(s1.x & kAbsent) && hit_filtered(s1.x, s1.y, s1.z, rf, og, dg, p.t_min, p.t_max);
        const bool h2 = !(s2.x & kAbsent) && hit_filtered(s2.x, s2.y, s2.z, rf, og, dg, p.t_min, p.t_max);
        const bool h3 = !(s3.x & kAbsent) && hit_filtered(s3.x, s3.y, s3.z, rf, og, dg, p.t_min, p.t_max);
        const bool left_first = dg[(s0.x >> 27) & 3u] > 0.0;
        const bool ll_first = dg[(s1.x >> 27) & 3u] > 0.0;  // meaningful when slot 1 exists
        const bool rl_first = dg[(s3.x >> 27) & 3u] > 0.0;  // meaningful when slot 3 exists
        // group L = slots (0, 1), group R = slots (2, 3), each in its own order
        const int la = (int)(ll_first ? s0.w : s1.w), lb = (int)(ll_first ? s1.w : s0.w);
        const bool hla = ll_first ? h0 : h1, hlb = ll_first ? h1 : h0;
        const int ra = (int)(rl_first ? s2.w : s3.w), rb = (int)(rl_first ? s3.w : s2.w);
        const bool hra = rl_first ? h2 : h3, hrb = rl_first ? h3 : h2;
        int o[4];
        bool oh[4];
        o[0] = left_first ? la : ra;
        oh[0] = left_first ? hla : hra;
        o[1] = left_first ? lb : rb;
        oh[1] = left_first ? hlb : hrb;
        o[2] = left_first ? ra : la;
        oh[2] = left_first ? hra : hla;
        o[3] = left_first ? rb : lb;
        oh[3] = left_first ? hrb : hlb;
        // compact the hit links in order
        int e0 = 0, e1 = 0, e2 = 0, e3 = 0, cnt = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (oh[j]) {
                if (cnt == 0) e0 = o[j];
                else if (cnt == 1) e1 = o[j];
                else if (cnt == 2) e2 = o[j];
                else e3 = o[j];
                ++cnt;
            }
        }
        auto ent = [&](int j) { return j == 0 ? e0 : j == 1 ? e1 : j == 2 ? e2 : e3; };
        int j = 0;
        while (j < cnt && ent(j) < 0 && nq < kQCap) {
            enqueue(~ent(j));
            ++j;
        }
        for (int t = cnt - 1; t >= j; --t) push(ent(t));
        cur = pop();
    };
    auto start_ray = [&](int64_t id) {
        ray = -1;
        double dw[3];
        if (kCamera) {
            const int64_t gi = id >> 5;
            if (kMulti) rv = (int)(gi % nv);
            const artemis_camera &cam = p.cam[rv];
            const int64_t t = tstart + (kMulti ? gi / nv : gi) * tstride;
            int64_t tile = order ? (int64_t)__ldg(order + t) : t;
            if (kMulti && p.view_shift) {  // views aligned by the grid centre's projection
                const int sh = __ldg(p.view_shift + rv) % p.tiles_x;
                if (sh) {
                    const int64_t tx = (tile % p.tiles_x + sh + p.tiles_x) % p.tiles_x;
                    tile = (tile / p.tiles_x) * p.tiles_x + tx;
                }
            }
            const int sl = (int)(id & 31);
            const int px = (int)(tile % p.tiles_x) * 8 + (sl & 7);
            const int py = (int)(tile / p.tiles_x) * 4 + (sl >> 3);
            if (py < cam.height && px < cam.width) {
                ARTEMIS_DCHECK(tile >= 0 && tile < n_tiles);
                ray = (int64_t)py * cam.width + px;
                if constexpr (kDDA && kMode == kRender && ARTEMIS_CULL) {
                    if (ray_misses_aabb(cam, px, py, p.bm.aabb)) {
                        // no leaf can be hit: the pixel's result is F = 0 (cleared),
                        // alpha = 0, depth = +inf, written now; the lane stays free
                        write_empty_pixel(p, ray, rv);
                        ray = -1;
                        return;
                    }
                }
                if constexpr (kFast && ARTEMIS_FAST_CAMRAY)
                    camera_ray_fast(cam, s_camr[rv], px, py, og, dg, dw);
                else
                    camera_ray(cam, px, py, og, dg, dw);
            }
        } else {
            ray = id;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                og[a] = p.og[3 * id + a];
                dg[a] = p.dg[3 * id + a];
                dw[a] = p.dw[3 * id + a];
            }
        }
        if (ray < 0) return;
        if (kMode != kCount)
#pragma unroll
            for (int a = 0; a < 3; ++a) s_dw[3 * tid + a] = dw[a];
        rf.exact_only = false;
        rf.cmax = 0.0f;
#pragma unroll
        for (int a = 0; a < 3 && !kDDA; ++a) {  // the fp32 box filter of the tree DFS
            if (dg[a] == 0.0) {
                rf.exact_only = true;
                rf.inv[a] = rf.o_inv[a] = 0.0f;
            } else {
                const double inv = 1.0 / dg[a];
                rf.inv[a] = (float)inv;
                rf.o_inv[a] = (float)(og[a] * inv);
                rf.cmax = fmaxf(rf.cmax, fabsf(rf.o_inv[a]));
            }
        }
        rf.tmin_up = __double2float_ru(p.t_min);
        rf.tmin_dn = __double2float_rd(p.t_min);
        rf.tmax_up = __double2float_ru(p.t_max);
        rf.tmax_dn = __double2float_rd(p.t_max);
        s_tad[0] = 1.0;
        s_tad[1] = 0.0;
        s_tad[2] = CUDART_INF;
        hits = 0;
        top = 0;
        nq = 0;
        trace_base = (kMode == kTrace) ? p.offsets[ray] : 0;
        cur = (n_leaves > 0 && p.t_min < p.t_max) ? super_root : kEnd;
        walking = true;
        if constexpr (kDDA) {
            // exact slab clip against the leaf AABB, then each axis's slab at
            // the clipped entry distance
            walking = false;
            if (!(n_leaves > 0 && p.t_min < p.t_max)) return;
            int aL[3], aU[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                aL[a] = __ldg(p.bm.aabb + a);
                aU[a] = __ldg(p.bm.aabb + 3 + a);
            }
            if constexpr (kFast) {
#pragma unroll
                for (int a = 0; a < 3; ++a) rg[a] = dg[a] != 0.0 ? __drcp_rn(dg[a]) : 0.0;
            }
            double t0 = p.t_min, t1 = p.t_max;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double lo = (double)aL[a], hi = (double)aU[a];
                if (dg[a] == 0.0) {
                    if (og[a] < lo || og[a] >= hi) return;
                } else {  // the slab test's exact plane distances (_core.pyx:252-285)
                    double ta = crossing<kFast>(aL[a], og[a], dg[a], rg[a]);
                    double tb = crossing<kFast>(aU[a], og[a], dg[a], rg[a]);
                    if (ta > tb) {
                        const double sw = ta;
                        ta = tb;
                        tb = sw;
                    }
                    if (ta > t0) t0 = ta;
                    if (tb < t1) t1 = tb;
                    if (t0 >= t1) return;
                }
            }
            t_end = t1;
            t_in = -CUDART_INF;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (dg[a] == 0.0) {
                    cs[a] = 0;
                    cc[a] = (int)floor(og[a]);
                    cX[a] = CUDART_INF;
                } else {
                    cs[a] = dg[a] > 0.0 ? 1 : -1;
                    double E;
                    sync_axis<kFast>(og[a], dg[a], rg[a], t0, aL[a], aU[a] - 1, cc[a], E, cX[a]);
                    t_in = fmax(t_in, E);
                }
                cb[a] = cc[a] >> 3;
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) cTb[a] = brick_exit(a);
            cbid = brick_lookup(p.bm, cb[0], cb[1], cb[2]);
            if (cbid >= 0) load_mask();
            walking = true;
        }
    };

    // cooperative shading geometry: lph lanes per hit, hpi hits per pass
    const int units = kVec ? C / 4 : C;
    int lph = 1;
    while (lph < units && lph < 32) lph <<= 1;
    const int hpi = 32 / lph;
    const int grp = lane / lph, q = lane % lph;

    while (true) {
        ARTEMIS_PHASE(0);
        // ---- refill idle lanes from the ray queue
        const unsigned idle = __ballot_sync(0xffffffffu, ray < 0);
        if (queue_open && __popc(idle) >= 8) {
            int64_t base = 0;
            if (lane == 0) base = (int64_t)atomicAdd(p.queue, (unsigned long long)__popc(idle));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base >= n_ids) queue_open = false;
            if (ray < 0) {
                const int64_t id = base + __popc(idle & lt);
                if (id < n_ids) start_ray(id);
            }
        }
        if (__ballot_sync(0xffffffffu, ray >= 0) == 0) {
            if (!queue_open) break;
            continue;
        }
        ARTEMIS_PHASE(1);
        // ---- phase A: uniform DFS steps until enough leaves are queued
        for (int it = 0; it < kMaxSteps; ++it) {
            const bool can = walking && nq < kQCap;
            if (__ballot_sync(0xffffffffu, can) == 0) break;
            if (can) step();
#if ARTEMIS_A_CHECK > 1
            // the warp's queued total is checked every ARTEMIS_A_CHECK steps
            // (a warp reduction per step sits on the walk's critical path)
            if ((it % ARTEMIS_A_CHECK) != ARTEMIS_A_CHECK - 1) continue;
#endif
            if (__reduce_add_sync(0xffffffffu, (unsigned)nq) >= (unsigned)kQThresh) break;
        }
        ARTEMIS_PHASE(2);
        // ---- phase B1: exact intervals and per-leaf terms, warp-cooperative:
        // all queued leaves of the warp are listed (lane | level << 5) and
        // handed out 32 at a time
        __syncwarp();
        int total = 0;
        for (int k = 0; k < kQCap; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, nq > k);
            if (!m) break;
            ARTEMIS_DCHECK(total + __popc(m) <= 32 * kQCap);
            if (nq > k) wl[total + __popc(m & lt)] = (uint16_t)(lane | (k << 5));
            total += __popc(m);
        }
        __syncwarp();
        for (int base = 0; base < total; base += 32) {
            const bool has = base + lane < total;
            const int entry = has ? (int)wl[base + lane] : lane;
            const int src = entry & 31, k = entry >> 5;
            double so[3], sd[3], sw[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if constexpr (!kDDA) {  // the cell walk already holds the exact interval
                    so[a] = __shfl_sync(0xffffffffu, og[a], src);
                    sd[a] = __shfl_sync(0xffffffffu, dg[a], src);
                } else {
                    so[a] = sd[a] = 0.0;
                }
                if (kMode != kCount) sw[a] = s_dw[3 * (wbase + src) + a];
            }
            if (has && kMode != kCount) {
                const int qi = k * kRenderThreads + wbase + src;
                const uint4 L = __ldg(p.leaves + 2 * (size_t)q_id[qi]);
                const uint4 L2 = __ldg(p.leaves + 2 * (size_t)q_id[qi] + 1);
                const uint32_t fidx = L.w;
                ARTEMIS_DCHECK(p.n_rows <= 0 || (int64_t)fidx < p.n_rows);
#if ARTEMIS_ROW_PREFETCH
                if (!p.no_row_prefetch) {  // the row's 9 x 128 B lines are read in phase C
                    const char *row = reinterpret_cast<const char *>(p.coef + (size_t)fidx * p.coef_stride);
#if ARTEMIS_ROW_PREFETCH == 4
                    // one bulk (TMA-engine) L2 prefetch of the whole row: vec rows are
                    // 16-B aligned with a multiple-of-16 length
                    if (kVec) {
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row),
                                     "r"((unsigned)(p.coef_stride * 4)));
                    } else
#endif
                    for (int off = 0; off < (ARTEMIS_ROW_PREFETCH == 2 ? 1 : p.coef_stride * 4); off += 128) {
#if ARTEMIS_ROW_PREFETCH == 3
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(row + off));
#else
                        prefetch_l2(row + off);
#endif
                    }
                }
#endif
                const double sigma = __longlong_as_double(((long long)L2.y << 32) | L2.x);
                q_id[qi] = fidx | (sigma > p.sigma_dep ? kDenseFlag : 0u);
                if constexpr (kDDA) {
                    // interval from the walk; q_em holds t1 - t0 (or t1 for the trace)
                    if (kMode != kTrace) q_em[qi] = exp(-sigma * q_em[qi]);
                } else {
                    double t0 = 0.0, t1 = 0.0;
                    clip_exact(L.x, L.y, L.z, so, sd, p.t_min, p.t_max, t0, t1);
                    q_t0[qi] = (T0)t0;
                    // trace mode keeps t1 for B2, which writes the CSR trace
                    q_em[qi] = kMode == kTrace ? t1 : exp(-sigma * (t1 - t0));
                }
                const double *R = p.rot_inv + 9 * L2.z;
                float4 v;
                v.x = 0.0f;
                v.y = (float)(R[0] * sw[0] + R[1] * sw[1] + R[2] * sw[2]);
                v.z = (float)(R[3] * sw[0] + R[4] * sw[1] + R[5] * sw[2]);
                v.w = (float)(R[6] * sw[0] + R[7] * sw[1] + R[8] * sw[2]);
                q_val[qi] = v;
            }
        }
        __syncwarp();
        ARTEMIS_PHASE(3);
        // ---- phase B2: sequential per-ray integration over own leaves
        double T = 1.0, acc = 0.0, depth = CUDART_INF;
        if (nq > 0 && kMode != kCount) {
            T = s_tad[0];
            acc = s_tad[1];
            depth = s_tad[2];
        }
        for (int k = 0; k < nq; ++k) {
            const int qi = k * kRenderThreads + tid;
            const uint32_t id = q_id[qi];
            if (kMode == kCount) {
                ++hits;
                continue;
            }
            const uint32_t fidx = id & ~kDenseFlag;
            const double t0 = (double)q_t0[qi];
            double em;
            if (kMode == kTrace) {
                const double t1 = q_em[qi];
                p.hit_idx[trace_base + hits] = (int64_t)fidx;
                p.hit_t0[trace_base + hits] = t0;
                p.hit_t1[trace_base + hits] = t1;
                em = exp(-__ldg(p.sigma + fidx) * (t1 - t0));  // trace mode: recompute
            } else {
                em = q_em[qi];
            }
            if (kMode == kRender && depth == CUDART_INF && (id & kDenseFlag)) depth = t0;
            const double a = T * (1.0 - em);
            float4 v = q_val[qi];
            v.x = 0.0f;
            if (a > 0.0) {
                v.x = (float)a;
                acc = acc + a;
            }
            q_val[qi] = v;
            T = T * em;
            ++hits;
            if (kMode == kRender && p.early_stop && acc > p.stop) {
                nq = k + 1;  // drop leaves queued past the stop
                walking = false;
                cur = kEnd;
                break;
            }
        }
        if (nq > 0 && kMode != kCount) {
            s_tad[0] = T;
            s_tad[1] = acc;
            s_tad[2] = depth;
        }
        ARTEMIS_PHASE(4);
        // ---- phase C: shade the visible queued leaves level by level (a ray
        // has at most one leaf per level, so its features accumulate in order).
        // Rays of a tile often hit the same leaf at the same level: lanes with
        // equal FLUT rows are grouped (__match_any_sync) and the row is read
        // once per group, then applied to every member ray.
#ifdef ARTEMIS_PHASE_CLOCKS
        if (kMode != kCount) {  // reuse statistics (instrumented build only)
            unsigned vis_n = 0, uniq = 0;
            for (int k = 0; k < kQCap; ++k) {
                const int qme = k * kRenderThreads + tid;
                const bool vis = nq > k && q_val[qme].x > 0.0f;
                const uint32_t key = vis ? (q_id[qme] & ~kDenseFlag) : 0xFFFFFFFFu;
                bool dup = false;
                for (int k2 = 0; k2 <= k; ++k2) {
                    const int q2 = k2 * kRenderThreads + tid;
                    const bool v2 = nq > k2 && q_val[q2].x > 0.0f;
                    const uint32_t key2 = v2 ? (q_id[q2] & ~kDenseFlag) : 0xFFFFFFFEu;
                    for (int src = 0; src < 32; ++src) {
                        const uint32_t o = __shfl_sync(0xffffffffu, key2, src);
                        if (vis && o == key && (k2 < k || src < lane)) dup = true;
                    }
                }
                vis_n += __popc(__ballot_sync(0xffffffffu, vis));
                uniq += __popc(__ballot_sync(0xffffffffu, vis && !dup));
            }
            if (lane == 0) {
                atomicAdd(&g_shade_stats[0], (unsigned long long)vis_n);
                atomicAdd(&g_shade_stats[2], (unsigned long long)uniq);
                atomicAdd(&g_shade_stats[3], 1ull);
            }
        }
#endif
#ifndef ARTEMIS_NOSHADE
#define ARTEMIS_NOSHADE 0
#endif
        if (kMode != kCount && !ARTEMIS_NOSHADE) {
            __syncwarp();
            for (int k = 0; k < kQCap; ++k) {
                if (!__any_sync(0xffffffffu, nq > k)) break;
                const int qme = k * kRenderThreads + tid;
                const bool vis = nq > k && q_val[qme].x > 0.0f;
                const uint32_t key = vis ? (q_id[qme] & ~kDenseFlag) : (0x80000000u | (uint32_t)lane);
#if ARTEMIS_DEDUP
                const unsigned grpm = __match_any_sync(0xffffffffu, key);
#else
                const unsigned grpm = 1u << lane;
                (void)key;
#endif
                const bool leader = vis && lane == __ffs(grpm) - 1;
#if ARTEMIS_FLAT_SHADE
                if (kVec) {
                    // flat member list: the level's visible lanes, groups of one FLUT
                    // row adjacent (leader-lane order), so every lane group shades a
                    // member each pass (no idle groups waiting on a long member
                    // list); members of one row in the same pass load the same
                    // addresses (one L1 request), later passes hit L1
                    const int nvis = __popc(__ballot_sync(0xffffffffu, vis));
                    const int x = leader ? __popc(grpm) : 0;
                    int incl = x;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const int goff = __shfl_sync(0xffffffffu, incl - x, __ffs(grpm) - 1);
                    if (vis) wl[goff + __popc(grpm & lt)] = (uint16_t)lane;
                    __syncwarp();
                    for (int m = grp; m - grp < nvis; m += hpi) {
                        if (m >= nvis) continue;
                        const int s = (int)wl[m];
                        const uint32_t bf = q_id[k * kRenderThreads + wbase + s] & ~kDenseFlag;
                        const float4 *row =
                            reinterpret_cast<const float4 *>(p.coef + (size_t)bf * p.coef_stride);
                        const float4 bv = q_val[k * kRenderThreads + wbase + s];
                        float Y[H];
                        sh_basis_f<kDeg>(bv.y, bv.z, bv.w, Y);
                        for (int c4 = q; c4 < units; c4 += lph) {
                            float4 v[H];
#pragma unroll
                            for (int h = 0; h < H; ++h) v[h] = ld_row(row + h * units + c4, l2pol);
                            float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f;
#pragma unroll
                            for (int h = 0; h < H; ++h) {
                                ax = fmaf(v[h].x, Y[h], ax);
                                ay = fmaf(v[h].y, Y[h], ay);
                                az = fmaf(v[h].z, Y[h], az);
                                aw = fmaf(v[h].w, Y[h], aw);
                            }
                            float4 *dst =
                                reinterpret_cast<float4 *>(reinterpret_cast<float *>(feat) + s * cp) + c4;
                            float4 f = *dst;
                            f.x += bv.x * ax;
                            f.y += bv.x * ay;
                            f.z += bv.x * az;
                            f.w += bv.x * aw;
                            *dst = f;
                        }
                    }
                    __syncwarp();
                    continue;
                }
#endif
#if ARTEMIS_SPLIT_M > 0
                // With an L2-resident FLUT a group's members, in lane order,
                // are dealt as items of <= M members (the head of each item is
                // the lane whose rank in the group is a multiple of M; its mask
                // is the next M members), so a pass no longer waits on one
                // large group: the items of one row re-read it from L1/L2,
                // which is cheap only when the row is L2-resident (configs[1]
                // 0.846 -> 0.803 ms; configs[2] +1 %, configs[4] +0.6 %, where
                // the member-count ranking below balances the passes instead).
                // Items of one level belong to different rays: exact.
                unsigned imask = 0;
                bool ihead = false;
                if (kVec && vis && (ARTEMIS_SPLIT_ALL || p.no_row_prefetch)) {
                    const int r = __popc(grpm & lt);
                    ihead = (r % ARTEMIS_SPLIT_M) == 0;
                    unsigned m = grpm & ~lt;
#pragma unroll
                    for (int j = 0; j < ARTEMIS_SPLIT_M; ++j) {
                        imask |= m & (0u - m);
                        m &= m - 1;
                    }
                } else {
                    ihead = leader;
                    imask = grpm;
                }
                const unsigned ml = __ballot_sync(0xffffffffu, ihead);
#define ARTEMIS_ITEM_MASK imask
#define ARTEMIS_ITEM_HEAD ihead
#else
                const unsigned ml = __ballot_sync(0xffffffffu, leader);
#define ARTEMIS_ITEM_MASK grpm
#define ARTEMIS_ITEM_HEAD leader
#endif
                const int cnt = __popc(ml);
#ifdef ARTEMIS_PHASE_CLOCKS
                if (lane == 0) atomicAdd(&g_shade_stats[1], (unsigned long long)cnt);
#endif
#if ARTEMIS_SORT_ITEMS
                // The lane groups of one pass run their member loops in
                // lockstep, so a pass costs its largest group: order the row
                // groups by member count (descending, capped at 8; ties by
                // lane) so each pass holds groups of similar size. Groups of
                // one level belong to different rays: any order is exact.
                // Only when the FLUT is not L2-resident (the passes wait on
                // L2 misses; with an L2-resident FLUT the ranking's ballots
                // cost more than they save: configs[1] 0.842 -> 0.854 ms).
                int slot = __popc(ml & lt);
                if (ARTEMIS_SORT_ITEMS == 2 || !p.no_row_prefetch) {
                    const unsigned key = 8u - (unsigned)min(__popc(ARTEMIS_ITEM_MASK), 8);  // 0..7
                    unsigned same = ml;
                    slot = 0;
#pragma unroll
                    for (int b = 2; b >= 0; --b) {
                        const unsigned bb = __ballot_sync(0xffffffffu, (key >> b) & 1u);
                        if ((key >> b) & 1u) {
                            slot += __popc(same & ~bb);
                            same &= bb;
                        } else {
                            same &= ~bb;
                        }
                    }
                    slot += __popc(same & lt);
                }
#else
                const int slot = __popc(ml & lt);
#endif
                if (ARTEMIS_ITEM_HEAD) {
                    wl[slot] = (uint16_t)lane;
                    wm[slot] = ARTEMIS_ITEM_MASK;
                }
#undef ARTEMIS_ITEM_MASK
#undef ARTEMIS_ITEM_HEAD
                __syncwarp();
                for (int item = grp; item - grp < cnt; item += hpi) {
                    if (item >= cnt) continue;
                    const int s0 = (int)wl[item];
                    unsigned members = wm[item];
                    const uint32_t bf = q_id[k * kRenderThreads + wbase + s0] & ~kDenseFlag;
                    if (kVec) {
                        const float4 *row = reinterpret_cast<const float4 *>(
                            p.coef + (size_t)bf * p.coef_stride);
                        for (int c4 = q; c4 < units; c4 += lph) {
                            float4 v[H];
#pragma unroll
                            for (int h = 0; h < H; ++h) v[h] = ld_row(row + h * units + c4, l2pol);
                            unsigned mm = members;
                            while (mm) {
                                const int s = __ffs(mm) - 1;
                                mm &= mm - 1;
                                const float4 bv = q_val[k * kRenderThreads + wbase + s];
                                float Y[H];
                                sh_basis_f<kDeg>(bv.y, bv.z, bv.w, Y);
                                float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f;
#pragma unroll
                                for (int h = 0; h < H; ++h) {
                                    ax = fmaf(v[h].x, Y[h], ax);
                                    ay = fmaf(v[h].y, Y[h], ay);
                                    az = fmaf(v[h].z, Y[h], az);
                                    aw = fmaf(v[h].w, Y[h], aw);
                                }
                                float4 *dst = reinterpret_cast<float4 *>(
                                                  reinterpret_cast<float *>(feat) + s * cp) + c4;
                                float4 f = *dst;
                                f.x += bv.x * ax;
                                f.y += bv.x * ay;
                                f.z += bv.x * az;
                                f.w += bv.x * aw;
                                *dst = f;
                            }
                        }
                    } else {
                        const float *row = p.coef + (size_t)bf * p.coef_stride;
                        while (members) {
                            const int s = __ffs(members) - 1;
                            members &= members - 1;
                            const float4 bv = q_val[k * kRenderThreads + wbase + s];
                            float Y[H];
                            sh_basis_f<kDeg>(bv.y, bv.z, bv.w, Y);
                            for (int c = q; c < C; c += lph) {
                                float acc_c = 0.0f;
#pragma unroll
                                for (int h = 0; h < H; ++h)
                                    acc_c = fmaf(__ldg(row + h * C + c), Y[h], acc_c);
                                reinterpret_cast<float *>(feat)[s * cp + c] += bv.x * acc_c;
                            }
                        }
                    }
                }
                __syncwarp();
            }
        }
        nq = 0;
        ARTEMIS_PHASE(5);
        // ---- retire finished rays: scalars per lane, features row by row
        const bool done = ray >= 0 && !walking;
        if (kMode != kCount && done) {
            acc = s_tad[1];
            depth = s_tad[2];
        }
        if (done) {
            if (kMode == kCount) {
                p.counts[ray] = hits;
            } else {
                if (kMulti) {  // per-view maps
                    if (p.A64) {
                        st_out(static_cast<double *>(p.Av[rv]) + ray, acc);
                        st_out(static_cast<double *>(p.Dv[rv]) + ray, depth);
                    } else {
                        st_out(static_cast<float *>(p.Av[rv]) + ray, (float)acc);
                        st_out(static_cast<float *>(p.Dv[rv]) + ray, (float)depth);
                    }
                } else {
                    if (p.A64) st_out(p.A64 + ray, acc);
                    if (p.A32) st_out(p.A32 + ray, (float)acc);
                    if (kMode == kRender) {
                        if (p.D64) st_out(p.D64 + ray, depth);
                        if (p.D32) st_out(p.D32 + ray, (float)depth);
                    }
                }
            }
        }
        if (kMode != kCount) {
            unsigned fm = __ballot_sync(0xffffffffu, done && acc > 0.0);
            __syncwarp();
            while (fm) {
                const int s = __ffs(fm) - 1;
                fm &= fm - 1;
                const int64_t r = __shfl_sync(0xffffffffu, ray, s);
                float *Fo = p.F;
                if (kMulti) Fo = p.Fv[__shfl_sync(0xffffffffu, rv, s)];
                for (int c = lane; c < C; c += 32) {
                    st_out(Fo + r * C + c, feat[s * cp + c]);
                    feat[s * cp + c] = FeatT(0);
                }
            }
            __syncwarp();
        }
        if (done) ray = -1;
    }
    ARTEMIS_PHASE(6);
#ifdef ARTEMIS_PHASE_CLOCKS
    if (lane == 0)
        for (int k = 0; k < 7; ++k) atomicAdd(&g_phase_clocks[k], ph_acc[k]);
#endif
}

// test hook (artemis_debug_set_render_blocks): cap the persistent render
// grid so a test can vary the ray-to-warp schedule; results must not change
static int g_render_block_cap = 0;
// test hook (artemis_debug_set_flut_l2_resident): -1 automatic, 0/1 force the
// "FLUT L2-resident" launch flag (1: no row prefetch, phase-C groups split;
// 0: row prefetch, phase-C member-count ranking)
static int g_flut_l2_resident = -1;

template <int kMode, int kRays, bool kVec, bool kDDA, bool kFast = false>
int launch_render_vec(int degree, const RenderArgs &a, int64_t warps, cudaStream_t st) {
    if (warps == 0) return ARTEMIS_OK;
    const int cp = kVec ? a.channels : (a.channels | 1);
    const size_t feat_bytes = 4;
    const size_t smem = stack_bytes(kDDA) + queue_bytes(kRays == 1 || kRays == 3) +
                        (kMode == kCount ? 0 : (size_t)kRenderWarps * 32 * cp * feat_bytes) +
                        (size_t)kRenderWarps * 32 * kQCap * (2 + 4) + (size_t)kRenderThreads * 6 * 8 +
                        (kDDA && ARTEMIS_SMEM_MASK ? (size_t)kRenderThreads * 64 : 0);
    const int64_t want = ceil_div<int64_t>(warps, kRenderWarps);
    int rc_launch = ARTEMIS_OK;
    switch (degree) {
#define ARTEMIS_LAUNCH(D)                                                                       \
    case D: {                                                                                   \
        auto kern = render_kernel<D, kMode, kRays, kVec, kDDA, kFast>;                          \
        if (smem > 48 * 1024)                                                                   \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        int occ = 0;                                                                            \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRenderThreads, smem);        \
        int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * (occ > 0 ? occ : 1)); \
        if (g_render_block_cap > 0 && blocks > g_render_block_cap) blocks = g_render_block_cap; \
        rc_launch = launch_pdl(kern, blocks, kRenderThreads, smem, st, a);                     \
        break;                                                                                  \
    }
        ARTEMIS_LAUNCH(0) ARTEMIS_LAUNCH(1) ARTEMIS_LAUNCH(2) ARTEMIS_LAUNCH(3) ARTEMIS_LAUNCH(4)
#undef ARTEMIS_LAUNCH
        default:
            return ARTEMIS_ERR_ARG;
    }
    return rc_launch;
}

template <int kMode, int kRays>
int launch_render_deg(int degree, const RenderArgs &a, int64_t warps, cudaStream_t st) {
    const bool vec = kMode != kCount && a.channels % 4 == 0 && a.coef_stride % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(a.coef) & 15) == 0;
    const bool dda = a.bm.table != nullptr;
    if (kRays != 0) {  // the device pipeline always has a brick map
        if (a.fast_div && ARTEMIS_RCP_CROSSING)  // cameras in div_fast's operand ranges
            return vec ? launch_render_vec<kMode, kRays, true, true, true>(degree, a, warps, st)
                       : launch_render_vec<kMode, kRays, false, true, true>(degree, a, warps, st);
        return vec ? launch_render_vec<kMode, kRays, true, true>(degree, a, warps, st)
                   : launch_render_vec<kMode, kRays, false, true>(degree, a, warps, st);
    }
    if (dda) {
        if (a.fast_div && ARTEMIS_RCP_CROSSING)  // rays vouched for by the caller
            return vec ? launch_render_vec<kMode, kRays, true, true, true>(degree, a, warps, st)
                       : launch_render_vec<kMode, kRays, false, true, true>(degree, a, warps, st);
        return vec ? launch_render_vec<kMode, kRays, true, true>(degree, a, warps, st)
                   : launch_render_vec<kMode, kRays, false, true>(degree, a, warps, st);
    }
    return vec ? launch_render_vec<kMode, kRays, true, false>(degree, a, warps, st)
               : launch_render_vec<kMode, kRays, false, false>(degree, a, warps, st);
}

static void fill_tree(RenderArgs &a, const artemis_tree_view *t) {
    a.nodes = static_cast<const WideNode *>(t->nodes);
    a.leaves = static_cast<const uint4 *>(t->leaves);
    a.n_leaves = t->n_leaves;
    a.n_leaves_dev = t->n_leaves_dev;
    a.coord_max = t->coord_max > 0.0 ? (float)t->coord_max : 2097152.0f;
    if (t->bricks) {
        a.bm.table = t->bricks->table;
        a.bm.recs = static_cast<const BrickRec *>(t->bricks->recs);
        a.bm.aabb = t->bricks->aabb;
        for (int k = 0; k < 3; ++k) {
            a.bm.org[k] = t->bricks->org[k];
            a.bm.dims[k] = t->bricks->dims[k];
        }
    }
}

static void fill_shade(RenderArgs &a, const artemis_shading *s) {
    a.coef = s->coef;
    a.sigma = s->sigma;
    a.rot_index = s->rot_index;
    a.rot_inv = s->rot_inv;
    a.channels = s->channels;
    a.coef_stride = s->coef_stride > 0 ? s->coef_stride : (s->degree + 1) * (s->degree + 1) * s->channels;
}

static void fill_rays(RenderArgs &a, const artemis_rays *r) {
    a.og = r->origins_g;
    a.dg = r->dirs_g;
    a.dw = r->dirs_w;
    a.n_rays = r->n_rays;
    a.t_min = r->t_min;
    a.t_max = r->t_max;
    a.fast_div = r->fast_div;
}

template <typename T>
__global__ void fill_alpha_depth(T *A, T *D, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        A[i] = T(0);
        D[i] = T(CUDART_INF);
    }
}

// Output clearing of render_camera, for callers that run it ahead on another
// stream (frame.cu: concurrent with the rebuild): F zero, and for sharded
// frames alpha 0 / depth +inf (other ranks' pixels).
int render_clear_outputs(float *F, void *A, void *D, int64_t n, int channels, int sharded,
                         int maps64, cudaStream_t st) {
    ARTEMIS_TRY(cudaMemsetAsync(F, 0, (size_t)n * channels * sizeof(float), st));
    if (sharded) {
        const int g = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 4 * 148);
        if (maps64)
            fill_alpha_depth<double><<<g, 256, 0, st>>>(static_cast<double *>(A),
                                                        static_cast<double *>(D), n);
        else
            fill_alpha_depth<float><<<g, 256, 0, st>>>(static_cast<float *>(A),
                                                       static_cast<float *>(D), n);
        return ARTEMIS_LAUNCHED();
    }
    return ARTEMIS_OK;
}

// Device-pipeline render with in-kernel camera rays (frame.cu). maps64:
// alpha/depth are double (exact fp64 maps, as the API path) instead of float.
int render_camera(const artemis_tree_view *tree, const artemis_shading *shade,
                  const artemis_camera *cam_dev, int width, int height, int sharded,
                  double lambda_th, double sigma_dep, int early_stop, int maps64, float *F,
                  void *A, void *D, unsigned long long *queue, const int32_t *tile_order,
                  const int32_t *order_on, void *const *peer_out, int n_views,
                  float *const *Fv, void *const *Av, void *const *Dv, int64_t flut_rows,
                  int outputs_ready, int fast_div, const int32_t *view_shift, cudaStream_t st) {
    RenderArgs a{};
    a.fast_div = fast_div;
    a.view_shift = n_views > 1 ? view_shift : nullptr;
    {   // a FLUT that fits in half the L2 stays resident: prefetching its rows only costs
        static int l2 = 0;
        if (!l2) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
            if (l2 <= 0) l2 = 126 << 20;
        }
        const int stride = shade->coef_stride > 0 ? shade->coef_stride
                                                  : (shade->degree + 1) * (shade->degree + 1) * shade->channels;
        a.no_row_prefetch = g_flut_l2_resident >= 0
                                ? g_flut_l2_resident
                                : flut_rows > 0 && (double)flut_rows * stride * 4.0 <= 0.5 * l2;
        a.n_rows = flut_rows;
    }
    if (n_views > 1) {  // several views of one tree in one launch (unsharded, own outputs)
        if (n_views > kMaxViews || sharded || (peer_out && peer_out[0])) return ARTEMIS_ERR_ARG;
        const int64_t n = (int64_t)width * height;
        for (int v = 0; v < n_views; ++v) {
            if (!outputs_ready)
                ARTEMIS_TRY(cudaMemsetAsync(Fv[v], 0, (size_t)n * shade->channels * sizeof(float), st));
            a.Fv[v] = Fv[v];
            a.Av[v] = Av[v];
            a.Dv[v] = Dv[v];
        }
        a.n_views = n_views;
        F = Fv[0];
        A = Av[0];
        D = Dv[0];
    }
    a.tile_order = sharded ? nullptr : tile_order;
    a.order_on = order_on;
    fill_tree(a, tree);
    fill_shade(a, shade);
    a.cam = cam_dev;
    a.queue = queue;
    const int64_t n = (int64_t)width * height;
    // peer outputs: another rank's full-frame buffers (initialised by their
    // owner); this launch writes exactly its own tiles' pixels into them
    const bool peer = peer_out && peer_out[0];
    if (peer) {
        F = static_cast<float *>(peer_out[0]);
        A = peer_out[1];
        D = peer_out[2];
    }
    if (!peer && n_views <= 1 && !outputs_ready)
        ARTEMIS_TRY(cudaMemsetAsync(F, 0, (size_t)n * shade->channels * sizeof(float), st));
    if (sharded && !peer && !outputs_ready) {  // pixels of other ranks' tiles: alpha 0, depth +inf
        const int g = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 4 * 148);
        if (maps64)
            fill_alpha_depth<double><<<g, 256, 0, st>>>(static_cast<double *>(A),
                                                        static_cast<double *>(D), n);
        else
            fill_alpha_depth<float><<<g, 256, 0, st>>>(static_cast<float *>(A),
                                                       static_cast<float *>(D), n);
    }
    a.tiles_x = (width + 7) / 8;
    a.tiles_y = (height + 3) / 4;
    a.n_rays = n;
    a.t_min = 0.0;
    a.t_max = HUGE_VAL;
    a.stop = 1.0 - lambda_th;
    a.sigma_dep = sigma_dep;
    a.early_stop = early_stop;
    a.F = F;
    if (maps64) {
        a.A64 = static_cast<double *>(A);
        a.D64 = static_cast<double *>(D);
    } else {
        a.A32 = static_cast<float *>(A);
        a.D32 = static_cast<float *>(D);
    }
    const int64_t warps = (int64_t)a.tiles_x * ((height + 3) / 4) * (n_views > 1 ? n_views : 1);
    // kRays: 1 / 2 camera rays with float / double maps, 3 / 4 the same over
    // several views
    if (n_views > 1)
        return maps64 ? launch_render_deg<kRender, 4>(shade->degree, a, warps, st)
                      : launch_render_deg<kRender, 3>(shade->degree, a, warps, st);
    return maps64 ? launch_render_deg<kRender, 2>(shade->degree, a, warps, st)
                  : launch_render_deg<kRender, 1>(shade->degree, a, warps, st);
}

__global__ void camera_rays_kernel(artemis_camera cam, double *og, double *dg, double *dw) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= (int64_t)cam.width * cam.height) return;
    double o[3], d[3], w[3];
    camera_ray(cam, (int)(p % cam.width), (int)(p / cam.width), o, d, w);
    for (int a = 0; a < 3; ++a) {
        og[3 * p + a] = o[a];
        dg[3 * p + a] = d[a];
        dw[3 * p + a] = w[a];
    }
}

template <typename Tin>
__global__ void flut_split_kernel(const Tin *__restrict__ flut, int64_t n, int width,
                                  float *__restrict__ coef, double *__restrict__ sigma) {
    const int64_t hc = width - 1;
    const int64_t total = n * width;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / width, c = i - r * width;
        const Tin v = flut[i];
        if (c == hc)
            sigma[r] = (double)v;
        else
            coef[r * hc + c] = (float)v;
    }
}

}  // namespace artemis

using namespace artemis;

// Launch helper for the API entry points: a stream-ordered 8-byte ray-queue
// counter around the launch.
template <typename Fn>
static int with_queue(RenderArgs &a, cudaStream_t st, Fn &&launch) {
    unsigned long long *q = nullptr;
    ARTEMIS_TRY(cudaMallocAsync(reinterpret_cast<void **>(&q), sizeof(*q), st));
    ARTEMIS_TRY(cudaMemsetAsync(q, 0, sizeof(*q), st));
    a.queue = q;
    int rc = launch();
    cudaFreeAsync(q, st);
    return rc;
}

static bool valid_common(const artemis_tree_view *t, const artemis_rays *r) {
    return t && r && t->nodes && t->leaves && r->n_rays >= 0 &&
           (r->n_rays == 0 || (r->origins_g && r->dirs_g));
}

extern "C" int artemis_render_rays(const artemis_tree_view *tree, const artemis_shading *shade,
                                   const artemis_rays *rays, double lambda_th, double sigma_dep,
                                   int early_stop, float *F, double *alpha, double *depth,
                                   artemis_stream stream) {
    if (!valid_common(tree, rays) || !shade || !rays->dirs_w || shade->channels < 1 ||
        shade->degree < 0 || shade->degree > 4 || !F || !alpha || !depth)
        return ARTEMIS_ERR_ARG;
    RenderArgs a{};
    fill_tree(a, tree);
    fill_shade(a, shade);
    fill_rays(a, rays);
    a.stop = 1.0 - lambda_th;
    a.sigma_dep = sigma_dep;
    a.early_stop = early_stop;
    a.F = F;
    a.A64 = alpha;
    a.D64 = depth;
    if (rays->n_rays == 0) return ARTEMIS_OK;
    ARTEMIS_TRY(cudaMemsetAsync(F, 0, (size_t)rays->n_rays * shade->channels * sizeof(float),
                                S(stream)));
    return with_queue(a, S(stream), [&] {
        return launch_render_deg<kRender, 0>(shade->degree, a,
                                                 ceil_div<int64_t>(rays->n_rays, 32), S(stream));
    });
}

extern "C" int artemis_count_hits(const artemis_tree_view *tree, const artemis_rays *rays,
                                  int64_t *counts, artemis_stream stream) {
    if (!valid_common(tree, rays) || !counts) return ARTEMIS_ERR_ARG;
    RenderArgs a{};
    fill_tree(a, tree);
    fill_rays(a, rays);
    a.channels = 1;
    a.counts = counts;
    if (rays->n_rays == 0) return ARTEMIS_OK;
    return with_queue(a, S(stream), [&] {
        return launch_render_deg<kCount, 0>(0, a, ceil_div<int64_t>(rays->n_rays, 32),
                                                S(stream));
    });
}

extern "C" int artemis_forward_fit(const artemis_tree_view *tree, const artemis_shading *shade,
                                   const artemis_rays *rays, const int64_t *offsets,
                                   int64_t *hit_idx, double *hit_t0, double *hit_t1, float *F,
                                   double *alpha, artemis_stream stream) {
    if (!valid_common(tree, rays) || !shade || !rays->dirs_w || !offsets || !F || !alpha ||
        shade->channels < 1 || shade->degree < 0 || shade->degree > 4)
        return ARTEMIS_ERR_ARG;
    RenderArgs a{};
    fill_tree(a, tree);
    fill_shade(a, shade);
    fill_rays(a, rays);
    a.stop = 2.0;
    a.sigma_dep = HUGE_VAL;
    a.early_stop = 0;
    a.F = F;
    a.A64 = alpha;
    a.offsets = offsets;
    a.hit_idx = hit_idx;
    a.hit_t0 = hit_t0;
    a.hit_t1 = hit_t1;
    if (rays->n_rays == 0) return ARTEMIS_OK;
    ARTEMIS_TRY(cudaMemsetAsync(F, 0, (size_t)rays->n_rays * shade->channels * sizeof(float),
                                S(stream)));
    return with_queue(a, S(stream), [&] {
        return launch_render_deg<kTrace, 0>(shade->degree, a,
                                                ceil_div<int64_t>(rays->n_rays, 32), S(stream));
    });
}

// Self-test of the reciprocal-corrected division the cell walk uses
// (bricks.cuh crossing): RN(q + (n - q d) r) with q = RN(n r), r = RN(1/d)
// must equal __ddiv_rn(n, d) bit for bit. Samples per thread cycle through
// regimes: walk-like (integer plane minus a grid-space origin over a grid
// direction), divisors with all-ones or all-zeros significands (the
// reciprocal's hardest cases), dividends one ulp off a divisor multiple,
// and random bit patterns over a wide normal exponent range.
__device__ __forceinline__ uint64_t splitmix(uint64_t &x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double rand_normal_bits(uint64_t &st, int emin, int emax) {
    const uint64_t b = splitmix(st);
    const int e = emin + (int)(splitmix(st) % (uint64_t)(emax - emin + 1));
    const uint64_t bits = ((uint64_t)(e + 1023) << 52) | (b & 0x000FFFFFFFFFFFFFull) |
                          (b & 0x8000000000000000ull);
    return __longlong_as_double((long long)bits);
}

__global__ void division_selftest_kernel(int64_t n, uint64_t seed,
                                         unsigned long long *mismatches, double *failed) {
    uint64_t st = seed ^ (0xD1B54A32D192ED03ull * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x));
    unsigned long long bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double num, d;
        switch (i & 3) {
            case 0: {  // walk-like: k - o over a grid-space direction
                const int k = (int)(splitmix(st) % 4096u) - 1024;
                const double o = (double)(splitmix(st) >> 11) * 0x1.0p-53 * 4096.0 - 1024.0;
                num = __dadd_rn((double)k, -o);
                d = rand_normal_bits(st, -12, 12);
                break;
            }
            case 1: {  // divisor significand all ones / all zeros
                const int e = (int)(splitmix(st) % 41u) - 20;
                const uint64_t mant = (splitmix(st) & 1) ? 0x000FFFFFFFFFFFFFull : 0ull;
                d = __longlong_as_double((long long)(((uint64_t)(e + 1023) << 52) | mant));
                if (splitmix(st) & 1) d = -d;
                num = rand_normal_bits(st, -30, 30);
                break;
            }
            case 2: {  // dividend one ulp off a multiple of the divisor
                d = rand_normal_bits(st, -20, 20);
                const double m = (double)(int64_t)(splitmix(st) % 100000u) - 50000.0;
                const double x = __dmul_rn(m, d);
                const int64_t step = (int64_t)(splitmix(st) % 3u) - 1;
                num = __longlong_as_double(__double_as_longlong(x) + step);
                break;
            }
            default:  // random patterns, wide normal range
                num = rand_normal_bits(st, -400, 400);
                d = rand_normal_bits(st, -400, 400);
        }
        if (d == 0.0 || !isfinite(num) || !isfinite(d)) continue;
        // div_fast where its operand-range contract holds (dividend 0 or in
        // [2^-400, 2^400], divisor in [2^-600, 2^600]), as the launches use it
        const bool in_range = div_operand_ok(num, 0x1p-400, 0x1p400) &&
                              div_operand_ok(d, 0x1p-600, 0x1p600);
        const double fast = in_range ? div_fast(num, d, __drcp_rn(d)) : __ddiv_rn(num, d);
        const double ref = __ddiv_rn(num, d);
        if (__double_as_longlong(fast) != __double_as_longlong(ref) && !(isnan(fast) && isnan(ref))) {
            ++bad;
            if (failed) {  // record a few (regime, n, d) for diagnosis
                const unsigned long long slot = atomicAdd(mismatches + 1, 1ull);
                if (slot < 16) {
                    failed[3 * slot] = (double)(i & 3);
                    failed[3 * slot + 1] = num;
                    failed[3 * slot + 2] = d;
                }
            }
        }
    }
    if (bad) atomicAdd(mismatches, bad);
}

extern "C" int artemis_debug_division_selftest(int64_t n, uint64_t seed,
                                               unsigned long long *mismatches_host,
                                               double *failed_host /* 48 doubles, may be NULL */) {
    if (n < 0 || !mismatches_host) return ARTEMIS_ERR_ARG;
    unsigned long long *d = nullptr;
    double *fd = nullptr;
    ARTEMIS_TRY(cudaMalloc(&d, 2 * sizeof(*d)));
    ARTEMIS_TRY(cudaMemset(d, 0, 2 * sizeof(*d)));
    ARTEMIS_TRY(cudaMalloc(&fd, 48 * sizeof(double)));
    ARTEMIS_TRY(cudaMemset(fd, 0, 48 * sizeof(double)));
    division_selftest_kernel<<<num_sms() * 8, 256>>>(n, seed, d, fd);
    int rc = ARTEMIS_LAUNCHED();
    if (!rc && failed_host)
        cudaMemcpy(failed_host, fd, 48 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(fd);
    if (!rc) {
        cudaError_t e = cudaMemcpy(mismatches_host, d, sizeof(*d), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            set_cuda_error(e);
            rc = ARTEMIS_ERR_CUDA;
        }
    }
    cudaFree(d);
    return rc;
}

extern "C" int artemis_debug_set_flut_l2_resident(int mode) {
    if (mode < -1 || mode > 1) return ARTEMIS_ERR_ARG;
    g_flut_l2_resident = mode;
    return ARTEMIS_OK;
}

extern "C" int artemis_debug_set_render_blocks(int max_blocks) {
    if (max_blocks < 0) return ARTEMIS_ERR_ARG;
    g_render_block_cap = max_blocks;
    return ARTEMIS_OK;
}

extern "C" int artemis_camera_rays(const artemis_camera *cam, double *og, double *dg, double *dw,
                                   artemis_stream stream) {
    if (!cam || !og || !dg || !dw || cam->width < 1 || cam->height < 1) return ARTEMIS_ERR_ARG;
    const int64_t n = (int64_t)cam->width * cam->height;
    camera_rays_kernel<<<(int)ceil_div<int64_t>(n, 256), 256, 0, S(stream)>>>(*cam, og, dg, dw);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_flut_split_f64(const double *flut, int64_t n, int width, float *coef,
                                      double *sigma, artemis_stream stream) {
    if (n < 0 || width < 1 || (n > 0 && (!flut || !sigma || (width > 1 && !coef))))
        return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_OK;
    const int blocks = (int)std::min<int64_t>(ceil_div<int64_t>(n * width, 256), 148 * 32);
    flut_split_kernel<double><<<blocks, 256, 0, S(stream)>>>(flut, n, width, coef, sigma);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_flut_split_f32(const float *flut, int64_t n, int width, float *coef,
                                      double *sigma, artemis_stream stream) {
    if (n < 0 || width < 1 || (n > 0 && (!flut || !sigma || (width > 1 && !coef))))
        return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_OK;
    const int blocks = (int)std::min<int64_t>(ceil_div<int64_t>(n * width, 256), 148 * 32);
    flut_split_kernel<float><<<blocks, 256, 0, S(stream)>>>(flut, n, width, coef, sigma);
    return ARTEMIS_LAUNCHED();
}
