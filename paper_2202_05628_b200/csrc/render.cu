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
#include <math_constants.h>

#include "common.cuh"
#include "tree.cuh"

namespace artemis {

namespace {
constexpr int kRenderWarps = 4;
constexpr int kRenderThreads = 32 * kRenderWarps;
constexpr int kSmemStack = 32;       // per-thread stack entries kept in shared memory
constexpr int kStack = 68;           // tree depth <= 64 key bits + super-root; overflow in local
constexpr int kStackBytes = kSmemStack * kRenderThreads * 4;
constexpr int kEnd = (int)0x80000000;  // empty-stack marker (never a node or ~leaf)
}  // namespace

enum RenderMode { kRender = 0, kTrace = 1, kCount = 2 };

struct RenderArgs {
    const PackedNode *nodes;
    const uint4 *leaves;  // {x, y, z, flut row}
    int64_t n_leaves;
    const int32_t *n_leaves_dev;
    // shading
    const float *coef;
    const double *sigma;
    const int32_t *rot_index;
    const double *rot_inv;
    int channels;
    int coef_stride;
    // rays: explicit arrays or a camera (device pointer, read once)
    const double *og, *dg, *dw;
    const artemis_camera *cam;
    int64_t n_rays;
    int tiles_x, tiles_y;  // camera mode: ceil(W / 8), ceil(H / 4)
    unsigned long long *queue;  // ray-id counter, zero at launch
    double t_min, t_max;
    double stop;  // 1 - lambda_th
    double sigma_dep;
    int early_stop;
    // outputs
    float *F;
    double *A64, *D64;
    float *A32, *D32;
    const int64_t *offsets;
    int64_t *hit_idx;
    double *hit_t0, *hit_t1;
    int64_t *counts;
};

// Ray/box overlap of the child box packed in (w0, w1, w2) within
// [t_min, t_max]; exact port of the slab test (_core.pyx:252-285).
__device__ __forceinline__ bool clip_exact(uint32_t w0, uint32_t w1, uint32_t w2,
                                           const double o[3], const double d[3], double t_min,
                                           double t_max, double &t0o, double &t1o) {
    const int fb = (int)((w0 >> 21) & 63u);
    const int lo_i[3] = {(int)(w0 & kCoordMask), (int)(w1 & kCoordMask), (int)(w2 & kCoordMask)};
    double t0 = t_min, t1 = t_max;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double lo = (double)lo_i[a];
        const double hi = (double)(lo_i[a] + box_size_axis(fb, a));
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

// Filtered hit test: the slab planes are scaled by a per-ray reciprocal
// instead of divided, which is within 3 ulp of the exact quotient; the
// decision t0 < t1 is taken from it only when the gap exceeds a bound far
// above that error (2^-50 relative), otherwise the exact test decides. So
// the answer always equals clip_exact's; only its cost differs.
__device__ __forceinline__ bool hit_filtered(uint32_t w0, uint32_t w1, uint32_t w2,
                                             const double o[3], const double d[3],
                                             const double inv[3], double t_min, double t_max) {
    const int fb = (int)((w0 >> 21) & 63u);
    const int lo_i[3] = {(int)(w0 & kCoordMask), (int)(w1 & kCoordMask), (int)(w2 & kCoordMask)};
    double t0 = t_min, t1 = t_max;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double lo = (double)lo_i[a];
        const double hi = (double)(lo_i[a] + box_size_axis(fb, a));
        if (d[a] == 0.0) {
            if (o[a] < lo || o[a] >= hi) return false;
        } else {
            double ta = (lo - o[a]) * inv[a];
            double tb = (hi - o[a]) * inv[a];
            t0 = fmax(t0, fmin(ta, tb));
            t1 = fmin(t1, fmax(ta, tb));
        }
    }
    const double m = 8.881784197001252e-16 * (fabs(t0) + (isinf(t1) ? 0.0 : fabs(t1)));
    if (t0 + m < t1) return true;
    if (t0 > t1 + m) return false;
    double e0, e1;
    return clip_exact(w0, w1, w2, o, d, t_min, t_max, e0, e1);
}

template <int kDeg>
__device__ __forceinline__ void sh_basis_f(float x, float y, float z, float *Y) {
    Y[0] = 0.28209479177387814f;
    if (kDeg >= 1) {
        Y[1] = 0.4886025119029199f * y;
        Y[2] = 0.4886025119029199f * z;
        Y[3] = 0.4886025119029199f * x;
    }
    if (kDeg >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        Y[4] = 1.0925484305920792f * x * y;
        Y[5] = 1.0925484305920792f * y * z;
        Y[6] = 0.31539156525252005f * (3.0f * zz - 1.0f);
        Y[7] = 1.0925484305920792f * x * z;
        Y[8] = 0.5462742152960396f * (xx - yy);
        if (kDeg >= 3) {
            Y[9] = 0.5900435899266435f * y * (3.0f * xx - yy);
            Y[10] = 2.890611442640554f * x * y * z;
            Y[11] = 0.4570457994644658f * y * (5.0f * zz - 1.0f);
            Y[12] = 0.3731763325901154f * z * (5.0f * zz - 3.0f);
            Y[13] = 0.4570457994644658f * x * (5.0f * zz - 1.0f);
            Y[14] = 1.445305721320277f * z * (xx - yy);
            Y[15] = 0.5900435899266435f * x * (xx - 3.0f * yy);
        }
        if (kDeg >= 4) {
            Y[16] = 2.5033429417967046f * x * y * (xx - yy);
            Y[17] = 1.7701307697799304f * y * z * (3.0f * xx - yy);
            Y[18] = 0.9461746957575601f * x * y * (7.0f * zz - 1.0f);
            Y[19] = 0.6690465435572892f * y * z * (7.0f * zz - 3.0f);
            Y[20] = 0.10578554691520431f * (zz * (35.0f * zz - 30.0f) + 3.0f);
            Y[21] = 0.6690465435572892f * x * z * (7.0f * zz - 3.0f);
            Y[22] = 0.47308734787878004f * (xx - yy) * (7.0f * zz - 1.0f);
            Y[23] = 1.7701307697799304f * x * z * (xx - 3.0f * yy);
            Y[24] = 0.6258357354491761f * (xx * (xx - 3.0f * yy) - yy * (3.0f * xx - yy));
        }
    }
}

// Exact per-pixel ray of rays_for_camera + _grid_rays (see artemis.h).
__device__ __forceinline__ void camera_ray(const artemis_camera &c, int u, int v, double og[3],
                                           double dg[3], double dw[3]) {
    const double c0 = __ddiv_rn(__dadd_rn(__dadd_rn((double)u, 0.5), -c.cx), c.fx);
    const double c1 = __ddiv_rn(__dadd_rn(__dadd_rn((double)v, 0.5), -c.cy), c.fy);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        d[a] = __fma_rn(1.0, c.R[3 * a + 2], __fma_rn(c1, c.R[3 * a + 1], __dmul_rn(c0, c.R[3 * a])));
    const double nrm = __dsqrt_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        dw[a] = __ddiv_rn(d[a], nrm);
        dg[a] = __ddiv_rn(dw[a], c.cell[a]);
        og[a] = __ddiv_rn(__dadd_rn(c.origin[a], -c.lo[a]), c.cell[a]);
    }
}

// Persistent warps pull rays from a global queue (ids in 8x4 pixel-tile order
// in camera mode) and refill idle lanes as rays finish, so SIMD lanes stay
// busy despite the ~6x spread of per-ray work. Each lane walks its ray's
// DFS with a stack in shared memory (column per thread, so lanes at
// different depths never bank-conflict). Child visiting order uses the
// split axis: the two children's octants are separated by the plane of the
// node's highest differing Morton bit, so when both are hit the one on the
// ray's side of that plane has the smaller entry distance -- the order the
// reference's `lt0 <= rt0` comparison yields (_core.pyx:345), without
// computing either distance. Internal-node tests use the filtered predicate;
// emitted leaves get exact fp64 intervals. Visible hits of a round are then
// shaded by lane groups.
template <int kDeg, int kMode, bool kCamera, bool kVec>
__global__ void __launch_bounds__(kRenderThreads) render_kernel(RenderArgs p) {
    constexpr int H = (kDeg + 1) * (kDeg + 1);
    extern __shared__ __align__(16) unsigned char s_raw[];
    int *s_stack = reinterpret_cast<int *>(s_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = p.channels;
    const int cp = kVec ? C + 4 : (C | 1);
    float *feat = reinterpret_cast<float *>(s_raw + kStackBytes) + (size_t)warp * 32 * cp;
    if (kMode != kCount)
        for (int i = lane; i < 32 * cp; i += 32) feat[i] = 0.0f;
    const int64_t n_leaves = p.n_leaves_dev ? (int64_t)*p.n_leaves_dev : p.n_leaves;
    const int super_root = (int)(n_leaves > 1 ? n_leaves - 1 : 0);
    const int64_t n_ids = kCamera ? (int64_t)p.tiles_x * p.tiles_y * 32 : p.n_rays;
    const unsigned lt = lanemask_lt();

    // per-lane ray state
    int64_t ray = -1;
    bool alive = false;
    double og[3], dg[3], dw[3], inv[3];
    double T = 1.0, acc = 0.0, depth = CUDART_INF;
    int64_t hits = 0, trace_base = 0;
    int cur = kEnd, top = 0;
    int ovf[kStack - kSmemStack];
    bool queue_open = true;

    auto push = [&](int v) {
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
    // next occupied leaf front to back (_core.pyx:307-355 order)
    auto next_hit = [&](int &leaf, double &t0, double &t1, uint32_t &fidx) -> bool {
        while (cur != kEnd) {
            if (cur >= 0) {
                const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p.nodes + cur));
                const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p.nodes + cur) + 1);
                const bool hl = hit_filtered(a.x, a.y, a.z, og, dg, inv, p.t_min, p.t_max);
                const bool hr = !(b.x & kAbsent) &&
                                hit_filtered(b.x, b.y, b.z, og, dg, inv, p.t_min, p.t_max);
                int nxt;
                uint4 nb;
                if (hl && hr) {
                    const bool left_first = dg[(a.x >> 27) & 3u] > 0.0;
                    push(left_first ? (int)b.w : (int)a.w);
                    nb = left_first ? a : b;
                } else if (hl) {
                    nb = a;
                } else if (hr) {
                    nb = b;
                } else {
                    cur = pop();
                    continue;
                }
                nxt = (int)nb.w;
                if (nxt >= 0) {
                    cur = nxt;  // internal nodes were just tested: expand directly
                    continue;
                }
                cur = pop();
                double e0, e1;
                if (clip_exact(nb.x, nb.y, nb.z, og, dg, p.t_min, p.t_max, e0, e1) && e1 > e0) {
                    leaf = ~nxt;
                    t0 = e0;
                    t1 = e1;
                    fidx = __ldg(&p.leaves[leaf].w);
                    return true;
                }
                continue;
            }
            leaf = ~cur;
            const uint4 L = __ldg(p.leaves + leaf);
            cur = pop();
            double e0, e1;
            if (clip_exact(L.x, L.y, L.z, og, dg, p.t_min, p.t_max, e0, e1) && e1 > e0) {
                t0 = e0;
                t1 = e1;
                fidx = L.w;
                return true;
            }
        }
        return false;
    };
    auto start_ray = [&](int64_t id) {
        ray = -1;
        if (kCamera) {
            const artemis_camera &cam = *p.cam;
            const int64_t tile = id >> 5;
            const int sl = (int)(id & 31);
            const int px = (int)(tile % p.tiles_x) * 8 + (sl & 7);
            const int py = (int)(tile / p.tiles_x) * 4 + (sl >> 3);
            if (py < cam.height && px < cam.width) {
                ray = (int64_t)py * cam.width + px;
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
#pragma unroll
        for (int a = 0; a < 3; ++a) inv[a] = dg[a] != 0.0 ? 1.0 / dg[a] : 0.0;
        T = 1.0;
        acc = 0.0;
        depth = CUDART_INF;
        hits = 0;
        top = 0;
        trace_base = (kMode == kTrace) ? p.offsets[ray] : 0;
        cur = n_leaves > 0 ? super_root : kEnd;
        alive = true;
    };
    auto finish_ray = [&]() {
        if (kMode == kCount) {
            p.counts[ray] = hits;
        } else {
            if (p.A64) p.A64[ray] = acc;
            if (p.A32) p.A32[ray] = (float)acc;
            if (kMode == kRender) {
                if (p.D64) p.D64[ray] = depth;
                if (p.D32) p.D32[ray] = (float)depth;
            }
        }
    };

    // cooperative shading geometry: lph lanes per hit, hpi hits per pass
    const int units = kVec ? C / 4 : C;
    int lph = 1;
    while (lph < units && lph < 32) lph <<= 1;
    const int hpi = 32 / lph;
    const int grp = lane / lph, q = lane % lph;

    while (true) {
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
        // ---- one traversal step per live lane
        int leaf = 0;
        double t0 = 0.0, t1 = 0.0;
        uint32_t fidx = 0;
        bool have = false;
        if (alive) {
            have = next_hit(leaf, t0, t1, fidx);
            if (!have) alive = false;
        }
        bool shade = false;
        float af = 0.0f, cx = 0.0f, cy = 0.0f, cz = 0.0f;
        if (have) {
            if (kMode == kCount) {
                ++hits;
            } else {
                const double sigma = __ldg(p.sigma + fidx);
                const double delta = t1 - t0;
                if (kMode == kRender && depth == CUDART_INF && sigma > p.sigma_dep) depth = t0;
                const double em = exp(-sigma * delta);
                const double a = T * (1.0 - em);
                if (a > 0.0) {
                    shade = true;
                    af = (float)a;
                    const double *R = p.rot_inv + 9 * __ldg(p.rot_index + fidx);
                    cx = (float)(R[0] * dw[0] + R[1] * dw[1] + R[2] * dw[2]);
                    cy = (float)(R[3] * dw[0] + R[4] * dw[1] + R[5] * dw[2]);
                    cz = (float)(R[6] * dw[0] + R[7] * dw[1] + R[8] * dw[2]);
                    acc = acc + a;
                }
                T = T * em;
                if (kMode == kTrace) {
                    p.hit_idx[trace_base + hits] = (int64_t)fidx;
                    p.hit_t0[trace_base + hits] = t0;
                    p.hit_t1[trace_base + hits] = t1;
                }
                ++hits;
                if (kMode == kRender && p.early_stop && acc > p.stop) alive = false;
            }
        }
        if (kMode != kCount) {
            unsigned m = __ballot_sync(0xffffffffu, shade);
            while (m) {
                const unsigned src = __fns(m, 0, grp + 1);
                const bool ok = src < 32;
                const int s = ok ? (int)src : 0;
                const uint32_t bf = __shfl_sync(0xffffffffu, fidx, s);
                const float ba = __shfl_sync(0xffffffffu, af, s);
                const float bx = __shfl_sync(0xffffffffu, cx, s);
                const float by = __shfl_sync(0xffffffffu, cy, s);
                const float bz = __shfl_sync(0xffffffffu, cz, s);
                if (ok) {
                    float Y[H];
                    sh_basis_f<kDeg>(bx, by, bz, Y);
                    if (kVec) {
                        const float4 *row =
                            reinterpret_cast<const float4 *>(p.coef + (size_t)bf * p.coef_stride);
                        float4 *dst = reinterpret_cast<float4 *>(feat + s * cp);
                        for (int c4 = q; c4 < units; c4 += lph) {
                            float4 v[H];
#pragma unroll
                            for (int h = 0; h < H; ++h) v[h] = __ldg(row + h * units + c4);
                            float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f;
#pragma unroll
                            for (int h = 0; h < H; ++h) {
                                ax = fmaf(v[h].x, Y[h], ax);
                                ay = fmaf(v[h].y, Y[h], ay);
                                az = fmaf(v[h].z, Y[h], az);
                                aw = fmaf(v[h].w, Y[h], aw);
                            }
                            float4 f = dst[c4];
                            f.x += ba * ax;
                            f.y += ba * ay;
                            f.z += ba * az;
                            f.w += ba * aw;
                            dst[c4] = f;
                        }
                    } else {
                        const float *row = p.coef + (size_t)bf * p.coef_stride;
                        for (int c = q; c < C; c += lph) {
                            float acc_c = 0.0f;
#pragma unroll
                            for (int h = 0; h < H; ++h)
                                acc_c = fmaf(__ldg(row + h * C + c), Y[h], acc_c);
                            feat[s * cp + c] += ba * acc_c;
                        }
                    }
                }
                for (int k = 0; k < hpi && m; ++k) m &= m - 1;
            }
        }
        // ---- retire finished rays: scalars per lane, features row by row
        const bool done = ray >= 0 && !alive;
        if (done) finish_ray();
        if (kMode != kCount) {
            unsigned fm = __ballot_sync(0xffffffffu, done && acc > 0.0);
            __syncwarp();
            while (fm) {
                const int s = __ffs(fm) - 1;
                fm &= fm - 1;
                const int64_t r = __shfl_sync(0xffffffffu, ray, s);
                for (int c = lane; c < C; c += 32) {
                    p.F[r * C + c] = feat[s * cp + c];
                    feat[s * cp + c] = 0.0f;
                }
            }
            __syncwarp();
            // a retired ray with acc == 0 never touched its row (rows start at
            // zero and F was cleared before the launch)
        }
        if (done) ray = -1;
    }
}

template <int kMode, bool kCamera, bool kVec>
int launch_render_vec(int degree, const RenderArgs &a, int64_t warps, cudaStream_t st) {
    if (warps == 0) return ARTEMIS_OK;
    const int cp = kVec ? a.channels + 4 : (a.channels | 1);
    const size_t smem = kStackBytes + (kMode == kCount ? 0 : (size_t)kRenderWarps * 32 * cp * 4);
    const int64_t want = ceil_div<int64_t>(warps, kRenderWarps);
    switch (degree) {
#define ARTEMIS_LAUNCH(D)                                                                       \
    case D: {                                                                                   \
        auto kern = render_kernel<D, kMode, kCamera, kVec>;                                     \
        if (smem > 48 * 1024)                                                                   \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        int occ = 0;                                                                            \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRenderThreads, smem);        \
        const int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * (occ > 0 ? occ : 1)); \
        kern<<<blocks, kRenderThreads, smem, st>>>(a);                                          \
        break;                                                                                  \
    }
        ARTEMIS_LAUNCH(0) ARTEMIS_LAUNCH(1) ARTEMIS_LAUNCH(2) ARTEMIS_LAUNCH(3) ARTEMIS_LAUNCH(4)
#undef ARTEMIS_LAUNCH
        default:
            return ARTEMIS_ERR_ARG;
    }
    return ARTEMIS_LAUNCHED();
}

template <int kMode, bool kCamera>
int launch_render_deg(int degree, const RenderArgs &a, int64_t warps, cudaStream_t st) {
    const bool vec = kMode != kCount && a.channels % 4 == 0 && a.coef_stride % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(a.coef) & 15) == 0;
    return vec ? launch_render_vec<kMode, kCamera, true>(degree, a, warps, st)
               : launch_render_vec<kMode, kCamera, false>(degree, a, warps, st);
}

static void fill_tree(RenderArgs &a, const artemis_tree_view *t) {
    a.nodes = static_cast<const PackedNode *>(t->nodes);
    a.leaves = static_cast<const uint4 *>(t->leaves);
    a.n_leaves = t->n_leaves;
    a.n_leaves_dev = t->n_leaves_dev;
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
}

// Device-pipeline render with in-kernel camera rays (frame.cu).
int render_camera(const artemis_tree_view *tree, const artemis_shading *shade,
                  const artemis_camera *cam_dev, int width, int height, double lambda_th,
                  double sigma_dep, int early_stop, float *F, float *A, float *D,
                  unsigned long long *queue, cudaStream_t st) {
    RenderArgs a{};
    fill_tree(a, tree);
    fill_shade(a, shade);
    a.cam = cam_dev;
    a.queue = queue;
    ARTEMIS_TRY(cudaMemsetAsync(F, 0, (size_t)width * height * shade->channels * sizeof(float), st));
    a.tiles_x = (width + 7) / 8;
    a.tiles_y = (height + 3) / 4;
    a.n_rays = (int64_t)width * height;
    a.t_min = 0.0;
    a.t_max = HUGE_VAL;
    a.stop = 1.0 - lambda_th;
    a.sigma_dep = sigma_dep;
    a.early_stop = early_stop;
    a.F = F;
    a.A32 = A;
    a.D32 = D;
    const int64_t warps = (int64_t)a.tiles_x * ((height + 3) / 4);
    return launch_render_deg<kRender, true>(shade->degree, a, warps, st);
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
        return launch_render_deg<kRender, false>(shade->degree, a,
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
        return launch_render_deg<kCount, false>(0, a, ceil_div<int64_t>(rays->n_rays, 32),
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
        return launch_render_deg<kTrace, false>(shade->degree, a,
                                                ceil_div<int64_t>(rays->n_rays, 32), S(stream));
    });
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
