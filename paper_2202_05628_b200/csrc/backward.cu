// Analytic FLUT gradients of a traced ray batch (training path, SURVEY.md
// section 8f row 1). Replaces animvox/_core.pyx:661-755 backward_rays
// (driven by fit.py:108-146 backward_batch and fit.py:474-492).
//
// Per ray the reference walks its CSR hit list front to back (alpha chain,
// coefficient gradients a * dL/dF_c * Y_h, the per-hit scalar
// g = dL/dalpha + sum_c dL/dF_c * s_c) and then back to front (density
// gradient delta * (g T e - suffix)). In deterministic mode it adds every
// contribution to grad[i, col] serially, rays in ascending order.
//
// B200 mapping, three stages, all deterministic:
//  1. bwd_ray_kernel: one warp per ray. Lanes split the channels to form
//     s_c (row gather, fp64, the reference's h order); lane 0 runs the ray's
//     sequential chains (g in channel order, T, alpha, then the reverse
//     suffix) and leaves per-hit records {a, g, T, e, delta, w_sigma, ray}.
//  2. a stable onesweep sort of the hits by FLUT row (sort.cu): within a
//     row the hits stay in CSR order, i.e. ascending ray -- exactly the
//     order the reference's serial loop adds them in.
//  3. bwd_accum_kernel: one warp per touched row (segment heads are listed
//     with an atomic counter; segment order is irrelevant, in-segment order
//     is the sorted order). Lane = column; each lane sums its column's
//     contributions in ray order in a real_t register and writes it once.
// No atomics touch gradient values, so the result is bit-reproducible and
// equals the reference's serial sum given the same per-hit terms. All fp64
// arithmetic uses explicitly rounded intrinsics (no FMA contraction), as the
// reference's x86-64 build (no -march) computes it; exp is CUDA's (<= 1 ulp
// from glibc's), the only source of difference.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace artemis {

template <typename K>
int sort_pairs(const K *keys_in, const uint32_t *vals_in, K *keys_out, uint32_t *vals_out,
               int64_t n, int key_bits, void *ws, size_t ws_bytes, cudaStream_t st);
size_t sort_workspace_bytes(int64_t n, int key_bits, int key_bytes);

namespace {

constexpr int kBwdWarps = 4;

#define DM __dmul_rn
#define DA __dadd_rn

// Real SH basis up to degree 4 (_core.pyx:420-451), each product and sum
// rounded as written there, left to right.
__device__ __forceinline__ void sh_basis_d(int degree, double x, double y, double z, double *Y) {
    Y[0] = 0.28209479177387814;
    if (degree >= 1) {
        Y[1] = DM(0.4886025119029199, y);
        Y[2] = DM(0.4886025119029199, z);
        Y[3] = DM(0.4886025119029199, x);
    }
    if (degree >= 2) {
        const double xx = DM(x, x), yy = DM(y, y), zz = DM(z, z);
        Y[4] = DM(DM(1.0925484305920792, x), y);
        Y[5] = DM(DM(1.0925484305920792, y), z);
        Y[6] = DM(0.31539156525252005, DA(DM(3.0, zz), -1.0));
        Y[7] = DM(DM(1.0925484305920792, x), z);
        Y[8] = DM(0.5462742152960396, DA(xx, -yy));
        if (degree >= 3) {
            Y[9] = DM(DM(0.5900435899266435, y), DA(DM(3.0, xx), -yy));
            Y[10] = DM(DM(DM(2.890611442640554, x), y), z);
            Y[11] = DM(DM(0.4570457994644658, y), DA(DM(5.0, zz), -1.0));
            Y[12] = DM(DM(0.3731763325901154, z), DA(DM(5.0, zz), -3.0));
            Y[13] = DM(DM(0.4570457994644658, x), DA(DM(5.0, zz), -1.0));
            Y[14] = DM(DM(1.445305721320277, z), DA(xx, -yy));
            Y[15] = DM(DM(0.5900435899266435, x), DA(xx, -DM(3.0, yy)));
        }
        if (degree >= 4) {
            Y[16] = DM(DM(DM(2.5033429417967046, x), y), DA(xx, -yy));
            Y[17] = DM(DM(DM(1.7701307697799304, y), z), DA(DM(3.0, xx), -yy));
            Y[18] = DM(DM(DM(0.9461746957575601, x), y), DA(DM(7.0, zz), -1.0));
            Y[19] = DM(DM(DM(0.6690465435572892, y), z), DA(DM(7.0, zz), -3.0));
            Y[20] = DM(0.10578554691520431, DA(DM(zz, DA(DM(35.0, zz), -30.0)), 3.0));
            Y[21] = DM(DM(DM(0.6690465435572892, x), z), DA(DM(7.0, zz), -3.0));
            Y[22] = DM(DM(0.47308734787878004, DA(xx, -yy)), DA(DM(7.0, zz), -1.0));
            Y[23] = DM(DM(DM(1.7701307697799304, x), z), DA(xx, -DM(3.0, yy)));
            Y[24] = DM(0.6258357354491761,
                       DA(DM(xx, DA(xx, -DM(3.0, yy))), -DM(yy, DA(DM(3.0, xx), -yy))));
        }
    }
}

// Canonical-frame direction of a world ray for FLUT row i (_core.pyx:741-743).
__device__ __forceinline__ void canon_dir(const double *R, const double *w, double &x, double &y,
                                          double &z) {
    x = DA(DA(DM(R[0], w[0]), DM(R[1], w[1])), DM(R[2], w[2]));
    y = DA(DA(DM(R[3], w[0]), DM(R[4], w[1])), DM(R[5], w[2]));
    z = DA(DA(DM(R[6], w[0]), DM(R[7], w[1])), DM(R[8], w[2]));
}

struct BwdArgs {
    const int64_t *off;
    int64_t n_rays;
    const int64_t *hit_idx;
    const double *t0, *t1;
    int64_t n_hits;
    const double *dw;
    const int32_t *rot_index;
    const double *rot_inv;
    const void *flut, *dldf, *dlda;
    int width, degree, channels;
    // per-hit records
    double *h_a, *h_g, *h_T, *h_e, *h_d, *h_ws;
    uint32_t *h_ray, *keys;
    // sorted
    const uint32_t *skeys, *sperm;
    uint32_t *heads;
    unsigned int *n_heads;
    void *grad;
};

template <typename R>
__global__ void __launch_bounds__(32 * kBwdWarps) bwd_ray_kernel(BwdArgs p) {
    extern __shared__ double s_prod[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int C = p.channels, W = p.width, hc = W - 1;
    const int H = (p.degree + 1) * (p.degree + 1);
    double *prod = s_prod + (size_t)wib * C;
    const R *flut = static_cast<const R *>(p.flut);
    const R *dldf = static_cast<const R *>(p.dldf);
    const R *dlda = static_cast<const R *>(p.dlda);
    const int64_t wstride = (int64_t)gridDim.x * kBwdWarps;
    for (int64_t r = blockIdx.x * (int64_t)kBwdWarps + wib; r < p.n_rays; r += wstride) {
        const int64_t s0 = p.off[r], m = p.off[r + 1] - s0;
        if (m <= 0) continue;
        for (int64_t k = lane; k < m; k += 32) {
            p.h_ray[s0 + k] = (uint32_t)r;
            p.keys[s0 + k] = (uint32_t)p.hit_idx[s0 + k];
        }
        const double w[3] = {p.dw[3 * r], p.dw[3 * r + 1], p.dw[3 * r + 2]};
        double T = 1.0;
        for (int64_t k = 0; k < m; ++k) {
            const int64_t i = p.hit_idx[s0 + k];
            double cx, cy, cz, Y[25];
            canon_dir(p.rot_inv + 9 * p.rot_index[i], w, cx, cy, cz);
            sh_basis_d(p.degree, cx, cy, cz, Y);
            const R *row = flut + i * (int64_t)W;
            for (int c = lane; c < C; c += 32) {
                double s = 0.0;
                for (int h = 0; h < H; ++h) s = DA(s, DM((double)row[h * C + c], Y[h]));
                prod[c] = DM((double)dldf[r * C + c], s);
            }
            __syncwarp();
            if (lane == 0) {
                double g = (double)dlda[r];
                for (int c = 0; c < C; ++c) g = DA(g, prod[c]);
                const double sigma = (double)row[hc];
                const double delta = DA(p.t1[s0 + k], -p.t0[s0 + k]);
                const double e = exp(DM(-sigma, delta));
                const double a = DM(T, DA(1.0, -e));
                p.h_a[s0 + k] = a;
                p.h_g[s0 + k] = g;
                p.h_T[s0 + k] = T;
                p.h_e[s0 + k] = e;
                p.h_d[s0 + k] = delta;
                T = DM(T, e);
            }
            __syncwarp();
        }
        if (lane == 0) {  // back to front: density gradient (_core.pyx:746-755)
            double suffix = 0.0;
            for (int64_t k = m - 1; k >= 0; --k) {
                const int64_t j = s0 + k;
                const double gt = DM(DM(p.h_g[j], p.h_T[j]), p.h_e[j]);
                p.h_ws[j] = DM(p.h_d[j], DA(gt, -suffix));
                suffix = DA(suffix, DM(p.h_g[j], p.h_a[j]));
            }
        }
        __syncwarp();
    }
}

// Segment heads of the row-sorted hits (order of the list is irrelevant).
__global__ void bwd_heads_kernel(const uint32_t *__restrict__ skeys, int64_t n,
                                 uint32_t *__restrict__ heads, unsigned int *__restrict__ count) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        if (j == 0 || skeys[j] != skeys[j - 1]) heads[atomicAdd(count, 1u)] = (uint32_t)j;
    }
}

template <typename R>
__global__ void __launch_bounds__(32 * kBwdWarps) bwd_accum_kernel(BwdArgs p) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int C = p.channels, W = p.width, hc = W - 1;
    const R *dldf = static_cast<const R *>(p.dldf);
    R *grad = static_cast<R *>(p.grad);
    const int64_t n_seg = *p.n_heads;
    const int64_t wstride = (int64_t)gridDim.x * kBwdWarps;
    for (int64_t s = blockIdx.x * (int64_t)kBwdWarps + wib; s < n_seg; s += wstride) {
        const int64_t start = p.heads[s];
        const uint32_t leaf = p.skeys[start];
        int64_t end = start + 1;
        while (end < p.n_hits && p.skeys[end] == leaf) ++end;
        const double *Rm = p.rot_inv + 9 * p.rot_index[leaf];
        for (int col0 = 0; col0 < W; col0 += 32) {
            const int col = col0 + lane;
            const int h = col < hc ? col / C : 0, c = col < hc ? col - h * C : 0;
            R acc = (R)0;
            for (int64_t j = start; j < end; ++j) {
                const uint32_t hit = p.sperm[j];
                double v;
                if (col < hc) {
                    const uint32_t r = p.h_ray[hit];
                    double cx, cy, cz, Y[25];
                    canon_dir(Rm, p.dw + 3 * (size_t)r, cx, cy, cz);
                    sh_basis_d(p.degree, cx, cy, cz, Y);
                    v = DM(DM(p.h_a[hit], (double)dldf[(size_t)r * C + c]), Y[h]);
                } else {
                    v = p.h_ws[hit];
                }
                acc = acc + (R)v;
            }
            if (col < W) grad[(size_t)leaf * W + col] = acc;
        }
    }
}

#undef DM
#undef DA

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

struct BwdWs {
    double *a, *g, *T, *e, *d, *ws;
    uint32_t *ray, *keys, *skeys, *sperm, *heads;
    unsigned int *count;
    void *sort_ws;
    size_t sort_bytes, total;
};

BwdWs carve(void *base, int64_t m, int key_bits) {
    BwdWs w{};
    char *p = static_cast<char *>(base);
    size_t o = 0;
    auto take = [&](size_t bytes) {
        char *q = p ? p + o : nullptr;
        o += align256(bytes);
        return q;
    };
    const size_t mm = (size_t)std::max<int64_t>(m, 1);
    w.a = reinterpret_cast<double *>(take(8 * mm));
    w.g = reinterpret_cast<double *>(take(8 * mm));
    w.T = reinterpret_cast<double *>(take(8 * mm));
    w.e = reinterpret_cast<double *>(take(8 * mm));
    w.d = reinterpret_cast<double *>(take(8 * mm));
    w.ws = reinterpret_cast<double *>(take(8 * mm));
    w.ray = reinterpret_cast<uint32_t *>(take(4 * mm));
    w.keys = reinterpret_cast<uint32_t *>(take(4 * mm));
    w.skeys = reinterpret_cast<uint32_t *>(take(4 * mm));
    w.sperm = reinterpret_cast<uint32_t *>(take(4 * mm));
    w.heads = reinterpret_cast<uint32_t *>(take(4 * mm));
    w.count = reinterpret_cast<unsigned int *>(take(8));
    w.sort_bytes = sort_workspace_bytes(m, key_bits, 4);
    w.sort_ws = take(w.sort_bytes);
    w.total = o;
    return w;
}

int key_bits_for(int64_t n_flut) {
    int b = 1;
    while (b < 32 && (int64_t(1) << b) < n_flut) ++b;
    return b;
}

}  // namespace
}  // namespace artemis

using namespace artemis;

extern "C" size_t artemis_backward_workspace_bytes(int64_t n_hits, int64_t n_flut) {
    return carve(nullptr, n_hits, key_bits_for(n_flut)).total;
}

extern "C" int artemis_backward_rays(const int64_t *offsets, int64_t n_rays,
                                     const int64_t *hit_idx, const double *hit_t0,
                                     const double *hit_t1, int64_t n_hits, const double *dirs_w,
                                     const int32_t *rot_index, const double *rot_inv,
                                     const void *flut, int64_t n_flut, int width,
                                     const void *dldf, const void *dlda, int real_bytes,
                                     int degree, int channels, int deterministic, void *grad,
                                     void *workspace, size_t workspace_bytes,
                                     artemis_stream stream) {
    (void)deterministic;  // one deterministic schedule serves both modes
    if (n_rays < 0 || n_hits < 0 || n_flut < 1 || width < 1 || channels < 1 || degree < 0 ||
        degree > 4 || width != (degree + 1) * (degree + 1) * channels + 1 ||
        (real_bytes != 4 && real_bytes != 8) || !grad || n_flut >= (int64_t(1) << 32) ||
        n_hits >= (int64_t(1) << 30))
        return ARTEMIS_ERR_ARG;
    cudaStream_t st = S(stream);
    ARTEMIS_TRY(cudaMemsetAsync(grad, 0, (size_t)n_flut * width * real_bytes, st));
    if (n_rays == 0 || n_hits == 0) return ARTEMIS_OK;
    if (!offsets || !hit_idx || !hit_t0 || !hit_t1 || !dirs_w || !rot_index || !rot_inv ||
        !flut || !dldf || !dlda || !workspace)
        return ARTEMIS_ERR_ARG;
    const int kb = key_bits_for(n_flut);
    const BwdWs w = carve(workspace, n_hits, kb);
    if (workspace_bytes < w.total) return ARTEMIS_ERR_WORKSPACE;
    BwdArgs a{};
    a.off = offsets;
    a.n_rays = n_rays;
    a.hit_idx = hit_idx;
    a.t0 = hit_t0;
    a.t1 = hit_t1;
    a.n_hits = n_hits;
    a.dw = dirs_w;
    a.rot_index = rot_index;
    a.rot_inv = rot_inv;
    a.flut = flut;
    a.dldf = dldf;
    a.dlda = dlda;
    a.width = width;
    a.degree = degree;
    a.channels = channels;
    a.h_a = w.a;
    a.h_g = w.g;
    a.h_T = w.T;
    a.h_e = w.e;
    a.h_d = w.d;
    a.h_ws = w.ws;
    a.h_ray = w.ray;
    a.keys = w.keys;
    a.skeys = w.skeys;
    a.sperm = w.sperm;
    a.heads = w.heads;
    a.n_heads = w.count;
    a.grad = grad;
    const int threads = 32 * kBwdWarps;
    const size_t smem = (size_t)kBwdWarps * channels * sizeof(double);
    if (smem > 48 * 1024) return ARTEMIS_ERR_ARG;
    const int ray_blocks =
        (int)std::min<int64_t>(ceil_div<int64_t>(n_rays, kBwdWarps), (int64_t)num_sms() * 16);
    if (real_bytes == 8)
        bwd_ray_kernel<double><<<ray_blocks, threads, smem, st>>>(a);
    else
        bwd_ray_kernel<float><<<ray_blocks, threads, smem, st>>>(a);
    int rc = ARTEMIS_LAUNCHED();
    if (rc) return rc;
    rc = sort_pairs<uint32_t>(w.keys, nullptr, w.skeys, w.sperm, n_hits, kb, w.sort_ws, w.sort_bytes, st);
    if (rc) return rc;
    ARTEMIS_TRY(cudaMemsetAsync(w.count, 0, sizeof(unsigned int), st));
    const int hb = (int)std::min<int64_t>(ceil_div<int64_t>(n_hits, 256), (int64_t)num_sms() * 16);
    bwd_heads_kernel<<<hb, 256, 0, st>>>(w.skeys, n_hits, w.heads, w.count);
    rc = ARTEMIS_LAUNCHED();
    if (rc) return rc;
    const int acc_blocks =
        (int)std::min<int64_t>(ceil_div<int64_t>(n_hits, kBwdWarps), (int64_t)num_sms() * 16);
    if (real_bytes == 8)
        bwd_accum_kernel<double><<<acc_blocks, threads, 0, st>>>(a);
    else
        bwd_accum_kernel<float><<<acc_blocks, threads, 0, st>>>(a);
    return ARTEMIS_LAUNCHED();
}
