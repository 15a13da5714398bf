// One training iteration's bookkeeping on the device (SURVEY.md section 8f
// row 1, around backward_rays): the L1 loss gradients, the collision-pair
// (VRT) gradient, the touched-row bitmap and the sparse Adam step, so a fit
// iteration (forward_fit -> gradients -> backward_rays -> optimiser) never
// moves the FLUT off the device.
//
//   artemis_l1_grads      fit.py:474-492 (np.sign(f - gt) / n_p) and
//                         loss_rgba fit.py:52-68
//   artemis_vrt_grads     fit.py:494-501 + GradBuffer.add (np.add.at order)
//   artemis_mark_touched  backward_batch's bitmap, fit.py:144-146
//   artemis_sparse_adam   SparseAdam.step fit.py:319-330 + FLUT.clamp_densities
//                         volume.py:166-167
//
// fp64 throughout with explicitly rounded intrinsics in numpy's evaluation
// order, so given the same inputs the results are the reference's bit for
// bit. The VRT sum follows np.add.at's order: a stable sort of the (row,
// pair) entries by row keeps, within each row, every `winner` entry (pair
// order) before every `loser` entry (pair order), one warp per row applies
// them in that order.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace artemis {

template <typename K>
int sort_pairs(const K *keys_in, const uint32_t *vals_in, K *keys_out, uint32_t *vals_out,
               int64_t n, int key_bits, void *ws, size_t ws_bytes, cudaStream_t st);
size_t sort_workspace_bytes(int64_t n, int key_bits, int key_bytes);

namespace {

#define DM __dmul_rn
#define DA __dadd_rn
#define DD __ddiv_rn

__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : x < 0.0 ? -1.0 : 0.0; }

// dL/dF = sign(F - gt_F) / n, dL/dalpha = sign(alpha - gt_alpha) / n; per-ray
// loss term sum_c |F - gt_F| + |alpha - gt_alpha| into loss_rays
__global__ void l1_kernel(const float *__restrict__ F, const double *__restrict__ A,
                          const double *__restrict__ gtF, const double *__restrict__ gtA,
                          int64_t n, int C, double n_p, double *__restrict__ dldf,
                          double *__restrict__ dlda, double *__restrict__ loss_rays) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        double l = 0.0;
        for (int c = 0; c < C; ++c) {
            const double d = DA((double)F[r * C + c], -gtF[r * C + c]);
            dldf[r * C + c] = DD(sgn(d), n_p);
            l = DA(l, fabs(d));
        }
        const double da = DA(A[r], -gtA[r]);
        dlda[r] = DD(sgn(da), n_p);
        loss_rays[r] = DA(l, fabs(da));
    }
}

// ordered sum of the per-ray loss terms (one block; deterministic)
__global__ void sum_kernel(const double *__restrict__ x, int64_t n, double *out) {
    __shared__ double part[256];
    const int64_t per = (n + 255) / 256;
    double s = 0.0;
    for (int64_t i = threadIdx.x * per; i < std::min<int64_t>(n, (threadIdx.x + 1) * per); ++i)
        s = DA(s, x[i]);
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 256; ++k) t = DA(t, part[k]);
        *out = t;
    }
}

__global__ void touched_kernel(const int64_t *__restrict__ hit_idx, int64_t m,
                               uint8_t *__restrict__ touched) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        touched[hit_idx[i]] = 1;
}

// entries 0..P-1: (winner row, pair p, +), P..2P-1: (loser row, pair p, -)
__global__ void vrt_keys_kernel(const int64_t *__restrict__ pairs, int64_t P,
                                uint32_t *__restrict__ keys, uint8_t *__restrict__ touched) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 2 * P;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e < P ? e : e - P;
        const int64_t row = pairs[2 * p + (e < P ? 0 : 1)];
        keys[e] = (uint32_t)row;
        touched[row] = 1;
    }
}

__global__ void vrt_heads_kernel(const uint32_t *__restrict__ skeys, int64_t n,
                                 uint32_t *__restrict__ heads, unsigned int *__restrict__ count) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        if (j == 0 || skeys[j] != skeys[j - 1]) heads[atomicAdd(count, 1u)] = (uint32_t)j;
}

// one warp per row: grad[row, c] += +-(sign(data[w, c] - data[l, c]) * scale)
// in sorted-entry order (np.add.at's order for this row)
__global__ void vrt_apply_kernel(const double *__restrict__ data, int width,
                                 const int64_t *__restrict__ pairs, int64_t P,
                                 const uint32_t *__restrict__ skeys,
                                 const uint32_t *__restrict__ sperm, const uint32_t *heads,
                                 const unsigned int *count, int64_t n, double scale,
                                 double *__restrict__ grad) {
    const int lane = threadIdx.x & 31;
    const int64_t n_seg = *count;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < n_seg;
         s += wstride) {
        const int64_t start = heads[s];
        const uint32_t row = skeys[start];
        int64_t end = start + 1;
        while (end < n && skeys[end] == row) ++end;
        for (int c = lane; c < width; c += 32) {
            double g = grad[(size_t)row * width + c];
            for (int64_t j = start; j < end; ++j) {
                const uint32_t e = sperm[j];
                const int64_t p = e < P ? e : e - P;
                const double d = DA(data[(size_t)pairs[2 * p] * width + c],
                                    -data[(size_t)pairs[2 * p + 1] * width + c]);
                const double v = DM(sgn(d), scale);
                g = DA(g, e < P ? v : -v);
            }
            grad[(size_t)row * width + c] = g;
        }
    }
}

// SparseAdam on touched rows, then the density clamp of every row
__global__ void adam_kernel(double *__restrict__ params, double *__restrict__ m,
                            double *__restrict__ v, const double *__restrict__ grad,
                            const uint8_t *__restrict__ touched, int64_t n_rows, int width,
                            double lr, double b1, double b2, double eps, double bc1,
                            double bc2) {
    const double ob1 = DA(1.0, -b1), ob2 = DA(1.0, -b2);
    const int64_t total = n_rows * width;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / width;
        if (!touched[row]) {
            // FLUT.clamp_densities clamps the whole density column every
            // iteration (volume.py:166-167), touched or not; np.maximum keeps NaN
            if ((int)(i - row * width) == width - 1 && params[i] < 0.0) params[i] = 0.0;
            continue;
        }
        const double g = grad[i];
        const double mi = DA(DM(b1, m[i]), DM(ob1, g));
        const double vi = DA(DM(b2, v[i]), DM(DM(ob2, g), g));
        m[i] = mi;
        v[i] = vi;
        const double m_hat = DD(mi, bc1), v_hat = DD(vi, bc2);
        double p = DA(params[i], -DD(DM(lr, m_hat), DA(__dsqrt_rn(v_hat), eps)));
        if ((int)(i - row * width) == width - 1 && !(p >= 0.0)) p = p < 0.0 ? 0.0 : p;
        params[i] = p;
    }
}

#undef DM
#undef DA
#undef DD

int grid(int64_t n) {
    return (int)std::min<int64_t>(std::max<int64_t>(ceil_div<int64_t>(n, 256), 1),
                                  (int64_t)num_sms() * 16);
}

}  // namespace
}  // namespace artemis

using namespace artemis;

extern "C" int artemis_l1_grads(const float *F, const double *alpha, const double *gt_F,
                                const double *gt_alpha, int64_t n_rays, int channels,
                                double *dldf, double *dlda, double *loss_rays, double *loss_sum,
                                artemis_stream stream) {
    if (n_rays < 1 || channels < 1 || !F || !alpha || !gt_F || !gt_alpha || !dldf || !dlda ||
        !loss_rays || !loss_sum)
        return ARTEMIS_ERR_ARG;
    l1_kernel<<<grid(n_rays), 256, 0, S(stream)>>>(F, alpha, gt_F, gt_alpha, n_rays, channels,
                                                   (double)n_rays, dldf, dlda, loss_rays);
    sum_kernel<<<1, 256, 0, S(stream)>>>(loss_rays, n_rays, loss_sum);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_mark_touched(const int64_t *hit_idx, int64_t n_hits, uint8_t *touched,
                                    artemis_stream stream) {
    if (n_hits < 0 || (n_hits && (!hit_idx || !touched))) return ARTEMIS_ERR_ARG;
    if (!n_hits) return ARTEMIS_OK;
    touched_kernel<<<grid(n_hits), 256, 0, S(stream)>>>(hit_idx, n_hits, touched);
    return ARTEMIS_LAUNCHED();
}

extern "C" size_t artemis_vrt_workspace_bytes(int64_t n_pairs, int64_t n_rows) {
    int kb = 1;
    while (kb < 32 && (int64_t(1) << kb) < n_rows) ++kb;
    const size_t e = (size_t)std::max<int64_t>(2 * n_pairs, 1);
    return 4 * e * 4 + 256 + sort_workspace_bytes((int64_t)e, kb, 4) + 1024;
}

extern "C" int artemis_vrt_grads(const double *data, int64_t n_rows, int width,
                                 const int64_t *pairs, int64_t n_pairs, double scale,
                                 double *grad, uint8_t *touched, void *workspace,
                                 size_t workspace_bytes, artemis_stream stream) {
    if (n_pairs < 0 || n_rows < 1 || width < 1 || !data || !grad || !touched) return ARTEMIS_ERR_ARG;
    if (n_pairs == 0) return ARTEMIS_OK;
    if (!pairs || !workspace || workspace_bytes < artemis_vrt_workspace_bytes(n_pairs, n_rows))
        return ARTEMIS_ERR_WORKSPACE;
    int kb = 1;
    while (kb < 32 && (int64_t(1) << kb) < n_rows) ++kb;
    const int64_t n = 2 * n_pairs;
    auto a256 = [](size_t b) { return (b + 255) & ~size_t(255); };
    char *w = static_cast<char *>(workspace);
    uint32_t *keys = reinterpret_cast<uint32_t *>(w);
    uint32_t *skeys = reinterpret_cast<uint32_t *>(w + a256(4 * n));
    uint32_t *sperm = reinterpret_cast<uint32_t *>(w + 2 * a256(4 * n));
    uint32_t *heads = reinterpret_cast<uint32_t *>(w + 3 * a256(4 * n));
    unsigned int *count = reinterpret_cast<unsigned int *>(w + 4 * a256(4 * n));
    void *sws = w + 4 * a256(4 * n) + 256;
    const size_t sbytes = sort_workspace_bytes(n, kb, 4);
    cudaStream_t st = S(stream);
    vrt_keys_kernel<<<grid(n), 256, 0, st>>>(pairs, n_pairs, keys, touched);
    int rc = ARTEMIS_LAUNCHED();
    if (rc) return rc;
    rc = sort_pairs<uint32_t>(keys, nullptr, skeys, sperm, n, kb, sws, sbytes, st);
    if (rc) return rc;
    ARTEMIS_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned int), st));
    vrt_heads_kernel<<<grid(n), 256, 0, st>>>(skeys, n, heads, count);
    vrt_apply_kernel<<<(int)std::min<int64_t>(ceil_div<int64_t>(n, 4), num_sms() * 16), 128, 0,
                       st>>>(data, width, pairs, n_pairs, skeys, sperm, heads, count, n, scale,
                             grad);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_sparse_adam(double *params, double *m, double *v, const double *grad,
                                   const uint8_t *touched, int64_t n_rows, int width, double lr,
                                   double beta1, double beta2, double eps, double bias1,
                                   double bias2, artemis_stream stream) {
    if (n_rows < 1 || width < 1 || !params || !m || !v || !grad || !touched) return ARTEMIS_ERR_ARG;
    adam_kernel<<<grid(n_rows * width), 256, 0, S(stream)>>>(params, m, v, grad, touched, n_rows,
                                                             width, lr, beta1, beta2, eps, bias1,
                                                             bias2);
    return ARTEMIS_LAUNCHED();
}
