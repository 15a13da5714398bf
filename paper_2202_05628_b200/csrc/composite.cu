// Post-render frame-buffer step: the
// consumers of a rendered frame, on the device while the frame is still
// resident, so only the final image leaves the GPU.
//
//   artemis_over_background   FrameBuffers.over_background   render.py:98-104
//   artemis_composite         composite (depth-resolved)     render.py:366-382
//   artemis_straight_rgba     frame_to_straight_rgba         assetio.py:265-275
//   artemis_rgba8             frame_to_straight_rgba + the 8-bit quantisation
//                             of save_png / encode_png       assetio.py:209-245
//
// The frame's F is fp32 (widened exactly to fp64 here), alpha/depth float
// or double (maps64). All arithmetic is fp64 with explicitly rounded
// intrinsics in the reference's operation order, so results equal numpy's
// on the same inputs bit for bit. One thread per output element; pure
// streaming work, HBM-bound.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace artemis {
namespace {

__device__ __forceinline__ double map_at(const void *m, int maps64, int64_t i) {
    return maps64 ? static_cast<const double *>(m)[i] : (double)static_cast<const float *>(m)[i];
}

int blocks_for(int64_t n) {
    return (int)std::min<int64_t>(std::max<int64_t>(ceil_div<int64_t>(n, 256), 1),
                                  (int64_t)num_sms() * 16);
}

#define GRID_STRIDE(i, n)                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
         i += (int64_t)gridDim.x * blockDim.x)

// out = F + (1 - alpha) * bg   (render.py:104, numpy broadcast order)
__global__ void over_background_kernel(const float *__restrict__ F, const void *alpha, int maps64,
                                       int64_t n_pix, int C, const double *__restrict__ color,
                                       double *__restrict__ out) {
    GRID_STRIDE(i, n_pix * C) {
        const int64_t p = i / C;
        const int c = (int)(i - p * C);
        const double t = __dadd_rn(1.0, -map_at(alpha, maps64, p));
        out[i] = __dadd_rn((double)F[i], __dmul_rn(t, color[c]));
    }
}

// front = depth <= bg_depth: out = F + (1 - alpha) * bg, else bg (render.py:378-382)
__global__ void composite_kernel(const float *__restrict__ F, const void *alpha,
                                 const void *depth, int maps64, int64_t n_pix, int C,
                                 const double *__restrict__ bg_color,
                                 const double *__restrict__ bg_depth, double *__restrict__ out) {
    GRID_STRIDE(i, n_pix * C) {
        const int64_t p = i / C;
        const double bg = bg_color[i];
        if (map_at(depth, maps64, p) <= bg_depth[p]) {
            const double t = __dadd_rn(1.0, -map_at(alpha, maps64, p));
            out[i] = __dadd_rn((double)F[i], __dmul_rn(t, bg));
        } else {
            out[i] = bg;
        }
    }
}

// straight-alpha RGBA (assetio.py:265-275): rgb = clip(F / a, 0, 1) where
// a > 0 else 0; A = alpha unclipped. C must be 3.
__device__ __forceinline__ void straight_px(const float *F, const void *alpha, int maps64,
                                            int64_t p, double v[4]) {
    const double a = map_at(alpha, maps64, p);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double x = 0.0;
        if (a > 0.0) x = fmin(fmax(__ddiv_rn((double)F[3 * p + c], a), 0.0), 1.0);
        v[c] = x;
    }
    v[3] = a;
}

__global__ void straight_rgba_kernel(const float *__restrict__ F, const void *alpha, int maps64,
                                     int64_t n_pix, double *__restrict__ out) {
    GRID_STRIDE(p, n_pix) {
        double v[4];
        straight_px(F, alpha, maps64, p, v);
        reinterpret_cast<double2 *>(out)[2 * p] = make_double2(v[0], v[1]);
        reinterpret_cast<double2 *>(out)[2 * p + 1] = make_double2(v[2], v[3]);
    }
}

// save_png quantisation: clip(round_half_even(v * 255), 0, 255) as uint8
__global__ void rgba8_kernel(const float *__restrict__ F, const void *alpha, int maps64,
                             int64_t n_pix, uchar4 *__restrict__ out) {
    GRID_STRIDE(p, n_pix) {
        double v[4];
        straight_px(F, alpha, maps64, p, v);
        unsigned char q[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
            q[c] = (unsigned char)fmin(fmax(rint(__dmul_rn(v[c], 255.0)), 0.0), 255.0);
        out[p] = make_uchar4(q[0], q[1], q[2], q[3]);
    }
}

#undef GRID_STRIDE

}  // namespace
}  // namespace artemis

using namespace artemis;

extern "C" int artemis_over_background(const float *F, const void *alpha, int maps64,
                                       int64_t n_pix, int channels, const double *color,
                                       double *out, artemis_stream stream) {
    if (n_pix < 0 || channels < 1 || (n_pix > 0 && (!F || !alpha || !color || !out)))
        return ARTEMIS_ERR_ARG;
    if (n_pix == 0) return ARTEMIS_OK;
    over_background_kernel<<<blocks_for(n_pix * channels), 256, 0, S(stream)>>>(
        F, alpha, maps64, n_pix, channels, color, out);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_composite(const float *F, const void *alpha, const void *depth, int maps64,
                                 int64_t n_pix, int channels, const double *bg_color,
                                 const double *bg_depth, double *out, artemis_stream stream) {
    if (n_pix < 0 || channels < 1 ||
        (n_pix > 0 && (!F || !alpha || !depth || !bg_color || !bg_depth || !out)))
        return ARTEMIS_ERR_ARG;
    if (n_pix == 0) return ARTEMIS_OK;
    composite_kernel<<<blocks_for(n_pix * channels), 256, 0, S(stream)>>>(
        F, alpha, depth, maps64, n_pix, channels, bg_color, bg_depth, out);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_straight_rgba(const float *F, const void *alpha, int maps64, int64_t n_pix,
                                     double *rgba, artemis_stream stream) {
    if (n_pix < 0 || (n_pix > 0 && (!F || !alpha || !rgba))) return ARTEMIS_ERR_ARG;
    if (n_pix == 0) return ARTEMIS_OK;
    straight_rgba_kernel<<<blocks_for(n_pix), 256, 0, S(stream)>>>(F, alpha, maps64, n_pix, rgba);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_rgba8(const float *F, const void *alpha, int maps64, int64_t n_pix,
                             uint8_t *rgba8, artemis_stream stream) {
    if (n_pix < 0 || (n_pix > 0 && (!F || !alpha || !rgba8))) return ARTEMIS_ERR_ARG;
    if (n_pix == 0) return ARTEMIS_OK;
    rgba8_kernel<<<blocks_for(n_pix), 256, 0, S(stream)>>>(F, alpha, maps64, n_pix,
                                                          reinterpret_cast<uchar4 *>(rgba8));
    return ARTEMIS_LAUNCHED();
}
