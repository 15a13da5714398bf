// Pieces shared by the render kernels (render.cu, all modes) and the
// gradient kernels: launch arguments, the exact camera ray, the fp32 SH
// basis, an L2 prefetch.
#pragma once
#include <math.h>

#include "bricks.cuh"
#include "common.cuh"
#include "tree.cuh"

namespace artemis {

constexpr int kMaxViews = 8;  // views one camera-mode launch renders together

enum RenderMode { kRender = 0, kTrace = 1, kCount = 2 };

constexpr uint32_t kDenseFlag = 1u << 31;  // queued row's density exceeds sigma_dep

struct RenderArgs {
    const WideNode *nodes;
    const uint4 *leaves;  // {x, y, z, flut row}
    BrickMap bm;          // exact cell walk (kDDA)
    int64_t n_leaves;
    const int32_t *n_leaves_dev;
    // shading
    const float *coef;
    const double *sigma;
    const int32_t *rot_index;
    const double *rot_inv;
    int channels;
    int coef_stride;
    int64_t n_rows;  // FLUT rows (0 = unknown; debug checks only)
    // rays: explicit arrays or a camera (device pointer, read once)
    const double *og, *dg, *dw;
    const artemis_camera *cam;
    int64_t n_rays;
    int tiles_x, tiles_y;  // camera mode: ceil(W / 8), ceil(H / 4)
    unsigned long long *queue;  // ray-id counter, zero at launch
    const int32_t *tile_order;  // camera mode, unsharded: the i-th 8x4 tile to visit (a permutation)
    const int32_t *order_on;    // device flag: use tile_order (else row-major); null = use it
    // camera mode: views rendered by this launch (cam[0 .. n_views), one
    // image size); with n_views > 1 the outputs of view v are Fv/Av/Dv[v]
    // (alpha/depth float, or double with A64/D64 set non-null)
    int n_views;
    const int32_t *view_shift;  // device, per view: x shift of the tile order (align_views)
    float *Fv[kMaxViews];
    void *Av[kMaxViews];
    void *Dv[kMaxViews];
    double t_min, t_max;
    double stop;  // 1 - lambda_th
    float coord_max;  // upper bound of every box coordinate (grid resolution)
    double sigma_dep;
    int early_stop;
    int fast_div;  // camera launch whose operand ranges allow div_fast (camera_fast_div_ok)
    int no_row_prefetch;  // skip the L2 prefetch of queued rows (FLUT already L2-resident)
    // outputs
    float *F;
    double *A64, *D64;
    float *A32, *D32;
    const int64_t *offsets;
    int64_t *hit_idx;
    double *hit_t0, *hit_t1;
    int64_t *counts;
};

__device__ __forceinline__ void prefetch_l2(const void *ptr) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
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

// Per-view constants of camera_ray_fast, computed once per block:
// reciprocals of fx, fy and the cell size, and the grid-space origin.
struct CamRecip {
    double rfx, rfy, rcell[3], og[3];
};

__device__ __forceinline__ CamRecip camera_recip(const artemis_camera &c) {
    CamRecip k;
    k.rfx = __drcp_rn(c.fx);
    k.rfy = __drcp_rn(c.fy);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        k.rcell[a] = __drcp_rn(c.cell[a]);
        k.og[a] = __ddiv_rn(__dadd_rn(c.origin[a], -c.lo[a]), c.cell[a]);
    }
    return k;
}

// camera_ray with every division by a per-view constant (and the per-ray
// norm) done by div_fast: the same bits, shorter dependent chains at ray
// start. Only for launches whose cameras passed camera_fast_div_ok (frame.cu):
// then (u + 0.5) - cx is 0 or >= 2^-353, |d[a]| is 0 or >= 2^-427 and the
// norm is >= 1, so every quotient stays far inside the normal range.
__device__ __forceinline__ void camera_ray_fast(const artemis_camera &c, const CamRecip &k,
                                                int u, int v, double og[3], double dg[3],
                                                double dw[3]) {
    const double c0 = div_fast(__dadd_rn(__dadd_rn((double)u, 0.5), -c.cx), c.fx, k.rfx);
    const double c1 = div_fast(__dadd_rn(__dadd_rn((double)v, 0.5), -c.cy), c.fy, k.rfy);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        d[a] = __fma_rn(1.0, c.R[3 * a + 2], __fma_rn(c1, c.R[3 * a + 1], __dmul_rn(c0, c.R[3 * a])));
    const double nrm = __dsqrt_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
    const double rn = __drcp_rn(nrm);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        dw[a] = div_fast(d[a], nrm, rn);
        dg[a] = div_fast(dw[a], c.cell[a], k.rcell[a]);
        og[a] = k.og[a];
    }
}

}  // namespace artemis
