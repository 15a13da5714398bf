// Sparse frame read-out: only the pixels a frame actually covers leave the
// GPU. At configs[2] about 16 % of the 1024^2 rays hit the character, so a
// dense F/alpha/depth copy (4(C+2) B/pixel, 142 MB) is mostly zeros; the
// compacted stream is ~6x smaller and the host rebuilds the dense maps.
//
//   artemis_frame_compact   device: pixels with alpha > 0 or finite depth,
//                           in pixel order, as records {u32 pixel, F[C],
//                           alpha, depth} (fp32) plus the record count, into
//                           device memory; the caller copies the count, then
//                           exactly `count` records, device -> host with the
//                           copy engine (no SMs held while PCIe drains).
//   artemis_host_expand     host: dense maps from records: the pixels the
//                           previous frame of this buffer covered are reset
//                           to (0, 0, +inf), then the new records written;
//                           both lists are pixel-ordered, split over threads.
//
// Compaction is order-preserving: per 1024-pixel block a ballot count, one
// scan of the block counts, then each warp writes its pixels' records at
// the scanned offsets, lane-contiguous across a record.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"

namespace artemis {
namespace {

constexpr int kCompactThreads = 1024;

__device__ __forceinline__ bool covered(const void *A, const void *D, int maps64, int64_t p) {
    if (maps64) {
        const double a = static_cast<const double *>(A)[p], d = static_cast<const double *>(D)[p];
        return a > 0.0 || d < HUGE_VAL;
    }
    const float a = static_cast<const float *>(A)[p], d = static_cast<const float *>(D)[p];
    return a > 0.0f || d < HUGE_VALF;
}

__global__ void __launch_bounds__(kCompactThreads) compact_count_kernel(
    const void *A, const void *D, int maps64, int64_t n, uint32_t *block_counts) {
    __shared__ uint32_t warp_counts[kCompactThreads / 32];
    const int64_t p = blockIdx.x * (int64_t)kCompactThreads + threadIdx.x;
    const bool hit = p < n && covered(A, D, maps64, p);
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0) warp_counts[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kCompactThreads / 32; ++w) t += warp_counts[w];
        block_counts[blockIdx.x] = t;
    }
}

// exclusive scan of the block counts in place (one block, any count)
__global__ void compact_scan_kernel(uint32_t *counts, int64_t nb, int64_t *total) {
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const uint32_t v = i < nb ? counts[i] : 0u;
        // block-wide inclusive scan (Hillis-Steele in shared memory)
        __shared__ uint32_t s[1024];
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < (int)blockDim.x; off <<= 1) {
            const uint32_t add = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0u;
            __syncthreads();
            s[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < nb) counts[i] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += s[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = (int64_t)carry;
}

__global__ void __launch_bounds__(kCompactThreads) compact_write_kernel(
    const float *__restrict__ F, const void *A, const void *D, int maps64, int64_t n, int C,
    const uint32_t *__restrict__ block_offsets, uint32_t *__restrict__ out) {
    __shared__ uint32_t warp_base[kCompactThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t p = blockIdx.x * (int64_t)kCompactThreads + threadIdx.x;
    const bool hit = p < n && covered(A, D, maps64, p);
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_base[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = block_offsets[blockIdx.x];
        for (int k = 0; k < kCompactThreads / 32; ++k) {
            const uint32_t c = warp_base[k];
            warp_base[k] = t;
            t += c;
        }
    }
    __syncthreads();
    const int R = C + 3;  // words per record
    uint32_t slot = warp_base[w];
    unsigned mm = m;
    while (mm) {  // the warp writes each of its covered pixels' records
        const int src = __ffs(mm) - 1;
        mm &= mm - 1;
        const int64_t q = blockIdx.x * (int64_t)kCompactThreads + w * 32 + src;
        uint32_t *rec = out + (size_t)slot * R;
        for (int k = lane; k < R; k += 32) {
            float v;
            if (k == 0) {
                rec[0] = (uint32_t)q;
                continue;
            } else if (k <= C) {
                v = F[q * C + (k - 1)];
            } else if (k == C + 1) {
                v = maps64 ? (float)static_cast<const double *>(A)[q] : static_cast<const float *>(A)[q];
            } else {
                v = maps64 ? (float)static_cast<const double *>(D)[q] : static_cast<const float *>(D)[q];
            }
            rec[k] = __float_as_uint(v);
        }
        ++slot;
    }
}

template <typename Fn>
void parallel_for(int64_t n, int threads, Fn &&fn) {
    threads = std::max(1, std::min<int>(threads, (int)((n + 4095) / 4096)));
    if (threads == 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
    }
    for (auto &th : pool) th.join();
}

}  // namespace
}  // namespace artemis

using namespace artemis;

extern "C" size_t artemis_compact_workspace_bytes(int64_t n_pix) {
    return (size_t)ceil_div<int64_t>(std::max<int64_t>(n_pix, 1), kCompactThreads) * 4 + 256;
}

extern "C" int artemis_frame_compact(const float *F, const void *alpha, const void *depth,
                                     int maps64, int64_t n_pix, int channels, void *records,
                                     int64_t *count, void *workspace, size_t workspace_bytes,
                                     artemis_stream stream) {
    if (n_pix < 1 || channels < 1 || !F || !alpha || !depth || !records || !count || !workspace)
        return ARTEMIS_ERR_ARG;
    if (workspace_bytes < artemis_compact_workspace_bytes(n_pix)) return ARTEMIS_ERR_WORKSPACE;
    cudaStream_t st = S(stream);
    const int64_t nb = ceil_div<int64_t>(n_pix, kCompactThreads);
    uint32_t *bc = static_cast<uint32_t *>(workspace);
    compact_count_kernel<<<(unsigned)nb, kCompactThreads, 0, st>>>(alpha, depth, maps64, n_pix, bc);
    compact_scan_kernel<<<1, 1024, 0, st>>>(bc, nb, count);
    compact_write_kernel<<<(unsigned)nb, kCompactThreads, 0, st>>>(
        F, alpha, depth, maps64, n_pix, channels, bc, static_cast<uint32_t *>(records));
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_host_expand(const void *records, int64_t count, int channels,
                                   const uint32_t *prev_pixels, int64_t prev_count, float *F,
                                   float *alpha, float *depth, uint32_t *pixels_out,
                                   int threads) {
    if (count < 0 || prev_count < 0 || channels < 1 || !F || !alpha || !depth ||
        (count && (!records || !pixels_out)) || (prev_count && !prev_pixels))
        return ARTEMIS_ERR_ARG;
    const int C = channels, R = C + 3;
    const uint32_t *rec = static_cast<const uint32_t *>(records);
    parallel_for(prev_count, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            const int64_t p = prev_pixels[i];
            std::fill(F + p * C, F + p * C + C, 0.0f);
            alpha[p] = 0.0f;
            depth[p] = HUGE_VALF;
        }
    });
    parallel_for(count, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            const uint32_t *r = rec + i * R;
            const int64_t p = r[0];
            pixels_out[i] = (uint32_t)p;
            memcpy(F + p * C, r + 1, sizeof(float) * C);
            memcpy(alpha + p, r + 1 + C, sizeof(float));
            memcpy(depth + p, r + 2 + C, sizeof(float));
        }
    });
    return ARTEMIS_OK;
}

// ---- covered-pixel bounding box + rectangle read-out ----------------------
namespace artemis {
namespace {
__global__ void bbox_kernel(const void *A, const void *D, int maps64, int width, int64_t n,
                            int32_t *box) {
    int x0 = INT32_MAX, y0 = INT32_MAX, x1 = -1, y1 = -1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (!covered(A, D, maps64, p)) continue;
        const int x = (int)(p % width), y = (int)(p / width);
        x0 = min(x0, x);
        x1 = max(x1, x);
        y0 = min(y0, y);
        y1 = max(y1, y);
    }
    for (int o = 16; o; o >>= 1) {
        x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
        y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
        x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
        y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    if ((threadIdx.x & 31) == 0 && x1 >= 0) {
        atomicMin(box + 0, x0);
        atomicMin(box + 1, y0);
        atomicMax(box + 2, x1);
        atomicMax(box + 3, y1);
    }
}
__global__ void bbox_init_kernel(int32_t *box) {
    box[0] = box[1] = INT32_MAX;
    box[2] = box[3] = -1;
}
}  // namespace
}  // namespace artemis

extern "C" int artemis_frame_bbox(const void *alpha, const void *depth, int maps64, int width,
                                  int height, int32_t *box, artemis_stream stream) {
    if (!alpha || !depth || !box || width < 1 || height < 1) return ARTEMIS_ERR_ARG;
    const int64_t n = (int64_t)width * height;
    bbox_init_kernel<<<1, 1, 0, S(stream)>>>(box);
    const int blocks = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), (int64_t)num_sms() * 8);
    bbox_kernel<<<blocks, 256, 0, S(stream)>>>(alpha, depth, maps64, width, n, box);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_copy_rect_d2h(void *dst_host, const void *src_dev, size_t row_pitch,
                                     size_t x_bytes, size_t width_bytes, int64_t y0,
                                     int64_t rows, artemis_stream stream) {
    if (!dst_host || !src_dev || rows < 0 || x_bytes + width_bytes > row_pitch)
        return ARTEMIS_ERR_ARG;
    if (rows == 0 || width_bytes == 0) return ARTEMIS_OK;
    const size_t off = (size_t)y0 * row_pitch + x_bytes;
    ARTEMIS_TRY(cudaMemcpy2DAsync(static_cast<char *>(dst_host) + off, row_pitch,
                                  static_cast<const char *>(src_dev) + off, row_pitch,
                                  width_bytes, (size_t)rows, cudaMemcpyDeviceToHost, S(stream)));
    return ARTEMIS_OK;
}

// Several views' covered-pixel boxes in one call (boxes: device, n_views x 4).
extern "C" int artemis_views_bbox(const void *const *alpha, const void *const *depth,
                                  int n_views, int maps64, int width, int height, int32_t *boxes,
                                  artemis_stream stream) {
    if (!alpha || !depth || !boxes || n_views < 1) return ARTEMIS_ERR_ARG;
    for (int v = 0; v < n_views; ++v) {
        const int rc = artemis_frame_bbox(alpha[v], depth[v], maps64, width, height, boxes + 4 * v,
                                          stream);
        if (rc) return rc;
    }
    return ARTEMIS_OK;
}

// Refresh n_views dense host frames (F fp32 (w*h, C), alpha/depth 4- or
// 8-byte maps) from their device frames: per view, the union of this frame's
// box (boxes, host) and the box that host buffer last received (prev, host,
// updated) as three 2-D copies on `stream`. Outside the union both frames are
// (0, 0, +inf), so the dense host maps equal the device maps bit for bit.
// *bytes receives the bytes moved.
extern "C" int artemis_views_copy_union_d2h(int n_views, const int32_t *boxes, int32_t *prev,
                                            const void *const *dev, void *const *host,
                                            int width, int height, int channels, int maps64,
                                            int64_t *bytes, artemis_stream stream) {
    if (n_views < 1 || !boxes || !prev || !dev || !host || width < 1 || height < 1 ||
        channels < 1)
        return ARTEMIS_ERR_ARG;
    int64_t moved = 0;
    const size_t per[3] = {(size_t)channels * 4, maps64 ? 8u : 4u, maps64 ? 8u : 4u};
    for (int v = 0; v < n_views; ++v) {
        const int32_t *b = boxes + 4 * v;
        int32_t *p = prev + 4 * v;
        const int ux0 = std::min(b[0], p[0]), uy0 = std::min(b[1], p[1]);
        const int ux1 = std::max(b[2], p[2]), uy1 = std::max(b[3], p[3]);
        // remember this frame's box (empty -> an empty box that unions to nothing)
        p[0] = b[2] >= 0 ? b[0] : width;
        p[1] = b[3] >= 0 ? b[1] : height;
        p[2] = b[2];
        p[3] = b[3];
        if (ux1 < 0 || uy1 < 0 || ux0 > ux1 || uy0 > uy1) continue;
        const int64_t rows = uy1 - uy0 + 1;
        for (int m = 0; m < 3; ++m) {
            const int rc = artemis_copy_rect_d2h(host[3 * v + m], dev[3 * v + m], width * per[m],
                                                 ux0 * per[m], (ux1 - ux0 + 1) * per[m], uy0, rows,
                                                 stream);
            if (rc) return rc;
            moved += (int64_t)(ux1 - ux0 + 1) * per[m] * rows;
        }
    }
    if (bytes) *bytes = moved;
    return ARTEMIS_OK;
}
