// Tile-shard packing for the multi-GPU image assembly.
//
// With tile sharding every rank renders the 8x4-pixel tiles t with
// t % stride == start of the same frame (render.cu, artemis_camera
// tile_start/tile_stride). Only those pixels are exchanged: each rank packs
// its tiles into one contiguous shard -- tile-major, 32 pixels per tile in
// tile-row order, (C + 2) floats per pixel: F[0..C), alpha, depth -- one
// NCCL gather moves the shards to the root, and the root unpacks each rank's
// shard into the image. Pixels of a tile that fall outside the image are
// packed as zeros and skipped on unpack.
//
// One thread per (tile pixel, float): consecutive threads read consecutive
// floats of a pixel's F row, so F is read/written in 4(C+2)-byte runs; the
// shard side is fully coalesced. Pure data movement, HBM-bound.
#include <algorithm>

#include "common.cuh"

namespace artemis {
namespace {

__device__ __forceinline__ bool tile_pixel(int64_t slot, int tiles_x, int width, int height,
                                           int start, int stride, int64_t &pix) {
    const int64_t t = start + (slot >> 5) * (int64_t)stride;
    const int s = (int)(slot & 31);
    const int px = (int)(t % tiles_x) * 8 + (s & 7);
    const int py = (int)(t / tiles_x) * 4 + (s >> 3);
    pix = (int64_t)py * width + px;
    return px < width && py < height;
}

__global__ void tiles_pack_kernel(const float *__restrict__ F, const float *__restrict__ A,
                                  const float *__restrict__ D, int width, int height, int C,
                                  int tiles_x, int start, int stride, int64_t n_slots,
                                  float *__restrict__ packed) {
    const int P = C + 2;
    const int64_t total = n_slots * P;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = i / P;
        const int k = (int)(i - slot * P);
        int64_t pix;
        float v = 0.0f;
        if (tile_pixel(slot, tiles_x, width, height, start, stride, pix))
            v = k < C ? F[pix * C + k] : k == C ? A[pix] : D[pix];
        packed[i] = v;
    }
}

__global__ void tiles_unpack_kernel(const float *__restrict__ packed, int width, int height,
                                    int C, int tiles_x, int start, int stride, int64_t n_slots,
                                    float *__restrict__ F, float *__restrict__ A,
                                    float *__restrict__ D) {
    const int P = C + 2;
    const int64_t total = n_slots * P;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = i / P;
        const int k = (int)(i - slot * P);
        int64_t pix;
        if (!tile_pixel(slot, tiles_x, width, height, start, stride, pix)) continue;
        const float v = packed[i];
        if (k < C)
            F[pix * C + k] = v;
        else if (k == C)
            A[pix] = v;
        else
            D[pix] = v;
    }
}

int64_t shard_tiles(int width, int height, int start, int stride) {
    const int64_t n = (int64_t)((width + 7) / 8) * ((height + 3) / 4);
    return start < n ? (n - start + stride - 1) / stride : 0;
}

bool tiles_args_ok(int width, int height, int channels, int start, int stride) {
    return width > 0 && height > 0 && channels > 0 && stride > 0 && start >= 0 && start < stride;
}

int grid_for(int64_t total) {
    return (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), (int64_t)num_sms() * 16);
}

}  // namespace
}  // namespace artemis

using namespace artemis;

extern "C" int64_t artemis_tiles_shard_floats(int width, int height, int channels,
                                              int tile_start, int tile_stride) {
    if (!tiles_args_ok(width, height, channels, tile_start, tile_stride)) return -1;
    return shard_tiles(width, height, tile_start, tile_stride) * 32 * (channels + 2);
}

extern "C" int artemis_tiles_pack(const float *F, const float *alpha, const float *depth,
                                  int width, int height, int channels, int tile_start,
                                  int tile_stride, float *packed, artemis_stream stream) {
    if (!tiles_args_ok(width, height, channels, tile_start, tile_stride) || !F || !alpha ||
        !depth || !packed)
        return ARTEMIS_ERR_ARG;
    const int64_t slots = shard_tiles(width, height, tile_start, tile_stride) * 32;
    if (slots == 0) return ARTEMIS_OK;
    tiles_pack_kernel<<<grid_for(slots * (channels + 2)), 256, 0, S(stream)>>>(
        F, alpha, depth, width, height, channels, (width + 7) / 8, tile_start, tile_stride, slots,
        packed);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_tiles_unpack(const float *packed, int width, int height, int channels,
                                    int tile_start, int tile_stride, float *F, float *alpha,
                                    float *depth, artemis_stream stream) {
    if (!tiles_args_ok(width, height, channels, tile_start, tile_stride) || !F || !alpha ||
        !depth || !packed)
        return ARTEMIS_ERR_ARG;
    const int64_t slots = shard_tiles(width, height, tile_start, tile_stride) * 32;
    if (slots == 0) return ARTEMIS_OK;
    tiles_unpack_kernel<<<grid_for(slots * (channels + 2)), 256, 0, S(stream)>>>(
        packed, width, height, channels, (width + 7) / 8, tile_start, tile_stride, slots, F, alpha,
        depth);
    return ARTEMIS_LAUNCHED();
}
