// Device-resident asset ingestion: the .nvo
// character container (animvox/assetio.py:49-202) straight into HBM.
//
// Layout (little-endian; assetio.py:37-41): a 54-byte header {magic "NVO1",
// version u32, resolution u32, count u64, degree u8, channels u8, bounds
// 6 x f32, rig offset u64}; the leaf table, count x {Morton code u64, FLUT
// row u32} sorted by code; the FLUT block, count x width f32 (column h*C+c,
// density last); optionally the rig block.
//
// The leaf table and the FLUT block are copied to the device as they lie in
// the file: one kernel decodes the codes and scatters the cells to their
// FLUT rows (cells[row] = decode(code), assetio.py:118-122) while checking
// that the rows form a permutation; artemis_flut_split_f32 turns the f32
// block into the render layout. The rig block is a sequential byte stream
// (u8 slot count, then (u16 joint, f32 weight) per slot, per voxel,
// assetio.py:158-202): it is decoded on the host, natively, in one pass.
// Validation order and failure classes follow load_asset (assetio.py:86-136):
// magic, version, zero count, truncated leaf table, truncated FLUT block,
// non-permutation, rig offset, truncated rig, trailing bytes.
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace artemis {
namespace {

constexpr size_t kHeader = 4 + 4 + 4 + 8 + 1 + 1 + 24 + 8;  // struct "<4sIIQBB6fQ" = 54
constexpr size_t kLeaf = 12;

template <typename T>
T rd(const uint8_t *p) {
    T v;
    memcpy(&v, p, sizeof(T));
    return v;
}

__global__ void leaves_kernel(const uint8_t *__restrict__ table, int64_t n,
                              int32_t *__restrict__ cells, uint32_t *__restrict__ seen,
                              int32_t *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t *rec = table + i * kLeaf;
        // records are 12-byte packed: assemble from 4-byte words
        const uint32_t w0 = (uint32_t)rec[0] | (uint32_t)rec[1] << 8 | (uint32_t)rec[2] << 16 |
                            (uint32_t)rec[3] << 24;
        const uint32_t w1 = (uint32_t)rec[4] | (uint32_t)rec[5] << 8 | (uint32_t)rec[6] << 16 |
                            (uint32_t)rec[7] << 24;
        const uint32_t row = (uint32_t)rec[8] | (uint32_t)rec[9] << 8 | (uint32_t)rec[10] << 16 |
                             (uint32_t)rec[11] << 24;
        const u64 code = (u64)w0 | ((u64)w1 << 32);
        if ((int64_t)row >= n || atomicExch(seen + row, 1u) != 0u) {
            atomicExch(bad, 1);
            continue;
        }
        cells[3 * (int64_t)row + 0] = (int32_t)compact_bits3(code);
        cells[3 * (int64_t)row + 1] = (int32_t)compact_bits3(code >> 1);
        cells[3 * (int64_t)row + 2] = (int32_t)compact_bits3(code >> 2);
    }
}

}  // namespace
}  // namespace artemis

using namespace artemis;

extern "C" int artemis_asset_probe(const uint8_t *data, size_t size, artemis_asset_info *info) {
    if (!data || !info) return ARTEMIS_ERR_ARG;
    memset(info, 0, sizeof(*info));
    if (size < kHeader) return ARTEMIS_ASSET_TRUNCATED_HEADER;
    if (memcmp(data, "NVO1", 4) != 0) return ARTEMIS_ASSET_BAD_MAGIC;
    info->version = rd<uint32_t>(data + 4);
    info->resolution = rd<uint32_t>(data + 8);
    info->count = (int64_t)rd<uint64_t>(data + 12);
    info->degree = data[20];
    info->channels = data[21];
    for (int a = 0; a < 3; ++a) {
        info->lo[a] = (double)rd<float>(data + 22 + 4 * a);
        info->hi[a] = (double)rd<float>(data + 34 + 4 * a);
    }
    info->rig_offset = (int64_t)rd<uint64_t>(data + 46);
    if (info->version != 1) return ARTEMIS_ASSET_BAD_VERSION;
    if (info->count == 0) return ARTEMIS_ASSET_ZERO_COUNT;
    info->width = (info->degree + 1) * (info->degree + 1) * info->channels + 1;
    info->leaf_offset = (int64_t)kHeader;
    const uint64_t cnt = (uint64_t)info->count;
    if (cnt > (uint64_t(1) << 40) || size < kHeader + cnt * kLeaf) return ARTEMIS_ASSET_TRUNCATED_LEAVES;
    info->flut_offset = (int64_t)(kHeader + cnt * kLeaf);
    const uint64_t flut_end = kHeader + cnt * kLeaf + cnt * (uint64_t)info->width * 4;
    if (size < flut_end) return ARTEMIS_ASSET_TRUNCATED_FLUT;
    info->flut_end = (int64_t)flut_end;
    return ARTEMIS_OK;
}

extern "C" int artemis_asset_decode_leaves(const uint8_t *leaf_table, int64_t count,
                                           int32_t *cells, void *workspace,
                                           size_t workspace_bytes, int32_t *bad_flag,
                                           artemis_stream stream) {
    if (!leaf_table || count < 1 || !cells || !bad_flag || !workspace ||
        workspace_bytes < (size_t)count * 4)
        return ARTEMIS_ERR_ARG;
    cudaStream_t st = S(stream);
    ARTEMIS_TRY(cudaMemsetAsync(workspace, 0, (size_t)count * 4, st));
    ARTEMIS_TRY(cudaMemsetAsync(bad_flag, 0, 4, st));
    const int blocks = (int)std::min<int64_t>(ceil_div<int64_t>(count, 256), (int64_t)num_sms() * 16);
    leaves_kernel<<<blocks, 256, 0, st>>>(leaf_table, count, cells,
                                          static_cast<uint32_t *>(workspace), bad_flag);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_asset_decode_rig(const uint8_t *data, size_t size,
                                        const artemis_asset_info *info, artemis_asset_rig *rig,
                                        int32_t *parents, double *bind, char *names,
                                        int32_t *name_offsets, int32_t *joint_idx,
                                        double *weights) {
    if (!data || !info || !rig) return ARTEMIS_ERR_ARG;
    if (info->rig_offset == 0) {
        memset(rig, 0, sizeof(*rig));
        return (uint64_t)info->flut_end == size ? ARTEMIS_OK : ARTEMIS_ASSET_TRAILING;
    }
    if (info->rig_offset != info->flut_end) return ARTEMIS_ASSET_RIG_OFFSET;
    const bool fill = parents != nullptr;
    size_t pos = (size_t)info->rig_offset;
    auto need = [&](size_t end) { return size >= end; };
    if (!need(pos + 4)) return ARTEMIS_ASSET_TRUNCATED_RIG;
    const uint32_t J = rd<uint32_t>(data + pos);
    pos += 4;
    size_t name_bytes = 0;
    for (uint32_t j = 0; j < J; ++j) {
        if (!need(pos + 2)) return ARTEMIS_ASSET_TRUNCATED_RIG;
        const uint16_t ln = rd<uint16_t>(data + pos);
        pos += 2;
        if (!need(pos + ln + 4 + 56)) return ARTEMIS_ASSET_TRUNCATED_RIG;
        if (fill) {
            name_offsets[j] = (int32_t)name_bytes;
            memcpy(names + name_bytes, data + pos, ln);
        }
        name_bytes += ln;
        pos += ln;
        if (fill) {
            parents[j] = rd<int32_t>(data + pos);
            for (int k = 0; k < 7; ++k) bind[7 * j + k] = rd<double>(data + pos + 4 + 8 * k);
        }
        pos += 60;
    }
    if (fill) name_offsets[J] = (int32_t)name_bytes;
    int k_max = 1;
    const int64_t n = info->count;
    const int km = fill ? rig->k_max : 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!need(pos + 1)) return ARTEMIS_ASSET_TRUNCATED_RIG;
        const int k = data[pos];
        pos += 1;
        if (!need(pos + 6 * (size_t)k)) return ARTEMIS_ASSET_TRUNCATED_RIG;
        if (fill) {
            for (int s = 0; s < km; ++s) {
                joint_idx[i * km + s] = s < k ? (int32_t)rd<uint16_t>(data + pos + 6 * s) : -1;
                weights[i * km + s] = s < k ? (double)rd<float>(data + pos + 6 * s + 2) : 0.0;
            }
        }
        k_max = std::max(k_max, k);
        pos += 6 * (size_t)k;
    }
    if (pos != size) return ARTEMIS_ASSET_TRAILING;
    rig->n_joints = (int32_t)J;
    rig->k_max = fill ? rig->k_max : k_max;
    rig->name_bytes = (int64_t)name_bytes;
    rig->end = (int64_t)pos;
    return ARTEMIS_OK;
}
