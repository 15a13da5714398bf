// Linear-blend-skinning warp of the canonical voxels.
//
// Replaces the numpy body of animvox/rigging.py:349-371 (warp_voxels). The
// warped keys must be bit-identical to the reference's, so the arithmetic is
// pinned with explicitly rounded intrinsics (no FMA contraction) in the
// order numpy evaluates it on the reference host (pinned by
// tests/test_oracle_golden.py against the reference's own positions):
//   centre  = lo + (cell_i + 0.5) * cell_size                (volume.py:82-85)
//   E_a     = (m_a0*x + m_a2*z) + m_a1*y    (np.einsum('nij,nj->ni') order)
//   pos_a  += w_k * (E_a + t_a)   over live slots k, from pos = 0
//   cell_a  = floor((pos_a - lo_a) / cell_size_a), in bounds iff in [0, res)
//   rotation joint = joint of the first maximal weight slot
// One thread per voxel; the per-joint 3x4 blocks sit in shared memory; the
// K = 4 slot rows are read as one int4 and two double2.
#include <algorithm>
#include <cmath>

#include "bricks.cuh"
#include "common.cuh"
#include "tree.cuh"

namespace artemis {

namespace {
constexpr int kWarpThreads = 256;
constexpr int kMaxJoints = 256;
constexpr int kWarpBlocksPerSM = 4;
}  // namespace

struct WarpArgs {
    const int32_t *cells;
    int64_t n;
    int slots;
    const int32_t *jidx;
    const double *w;
    const double *aff;    // (J, 12)
    int n_joints;
    double lo[3], cell[3];
    double rcell[3];      // RN(1 / cell): the floor division as div_exact (bit-identical)
    int res;
    // API outputs
    double *positions;
    int32_t *cells_out;
    uint8_t *in_bounds;
    int32_t *rot_joint;
    // device-pipeline outputs
    void *keys;           // u32 or u64 Morton keys, sentinel when out of bounds
    uint32_t *vals;       // canonical index
    int32_t *n_in;        // in-bounds counter
    uint64_t sentinel;
    int identity;         // 1 = no warp: canonical cells, rotation joint 0
    // counting rebuild (rebuild.cu; 32-bit keys): dense per-brick cell masks
    // and the brick-occupancy bitmap, both indexed by Morton code
    uint32_t *bmask;
    uint32_t *bocc;
};

// One voxel's input rows (loaded one iteration ahead of their use).
struct VoxelIn {
    int32_t ci[3];
    int4 jj;
    double2 w01, w23;
};

__device__ __forceinline__ void load_voxel(const WarpArgs &a, int64_t i, VoxelIn &v) {
    v.ci[0] = v.ci[1] = v.ci[2] = 0;
    v.jj = make_int4(-1, -1, -1, -1);
    v.w01 = v.w23 = make_double2(0.0, 0.0);
    if (i >= a.n) return;
    v.ci[0] = __ldg(a.cells + 3 * i);
    v.ci[1] = __ldg(a.cells + 3 * i + 1);
    v.ci[2] = __ldg(a.cells + 3 * i + 2);
    if (!a.identity && a.slots == 4) {
        v.jj = __ldg(reinterpret_cast<const int4 *>(a.jidx) + i);
        v.w01 = __ldg(reinterpret_cast<const double2 *>(a.w) + 2 * i);
        v.w23 = __ldg(reinterpret_cast<const double2 *>(a.w) + 2 * i + 1);
    }
}

// Persistent blocks (a few per SM): the joint table is staged once per
// block, and each thread loads its next voxel's rows before it computes the
// current one, so the loads of one iteration overlap the fp64 work of the
// previous (one block per 256 voxels spent most of its life on the staging,
// the barrier and the first load's latency).
template <typename K, bool kPipeline>
__global__ void __launch_bounds__(kWarpThreads) lbs_warp_kernel(WarpArgs a) {
    __shared__ double s_aff[kMaxJoints * 12];
    __shared__ int s_in;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    VoxelIn nx;
    load_voxel(a, i, nx);
    if (!a.identity)
        for (int t = threadIdx.x; t < a.n_joints * 12; t += blockDim.x) s_aff[t] = a.aff[t];
    if (threadIdx.x == 0) s_in = 0;
    __syncthreads();
    int n_ok = 0;  // in-bounds voxels of this thread's warp (lane 0 counts)
    // uniform trip count over the block: every lane runs the warp collectives
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < a.n; base += stride, i += stride) {
        const VoxelIn v = nx;
        load_voxel(a, i + stride, nx);
        const bool live = i < a.n;
        bool ok = false;
        int64_t g[3] = {0, 0, 0};
        if (live) {
            if (a.identity) {
                ok = true;
                for (int k = 0; k < 3; ++k) g[k] = v.ci[k];
                if (a.rot_joint) a.rot_joint[i] = 0;
            } else {
                double c[3];
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    c[k] = __dadd_rn(a.lo[k], __dmul_rn(__dadd_rn((double)v.ci[k], 0.5), a.cell[k]));
                double p[3] = {0.0, 0.0, 0.0};
                int best_j = -1;
                double best_w = 0.0;
                auto slot = [&](int k, int j, double wk) {
                    if (k == 0 || wk > best_w) {
                        best_w = wk;
                        best_j = j;
                    }
                    if (j < 0) return;
                    const double *m = s_aff + 12 * j;
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        double e = __dadd_rn(__dadd_rn(__dmul_rn(m[4 * r], c[0]), __dmul_rn(m[4 * r + 2], c[2])),
                                             __dmul_rn(m[4 * r + 1], c[1]));
                        p[r] = __dadd_rn(p[r], __dmul_rn(wk, __dadd_rn(e, m[4 * r + 3])));
                    }
                };
                if (a.slots == 4) {
                    slot(0, v.jj.x, v.w01.x);
                    slot(1, v.jj.y, v.w01.y);
                    slot(2, v.jj.z, v.w23.x);
                    slot(3, v.jj.w, v.w23.y);
                } else {
                    for (int k = 0; k < a.slots; ++k)
                        slot(k, a.jidx[i * a.slots + k], a.w[i * a.slots + k]);
                }
                ok = true;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    // RN((p - lo) / cell) via the cell's reciprocal (div_exact: exact
                    // when the dividend is in range; else __ddiv_rn)
                    const double n = __dadd_rn(p[k], -a.lo[k]);
                    const double an = fabs(n);
                    const bool ok_n = n == 0.0 || (an >= 0x1p-400 && an <= 0x1p400);
                    double f = floor(div_exact(n, a.cell[k], ok_n ? a.rcell[k] : 0.0));
                    // NaN and out-of-range both fail this test, like the reference's
                    // int64 cast + range check (rigging.py:369-371)
                    if (!(f >= 0.0 && f < (double)a.res)) ok = false;
                    g[k] = ok ? (int64_t)f : 0;
                }
                if (a.positions) {
                    a.positions[3 * i] = p[0];
                    a.positions[3 * i + 1] = p[1];
                    a.positions[3 * i + 2] = p[2];
                }
                if (a.rot_joint) a.rot_joint[i] = best_j < 0 ? 0 : best_j;
            }
            if (a.cells_out) {
                a.cells_out[3 * i] = ok ? (int32_t)g[0] : -1;
                a.cells_out[3 * i + 1] = ok ? (int32_t)g[1] : -1;
                a.cells_out[3 * i + 2] = ok ? (int32_t)g[2] : -1;
            }
            if (a.in_bounds) a.in_bounds[i] = ok ? 1 : 0;
            if (kPipeline) {
                K key = ok ? (K)morton3((u64)g[0], (u64)g[1], (u64)g[2]) : (K)a.sentinel;
                reinterpret_cast<K *>(a.keys)[i] = key;
                if (!a.bmask) a.vals[i] = (uint32_t)i;  // sort values (the counting rebuild has none)
            }
        }
        if (kPipeline) {
            n_ok += __popc(__ballot_sync(0xffffffffu, live && ok));
            if (sizeof(K) == 4 && a.bmask) {
                // mark the cell in its brick mask (word = key >> 5: at most 32
                // cells, so per-lane atomics barely contend) and the brick in the
                // bitmap (word = key >> 14: shared by thousands of voxels, so one
                // atomicOr per distinct brick per warp -- lanes hold neighbouring
                // canonical voxels)
                const bool on = live && ok;
                const uint32_t key = on ? (uint32_t)morton3((u64)g[0], (u64)g[1], (u64)g[2]) : 0u;
                const int lane = threadIdx.x & 31;
                if (on) atomicOr(a.bmask + (key >> 5), 1u << (key & 31u));
                const uint32_t brick = on ? key >> 9 : 0xFFFFFFFFu;
                const unsigned g2 = __match_any_sync(0xffffffffu, brick);
                if (on && lane == __ffs(g2) - 1) atomicOr(a.bocc + (brick >> 5), 1u << (brick & 31u));
            }
        }
    }
    if (kPipeline) {
        // in-bounds count: one global atomic per block (a per-warp atomic on the
        // one counter serialises tens of thousands of same-address atomics in L2)
        if ((threadIdx.x & 31) == 0 && n_ok) atomicAdd(&s_in, n_ok);
        __syncthreads();
        if (threadIdx.x == 0 && s_in) atomicAdd(a.n_in, s_in);
    }
}

template <typename K>
int launch_warp(const WarpArgs &a, bool pipeline, cudaStream_t st) {
    int blocks = (int)ceil_div<int64_t>(a.n, kWarpThreads);
    if (blocks == 0) return ARTEMIS_OK;
    blocks = std::min(blocks, num_sms() * kWarpBlocksPerSM);  // persistent (see the kernel)
    if (pipeline)
        lbs_warp_kernel<K, true><<<blocks, kWarpThreads, 0, st>>>(a);
    else
        lbs_warp_kernel<K, false><<<blocks, kWarpThreads, 0, st>>>(a);
    return ARTEMIS_LAUNCHED();
}

// Device-pipeline entry used by frame.cu.
int warp_pipeline(const int32_t *cells, int64_t n, int slots, const int32_t *jidx,
                  const double *w, const double *aff, int n_joints, const double lo[3],
                  const double cell[3], int res, int key_bytes, void *keys, uint32_t *vals,
                  int32_t *rot_joint, int32_t *n_in, uint64_t sentinel, int identity,
                  uint32_t *bmask, uint32_t *bocc, cudaStream_t st) {
    if (n_joints > kMaxJoints) return ARTEMIS_ERR_ARG;
    WarpArgs a{};
    a.cells = cells;
    a.n = n;
    a.slots = slots;
    a.jidx = jidx;
    a.w = w;
    a.aff = aff;
    a.n_joints = n_joints;
    for (int k = 0; k < 3; ++k) {
        a.lo[k] = lo[k];
        a.cell[k] = cell[k];
        // IEEE double division (correctly rounded); 0 leaves div_exact on __ddiv_rn
        a.rcell[k] = (std::fabs(cell[k]) >= 0x1p-400 && std::fabs(cell[k]) <= 0x1p400) ? 1.0 / cell[k] : 0.0;
    }
    a.res = res;
    a.keys = keys;
    a.vals = vals;
    a.rot_joint = rot_joint;
    a.n_in = n_in;
    a.sentinel = sentinel;
    a.identity = identity;
    a.bmask = bmask;
    a.bocc = bocc;
    return key_bytes == 4 ? launch_warp<uint32_t>(a, true, st) : launch_warp<u64>(a, true, st);
}

}  // namespace artemis

using namespace artemis;

extern "C" int artemis_warp(const int32_t *cells, int64_t n, int slots, const int32_t *joint_idx,
                            const double *weights, const double *joint_aff, int n_joints,
                            const double *lo, const double *cell, int resolution,
                            double *positions, int32_t *cells_out, uint8_t *in_bounds,
                            int32_t *rotation_joint, artemis_stream stream) {
    if (n < 0 || slots < 1 || n_joints < 1 || n_joints > kMaxJoints || !lo || !cell)
        return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_OK;
    if (!cells || !joint_idx || !weights || !joint_aff) return ARTEMIS_ERR_ARG;
    WarpArgs a{};
    a.cells = cells;
    a.n = n;
    a.slots = slots;
    a.jidx = joint_idx;
    a.w = weights;
    a.aff = joint_aff;
    a.n_joints = n_joints;
    // lo / cell are host pointers (3 doubles each)
    for (int k = 0; k < 3; ++k) {
        a.lo[k] = lo[k];
        a.cell[k] = cell[k];
        // IEEE double division (correctly rounded); 0 leaves div_exact on __ddiv_rn
        a.rcell[k] = (std::fabs(cell[k]) >= 0x1p-400 && std::fabs(cell[k]) <= 0x1p400) ? 1.0 / cell[k] : 0.0;
    }
    a.res = resolution;
    a.positions = positions;
    a.cells_out = cells_out;
    a.in_bounds = in_bounds;
    a.rot_joint = rotation_joint;
    return launch_warp<u64>(a, false, S(stream));
}
