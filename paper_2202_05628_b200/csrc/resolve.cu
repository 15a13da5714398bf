// Collision resolve over stably-sorted warped keys.
//
// Replaces animvox/rigging.py:433-459 (resolve_collisions): the reference
// lexsorts (code, -sigma, canonical index), keeps the first row of every
// code group as the winner and emits (winner, loser) pairs in that order.
// Here the keys arrive sorted stably by code with canonical indices
// ascending inside each group (the sort is stable and the warp kernel
// emits indices in order), so a group is a contiguous run; every entry
// ranks itself inside its run by (-sigma, index) -- runs are a handful of
// voxels -- and the live-cell index u of its run comes from an inclusive
// scan of run heads.
//   pass 1  per-block run-head counts
//   pass 2  one block scans the block counts (and writes n_live)
//   pass 3  per entry: u, rank; rank 0 writes (live code, winner), others
//           write their pair row (group start - u + rank - 1)
#include "common.cuh"
#include "tree.cuh"

namespace artemis {

namespace {
constexpr int kBlock = 256;
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

template <typename K>
__device__ __forceinline__ bool run_head(const K *c, int64_t i) {
    return i == 0 || c[i] != c[i - 1];
}

template <typename K>
__global__ void __launch_bounds__(kBlock) head_count_kernel(const K *__restrict__ codes,
                                                            int64_t n_host,
                                                            const int32_t *__restrict__ n_dev,
                                                            uint32_t *__restrict__ block_counts) {
    int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    bool h = i < n && run_head(codes, i);
    int c = __syncthreads_count(h);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = (uint32_t)c;
}

__global__ void __launch_bounds__(1024) block_scan_kernel(uint32_t *counts, int64_t nb,
                                                          int32_t *n_live) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
        int64_t b = b0 + threadIdx.x;
        uint32_t v = b < nb ? counts[b] : 0u, x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[w] = x;
        __syncthreads();
        uint32_t off = carry;
        for (int k = 0; k < w; ++k) off += warp_tot[k];
        if (b < nb) counts[b] = off + x - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = off + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_live = (int32_t)carry;
}

// Order of a collision group in the reference's np.lexsort((idx, -sigma,
// code)) (rigging.py:435): larger density first, ties by lower canonical
// index; NaN densities sort last (numpy puts NaN after every number), among
// themselves by index. A strict total order, so exactly one entry has rank 0
// even when densities are NaN.
__device__ __forceinline__ bool precedes(double sa, uint32_t a, double sb, uint32_t b) {
    const bool na = isnan(sa), nb = isnan(sb);
    if (na != nb) return nb;  // the number precedes the NaN
    if (na) return a < b;
    return sa > sb || (sa == sb && a < b);
}

template <typename K, bool kPairs>
__global__ void __launch_bounds__(kBlock) resolve_kernel(
    const K *__restrict__ codes, const uint32_t *__restrict__ idx, int64_t n_host,
    const int32_t *__restrict__ n_dev, const double *__restrict__ sigma,
    const uint32_t *__restrict__ block_offsets, K *__restrict__ live_codes,
    uint32_t *__restrict__ winners, int64_t *__restrict__ pairs) {
    __shared__ uint32_t warp_tot[kBlock / 32];
    int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    bool valid = i < n;
    uint32_t h = valid && run_head(codes, i) ? 1u : 0u, x = h;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (!valid) return;
    uint32_t incl = block_offsets[blockIdx.x] + x;
    for (int k = 0; k < w; ++k) incl += warp_tot[k];
    const int64_t u = (int64_t)incl - 1;  // live-cell index of i's run

    const K c = codes[i];
    int64_t s = i, e = i + 1;
    while (s > 0 && codes[s - 1] == c) --s;
    while (e < n && codes[e] == c) ++e;
    const uint32_t me = idx[i];
    const double sm = sigma[me];
    int64_t rank = 0;
    uint32_t best = me;
    double best_s = sm;
    for (int64_t m = s; m < e; ++m) {
        uint32_t o = idx[m];
        double so = sigma[o];
        if (precedes(so, o, sm, me)) ++rank;
        if (precedes(so, o, best_s, best)) {
            best = o;
            best_s = so;
        }
    }
    ARTEMIS_DCHECK(u >= 0 && u < n && u <= i);
    if (rank == 0) {
        live_codes[u] = c;
        winners[u] = me;
    } else if (kPairs) {
        int64_t row = s - u + rank - 1;
        ARTEMIS_DCHECK(row >= 0 && row < n);
        pairs[2 * row] = (int64_t)best;
        pairs[2 * row + 1] = (int64_t)me;
    }
}

size_t resolve_workspace_bytes(int64_t n) {
    return align256((size_t)ceil_div<int64_t>(n > 0 ? n : 1, kBlock) * 4);
}

template <typename K>
int resolve(const K *sorted_codes, const uint32_t *sorted_idx, int64_t n_host,
            const int32_t *n_dev, const double *sigma, K *live_codes, uint32_t *winners,
            int64_t *pairs, int32_t *n_live, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (n_host < 0 || !n_live) return ARTEMIS_ERR_ARG;
    if (n_host == 0) {
        ARTEMIS_TRY(cudaMemsetAsync(n_live, 0, 4, st));
        return ARTEMIS_OK;
    }
    if (!sorted_codes || !sorted_idx || !sigma || !live_codes || !winners) return ARTEMIS_ERR_ARG;
    if (!ws || ws_bytes < resolve_workspace_bytes(n_host)) return ARTEMIS_ERR_WORKSPACE;
    int64_t nb = ceil_div<int64_t>(n_host, kBlock);
    uint32_t *counts = static_cast<uint32_t *>(ws);
    head_count_kernel<K><<<(int)nb, kBlock, 0, st>>>(sorted_codes, n_host, n_dev, counts);
    block_scan_kernel<<<1, 1024, 0, st>>>(counts, nb, n_live);
    if (pairs)
        resolve_kernel<K, true><<<(int)nb, kBlock, 0, st>>>(sorted_codes, sorted_idx, n_host, n_dev,
                                                            sigma, counts, live_codes, winners,
                                                            pairs);
    else
        resolve_kernel<K, false><<<(int)nb, kBlock, 0, st>>>(sorted_codes, sorted_idx, n_host,
                                                             n_dev, sigma, counts, live_codes,
                                                             winners, nullptr);
    return ARTEMIS_LAUNCHED();
}

template int resolve<u64>(const u64 *, const uint32_t *, int64_t, const int32_t *, const double *,
                          u64 *, uint32_t *, int64_t *, int32_t *, void *, size_t, cudaStream_t);
template int resolve<uint32_t>(const uint32_t *, const uint32_t *, int64_t, const int32_t *,
                               const double *, uint32_t *, uint32_t *, int64_t *, int32_t *,
                               void *, size_t, cudaStream_t);

}  // namespace artemis

using namespace artemis;

extern "C" size_t artemis_resolve_workspace_bytes(int64_t n_sorted) {
    return resolve_workspace_bytes(n_sorted);
}

extern "C" int artemis_resolve_u64(const uint64_t *sorted_codes, const uint32_t *sorted_idx,
                                   int64_t n_sorted, const int32_t *n_sorted_dev,
                                   const double *sigma, uint64_t *live_codes, uint32_t *winners,
                                   int64_t *pairs, int32_t *n_live_out, void *workspace,
                                   size_t workspace_bytes, artemis_stream stream) {
    return resolve<u64>(reinterpret_cast<const u64 *>(sorted_codes), sorted_idx, n_sorted,
                        n_sorted_dev, sigma, reinterpret_cast<u64 *>(live_codes), winners, pairs,
                        n_live_out, workspace, workspace_bytes, S(stream));
}
