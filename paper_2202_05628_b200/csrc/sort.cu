// Stable LSD radix sort of (key, value) pairs: one upfront histogram pass
// for every digit, then one "onesweep" pass per 8-bit digit with decoupled
// look-back across tiles (Adinets & Merrill's single-pass scheme), no CUB.
//
// Replaces animvox/_core.pyx:111-167 sort_order: same digit width, same
// number of passes (ceil(bits/8) of the largest key) and the same stability
// (equal keys keep their input order), so the permutation is identical.
//
// Tile = 8 warps x 16 items x 32 lanes = 4096 keys. Warp w owns the
// contiguous 512-key chunk w of the tile and walks it in 16 coalesced rows;
// ranks are built row by row (peer lanes from 8 bit-plane ballots) so the (warp, row, lane)
// order -- i.e. input order -- is preserved inside each digit. Thread d of
// the CTA then owns digit d: it prefixes the 8 warp counts, publishes the
// tile aggregate, and walks back over earlier tiles' published values
// (flag in the top 2 bits of one 32-bit word: 0 = pending, 1 = aggregate,
// 2 = inclusive prefix) until it meets an inclusive prefix, reading the
// statuses of kLook predecessors per memory round trip.
#include "common.cuh"
#include "tree.cuh"

namespace artemis {

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kWarpTile = 32 * kItems;
constexpr int kRadix = 256;
constexpr uint32_t kValMask = (1u << 30) - 1;
constexpr int kLook = 32;  // look-back window (tiles whose status is read at once)

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct SortLayout {
    int passes;
    int64_t tiles;
    size_t alt_keys, alt_vals, hist, status, counters, total;
};

SortLayout layout(int64_t n, int key_bits, int key_bytes) {
    SortLayout L;
    L.passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
    L.tiles = ceil_div<int64_t>(n > 0 ? n : 1, kTile);
    size_t off = 0;
    L.alt_keys = off;
    off += align256((size_t)n * key_bytes);
    L.alt_vals = off;
    off += align256((size_t)n * 4);
    L.hist = off;  // hist, status and counters are zeroed by one memset
    off += align256((size_t)L.passes * kRadix * 4);
    L.status = off;
    off += align256((size_t)L.passes * L.tiles * kRadix * 4);
    L.counters = off;
    off += align256((size_t)L.passes * 4);
    L.total = off;
    return L;
}

__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
}  // namespace

template <typename K>
__global__ void __launch_bounds__(kThreads) radix_hist_kernel(const K *__restrict__ keys, int64_t n,
                                                              int passes, uint32_t *hist) {
    __shared__ uint32_t sh[8 * kRadix];
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        K k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * kRadix + (int)((k >> (8 * p)) & 0xFF)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// exclusive scan of each pass's 256 counts, in place; one block per pass
__global__ void __launch_bounds__(kRadix) radix_scan_kernel(uint32_t *hist) {
    __shared__ uint32_t warp_sum[kRadix / 32];
    uint32_t *h = hist + blockIdx.x * kRadix;
    int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v = h[t], x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    uint32_t base = 0;
    for (int i = 0; i < w; ++i) base += warp_sum[i];
    h[t] = base + x - v;
}

template <typename K, bool kIota>
__global__ void __launch_bounds__(kThreads) onesweep_kernel(
    const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const uint32_t *__restrict__ digit_offsets,
    uint32_t *status, uint32_t *tile_counter) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t whist[kWarps][kRadix];
    __shared__ uint32_t dbase[kRadix];
    __shared__ uint32_t tpre[kRadix];   // tile-local exclusive prefix per digit
    __shared__ uint32_t wsum[kWarps];
    extern __shared__ __align__(16) unsigned char s_stage[];  // tile reordered by digit
    K *skey = reinterpret_cast<K *>(s_stage);
    uint32_t *sval = reinterpret_cast<uint32_t *>(s_stage + kTile * sizeof(K));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int i = tid; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kTile + (int64_t)warp * kWarpTile;

    K key[kItems];
    uint32_t val[kItems];
    uint32_t rank[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        int64_t idx = base + j * 32 + lane;
        bool ok = idx < n;
        key[j] = ok ? kin[idx] : K(0);
        val[j] = ok ? (kIota ? (uint32_t)idx : vin[idx]) : 0u;
    }
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        int64_t idx = base + j * 32 + lane;
        unsigned valid = __ballot_sync(0xffffffffu, idx < n);
        // lanes holding the same digit: 8 bit-plane ballots (cheaper than
        // __match_any_sync when a row holds many distinct digits)
        const uint32_t dj = (uint32_t)((key[j] >> shift) & 0xFF);
        unsigned peers = valid;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const unsigned bb = __ballot_sync(0xffffffffu, (dj >> b) & 1u);
            peers &= ((dj >> b) & 1u) ? bb : ~bb;
        }
        if (idx < n) {
            uint32_t d = dj;
            uint32_t prev = whist[warp][d];
            __syncwarp(valid);
            if (lane == __ffs(peers) - 1) whist[warp][d] = prev + __popc(peers);
            __syncwarp(valid);
            rank[j] = prev + __popc(peers & lt);
        }
    }
    __syncthreads();
    const int d = tid;  // kThreads == kRadix: thread d owns digit d
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        uint32_t x = whist[w][d];
        whist[w][d] = tot;
        tot += x;
    }
    uint32_t *mine = status + tile * kRadix + d;
    // publish this tile's aggregate first: later tiles sum it while this one
    // stages its keys and looks back
    st_relaxed(mine, (tile == 0 ? 2u << 30 : 1u << 30) | tot);
    {   // tile-local digit offsets (block exclusive scan of the counts)
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += wsum[w];
        tpre[d] = wpre + x - tot;
    }
    __syncthreads();
    // stage the tile in digit order (frees the key/value registers for the
    // look-back); each digit's run is written out with consecutive threads
    // on consecutive addresses below
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        int64_t idx = base + j * 32 + lane;
        if (idx < n) {
            uint32_t dd = (uint32_t)((key[j] >> shift) & 0xFF);
            uint32_t lp = tpre[dd] + whist[warp][dd] + rank[j];
            ARTEMIS_DCHECK(lp < (uint32_t)kTile);
            skey[lp] = key[j];
            sval[lp] = val[j];
        }
    }
    {
        uint32_t excl = 0;
        if (tile > 0) {
            // look back kLook predecessors at a time: their statuses are
            // loaded together (one memory round trip per window, not per
            // tile -- every tile of a small sort is resident at once, so
            // the walk back can be long), then consumed nearest first
            bool done = false;
            for (int64_t k = tile - 1; !done; k -= kLook) {
                uint32_t w[kLook];
#pragma unroll
                for (int i = 0; i < kLook; ++i)
                    w[i] = k - i >= 0 ? ld_relaxed(status + (k - i) * kRadix + d) : (2u << 30);
#pragma unroll
                for (int i = 0; i < kLook; ++i) {
                    if (done) break;
                    uint32_t sv = w[i];
                    while ((sv >> 30) == 0) sv = ld_relaxed(status + (k - i) * kRadix + d);
                    excl += sv & kValMask;
                    if ((sv >> 30) == 2) done = true;
                }
            }
            st_relaxed(mine, (2u << 30) | (excl + tot));
        }
        dbase[d] = digit_offsets[d] + excl - tpre[d];
    }
    __syncthreads();
    const int tile_n = (int)std::min<int64_t>(kTile, n - tile * kTile);
    for (int i = tid; i < tile_n; i += kThreads) {
        const K k = skey[i];
        const uint32_t pos = dbase[(uint32_t)((k >> shift) & 0xFF)] + (uint32_t)i;
        ARTEMIS_DCHECK((int64_t)pos < n);
        kout[pos] = k;
        vout[pos] = sval[i];
    }
}

size_t sort_workspace_bytes(int64_t n, int key_bits, int key_bytes) {
    return layout(n, key_bits, key_bytes).total;
}

template <typename K>
int sort_pairs(const K *keys_in, const uint32_t *vals_in, K *keys_out, uint32_t *vals_out,
               int64_t n, int key_bits, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (n < 0 || n >= (int64_t(1) << 30) || key_bits < 0 || key_bits > 8 * (int)sizeof(K))
        return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_OK;
    if (!keys_in || !keys_out || !vals_out) return ARTEMIS_ERR_ARG;
    SortLayout L = layout(n, key_bits, (int)sizeof(K));
    if (!ws || ws_bytes < L.total) return ARTEMIS_ERR_WORKSPACE;
    char *w = static_cast<char *>(ws);
    K *alt_k = reinterpret_cast<K *>(w + L.alt_keys);
    uint32_t *alt_v = reinterpret_cast<uint32_t *>(w + L.alt_vals);
    uint32_t *hist = reinterpret_cast<uint32_t *>(w + L.hist);
    uint32_t *status = reinterpret_cast<uint32_t *>(w + L.status);
    uint32_t *counters = reinterpret_cast<uint32_t *>(w + L.counters);
    ARTEMIS_TRY(cudaMemsetAsync(w + L.hist, 0, L.total - L.hist, st));
    int hist_blocks = (int)std::min<int64_t>(ceil_div<int64_t>(n, kThreads * 8),
                                             (int64_t)num_sms() * 4);
    radix_hist_kernel<K><<<hist_blocks, kThreads, 0, st>>>(keys_in, n, L.passes, hist);
    radix_scan_kernel<<<L.passes, kRadix, 0, st>>>(hist);
    const size_t stage = (size_t)kTile * (sizeof(K) + 4);
    // the opt-in is per device (and context): set it on every call, as the
    // render launches do -- it costs ~1 us and is legal during graph capture
    ARTEMIS_TRY(cudaFuncSetAttribute(onesweep_kernel<K, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage));
    ARTEMIS_TRY(cudaFuncSetAttribute(onesweep_kernel<K, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage));
    const K *src_k = keys_in;
    const uint32_t *src_v = vals_in;
    for (int p = 0; p < L.passes; ++p) {
        bool to_out = ((L.passes - 1 - p) % 2) == 0;
        K *dk = to_out ? keys_out : alt_k;
        uint32_t *dv = to_out ? vals_out : alt_v;
        uint32_t *stp = status + (size_t)p * L.tiles * kRadix;
        if (p == 0 && !vals_in)
            onesweep_kernel<K, true><<<(int)L.tiles, kThreads, stage, st>>>(
                src_k, nullptr, dk, dv, n, 8 * p, hist + p * kRadix, stp, counters + p);
        else
            onesweep_kernel<K, false><<<(int)L.tiles, kThreads, stage, st>>>(
                src_k, src_v, dk, dv, n, 8 * p, hist + p * kRadix, stp, counters + p);
        src_k = dk;
        src_v = dv;
    }
    return ARTEMIS_LAUNCHED();
}

template int sort_pairs<u64>(const u64 *, const uint32_t *, u64 *, uint32_t *, int64_t, int,
                             void *, size_t, cudaStream_t);
template int sort_pairs<uint32_t>(const uint32_t *, const uint32_t *, uint32_t *, uint32_t *,
                                  int64_t, int, void *, size_t, cudaStream_t);

}  // namespace artemis

using namespace artemis;

extern "C" size_t artemis_sort_workspace_bytes(int64_t n, int key_bits, int key_bytes) {
    return sort_workspace_bytes(n, key_bits, key_bytes);
}

extern "C" int artemis_sort_pairs_u64(const uint64_t *keys_in, const uint32_t *vals_in,
                                      uint64_t *keys_out, uint32_t *vals_out, int64_t n,
                                      int key_bits, void *workspace, size_t workspace_bytes,
                                      artemis_stream stream) {
    return sort_pairs<u64>(reinterpret_cast<const u64 *>(keys_in), vals_in,
                           reinterpret_cast<u64 *>(keys_out), vals_out, n, key_bits, workspace,
                           workspace_bytes, S(stream));
}

extern "C" int artemis_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in,
                                      uint32_t *keys_out, uint32_t *vals_out, int64_t n,
                                      int key_bits, void *workspace, size_t workspace_bytes,
                                      artemis_stream stream) {
    return sort_pairs<uint32_t>(keys_in, vals_in, keys_out, vals_out, n, key_bits, workspace,
                                workspace_bytes, S(stream));
}
