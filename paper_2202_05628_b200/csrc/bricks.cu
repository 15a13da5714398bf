// Per-frame occupancy brick map (see bricks.cuh). Leaves are Morton-sorted,
// so the leaves of one 8^3 brick (9 Morton bits) are one contiguous run:
// a brick record only needs the run's start, a 512-bit occupancy mask and
// per-word prefix counts to turn a cell into its leaf index.
//   pass 1 (per leaf): run heads claim a record and register it in the
//                      dense brick table; warp-reduced AABB of the leaves
//   pass 2 (per leaf): set the occupancy bit; first leaf of each mask word
//                      stores the word's prefix count
#include "bricks.cuh"
#include "tree.cuh"

namespace artemis {

template <typename K>
__global__ void brick_heads_kernel(const K *__restrict__ codes, int64_t n_host,
                                   const int32_t *__restrict__ n_dev, int32_t *table, int ox,
                                   int oy, int oz, int dx, int dy, int dz, BrickRec *recs,
                                   int32_t *counter, int32_t *aabb) {
    const int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool ok = i < n;
    const u64 c = ok ? (u64)codes[i] : 0ull;
    const int x = (int)compact_bits3(c), y = (int)compact_bits3(c >> 1), z = (int)compact_bits3(c >> 2);
    // leaf AABB: warp reduce, block reduce in shared memory, one atomic per
    // block and bound (global atomics on 6 words would serialise otherwise)
    __shared__ int red[6][8];
    const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
    int v[6] = {ok ? x : INT32_MAX, ok ? y : INT32_MAX, ok ? z : INT32_MAX,
                ok ? x + 1 : INT32_MIN, ok ? y + 1 : INT32_MIN, ok ? z + 1 : INT32_MIN};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        v[k] = __reduce_min_sync(0xffffffffu, v[k]);
        v[k + 3] = __reduce_max_sync(0xffffffffu, v[k + 3]);
    }
    if (ln == 0)
#pragma unroll
        for (int k = 0; k < 6; ++k) red[k][wid] = v[k];
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        int r = red[k][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            r = k < 3 ? min(r, red[k][w]) : max(r, red[k][w]);
        if (k < 3 ? r != INT32_MAX : r != INT32_MIN) {
            if (k < 3)
                atomicMin(aabb + k, r);
            else
                atomicMax(aabb + k, r);
        }
    }
    if (!ok) return;
    if (i > 0 && ((u64)codes[i - 1] >> 9) == (c >> 9)) return;
    const int bid = atomicAdd(counter, 1);
    const int bx = (x >> 3) - ox, by = (y >> 3) - oy, bz = (z >> 3) - oz;
    table[((size_t)bz * dy + by) * dx + bx] = bid;
    BrickRec &r = recs[bid];
    uint4 *m = reinterpret_cast<uint4 *>(r.mask);
    m[0] = m[1] = m[2] = m[3] = make_uint4(0, 0, 0, 0);
    uint4 *pf = reinterpret_cast<uint4 *>(r.prefix);
    pf[0] = pf[1] = make_uint4(0, 0, 0, 0);
    r.first = (uint32_t)i;
}

template <typename K>
__global__ void brick_bits_kernel(const K *__restrict__ codes, int64_t n_host,
                                  const int32_t *__restrict__ n_dev,
                                  const int32_t *__restrict__ table, int ox, int oy, int oz,
                                  int dx, int dy, int dz, BrickRec *recs) {
    const int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u64 c = (u64)codes[i];
    const int x = (int)compact_bits3(c), y = (int)compact_bits3(c >> 1), z = (int)compact_bits3(c >> 2);
    const int bx = (x >> 3) - ox, by = (y >> 3) - oy, bz = (z >> 3) - oz;
    const int bid = table[((size_t)bz * dy + by) * dx + bx];
    BrickRec &r = recs[bid];
    const uint32_t m = (uint32_t)(c & 511u), w = m >> 5;
    atomicOr(&r.mask[w], 1u << (m & 31u));
    // the first leaf of each mask word records how many of the brick's
    // leaves precede that word (brick + word = the code without its low 5 bits)
    if (i == (int64_t)r.first || ((u64)codes[i - 1] >> 5) != (c >> 5))
        r.prefix[w] = (uint16_t)(i - r.first);
}

template <typename K>
int build_bricks(const K *codes, int64_t n_host, const int32_t *n_dev, int64_t n_cap,
                 const int org[3], const int dims[3], int32_t *table, BrickRec *recs,
                 int32_t *counter, int32_t *aabb, cudaStream_t st) {
    const size_t cells = (size_t)dims[0] * dims[1] * dims[2];
    ARTEMIS_TRY(cudaMemsetAsync(table, 0xFF, cells * sizeof(int32_t), st));
    ARTEMIS_TRY(cudaMemsetAsync(counter, 0, sizeof(int32_t), st));
    ARTEMIS_TRY(cudaMemsetAsync(aabb, 0x7F, 3 * sizeof(int32_t), st));      // INT-ish max
    ARTEMIS_TRY(cudaMemsetAsync(aabb + 3, 0x80, 3 * sizeof(int32_t), st));  // negative
    if (n_cap <= 0) return ARTEMIS_OK;
    const int blocks = (int)ceil_div<int64_t>(n_cap, 256);
    brick_heads_kernel<K><<<blocks, 256, 0, st>>>(codes, n_host, n_dev, table, org[0], org[1],
                                                   org[2], dims[0], dims[1], dims[2], recs,
                                                   counter, aabb);
    brick_bits_kernel<K><<<blocks, 256, 0, st>>>(codes, n_host, n_dev, table, org[0], org[1],
                                                  org[2], dims[0], dims[1], dims[2], recs);
    return ARTEMIS_LAUNCHED();
}

template int build_bricks<u64>(const u64 *, int64_t, const int32_t *, int64_t, const int *,
                               const int *, int32_t *, BrickRec *, int32_t *, int32_t *,
                               cudaStream_t);
template int build_bricks<uint32_t>(const uint32_t *, int64_t, const int32_t *, int64_t,
                                    const int *, const int *, int32_t *, BrickRec *, int32_t *,
                                    int32_t *, cudaStream_t);

}  // namespace artemis

using namespace artemis;

extern "C" size_t artemis_brickmap_bytes(int64_t n_leaves, const int32_t *dims) {
    if (!dims || n_leaves < 1) return 0;
    const size_t cells = (size_t)dims[0] * dims[1] * dims[2];
    return ((cells * 4 + 255) & ~size_t(255)) + (size_t)n_leaves * sizeof(BrickRec) + 256;
}

extern "C" int artemis_brickmap_build(const uint64_t *codes, int64_t n, const int32_t *org,
                                      const int32_t *dims, void *storage, size_t storage_bytes,
                                      artemis_brickmap *out, artemis_stream stream) {
    if (!codes || n < 1 || !org || !dims || !storage || !out) return ARTEMIS_ERR_ARG;
    if (storage_bytes < artemis_brickmap_bytes(n, dims)) return ARTEMIS_ERR_WORKSPACE;
    const size_t cells = (size_t)dims[0] * dims[1] * dims[2];
    char *base = static_cast<char *>(storage);
    int32_t *table = reinterpret_cast<int32_t *>(base);
    BrickRec *recs = reinterpret_cast<BrickRec *>(base + ((cells * 4 + 255) & ~size_t(255)));
    int32_t *meta = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(recs) + n * sizeof(BrickRec));
    const int o[3] = {org[0], org[1], org[2]}, dm[3] = {dims[0], dims[1], dims[2]};
    out->table = table;
    out->recs = recs;
    out->aabb = meta + 1;
    for (int a = 0; a < 3; ++a) {
        out->org[a] = org[a];
        out->dims[a] = dims[a];
    }
    return build_bricks<u64>(reinterpret_cast<const u64 *>(codes), n, nullptr, n, o, dm, table,
                             recs, meta, meta + 1, S(stream));
}

