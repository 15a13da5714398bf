// Morton codes, Karras radix-tree build and the packed traversal layout.
//
// build_tree follows animvox/_core.pyx:193-246 node for node: direction from
// the neighbouring prefix lengths, exponential then binary range search,
// split bisection, ~leaf child links, octant boxes from the common prefix.
// One thread per internal node; the same thread also writes the node's
// 32-byte packed record (both children's boxes) for the render kernels, so
// the device pipeline never re-derives boxes at traversal time.
#include "common.cuh"
#include "tree.cuh"

namespace artemis {

__global__ void morton_encode_kernel(const int64_t *__restrict__ xyz, int64_t n,
                                     u64 *__restrict__ codes, int32_t *__restrict__ range_flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    const int64_t lim = int64_t(1) << 21;
    if (range_flag && (x < 0 || y < 0 || z < 0 || x >= lim || y >= lim || z >= lim))
        *range_flag = 1;
    codes[i] = morton3((u64)x, (u64)y, (u64)z);
}

__global__ void morton_decode_kernel(const u64 *__restrict__ codes, int64_t n,
                                     int64_t *__restrict__ xyz) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    u64 c = codes[i];
    xyz[3 * i] = (int64_t)compact_bits3(c);
    xyz[3 * i + 1] = (int64_t)compact_bits3(c >> 1);
    xyz[3 * i + 2] = (int64_t)compact_bits3(c >> 2);
}

template <typename K>
__device__ __forceinline__ int prefix_len(const K *__restrict__ c, int64_t n, int64_t i,
                                          int64_t j) {
    if (j < 0 || j >= n) return -1;
    u64 x = (u64)c[i] ^ (u64)c[j];
    return x ? __clzll((long long)x) : 64;
}

// 32-byte leaf record: {x, y, z, FLUT row} + {density (fp64), rotation
// index, 0}, so the render kernel gets everything a hit needs in one sector.
__device__ __forceinline__ void write_leaf(uint4 *leaves, int64_t i, u64 c, uint32_t row,
                                           const double *sigma, const int32_t *rot_index) {
    const double sg = sigma ? sigma[row] : 0.0;
    const unsigned long long sb = (unsigned long long)__double_as_longlong(sg);
    leaves[2 * i] = make_uint4((uint32_t)compact_bits3(c), (uint32_t)compact_bits3(c >> 1),
                               (uint32_t)compact_bits3(c >> 2), row);
    leaves[2 * i + 1] = make_uint4((uint32_t)sb, (uint32_t)(sb >> 32),
                                   rot_index ? (uint32_t)rot_index[row] : 0u, 0u);
}

// Split of the Karras node covering the sorted range [first, last]
// (_core.pyx:233-242): the last index sharing more than the range's common
// prefix with `first`.
template <typename K>
__device__ __forceinline__ int64_t range_split(const K *__restrict__ c, int64_t n, int64_t first,
                                               int64_t last) {
    const int node_len = prefix_len(c, n, first, last);
    int64_t split = first, step = last - first;
    do {
        step = (step + 1) >> 1;
        if (split + step < last && prefix_len(c, n, first, split + step) > node_len)
            split += step;
    } while (step > 1);
    return split;
}

// The two grandchild slots contributed by child range [a, b].
template <typename K>
__device__ __forceinline__ void wide_group(const K *__restrict__ c, int64_t n, int64_t a,
                                           int64_t b, uint32_t *w) {
    if (a == b) {  // the child is a leaf: one slot, the other absent
        pack_child(w, (u64)c[a], (u64)c[a], ~(int32_t)a);
        w[4] = kAbsent;
        w[5] = w[6] = w[7] = 0;
        return;
    }
    const int64_t s = range_split(c, n, a, b);
    pack_child(w, (u64)c[a], (u64)c[s], s == a ? ~(int32_t)s : (int32_t)s);
    pack_child(w + 4, (u64)c[s + 1], (u64)c[b], s + 1 == b ? ~(int32_t)(s + 1) : (int32_t)(s + 1));
    w[4] |= (uint32_t)split_axis_of(range_free_bits((u64)c[a], (u64)c[b])) << 27;
}

__device__ __forceinline__ void store_wide(WideNode *dst, const uint32_t *w) {
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
    d[2] = make_uint4(w[8], w[9], w[10], w[11]);
    d[3] = make_uint4(w[12], w[13], w[14], w[15]);
}

// Karras node i (i < n-1). Writes reference arrays (when non-null) and the
// traversal record; node 0 also writes the super-root record at index n-1.
template <typename K>
__device__ void build_node(const K *__restrict__ c, int64_t n, int64_t i, int32_t *left,
                           int32_t *right, int32_t *bmin, int32_t *bsize, WideNode *nodes,
                           int32_t *dup_flag) {
    int dir = prefix_len(c, n, i, i + 1) > prefix_len(c, n, i, i - 1) ? 1 : -1;
    int floor_len = prefix_len(c, n, i, i - dir);
    int64_t hi = 2;
    while (prefix_len(c, n, i, i + hi * dir) > floor_len) hi <<= 1;
    int64_t len = 0;
    for (int64_t t = hi >> 1; t >= 1; t >>= 1)
        if (prefix_len(c, n, i, i + (len + t) * dir) > floor_len) len += t;
    int64_t j = i + len * dir;
    int64_t first = dir > 0 ? i : j, last = dir > 0 ? j : i;
    int node_len = prefix_len(c, n, first, last);
    int64_t split = first, step = last - first;
    do {
        step = (step + 1) >> 1;
        if (split + step < last && prefix_len(c, n, first, split + step) > node_len)
            split += step;
    } while (step > 1);
    int32_t l = split == first ? ~(int32_t)split : (int32_t)split;
    int32_t r = split + 1 == last ? ~(int32_t)(split + 1) : (int32_t)(split + 1);
    u64 cf = (u64)c[first], cl = (u64)c[last];
    if (left) {
        left[i] = l;
        right[i] = r;
        int fb = range_free_bits(cf, cl);
        u64 base = fb >= 64 ? 0ull : (cf >> fb) << fb;
        bmin[3 * i] = (int32_t)compact_bits3(base);
        bmin[3 * i + 1] = (int32_t)compact_bits3(base >> 1);
        bmin[3 * i + 2] = (int32_t)compact_bits3(base >> 2);
        bsize[3 * i] = box_size_axis(fb, 0);
        bsize[3 * i + 1] = box_size_axis(fb, 1);
        bsize[3 * i + 2] = box_size_axis(fb, 2);
    }
    if (nodes) {
        uint32_t w[16];
        wide_group(c, n, first, split, w);
        wide_group(c, n, split + 1, last, w + 8);
        w[0] |= (uint32_t)split_axis_of(range_free_bits(cf, cl)) << 27;
        store_wide(nodes + i, w);
        if (i == 0) {  // super-root: slot 0 = the root, the rest absent
            uint32_t sr[16] = {0};
            pack_child(sr, (u64)c[0], (u64)c[n - 1], 0);
            sr[4] = sr[8] = sr[12] = kAbsent;
            store_wide(nodes + (n - 1), sr);
        }
    }
    if (dup_flag && c[i] == c[i + 1]) atomicMin(dup_flag, (int32_t)i);
}

template <typename K>
__global__ void build_tree_kernel(const K *__restrict__ codes, int64_t n_host,
                                  const int32_t *__restrict__ n_dev, int32_t *left, int32_t *right,
                                  int32_t *bmin, int32_t *bsize, WideNode *nodes,
                                  uint4 *leaves, const uint32_t *__restrict__ leaf_flut,
                                  const double *__restrict__ sigma,
                                  const int32_t *__restrict__ rot_index, int32_t *dup_flag) {
    int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (leaves && i < n) write_leaf(leaves, i, (u64)codes[i], leaf_flut[i], sigma, rot_index);
    if (n == 1 && i == 0 && nodes) {
        // single leaf: root = ~0, only the super-root record exists
        uint32_t sr[16] = {0};
        const u64 c0 = (u64)codes[0];
        pack_child(sr, c0, c0, ~0);
        sr[4] = sr[8] = sr[12] = kAbsent;
        store_wide(nodes, sr);
        return;
    }
    if (i >= n - 1) return;
    build_node(codes, n, i, left, right, bmin, bsize, nodes, dup_flag);
}

// API path: traversal records from the reference arrays (any valid tree).
__global__ void pack_tree_kernel(const u64 *__restrict__ codes,
                                 const uint32_t *__restrict__ flut_idx, int64_t n, int32_t root,
                                 const int32_t *__restrict__ left, const int32_t *__restrict__ right,
                                 const int32_t *__restrict__ bmin,
                                 const int32_t *__restrict__ bsize, WideNode *nodes,
                                 uint4 *leaves, const double *__restrict__ sigma,
                                 const int32_t *__restrict__ rot_index) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) write_leaf(leaves, i, codes[i], flut_idx[i], sigma, rot_index);
    auto log2i = [](int32_t v) { return (uint32_t)(__ffs(v) - 1); };
    auto axis_of = [&](int32_t node) {
        const int32_t *s = bsize + 3 * node;
        return (uint32_t)split_axis_of((int)(log2i(s[0]) + log2i(s[1]) + log2i(s[2]))) << 27;
    };
    auto slot = [&](uint32_t *w, int32_t link) {
        if (link < 0) {
            u64 c = codes[~link];
            w[0] = (uint32_t)compact_bits3(c);
            w[1] = (uint32_t)compact_bits3(c >> 1);
            w[2] = (uint32_t)compact_bits3(c >> 2);
        } else {
            const int32_t *m = bmin + 3 * link, *s = bsize + 3 * link;
            w[0] = (uint32_t)m[0] | (log2i(s[0]) << 21);
            w[1] = (uint32_t)m[1] | (log2i(s[1]) << 21);
            w[2] = (uint32_t)m[2] | (log2i(s[2]) << 21);
        }
        w[3] = (uint32_t)link;
    };
    auto group = [&](uint32_t *w, int32_t child) {
        if (child < 0) {
            slot(w, child);
            w[4] = kAbsent;
            w[5] = w[6] = w[7] = 0;
        } else {
            slot(w, left[child]);
            slot(w + 4, right[child]);
            w[4] |= axis_of(child);
        }
    };
    uint32_t w[16] = {0};
    if (i < n - 1) {
        group(w, left[i]);
        group(w + 8, right[i]);
        w[0] |= axis_of((int32_t)i);
    } else if (i == (n > 1 ? n - 1 : 0)) {
        slot(w, root);
        w[4] = w[8] = w[12] = kAbsent;
    } else {
        return;
    }
    store_wide(nodes + i, w);
}

// 32-bit Morton codes (grids up to 2^10 per axis: the frame pipeline) and
// fewer than 2^30 leaves, reference arrays + leaf records only: the same
// node-for-node construction as build_node (_core.pyx:193-246) in 32-bit
// integer arithmetic -- prefix lengths are clz of the 32-bit XOR (the 64-bit
// lengths minus 32, the same comparisons), indices are int, the bisections
// compare codes against the split threshold instead of recomputing prefix
// lengths. The 64-bit build spent most of its issue slots on emulated
// 64-bit index and bit arithmetic.
__device__ __forceinline__ uint32_t compact_bits3_32(uint32_t v) {
    // compact_bits3 restricted to 32-bit inputs (the same masks, truncated)
    v &= 0x49249249u;
    v = (v ^ (v >> 2)) & 0xC30C30C3u;
    v = (v ^ (v >> 4)) & 0x0F00F00Fu;
    v = (v ^ (v >> 8)) & 0xFF0000FFu;
    v = (v ^ (v >> 16)) & 0x0000FFFFu;
    return v;
}

__global__ void __launch_bounds__(256) build_tree32_kernel(
    const uint32_t *__restrict__ c, int n_host, const int32_t *__restrict__ n_dev, int32_t *left,
    int32_t *right, int32_t *bmin, int32_t *bsize, uint4 *leaves,
    const uint32_t *__restrict__ leaf_flut, const double *__restrict__ sigma,
    const int32_t *__restrict__ rot_index) {
    griddep_wait();
    griddep_launch_dependents();
    const int n = n_dev ? *n_dev : n_host;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t ci = __ldg(c + i);
    if (leaves) {
        const uint32_t row = __ldg(leaf_flut + i);
        const double sg = sigma ? __ldg(sigma + row) : 0.0;
        const unsigned long long sb = (unsigned long long)__double_as_longlong(sg);
        leaves[2 * (size_t)i] =
            make_uint4(compact_bits3_32(ci), compact_bits3_32(ci >> 1), compact_bits3_32(ci >> 2), row);
        leaves[2 * (size_t)i + 1] = make_uint4((uint32_t)sb, (uint32_t)(sb >> 32),
                                               rot_index ? (uint32_t)__ldg(rot_index + row) : 0u, 0u);
    }
    if (i >= n - 1) return;
    // prefix length of codes i and j (-1 outside the array; 32 = equal)
    auto pl = [&](int j) -> int {
        if ((unsigned)j >= (unsigned)n) return -1;
        const uint32_t x = ci ^ __ldg(c + j);
        return x ? __clz(x) : 32;
    };
    const int dir = pl(i + 1) > pl(i - 1) ? 1 : -1;
    const int floor_len = pl(i - dir);
    int hi = 2;
    while (pl(i + hi * dir) > floor_len) hi <<= 1;
    int len = 0;
    for (int t = hi >> 1; t >= 1; t >>= 1)
        if (pl(i + (len + t) * dir) > floor_len) len += t;
    const int j = i + len * dir;
    const int first = dir > 0 ? i : j, last = dir > 0 ? j : i;
    const uint32_t cf = dir > 0 ? ci : __ldg(c + first), cl = dir > 0 ? __ldg(c + last) : ci;
    // split = the last index sharing more than the range's common prefix with
    // `first`: the last code below the prefix followed by a 1 bit (the codes
    // of a range are sorted and share its prefix)
    const uint32_t x = cf ^ cl;
    const int fb = x ? 32 - __clz(x) : 0;  // range_free_bits
    int split = first;
    if (x) {
        const uint32_t thr = (cl >> (fb - 1)) << (fb - 1);
        int step = last - first;
        do {
            step = (step + 1) >> 1;
            if (split + step < last && __ldg(c + split + step) < thr) split += step;
        } while (step > 1);
    }  // equal codes (duplicates): no longer prefix exists, split = first
    left[i] = split == first ? ~split : split;
    right[i] = split + 1 == last ? ~(split + 1) : split + 1;
    const uint32_t base = fb >= 32 ? 0u : (cf >> fb) << fb;
    bmin[3 * i] = (int32_t)compact_bits3_32(base);
    bmin[3 * i + 1] = (int32_t)compact_bits3_32(base >> 1);
    bmin[3 * i + 2] = (int32_t)compact_bits3_32(base >> 2);
    bsize[3 * i] = box_size_axis(fb, 0);
    bsize[3 * i + 1] = box_size_axis(fb, 1);
    bsize[3 * i + 2] = box_size_axis(fb, 2);
}

template <typename K>
int launch_build_tree(const K *codes, int64_t n_host, const int32_t *n_dev, int64_t n_cap,
                      int32_t *left, int32_t *right, int32_t *bmin, int32_t *bsize,
                      WideNode *nodes, uint4 *leaves, const uint32_t *leaf_flut,
                      const double *sigma, const int32_t *rot_index, int32_t *dup_flag,
                      cudaStream_t st) {
    int64_t threads = n_cap > 1 ? n_cap : 1;
    int blocks = (int)ceil_div<int64_t>(threads, 256);
    if (sizeof(K) == 4 && !nodes && !dup_flag && left && n_cap < (int64_t(1) << 30)) {
        return launch_pdl(build_tree32_kernel, blocks, 256, 0, st,
                          reinterpret_cast<const uint32_t *>(codes), (int)n_host, n_dev, left,
                          right, bmin, bsize, leaves, leaf_flut, sigma, rot_index);
    }
    build_tree_kernel<K><<<blocks, 256, 0, st>>>(codes, n_host, n_dev, left, right, bmin, bsize,
                                                  nodes, leaves, leaf_flut, sigma, rot_index,
                                                  dup_flag);
    return ARTEMIS_LAUNCHED();
}

template int launch_build_tree<u64>(const u64 *, int64_t, const int32_t *, int64_t, int32_t *,
                                    int32_t *, int32_t *, int32_t *, WideNode *, uint4 *,
                                    const uint32_t *, const double *, const int32_t *, int32_t *,
                                    cudaStream_t);
template int launch_build_tree<uint32_t>(const uint32_t *, int64_t, const int32_t *, int64_t,
                                         int32_t *, int32_t *, int32_t *, int32_t *,
                                         WideNode *, uint4 *, const uint32_t *, const double *,
                                         const int32_t *, int32_t *, cudaStream_t);

}  // namespace artemis

using namespace artemis;

extern "C" int artemis_morton_encode(const int64_t *coords, int64_t n, uint64_t *codes,
                                     int32_t *range_flag, artemis_stream stream) {
    if (n < 0 || (n > 0 && (!coords || !codes))) return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_OK;
    morton_encode_kernel<<<(int)ceil_div<int64_t>(n, 256), 256, 0, S(stream)>>>(
        coords, n, reinterpret_cast<u64 *>(codes), range_flag);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_morton_decode(const uint64_t *codes, int64_t n, int64_t *coords,
                                     artemis_stream stream) {
    if (n < 0 || (n > 0 && (!coords || !codes))) return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_OK;
    morton_decode_kernel<<<(int)ceil_div<int64_t>(n, 256), 256, 0, S(stream)>>>(
        reinterpret_cast<const u64 *>(codes), n, coords);
    return ARTEMIS_LAUNCHED();
}

extern "C" int artemis_build_tree(const uint64_t *codes, int64_t n, int32_t *left, int32_t *right,
                                  int32_t *box_min, int32_t *box_size, int32_t *dup_flag,
                                  artemis_stream stream) {
    if (n < 0 || !codes) return ARTEMIS_ERR_ARG;
    if (n == 0) return ARTEMIS_ERR_EMPTY;
    if (n == 1) return ARTEMIS_OK;
    if (!left || !right || !box_min || !box_size) return ARTEMIS_ERR_ARG;
    return launch_build_tree<u64>(reinterpret_cast<const u64 *>(codes), n, nullptr, n, left,
                                  right, box_min, box_size, nullptr, nullptr, nullptr, nullptr,
                                  nullptr, dup_flag, S(stream));
}

extern "C" int artemis_pack_tree(const uint64_t *codes, const uint32_t *flut_idx, int64_t n,
                                 int32_t root, const int32_t *left, const int32_t *right,
                                 const int32_t *box_min, const int32_t *box_size,
                                 const double *sigma, const int32_t *rot_index, void *nodes,
                                 void *leaves, artemis_stream stream) {
    if (n < 1 || !codes || !flut_idx || !nodes || !leaves) return ARTEMIS_ERR_ARG;
    if (n > 1 && (!left || !right || !box_min || !box_size)) return ARTEMIS_ERR_ARG;
    pack_tree_kernel<<<(int)ceil_div<int64_t>(n, 256), 256, 0, S(stream)>>>(
        reinterpret_cast<const u64 *>(codes), flut_idx, n, root, left, right, box_min, box_size,
        reinterpret_cast<WideNode *>(nodes), reinterpret_cast<uint4 *>(leaves), sigma,
        rot_index);
    return ARTEMIS_LAUNCHED();
}
