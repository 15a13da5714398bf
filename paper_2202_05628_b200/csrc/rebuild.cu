// Counting rebuild of the posed leaf set (frame pipeline, grids <= 1024^3).
//
// Replaces, for the device frame, the reference's stable radix sort of the
// warped Morton keys (volume.build_octree -> sort_order, _core.pyx:111-167)
// and its collision resolve (rigging.resolve_collisions, rigging.py:419-459:
// np.lexsort((idx, -sigma, code)), the first entry of each code wins). The
// output is the same: the live codes strictly ascending, each with its
// winner (largest density, ties to the lowest canonical index, NaN
// densities last) -- plus the occupancy brick map the renderer walks.
//
// A Morton code is (brick code << 9) | (cell code within the 8^3 brick), so
// ascending codes are bricks in Morton order and, inside a brick, the
// 512-bit occupancy mask in bit order. The sort is therefore a two-digit
// counting sort over the key space instead of four 8-bit scatter passes:
//   warp kernel   sets the cell's bit in a dense per-brick mask and the
//                 brick's bit in a brick-occupancy bitmap (warp-aggregated
//                 atomicOr: order-independent)
//   count         per bitmap word: occupied bricks, live cells (popcounts)
//   scan          exclusive scans of both (one block)
//   emit          per occupied brick, in Morton order: its record (mask,
//                 per-word prefix, first leaf), the dense brick table entry,
//                 the leaf-cell AABB; clears the dense masks for the next frame
//   slot          per in-bounds voxel: its live-cell rank = record.first +
//                 prefix + popc(mask below the bit); live code; 128-bit
//                 atomic max of (density total-order key, ~index) -> the
//                 winner (largest density, then lowest index)
//   finish        winners out of the max scratch, scratch reset
// Integer atomics (or / max) commute, so the result is deterministic and
// equals the reference's order, with no per-entry sort at all.
#include <algorithm>

#include "bricks.cuh"
#include "tree.cuh"

namespace artemis {

namespace {
constexpr int kCountThreads = 256;
}

// Density total order of the reference's lexsort on -sigma: larger first,
// -0.0 == +0.0, NaN after every number (key 0).
__device__ __forceinline__ unsigned long long density_key(double s) {
    if (isnan(s)) return 0ull;
    if (s == 0.0) s = 0.0;  // -0.0 ties with +0.0, as in the lexsort
    const unsigned long long b = (unsigned long long)__double_as_longlong(s);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// live cells of brick b (popcount of its 512-bit mask)
__device__ __forceinline__ uint32_t brick_cells(const uint32_t *__restrict__ bmask, u64 b) {
    const uint4 *m = reinterpret_cast<const uint4 *>(bmask + b * 16);
    uint32_t cells = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 v = m[q];
        cells += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    return cells;
}

// exact leaf-cell AABB of the cells in mask word q (local Morton index
// l = 32 q + i: x = l0 + 2 l3 + 4 l6, y = l1 + 2 l4 + 4 l7, z = l2 + 2 l5 +
// 4 l8, l5..l8 = bits of q) from bit patterns, no loop over the bits
__device__ __forceinline__ void word_aabb(uint32_t m, int q, int bx, int by, int bz, int lo[3],
                                          int hi[3]) {
    if (!m) return;
    const uint32_t X[4] = {0x550055u, 0xaa00aau, 0x55005500u, 0xaa00aa00u};
    const uint32_t Y[4] = {0x3333u, 0xccccu, 0x33330000u, 0xcccc0000u};
    int xl = 3, xh = 0, yl = 3, yh = 0;
#pragma unroll
    for (int v = 3; v >= 0; --v) {
        if (m & X[v]) xl = v;
        if (m & Y[v]) yl = v;
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        if (m & X[v]) xh = v;
        if (m & Y[v]) yh = v;
    }
    const int zl = (m & 0x0f0f0f0fu) ? 0 : 1, zh = (m & 0xf0f0f0f0u) ? 1 : 0;
    const int xo = bx * 8 + 4 * ((q >> 1) & 1), yo = by * 8 + 4 * ((q >> 2) & 1),
              zo = bz * 8 + 2 * (q & 1) + 4 * ((q >> 3) & 1);
    lo[0] = min(lo[0], xo + xl);
    hi[0] = max(hi[0], xo + xh + 1);
    lo[1] = min(lo[1], yo + yl);
    hi[1] = max(hi[1], yo + yh + 1);
    lo[2] = min(lo[2], zo + zl);
    hi[2] = max(hi[2], zo + zh + 1);
}

// one warp per bitmap word (lane j = brick 32 w + j): the word's occupied
// bricks and live cells, each brick's cell offset within the word, and the
// exact leaf-cell AABB (block-reduced, then one atomic per bound and block)
__global__ void count_kernel(const uint32_t *__restrict__ bocc,
                             const uint32_t *__restrict__ bmask, int64_t n_words,
                             uint32_t *__restrict__ n_bricks, uint32_t *__restrict__ n_cells,
                             uint32_t *__restrict__ bpre, uint32_t *__restrict__ blk_bricks,
                             uint32_t *__restrict__ blk_cells, int32_t *aabb) {
    griddep_wait();
    griddep_launch_dependents();
    __shared__ int red[6][kCountThreads / 32];
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    const uint32_t occ = w < n_words ? bocc[w] : 0u;
    uint32_t c = 0;
    if ((occ >> lane) & 1u) {
        const u64 b = (u64)(32 * w + lane);
        const int bx = (int)compact_bits3(b), by = (int)compact_bits3(b >> 1),
                  bz = (int)compact_bits3(b >> 2);
        const uint4 *m4 = reinterpret_cast<const uint4 *>(bmask + b * 16);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 v = m4[q4];
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            word_aabb(v.x, 4 * q4, bx, by, bz, lo, hi);
            word_aabb(v.y, 4 * q4 + 1, bx, by, bz, lo, hi);
            word_aabb(v.z, 4 * q4 + 2, bx, by, bz, lo, hi);
            word_aabb(v.w, 4 * q4 + 3, bx, by, bz, lo, hi);
        }
    }
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    // block-level exclusive offsets of the block's words (8 words per block);
    // the block totals are scanned across blocks by scan2_kernel
    __shared__ uint32_t s_nb[kCountThreads / 32], s_nc[kCountThreads / 32];
    if (lane == 31) {
        s_nb[wid] = __popc(occ);
        s_nc[wid] = incl;
    }
    __syncthreads();
    if (w < n_words) {
        bpre[32 * w + lane] = incl - c;
        if (lane == 0) {
            uint32_t ob = 0, oc = 0;
            for (int v = 0; v < wid; ++v) {
                ob += s_nb[v];
                oc += s_nc[v];
            }
            n_bricks[w] = ob;  // exclusive within the block
            n_cells[w] = oc;
        }
    }
    if (threadIdx.x == 0) {
        uint32_t tb = 0, tc = 0;
        for (int v = 0; v < kCountThreads / 32; ++v) {
            tb += s_nb[v];
            tc += s_nc[v];
        }
        blk_bricks[blockIdx.x] = tb;
        blk_cells[blockIdx.x] = tc;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
    }
    if (lane == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            red[a][wid] = lo[a];
            red[3 + a][wid] = hi[a];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        int r = red[k][0];
        for (int v = 1; v < kCountThreads / 32; ++v) r = k < 3 ? min(r, red[k][v]) : max(r, red[k][v]);
        if (k < 3 ? r != INT32_MAX : r != INT32_MIN) {
            if (k < 3)
                atomicMin(aabb + k, r);
            else
                atomicMax(aabb + k, r);
        }
    }
}

// exclusive scans of both count arrays (one block), totals to n_live / n_recs
__global__ void __launch_bounds__(1024) scan2_kernel(uint32_t *a, uint32_t *b, int64_t n,
                                                     int32_t *total_b, int32_t *total_a) {
    griddep_wait();
    griddep_launch_dependents();
    __shared__ uint32_t sa[32], sb[32];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int64_t per = (n + 1023) / 1024;
    const int64_t lo = t * per, hi = min(n, lo + per);
    uint32_t xa = 0, xb = 0;
    for (int64_t base = lo; base < hi; base += 8) {  // batches of 8 independent loads
        uint32_t ta[8], tb[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ta[k] = base + k < hi ? a[base + k] : 0u;
            tb[k] = base + k < hi ? b[base + k] : 0u;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            xa += ta[k];
            xb += tb[k];
        }
    }
    uint32_t ia = xa, ib = xb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
        const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += ya;
            ib += yb;
        }
    }
    if (lane == 31) {
        sa[wid] = ia;
        sb[wid] = ib;
    }
    __syncthreads();
    if (wid == 0) {
        uint32_t va = sa[lane], vb = sb[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, va, o);
            const uint32_t yb = __shfl_up_sync(0xffffffffu, vb, o);
            if (lane >= o) {
                va += ya;
                vb += yb;
            }
        }
        sa[lane] = va;
        sb[lane] = vb;
    }
    __syncthreads();
    uint32_t ea = (wid ? sa[wid - 1] : 0u) + ia - xa;
    uint32_t eb = (wid ? sb[wid - 1] : 0u) + ib - xb;
    for (int64_t base = lo; base < hi; base += 8) {
        uint32_t ta[8], tb[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ta[k] = base + k < hi ? a[base + k] : 0u;
            tb[k] = base + k < hi ? b[base + k] : 0u;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (base + k < hi) {
                a[base + k] = ea;
                b[base + k] = eb;
            }
            ea += ta[k];
            eb += tb[k];
        }
    }
    if (t == 1023) {
        *total_a = (int32_t)ea;
        *total_b = (int32_t)eb;
    }
}

// one warp per bitmap word, one lane per brick (all bricks of the word in
// parallel): an occupied brick's record (mask, per-word prefix, first leaf),
// its table entry, and its dense mask cleared for the next frame. The live
// slots' winner keys need no initialisation here: finish_kernel resets the
// ones a frame used after the tree is built (they start zeroed at creation).
__global__ void emit_kernel(const uint32_t *__restrict__ bocc, uint32_t *__restrict__ bmask,
                            int64_t n_words, const uint32_t *__restrict__ rec_base,
                            const uint32_t *__restrict__ cell_base,
                            const uint32_t *__restrict__ blk_bricks,
                            const uint32_t *__restrict__ blk_cells,
                            const uint32_t *__restrict__ bpre, BrickRec *__restrict__ recs,
                            int32_t *__restrict__ table, int dx, int dy) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_words) return;
    const uint32_t occ = bocc[w];
    if (!((occ >> lane) & 1u)) return;
    const int64_t blk = w / (kCountThreads / 32);
    const uint32_t rec = blk_bricks[blk] + rec_base[w] + __popc(occ & ((1u << lane) - 1u));
    const u64 b = (u64)(32 * w + lane);
    uint4 *mk = reinterpret_cast<uint4 *>(bmask + b * 16);
    BrickRec &R = recs[rec];
    uint4 *rm = reinterpret_cast<uint4 *>(R.mask);
    uint32_t pf[16];
    uint32_t run = 0;
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
        const uint4 v = mk[q4];
        rm[q4] = v;
        mk[q4] = make_uint4(0u, 0u, 0u, 0u);  // ready for the next frame
        pf[4 * q4] = run;
        run += __popc(v.x);
        pf[4 * q4 + 1] = run;
        run += __popc(v.y);
        pf[4 * q4 + 2] = run;
        run += __popc(v.z);
        pf[4 * q4 + 3] = run;
        run += __popc(v.w);
    }
    uint4 *rp = reinterpret_cast<uint4 *>(R.prefix);
    rp[0] = make_uint4(pf[0] | (pf[1] << 16), pf[2] | (pf[3] << 16), pf[4] | (pf[5] << 16),
                       pf[6] | (pf[7] << 16));
    rp[1] = make_uint4(pf[8] | (pf[9] << 16), pf[10] | (pf[11] << 16), pf[12] | (pf[13] << 16),
                       pf[14] | (pf[15] << 16));
    R.first = blk_cells[blk] + cell_base[w] + bpre[b];
    const int bx = (int)compact_bits3(b), by = (int)compact_bits3(b >> 1),
              bz = (int)compact_bits3(b >> 2);
    table[((size_t)bz * dy + by) * dx + bx] = (int32_t)rec;
}

// the winners out of the 128-bit max scratch (low word = 2^32 - 1 - index)
// into the frame's winner array, and the scratch slots the frame used reset
// for the next frame (a zero entry loses to every voxel)
// With `leaves`, also the renderer's leaf records (cell, FLUT row, density,
// rotation joint: the record build_tree32_kernel writes), so the render
// depends on this pass only and the Karras tree arrays can be built beside it.
__global__ void finish_kernel(const int32_t *__restrict__ n_live, ulonglong2 *__restrict__ wmax,
                              uint32_t *__restrict__ winners, const uint32_t *__restrict__ codes,
                              uint4 *__restrict__ leaves, const double *__restrict__ sigma,
                              const int32_t *__restrict__ rot_index) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t n = *n_live;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t row = 0xFFFFFFFFu - (uint32_t)wmax[i].x;
        winners[i] = row;
        wmax[i] = make_ulonglong2(0ull, 0ull);
        if (leaves) {
            const uint32_t c = codes[i];
            const unsigned long long sb =
                (unsigned long long)__double_as_longlong(sigma ? __ldg(sigma + row) : 0.0);
            leaves[2 * i] = make_uint4((uint32_t)compact_bits3(c), (uint32_t)compact_bits3(c >> 1),
                                       (uint32_t)compact_bits3(c >> 2), row);
            leaves[2 * i + 1] = make_uint4((uint32_t)sb, (uint32_t)(sb >> 32),
                                           rot_index ? (uint32_t)__ldg(rot_index + row) : 0u, 0u);
        }
    }
}

int counting_finish(const int32_t *n_live, int64_t n_cap, unsigned long long *wmax,
                    uint32_t *winners, const uint32_t *codes, uint4 *leaves, const double *sigma,
                    const int32_t *rot_index, cudaStream_t st) {
    // leaf records: one thread per possible leaf (more loads in flight than a
    // grid-stride loop over 4 blocks per SM)
    const int blocks = leaves ? (int)ceil_div<int64_t>(n_cap, 256) : num_sms() * 4;
    return launch_pdl(finish_kernel, blocks, 256, 0, st, n_live,
                      reinterpret_cast<ulonglong2 *>(wmax), winners, codes, leaves, sigma,
                      rot_index);
}

// live-cell rank of an in-bounds voxel's key (from its brick record)
__device__ __forceinline__ uint32_t live_rank(uint32_t key, const int32_t *__restrict__ table,
                                              const BrickRec *__restrict__ recs, int dx,
                                              int dy) {
    const u64 b = (u64)(key >> 9);
    const int bx = (int)compact_bits3(b), by = (int)compact_bits3(b >> 1),
              bz = (int)compact_bits3(b >> 2);
    const BrickRec &R = recs[table[((size_t)bz * dy + by) * dx + bx]];
    const uint32_t l = key & 511u, q = l >> 5;
    return R.first + R.prefix[q] + (uint32_t)__popc(R.mask[q] & ((1u << (l & 31u)) - 1u));
}

// 128-bit atomic max of (density key, 2^32 - 1 - index): the winner rule in
// one pass -- largest density first, ties to the lowest canonical index
// (_core / rigging.py:435 lexsort order). A compare-and-swap loop; most
// cells hold one voxel, so most slots take one CAS.
__device__ __forceinline__ void winner_max(ulonglong2 *slot, unsigned long long key, uint32_t i) {
    unsigned __int128 *p = reinterpret_cast<unsigned __int128 *>(slot);
    const unsigned __int128 v = ((unsigned __int128)key << 64) | (unsigned __int128)(0xFFFFFFFFu - i);
    unsigned __int128 cur = *p;
    while (cur < v) {
        const unsigned __int128 seen = atomicCAS(p, cur, v);
        if (seen == cur) break;
        cur = seen;
    }
}

__global__ void slot_kernel(const uint32_t *__restrict__ keys, int64_t n, uint32_t sentinel,
                            const double *__restrict__ sigma, const int32_t *__restrict__ table,
                            const BrickRec *__restrict__ recs, int dx, int dy,
                            uint32_t *__restrict__ live_codes, ulonglong2 *__restrict__ wmax,
                            uint32_t *__restrict__ bocc, int64_t n_words) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n_words) bocc[i] = 0u;  // emit has read the bitmap: clear it for the next frame
    if (i >= n) return;
    const uint32_t key = keys[i];
    if (key == sentinel) return;
    const uint32_t s = live_rank(key, table, recs, dx, dy);
    live_codes[s] = key;  // every voxel of the cell writes the same code
    winner_max(wmax + s, density_key(sigma[i]), (uint32_t)i);
}

// The counting rebuild after the warp kernel marked bmask / bocc: leaves
// (codes ascending, winners) + brick map. keys are indexed by canonical voxel
// (sentinel = out of bounds); n_live / n_recs receive the counts.
int counting_rebuild(const uint32_t *keys, int64_t n, uint32_t sentinel, const double *sigma,
                     uint32_t *bocc, uint32_t *bmask, int64_t n_words, uint32_t *wtmp,
                     BrickRec *recs, int32_t *table, const int dims[3], int32_t *aabb,
                     uint32_t *live_codes, unsigned long long *wmax,
                     int32_t *n_live, int32_t *n_recs, cudaStream_t st, int *launches) {
    uint32_t *nb = wtmp, *nc = wtmp + n_words;
    const size_t cells = (size_t)dims[0] * dims[1] * dims[2];
    (void)cells;  // the table and AABB were reset by counting_prepare
    const int wb = (int)ceil_div<int64_t>(n_words * 32, kCountThreads);
    uint32_t *bpre = wtmp + 2 * n_words;  // per dense brick: cells before it in its word
    uint32_t *bb = bpre + 32 * n_words, *bc = bb + wb;  // per count block: bricks, cells
    int rc = launch_pdl(count_kernel, wb, kCountThreads, 0, st, bocc, bmask, n_words, nb, nc,
                        bpre, bb, bc, aabb);
    if (rc) return rc;
    rc = launch_pdl(scan2_kernel, 1, 1024, 0, st, bc, bb, (int64_t)wb, n_recs, n_live);
    if (rc) return rc;
    rc = launch_pdl(emit_kernel, wb, kCountThreads, 0, st, bocc, bmask, n_words, nb, nc, bb, bc,
                    bpre, recs, table, dims[0], dims[1]);
    if (rc) return rc;
    const int vb = (int)ceil_div<int64_t>(std::max<int64_t>(n, n_words), kCountThreads);
    rc = launch_pdl(slot_kernel, vb, kCountThreads, 0, st, keys, n, sentinel, sigma, table, recs,
                    dims[0], dims[1], live_codes, reinterpret_cast<ulonglong2 *>(wmax), bocc,
                    n_words);
    if (launches) *launches += 4;
    return rc;
}

// Frame start, one kernel instead of four memset nodes (a graph ran them one
// after another, behind the side stream's output clear): the frame counters
// zeroed, the dense brick table to -1 and the leaf AABB to (+max, -max).
__global__ void frame_prepare_kernel(int32_t *__restrict__ counters, int n_counters,
                                     int4 *__restrict__ table4, int64_t n4,
                                     int32_t *__restrict__ aabb) {
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i0 < n_counters) counters[i0] = 0;
    if (aabb && i0 < 6) aabb[i0] = i0 < 3 ? 0x7F7F7F7F : (int32_t)0x80808080;
    for (int64_t i = i0; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        table4[i] = make_int4(-1, -1, -1, -1);
}

int counting_prepare(int32_t *counters, int n_counters, int32_t *table, const int dims[3],
                     int32_t *aabb, cudaStream_t st) {
    const size_t cells = table ? (size_t)dims[0] * dims[1] * dims[2] : 0;
    if (cells % 4) {  // not a whole number of int4 (never for 8^3-brick grids)
        ARTEMIS_TRY(cudaMemsetAsync(table, 0xFF, cells * sizeof(int32_t), st));
    }
    const int64_t n4 = cells % 4 ? 0 : (int64_t)(cells / 4);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(n4, 256),
                                                                   num_sms() * 4));
    frame_prepare_kernel<<<blocks, 256, 0, st>>>(counters, n_counters,
                                                  reinterpret_cast<int4 *>(table), n4, aabb);
    return ARTEMIS_LAUNCHED();
}

}  // namespace artemis
