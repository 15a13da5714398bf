// Occupancy brick map over the sorted unique leaf codes, and the exact cell
// walk that enumerates a ray's hit leaves with it.
//
// Why a cell walk reproduces the reference's tree traversal exactly
// (_core.pyx:252-355): a leaf is emitted iff its unit cell passes the fp64
// slab test with t1 > t0 -- every ancestor box contains the cell, so its
// (monotone, correctly rounded) slab test passes too and the DFS reaches
// it -- and emitted leaves come out in increasing t0: sibling octants are
// separated by a plane the ray crosses once, and two distinct cells with
// positive-length intervals cannot share an entry distance. So the hit
// sequence is "occupied cells whose exact slab interval is non-empty, in
// entry order". The walk steps cell to cell across exactly computed plane
// crossings fl((k - o) / d), the very values the reference's slab test
// computes, so each visited cell's [max(entries), min(exits)] IS its slab
// interval; cells are visited in crossing order, tied crossings skip only
// zero-length cells. Empty 8^3 bricks are skipped in one step: the walk
// jumps to the brick's exact exit distance and re-derives each axis's slab
// there with exact crossings.
#pragma once
#include "common.cuh"

namespace artemis {

struct BrickRec {
    uint32_t mask[16];    // 512 occupancy bits, bit = local Morton index (9 bits)
    uint16_t prefix[16];  // leaves of this brick before word w (valid for words with bits)
    uint32_t first;       // index of the brick's first leaf in the sorted leaf array
    uint32_t pad[7];
};

struct BrickMap {
    const int32_t *table;  // dense brick table over [org, org + dims) brick coords, -1 = empty
    const BrickRec *recs;
    const int32_t *aabb;   // [6] leaf-cell bounds: lo xyz inclusive, hi xyz exclusive
    int org[3];
    int dims[3];
};

__device__ __forceinline__ uint32_t spread3_small(uint32_t v) {  // 3 bits -> slots 0, 3, 6
    return (v & 1u) | ((v & 2u) << 2) | ((v & 4u) << 4);
}

__device__ __forceinline__ int brick_lookup(const BrickMap &bm, int bx, int by, int bz) {
    const int x = bx - bm.org[0], y = by - bm.org[1], z = bz - bm.org[2];
    if ((unsigned)x >= (unsigned)bm.dims[0] || (unsigned)y >= (unsigned)bm.dims[1] ||
        (unsigned)z >= (unsigned)bm.dims[2])
        return -1;
    return __ldg(bm.table + ((size_t)z * bm.dims[1] + y) * bm.dims[0] + x);
}

// Exact plane crossing fl((k - o) / d) -- the same double the reference's
// slab test computes for the plane k of a unit cell.
#ifdef ARTEMIS_PHASE_CLOCKS
__device__ unsigned long long g_walk_stats[4];  // crossings, cell steps, brick skips, syncs
#define ARTEMIS_STAT(i) atomicAdd(&g_walk_stats[i], 1ull)
#else
#define ARTEMIS_STAT(i) \
    do {                \
    } while (0)
#endif

#ifndef ARTEMIS_RCP_CROSSING
#define ARTEMIS_RCP_CROSSING 1  // 0: __ddiv_rn for every crossing (round 1; same results, slower)
#endif

// RN(n / d) from r = RN(1/d) (Markstein): q = RN(n r) corrected once with
// the exact residual n - q d, RN(q + (n - q d) r), equals RN(n / d) --
// __ddiv_rn's bits in three dependent fp64 ops -- as long as nothing
// underflows or overflows (n, d, n / d well inside the normal range). The
// GPU self-test (artemis_debug_division_selftest) found the failure mode
// outside it: a subnormal dividend. div_fast is used where the caller has
// established the operand ranges for the whole launch (camera frames:
// camera_fast_div_ok in frame.cu); div_exact checks per call.
__device__ __forceinline__ double div_fast(double n, double d, double r) {
    const double q = __dmul_rn(n, r);
    return __fma_rn(__fma_rn(-q, d, n), r, q);
}

static __device__ __noinline__ double div_slow(double n, double d) { return __ddiv_rn(n, d); }

// safe-range predicate of div_fast's operands (0 is always fine)
__device__ __forceinline__ bool div_operand_ok(double x, double lo, double hi) {
    const double a = fabs(x);
    return x == 0.0 || (a >= lo && a <= hi);
}

__device__ __forceinline__ double div_exact(double n, double d, double r) {
    if (r != 0.0 && div_operand_ok(n, 0x1p-400, 0x1p400)) return div_fast(n, d, r);
    return div_slow(n, d);
}

// r for div_exact / div_fast (0 = divisor out of range: div_exact falls back)
__device__ __forceinline__ double recip_for_div(double d) {
    const double ad = fabs(d);
    return (ad >= 0x1p-600 && ad <= 0x1p600) ? __drcp_rn(d) : 0.0;
}

// Exact plane crossing fl((k - o) / d) -- the same double the reference's
// slab test computes for the plane k of a unit cell. kFast: the launch's
// operand ranges are established (k - o is 0 or in [2^-353, 2^301], d in
// [2^-487, 2^60]: every quotient, product and residual normal), r = RN(1/d).
template <bool kFast>
__device__ __forceinline__ double crossing(int k, double o, double d, double r) {
    ARTEMIS_STAT(0);
    if constexpr (kFast) {
        return div_fast(__dadd_rn((double)k, -o), d, r);
    } else {
        (void)r;
        return __ddiv_rn(__dadd_rn((double)k, -o), d);
    }
}

// Slab of one axis that contains distance t (entry <= t < exit), searched
// from an estimate inside [cmin, cmax]; returns its exact entry/exit.
template <bool kFast>
__device__ __forceinline__ void sync_axis(double o, double d, double r, double t, int cmin,
                                          int cmax, int &c, double &E, double &X) {
    ARTEMIS_STAT(3);
    const double est = floor(o + t * d);
    c = est < (double)cmin ? cmin : est > (double)cmax ? cmax : (int)est;
    if (d > 0.0) {  // slab c = [cross(c), cross(c+1))
        double lo = crossing<kFast>(c, o, d, r);
        while (c > cmin && lo > t) {
            --c;
            lo = crossing<kFast>(c, o, d, r);
        }
        double hi = crossing<kFast>(c + 1, o, d, r);
        while (c < cmax && hi <= t) {
            ++c;
            lo = hi;
            hi = crossing<kFast>(c + 1, o, d, r);
        }
        E = lo;
        X = hi;
    } else {  // slab c = [cross(c+1), cross(c))
        double en = crossing<kFast>(c + 1, o, d, r);
        while (c < cmax && en > t) {
            ++c;
            en = crossing<kFast>(c + 1, o, d, r);
        }
        double ex = crossing<kFast>(c, o, d, r);
        while (c > cmin && ex <= t) {
            --c;
            en = ex;
            ex = crossing<kFast>(c, o, d, r);
        }
        E = en;
        X = ex;
    }
}

}  // namespace artemis
