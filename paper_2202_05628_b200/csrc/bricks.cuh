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
#define ARTEMIS_RCP_CROSSING 1  // 0: __ddiv_rn per crossing (round 1; same results, slower)
#endif

// RN(n / d). Markstein: with r = RN(1/d) and n, d, n/d well inside the
// normal range, q = RN(n r) corrected once with the exact residual n - q d,
// RN(q + (n - q d) r), is RN(n / d) -- __ddiv_rn's bits in three dependent
// fp64 ops. Outside that range it can differ (a subnormal dividend did, in
// the GPU self-test), so the range is established by the CALLER, once per
// divisor: r != 0 asserts that every dividend it will see is 0 or has
// magnitude in [2^-400, 2^400] and that |d| is in [2^-400, 2^400]; r == 0
// takes __ddiv_rn (out of line: it never runs on real rays).
static __device__ __noinline__ double div_slow(double n, double d) { return __ddiv_rn(n, d); }

__device__ __forceinline__ double div_exact(double n, double d, double r) {
    if (r != 0.0) {
        const double q = __dmul_rn(n, r);
        return __fma_rn(__fma_rn(-q, d, n), r, q);
    }
    return div_slow(n, d);
}

// r for div_exact when every dividend is known to be 0 or in [2^-400, 2^400]
__device__ __forceinline__ double recip_for_div(double d) {
    const double ad = fabs(d);
    return (ad >= 0x1p-400 && ad <= 0x1p400) ? __drcp_rn(d) : 0.0;
}

// r for the plane crossings of one ray axis: dividends k - o with integer
// |k| <= 2^22 are 0 or in [2^-353, 2^301] whenever o is 0 or |o| is in
// [2^-300, 2^300] (a nonzero k - o is a multiple of ulp(o) > 2^-353)
__device__ __forceinline__ double recip_for_crossings(double o, double d) {
    const double ao = fabs(o);
    return (o == 0.0 || (ao >= 0x1p-300 && ao <= 0x1p300)) ? recip_for_div(d) : 0.0;
}

// Exact plane crossing fl((k - o) / d) -- the same double the reference's
// slab test computes for the plane k of a unit cell; r = recip_for_crossings.
__device__ __forceinline__ double crossing(int k, double o, double d, double r) {
    ARTEMIS_STAT(0);
#if ARTEMIS_RCP_CROSSING
    return div_exact(__dadd_rn((double)k, -o), d, r);
#else
    (void)r;
    return __ddiv_rn(__dadd_rn((double)k, -o), d);
#endif
}

// Slab of one axis that contains distance t (entry <= t < exit), searched
// from an estimate inside [cmin, cmax]; returns its exact entry/exit.
__device__ __forceinline__ void sync_axis(double o, double d, double r, double t, int cmin,
                                          int cmax, int &c, double &E, double &X) {
    ARTEMIS_STAT(3);
    const double est = floor(o + t * d);
    c = est < (double)cmin ? cmin : est > (double)cmax ? cmax : (int)est;
    if (d > 0.0) {  // slab c = [cross(c), cross(c+1))
        double lo = crossing(c, o, d, r);
        while (c > cmin && lo > t) {
            --c;
            lo = crossing(c, o, d, r);
        }
        double hi = crossing(c + 1, o, d, r);
        while (c < cmax && hi <= t) {
            ++c;
            lo = hi;
            hi = crossing(c + 1, o, d, r);
        }
        E = lo;
        X = hi;
    } else {  // slab c = [cross(c+1), cross(c))
        double en = crossing(c + 1, o, d, r);
        while (c < cmax && en > t) {
            ++c;
            en = crossing(c + 1, o, d, r);
        }
        double ex = crossing(c, o, d, r);
        while (c > cmin && ex <= t) {
            --c;
            en = ex;
            ex = crossing(c, o, d, r);
        }
        E = en;
        X = ex;
    }
}

}  // namespace artemis
