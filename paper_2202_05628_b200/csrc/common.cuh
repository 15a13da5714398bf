// Shared device helpers for libartemis (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "artemis.h"

namespace artemis {

typedef unsigned long long u64;

// ---- debug checks (scripts/build_variants.py "checks": -DARTEMIS_DEBUG_CHECKS)
// compute-sanitizer is not available on the GPU pool, so index bounds of the
// shared-memory queues, stacks and scatter targets are asserted in a checking
// build instead; a violation prints its site and traps.
#ifdef ARTEMIS_DEBUG_CHECKS
#define ARTEMIS_DCHECK(c)                                                          \
    do {                                                                           \
        if (!(c)) {                                                                \
            printf("ARTEMIS_DCHECK failed: %s at %s:%d\n", #c, __FILE__, __LINE__); \
            __trap();                                                              \
        }                                                                          \
    } while (0)
#else
#define ARTEMIS_DCHECK(c) \
    do {                  \
    } while (0)
#endif

// ---- status plumbing ------------------------------------------------------
void set_cuda_error(cudaError_t e);
int check_launch();  // ARTEMIS_OK or ARTEMIS_ERR_CUDA after a launch

#define ARTEMIS_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) {                            \
            ::artemis::set_cuda_error(_e);                  \
            return _e == cudaErrorMemoryAllocation ? ARTEMIS_ERR_OOM : ARTEMIS_ERR_CUDA; \
        }                                                   \
    } while (0)

#define ARTEMIS_LAUNCHED() ::artemis::check_launch()

// ---- programmatic dependent launch ------------------------------------------
// The frame's kernel chain (counting rebuild -> Karras build -> finish ->
// render) is launched with programmatic stream serialization: the next grid
// is scheduled while the previous one drains (once all of its blocks have
// called griddep_launch_dependents or exited) instead of after a full
// launch round trip. A kernel launched this way MUST call griddep_wait()
// before its first access to memory an earlier launch wrote; both are no-ops
// for a normal launch. ARTEMIS_PDL=0 launches them normally (A/B).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("ARTEMIS_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// Launch priority of the launches made through launch_pdl on this host
// thread (0 = the stream's own); PriorityScope raises it for one launch.
inline int &launch_priority() {
    static thread_local int p = 0;
    return p;
}
struct PriorityScope {
    int saved;
    explicit PriorityScope(bool on) : saved(launch_priority()) {
        if (on) {
            int least = 0, greatest = 0;
            cudaDeviceGetStreamPriorityRange(&least, &greatest);
            launch_priority() = greatest;
        }
    }
    ~PriorityScope() { launch_priority() = saved; }
};

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (launch_priority() != 0) {  // set around a launch by PriorityScope
        at[na].id = cudaLaunchAttributePriority;
        at[na].val.priority = launch_priority();
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return ARTEMIS_ERR_CUDA;
    }
    return check_launch();
}

inline cudaStream_t S(artemis_stream s) { return reinterpret_cast<cudaStream_t>(s); }

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <typename T>
inline T ceil_div(T a, T b) { return (a + b - 1) / b; }

// ---- Morton (21 bits per axis, x lowest; animvox/_core.pyx:51-76) ----------
__host__ __device__ __forceinline__ u64 spread_bits3(u64 v) {
    v &= 0x1FFFFFull;
    v = (v | (v << 32)) & 0x1F00000000FFFFull;
    v = (v | (v << 16)) & 0x1F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

__host__ __device__ __forceinline__ u64 compact_bits3(u64 v) {
    v &= 0x1249249249249249ull;
    v = (v ^ (v >> 2)) & 0x10C30C30C30C30C3ull;
    v = (v ^ (v >> 4)) & 0x100F00F00F00F00Full;
    v = (v ^ (v >> 8)) & 0x1F0000FF0000FFull;
    v = (v ^ (v >> 16)) & 0x1F00000000FFFFull;
    v = (v ^ (v >> 32)) & 0x1FFFFFull;
    return v;
}

__host__ __device__ __forceinline__ u64 morton3(u64 x, u64 y, u64 z) {
    return spread_bits3(x) | (spread_bits3(y) << 1) | (spread_bits3(z) << 2);
}

// ---- packed traversal node --------------------------------------------------
// One internal node = 32 bytes: both children's octant boxes (min corner
// plus the number of free Morton bits, which fixes the per-axis power-of-two
// size exactly as _core.pyx:182-190 does) and the child links.
// word[0] = L.x | L.sx << 21 | split_axis << 27, word[1] = L.y | L.sy << 21,
// word[2] = L.z | L.sz << 21, word[3] = left
// word[4] = R.x | R.sx << 21 | absent << 31, word[5] = R.y | R.sy << 21,
// word[6] = R.z | R.sz << 21, word[7] = right
// with s_a = log2 of the box size on axis a (box_size_axis of the free bits).
// split_axis is the axis of the node's highest differing Morton bit: the
// plane that separates the two children's octants. kAbsent marks a missing
// child (the super-root's right).
constexpr uint32_t kAbsent = 1u << 31;
constexpr uint32_t kCoordMask = 0x1FFFFFu;

__host__ __device__ __forceinline__ int split_axis_of(int free_bits) {
    return (free_bits - 1) % 3;
}

struct PackedNode {
    uint32_t w[8];
};

// Traversal record of one internal node (64 bytes): its four grandchild
// slots in left-to-right order {LL, LR, RL, RR}, each a packed box + link
// (when a child is a leaf it takes slot 0 or 2 and slot 1 or 3 is absent).
// Split axes: the node's in slot 0 bits 27-28, the left child's in slot 1,
// the right child's in slot 3. One visit covers two binary levels.
struct WideNode {
    uint4 s[4];
};

__host__ __device__ __forceinline__ int box_size_axis(int free_bits, int axis) {
    return 1 << ((free_bits + 2 - axis) / 3);
}

// number of differing low bits between the first and last code of a range
__device__ __forceinline__ int range_free_bits(u64 a, u64 b) {
    return a == b ? 0 : 64 - __clzll(static_cast<long long>(a ^ b));
}

__host__ __device__ __forceinline__ int log_size_axis(int free_bits, int axis) {
    return (free_bits + 2 - axis) / 3;
}

__device__ __forceinline__ void pack_box(uint32_t *w, uint32_t x, uint32_t y, uint32_t z,
                                         int free_bits) {
    w[0] = x | ((uint32_t)log_size_axis(free_bits, 0) << 21);
    w[1] = y | ((uint32_t)log_size_axis(free_bits, 1) << 21);
    w[2] = z | ((uint32_t)log_size_axis(free_bits, 2) << 21);
}

__device__ __forceinline__ void pack_child(uint32_t *w, u64 c_first, u64 c_last, int link) {
    int fb = range_free_bits(c_first, c_last);
    u64 base = fb >= 64 ? 0ull : (c_first >> fb) << fb;
    pack_box(w, static_cast<uint32_t>(compact_bits3(base)),
             static_cast<uint32_t>(compact_bits3(base >> 1)),
             static_cast<uint32_t>(compact_bits3(base >> 2)), fb);
    w[3] = static_cast<uint32_t>(link);
}

// ---- warp helpers -----------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace artemis
