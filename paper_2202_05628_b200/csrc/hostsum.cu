// Host-side content checksum of caller arrays (the kernel-contract shim's
// device cache key: "device-cached tree and FLUT keyed
// by array identity plus a content check, no per-call re-upload").
//
// The reference re-reads its numpy arguments on every call
// (_core.pyx:473-559), so an in-place edit of the FLUT between two calls
// must change the result. The shim therefore keys its device copies by the
// full content of the arrays, not a sample: 128 bits from an xxh64-style
// multiply-rotate over every 8-byte word, computed in 64 KB blocks on
// several host threads (memory-bandwidth bound) and combined in block order,
// so the digest does not depend on the thread count.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

constexpr uint64_t P1 = 0x9E3779B185EBCA87ull;
constexpr uint64_t P2 = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t P3 = 0x165667B19E3779F9ull;
constexpr uint64_t P4 = 0x85EBCA77C2B2AE63ull;
constexpr size_t kBlock = 64 << 10;

inline uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline uint64_t round1(uint64_t acc, uint64_t w) { return rotl(acc + w * P2, 31) * P1; }
inline uint64_t avalanche(uint64_t h) {
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

// digest of one block (bytes <= kBlock), seeded by its index
uint64_t block_digest(const unsigned char *p, size_t bytes, uint64_t index) {
    uint64_t a0 = P1 + P2 + index, a1 = P2 + index, a2 = index, a3 = index - P1;
    size_t i = 0;
    for (; i + 32 <= bytes; i += 32) {
        uint64_t w[4];
        memcpy(w, p + i, 32);
        a0 = round1(a0, w[0]);
        a1 = round1(a1, w[1]);
        a2 = round1(a2, w[2]);
        a3 = round1(a3, w[3]);
    }
    uint64_t h = rotl(a0, 1) + rotl(a1, 7) + rotl(a2, 12) + rotl(a3, 18);
    for (; i + 8 <= bytes; i += 8) {
        uint64_t w;
        memcpy(&w, p + i, 8);
        h = rotl(h ^ round1(0, w), 27) * P1 + P4;
    }
    if (i < bytes) {
        uint64_t w = 0;
        memcpy(&w, p + i, bytes - i);
        h = rotl(h ^ (w * P1), 23) * P2 + P3;
    }
    return avalanche(h ^ (uint64_t)bytes);
}

}  // namespace

extern "C" int artemis_host_checksum(const void *data, size_t bytes, int threads,
                                     uint64_t *out /* host, 2 words */) {
    if (!out || (bytes && !data)) return ARTEMIS_ERR_ARG;
    const unsigned char *p = static_cast<const unsigned char *>(data);
    const size_t nblocks = (bytes + kBlock - 1) / kBlock;
    std::vector<uint64_t> dig(nblocks);
    auto work = [&](size_t b0, size_t b1) {
        for (size_t b = b0; b < b1; ++b) {
            const size_t off = b * kBlock;
            dig[b] = block_digest(p + off, std::min(kBlock, bytes - off), b);
        }
    };
    // one thread per >= 8 MB; thread start-up would dominate small arrays
    size_t nt = std::max<size_t>(1, std::min<size_t>(threads > 0 ? (size_t)threads : 1,
                                                     bytes / (8u << 20)));
    if (nt <= 1) {
        work(0, nblocks);
    } else {
        std::vector<std::thread> pool;
        const size_t per = (nblocks + nt - 1) / nt;
        for (size_t t = 0; t < nt; ++t) {
            const size_t b0 = t * per, b1 = std::min(nblocks, b0 + per);
            if (b0 < b1) pool.emplace_back(work, b0, b1);
        }
        for (auto &th : pool) th.join();
    }
    uint64_t h0 = P3 ^ (uint64_t)bytes, h1 = P4 + (uint64_t)bytes * P1;
    for (size_t b = 0; b < nblocks; ++b) {
        h0 = rotl(h0 ^ dig[b], 29) * P1 + P2;
        h1 += avalanche(dig[b] + (uint64_t)b * P3);
    }
    out[0] = avalanche(h0);
    out[1] = avalanche(h1 ^ h0);
    return ARTEMIS_OK;
}

// fp32 -> fp64 widening of a row-strided block on several host threads (the
// reference returns FrameBuffers.features as float64, render.py:359-363):
// rows x cols floats at src (row pitch src_pitch floats) into dst (row pitch
// dst_pitch doubles). Exact (every float is a double).
extern "C" int artemis_host_widen_f32(const float *src, int64_t rows, int64_t cols,
                                      int64_t src_pitch, double *dst, int64_t dst_pitch,
                                      int threads) {
    if (rows < 0 || cols < 0 || (rows && cols && (!src || !dst))) return ARTEMIS_ERR_ARG;
    if (!rows || !cols) return ARTEMIS_OK;
    auto work = [&](int64_t r0, int64_t r1) {
        for (int64_t r = r0; r < r1; ++r) {
            const float *s = src + r * src_pitch;
            double *d = dst + r * dst_pitch;
            for (int64_t c = 0; c < cols; ++c) d[c] = (double)s[c];
        }
    };
    const int64_t total = rows * cols;
    int64_t nt = std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : 1,
                                                        total / (1 << 18)));
    nt = std::min<int64_t>(nt, rows);
    if (nt <= 1) {
        work(0, rows);
        return ARTEMIS_OK;
    }
    std::vector<std::thread> pool;
    const int64_t per = (rows + nt - 1) / nt;
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t r0 = t * per, r1 = std::min(rows, r0 + per);
        if (r0 < r1) pool.emplace_back(work, r0, r1);
    }
    for (auto &th : pool) th.join();
    return ARTEMIS_OK;
}
