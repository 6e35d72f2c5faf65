// lu_common.cuh -- shared pieces of the sm_100a transcode/validate kernels.
//
// Geometry (all kernels): one CTA = 8 warps = one 16 KiB tile of input
// bytes, staged in shared memory with a 4-byte halo on each side.  Warp w
// owns the contiguous 2 KiB chunk [w*2048, (w+1)*2048) of the tile and walks
// it in 16 steps of 128 B (one 32-bit "quad" per lane), grouped by 4 so one
// packed warp scan serves 4 steps.  Tiles are scanned with a single-pass
// decoupled look-back (tile id = blockIdx.x, as in CUB's single-pass scan).
//
// Tile status word (uint64, one per tile, zeroed before each launch):
//   bits 63..62  flag: 0 not ready, 1 aggregate, 2 inclusive prefix
//   bit  61      error: an invalid unit lies in (or before) this span
//   bits 60..0   output units before the first error (or all of them)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lu {

struct Outcome {
    int32_t status;
    int32_t pad;
    uint64_t consumed;
    uint64_t written;
};

enum : int32_t { kStatusOk = 0, kStatusMalformed = 1, kStatusOutputTooSmall = 2 };

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileBytes = 16384;
constexpr int kTileWords32 = kTileBytes / 4;          // 4096 quads per tile
constexpr int kChunkBytes = kTileBytes / kWarps;      // 2048 B per warp
constexpr int kChunkQuads = kChunkBytes / 4;          // 512
constexpr int kSteps = kChunkQuads / 32;              // 16 steps of 128 B
constexpr int kGroup = 4;                             // steps per packed scan
constexpr int kGroups = kSteps / kGroup;              // 4
// staged input: [4 pad words | halo word | 4096 tile words | halo word | pad]
constexpr int kInHead = 4;                            // tile word t lives at in_s[kInHead + t]
constexpr int kInWords = kInHead + kTileWords32 + 4;

constexpr uint32_t H8 = 0x80808080u;

constexpr uint64_t kFlagShift = 62;
constexpr uint64_t kFlagAgg = 1ull << kFlagShift;
constexpr uint64_t kFlagInc = 2ull << kFlagShift;
constexpr uint64_t kErrBit = 1ull << 61;
constexpr uint64_t kValMask = (1ull << 61) - 1;

// ---------------------------------------------------------------- bit helpers

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// 0xFF in every byte whose bit 7 is set, 0x00 elsewhere (prmt sign mode).
__device__ __forceinline__ uint32_t sgn8(uint32_t f) { return prmt(f, 0u, 0xBA98u); }

// stream shifts over little-endian byte streams: lo = earlier quad, hi = later
// quad.  fsl(prev, cur, 8*k): byte j of result = stream byte (j - k) (look-behind).
// fsr(cur, next, 8*k): byte j of result = stream byte (j + k) (look-ahead).
__device__ __forceinline__ uint32_t fsl(uint32_t lo, uint32_t hi, uint32_t s)
{
    return __funnelshift_l(lo, hi, s);
}
__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t s)
{
    return __funnelshift_r(lo, hi, s);
}

__device__ __forceinline__ uint32_t lane_id()
{
    uint32_t l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

// ----------------------------------------------------------- status words

// The status word is the only datum published through it (flag, error bit
// and count live in one 64-bit atomic word), so relaxed gpu-scope atomics
// suffice: no acquire/release fences on the look-back critical path.
__device__ __forceinline__ void st_release(uint64_t *p, uint64_t v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// (a then b): counts stop growing at the first error.
__device__ __forceinline__ uint64_t seq_combine(uint64_t a, uint64_t b)
{
    if (a & kErrBit)
        return a & (kErrBit | kValMask);
    return (b & kErrBit) | (((a & kValMask) + (b & kValMask)) & kValMask);
}

// Decoupled look-back, executed by one whole warp.  Publishes this tile's
// aggregate, accumulates predecessors (32 at a time, nearest first) until an
// inclusive prefix is found, publishes the inclusive prefix and returns the
// exclusive one (flag bits clear).
__device__ __forceinline__ uint64_t lookback(uint64_t *status, uint32_t tile, uint64_t agg)
{
    const uint32_t lane = lane_id();
    if (tile == 0) {
        if (lane == 0)
            st_release(&status[0], kFlagInc | agg);
        return 0;
    }
    if (lane == 0)
        st_release(&status[tile], kFlagAgg | agg);
    // Each lane inspects kPerLane consecutive predecessors, so one L2 round
    // trip covers 32*kPerLane tiles: the inclusive-prefix frontier then moves
    // 256 tiles (4 MiB of input) per round trip instead of 32.
    constexpr int kPerLane = 4;
    uint64_t excl = 0;
    int64_t pred = (int64_t)tile - 1;
    while (true) {
        uint64_t s[kPerLane];
#pragma unroll
        for (int j = 0; j < kPerLane; ++j) {
            const int64_t t = pred - (int64_t)(kPerLane * lane + j);
            s[j] = (t >= 0) ? ld_acquire(&status[t]) : kFlagInc; // before tile 0: identity, inclusive
        }
#pragma unroll
        for (int j = 0; j < kPerLane; ++j) {
            const int64_t t = pred - (int64_t)(kPerLane * lane + j);
            uint32_t spins = 0;
            while ((s[j] >> kFlagShift) == 0) {
                if (++spins > 64)
                    __nanosleep(20);
                s[j] = ld_acquire(&status[t]);
            }
        }
        // closest inclusive inside this lane's slice
        int jinc = kPerLane;
#pragma unroll
        for (int j = kPerLane - 1; j >= 0; --j)
            if ((s[j] >> kFlagShift) == 2)
                jinc = j;
        uint64_t v = 0;
#pragma unroll
        for (int j = kPerLane - 1; j >= 0; --j)
            if (j <= jinc)
                v = seq_combine(v, s[j] & (kErrBit | kValMask));
        const uint32_t inc = __ballot_sync(0xffffffffu, jinc < kPerLane);
        const uint32_t stop = inc ? (uint32_t)(__ffs(inc) - 1) : 31u;
        if (lane > stop)
            v = 0;
        // ordered reduction: higher lane = earlier tile
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint64_t o = __shfl_down_sync(0xffffffffu, v, d);
            if (lane + d < 32)
                v = seq_combine(o, v);
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        excl = seq_combine(v, excl);
        if (inc)
            break;
        pred -= 32 * kPerLane;
    }
    if (lane == 0)
        st_release(&status[tile], kFlagInc | seq_combine(excl, agg));
    return excl;
}

// Central scanner, run by one warp for the whole grid.  Tiles publish only
// their aggregate (flag 1); the scanner sweeps the status array in tile order,
// 32*K entries per pass, and replaces each ready entry by flag 2 | EXCLUSIVE
// prefix.  One pass covers up to 32*K tiles per L2 round trip, and no tile
// ever waits on an inclusive-prefix chain: a tile's owner just polls its own
// status word.  It stops at the first tile whose aggregate is not yet
// published, so every claimed tile must publish without waiting on anything.
template <int K>
__device__ __forceinline__ void scan_tiles(uint64_t *status, uint32_t ntiles)
{
    const uint32_t lane = lane_id();
    uint32_t next = 0;
    uint64_t acc = 0;
    while (next < ntiles) {
        uint64_t s[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint32_t t = next + lane * K + j;
            s[j] = t < ntiles ? ld_acquire(&status[t]) : 0ull;
        }
        uint32_t r = K; // leading ready entries of this lane's slice
#pragma unroll
        for (int j = K - 1; j >= 0; --j)
            if ((s[j] >> kFlagShift) == 0)
                r = j;
        const uint32_t full = __ballot_sync(0xffffffffu, r == K);
        const uint32_t f = full == 0xffffffffu ? 32u : (uint32_t)__ffs(~full) - 1;
        const uint32_t myr = lane < f ? K : (lane == f ? r : 0u);
        const uint32_t total = __reduce_add_sync(0xffffffffu, myr);
        if (total == 0) {
            __nanosleep(64);
            continue;
        }
        uint64_t sum = 0;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((uint32_t)j < myr)
                sum = seq_combine(sum, s[j] & (kErrBit | kValMask));
        uint64_t inc = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (uint32_t)d)
                inc = seq_combine(o, inc);
        }
        uint64_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0)
            ex = 0;
        uint64_t run = seq_combine(acc, ex);
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((uint32_t)j < myr) {
                st_release(&status[next + lane * K + j], kFlagInc | run);
                run = seq_combine(run, s[j] & (kErrBit | kValMask));
            }
        acc = seq_combine(acc, __shfl_sync(0xffffffffu, inc, 31));
        next += total;
    }
}

// ------------------------------------------------------- tile staging loads

// Loads the 16 KiB tile at aligned byte offset tile_off (relative to the
// 16-byte aligned base) plus a 4-byte halo on each side into in_s.  Bytes
// whose logical position (aligned offset - lead) is outside [0, n_bytes) read
// as 0x00, which every kernel treats as "no unit here" (ASCII / non-surrogate,
// never a continuation): exactly the reference's start/end-of-input rules.
__device__ __forceinline__ uint32_t load_u32_masked(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    if (a >= lo && a + 4 <= hi)
        return *reinterpret_cast<const uint32_t *>(base + a);
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int64_t p = a + k;
        if (p >= lo && p < hi)
            v |= (uint32_t)base[p] << (8 * k);
    }
    return v;
}

__device__ __forceinline__ uint4 load_u128_masked(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    if (a >= lo && a + 16 <= hi)
        return __ldcs(reinterpret_cast<const uint4 *>(base + a));
    uint4 v;
    v.x = load_u32_masked(base, a, lo, hi);
    v.y = load_u32_masked(base, a + 4, lo, hi);
    v.z = load_u32_masked(base, a + 8, lo, hi);
    v.w = load_u32_masked(base, a + 12, lo, hi);
    return v;
}

// Returns true when the tile (with halos) lies entirely inside the input.
__device__ __forceinline__ bool stage_tile(uint32_t *in_s, const uint8_t *base, int64_t tile_off, int64_t lo,
                                           int64_t hi)
{
    const bool interior = (tile_off - 4 >= lo) && (tile_off + kTileBytes + 4 <= hi);
    uint4 *dst = reinterpret_cast<uint4 *>(in_s + kInHead);
    const uint4 *src = reinterpret_cast<const uint4 *>(base + tile_off);
    if (interior) {
        uint4 v[kTileBytes / 16 / kThreads];
#pragma unroll
        for (int m = 0; m < kTileBytes / 16 / kThreads; ++m)
            v[m] = __ldcs(src + threadIdx.x + m * kThreads);
#pragma unroll
        for (int m = 0; m < kTileBytes / 16 / kThreads; ++m)
            dst[threadIdx.x + m * kThreads] = v[m];
        if (threadIdx.x == 0)
            in_s[kInHead - 1] = *reinterpret_cast<const uint32_t *>(base + tile_off - 4);
        if (threadIdx.x == 1)
            in_s[kInHead + kTileWords32] = *reinterpret_cast<const uint32_t *>(base + tile_off + kTileBytes);
    } else {
#pragma unroll 1
        for (int m = 0; m < kTileBytes / 16 / kThreads; ++m) {
            int64_t a = tile_off + 16 * (int64_t)(threadIdx.x + m * kThreads);
            uint4 v = make_uint4(0, 0, 0, 0);
            if (a + 16 > lo && a < hi)
                v = load_u128_masked(base, a, lo, hi);
            dst[threadIdx.x + m * kThreads] = v;
        }
        if (threadIdx.x == 0)
            in_s[kInHead - 1] = (tile_off - 4 + 4 > lo && tile_off - 4 < hi)
                                    ? load_u32_masked(base, tile_off - 4, lo, hi)
                                    : 0u;
        if (threadIdx.x == 1) {
            int64_t a = tile_off + kTileBytes;
            in_s[kInHead + kTileWords32] = (a + 4 > lo && a < hi) ? load_u32_masked(base, a, lo, hi) : 0u;
        }
    }
    return interior;
}

// Per-quad validity mask (bit 7 of each byte whose logical position is in
// [0, n)) for boundary tiles.
__device__ __forceinline__ uint32_t valid_mask(int64_t a, int64_t lo, int64_t hi)
{
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (a + k >= lo && a + k < hi)
            m |= 0x80u << (8 * k);
    return m;
}

// Warp inclusive scan of packed 8-bit lanes (no lane overflows 255).
__device__ __forceinline__ uint32_t warp_scan_packed(uint32_t v)
{
    const uint32_t lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= (uint32_t)d)
            v += o;
    }
    return v;
}

} // namespace lu
