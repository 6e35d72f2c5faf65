// lu_common.cuh -- shared pieces of the sm_100a transcode/validate kernels.
//
// Geometry (all kernels): a warp owns a contiguous 2 KiB chunk of input and
// walks it in 4 rounds of 512 B, lane l holding bytes [16l, 16l+16) of the
// round in registers (neighbours by shuffle).  The transcode kernels group 4
// chunks into an 8 KiB tile; tiles are ordered by a central scanner warp
// (scan_tiles) rather than a per-tile look-back.
//
// Tile status word (uint64, one per tile, zeroed before each launch):
//   bits 63..62  flag: 0 not ready, 1 aggregate, 2 exclusive prefix
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
constexpr int kChunkBytes = kTileBytes / kWarps;      // 2048 B per warp

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

// Bytes whose logical position (aligned offset - lead) is outside
// [0, n_bytes) read as 0x00, which every kernel treats as "no unit here"
// (ASCII / non-surrogate, never a continuation): exactly the reference's
// start/end-of-input rules.
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


} // namespace lu
