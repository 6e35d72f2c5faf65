// lu_kernels.cu -- sm_100a kernels K1..K4 and the C-ABI entry points of
// liblaneutf_b200.so (declared in include/laneutf_b200.h).
//
// One launch per call: K1/K2 are single-pass (classify/validate -> central
// scanner orders 8 KiB tiles -> staged scatter) persistent kernels; K3/K4 are
// warp-persistent read-only validators that reduce the first bad position
// with one atomic and finalize in the last warp.  Stream-ordered; the library
// allocates nothing and keeps no mutable global state (per-call workspace,
// thread-local error string).
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "lu_common.cuh"
#include "lu_utf16.cuh"
#include "lu_utf8.cuh"
#include "lu_utf8_lc.cuh"

#include "../../include/laneutf_b200.h"

namespace lu {

constexpr int kOutStrideU16 = kChunkBytes + 16;      // words per warp staging region (<= 1 word per byte)
constexpr int kOutStrideU8 = 3 * kChunkBytes / 2 + 32; // bytes per warp region (<= 3 bytes per word)

// staging buffers per group: K1 double-buffered (its 8.2 KiB of words per
// warp leave no room for a third buffer at 3 CTAs/SM), K2 triple-buffered
// (more slack for the scanner's prefix before a buffer is reused)
constexpr int kBufsK1 = 2, kBufsK2 = 3;
constexpr size_t kSmemK1 = kBufsK1 * sizeof(uint16_t) * kOutStrideU16 * kWarps; // 2 groups x 2 buffers x 4 warps
constexpr size_t kSmemK2 = kBufsK2 * kOutStrideU8 * kWarps; // 2 groups x 3 buffers x 4 warps

// ------------------------------------------------------------- copy-out

// Copy cnt UTF-16 words from a warp's shared staging region (16-byte aligned)
// to out_a[g0 ..) (out_a 16-byte aligned).  Interior 16-byte chunks use vector
// stores; the partial head/tail chunks are written word-parallel by lanes
// 0..15.  All index math is 32-bit relative to the aligned chunk start.
__device__ __forceinline__ void copy_out_u16(const uint16_t *src, uint32_t cnt, uint16_t *out_a, uint64_t g0)
{
    if (cnt == 0)
        return;
    const uint32_t lane = lane_id();
    const uint32_t shift = (uint32_t)(g0 & 7);
    uint16_t *dst = out_a + (g0 - shift); // 16-byte aligned
    const uint32_t total = shift + cnt;   // words from the aligned start
    const uint32_t full_lo = shift ? 1u : 0u, full_hi = total >> 3;
    // Each output chunk straddles two aligned 16-byte staging vectors; read
    // both with conflict-free LDS.128 and select the window (warp-uniform
    // word offset r) in registers.
    const uint4 *s128 = reinterpret_cast<const uint4 *>(src);
    const uint32_t r = (8u - shift) & 7u;
    uint4 *d128 = reinterpret_cast<uint4 *>(dst);
    // the word shift is warp-uniform: one specialised loop per value
    switch (r) {
    case 0:
#pragma unroll 1
        for (uint32_t c = full_lo + lane; c < full_hi; c += 32)
            __stcs(d128 + c, s128[c]);
        break;
#define LU_COPY_CASE(R, BODY)                                                                                          \
    case R:                                                                                                            \
        _Pragma("unroll 1") for (uint32_t c = full_lo + lane; c < full_hi; c += 32) {                                  \
            const uint32_t v = c - 1;                                                                                  \
            const uint4 a = s128[v], b = s128[v + 1];                                                                  \
            const uint32_t w0 = a.x, w1 = a.y, w2 = a.z, w3 = a.w, w4 = b.x, w5 = b.y, w6 = b.z, w7 = b.w;             \
            (void)w0, (void)w1, (void)w2, (void)w3, (void)w4, (void)w5, (void)w6, (void)w7;                            \
            __stcs(d128 + c, BODY);                                                                                    \
        }                                                                                                              \
        break;
        LU_COPY_CASE(1, make_uint4(prmt(w0, w1, 0x5432), prmt(w1, w2, 0x5432), prmt(w2, w3, 0x5432),
                                   prmt(w3, w4, 0x5432)))
        LU_COPY_CASE(2, make_uint4(w1, w2, w3, w4))
        LU_COPY_CASE(3, make_uint4(prmt(w1, w2, 0x5432), prmt(w2, w3, 0x5432), prmt(w3, w4, 0x5432),
                                   prmt(w4, w5, 0x5432)))
        LU_COPY_CASE(4, make_uint4(w2, w3, w4, w5))
        LU_COPY_CASE(5, make_uint4(prmt(w2, w3, 0x5432), prmt(w3, w4, 0x5432), prmt(w4, w5, 0x5432),
                                   prmt(w5, w6, 0x5432)))
        LU_COPY_CASE(6, make_uint4(w3, w4, w5, w6))
        LU_COPY_CASE(7, make_uint4(prmt(w3, w4, 0x5432), prmt(w4, w5, 0x5432), prmt(w5, w6, 0x5432),
                                   prmt(w6, w7, 0x5432)))
#undef LU_COPY_CASE
    }
    // partial chunks: head (chunk 0 when shift > 0) and tail (chunk full_hi)
    if (lane < 16) {
        uint32_t chunk;
        if (lane < 8)
            chunk = shift ? 0u : 0xffffffffu;
        else
            chunk = (total & 7) && !(shift && full_hi == 0) ? full_hi : 0xffffffffu;
        if (chunk != 0xffffffffu) {
            const uint32_t i = 8 * chunk + (lane & 7);
            if (i >= shift && i < total)
                dst[i] = src[i - shift];
        }
    }
}

// Same for bytes (UTF-8 output), 16-byte chunks; head/tail by lanes 0..31.
__device__ __forceinline__ void copy_out_u8(const uint8_t *src, uint32_t cnt, uint8_t *out_a, uint64_t g0)
{
    if (cnt == 0)
        return;
    const uint32_t lane = lane_id();
    const uint32_t shift = (uint32_t)(g0 & 15);
    uint8_t *dst = out_a + (g0 - shift);
    const uint32_t total = shift + cnt;
    const uint32_t full_lo = shift ? 1u : 0u, full_hi = total >> 4;
    // Output chunk c holds staging bytes [16c - shift, +16): for shift > 0
    // that is byte r = 16 - shift of staging vector c - 1 onwards.  Read the
    // two aligned vectors with conflict-free LDS.128 (5 LDS.32 per chunk were
    // 4-way bank conflicted) and funnel-shift by the warp-uniform word offset
    // q = r / 4 (one specialised loop per value) and byte shift sh.
    const uint4 *s128 = reinterpret_cast<const uint4 *>(src);
    uint4 *d128 = reinterpret_cast<uint4 *>(dst);
    if (shift == 0) {
#pragma unroll 1
        for (uint32_t c = lane; c < full_hi; c += 32)
            __stcs(d128 + c, s128[c]);
    } else {
        const uint32_t r = 16u - shift, sh = 8u * (r & 3u);
        switch (r >> 2) {
#define LU_COPY8_CASE(Q, BODY)                                                                                         \
    case Q:                                                                                                            \
        _Pragma("unroll 1") for (uint32_t c = full_lo + lane; c < full_hi; c += 32) {                                  \
            const uint4 a = s128[c - 1], b = s128[c];                                                                  \
            const uint32_t w0 = a.x, w1 = a.y, w2 = a.z, w3 = a.w, w4 = b.x, w5 = b.y, w6 = b.z, w7 = b.w;             \
            (void)w0, (void)w1, (void)w2, (void)w3, (void)w4, (void)w5, (void)w6, (void)w7;                            \
            __stcs(d128 + c, BODY);                                                                                    \
        }                                                                                                              \
        break;
            LU_COPY8_CASE(0, make_uint4(fsr(w0, w1, sh), fsr(w1, w2, sh), fsr(w2, w3, sh), fsr(w3, w4, sh)))
            LU_COPY8_CASE(1, make_uint4(fsr(w1, w2, sh), fsr(w2, w3, sh), fsr(w3, w4, sh), fsr(w4, w5, sh)))
            LU_COPY8_CASE(2, make_uint4(fsr(w2, w3, sh), fsr(w3, w4, sh), fsr(w4, w5, sh), fsr(w5, w6, sh)))
            LU_COPY8_CASE(3, make_uint4(fsr(w3, w4, sh), fsr(w4, w5, sh), fsr(w5, w6, sh), fsr(w6, w7, sh)))
#undef LU_COPY8_CASE
        }
    }
    uint32_t chunk;
    if (lane < 16)
        chunk = shift ? 0u : 0xffffffffu;
    else
        chunk = (total & 15) && !(shift && full_hi == 0) ? full_hi : 0xffffffffu;
    if (chunk != 0xffffffffu) {
        const uint32_t i = 16 * chunk + (lane & 15);
        if (i >= shift && i < total)
            dst[i] = src[i - shift];
    }
}

__device__ __forceinline__ void sel_table_init(SelPair *sel)
{
    if (threadIdx.x < 16) {
        const uint32_t idx = threadIdx.x;
        uint32_t s[2] = {0, 0};
        uint32_t j = 0;
        for (uint32_t p = 0; p < 4; ++p) {
            if (idx & (1u << p)) {
                const uint32_t nib = p | ((4 + p) << 4);
                s[j >> 1] |= nib << (8 * (j & 1));
                ++j;
            }
        }
        sel[idx].s01 = s[0];
        sel[idx].s23 = s[1];
    } else if (threadIdx.x < 32) {
        // K2 path C (u16u8_warp_r): entry (c0 | c1 << 2) for the classes of a
        // word pair (0 ASCII, 1 low surrogate, 2 high surrogate; T0 / T1 =
        // their 4-byte strings, bytes 0-3 / 4-7 of prmt): s01 = selector of
        // the first four bytes, s23 = selector of the fifth | byte count << 16.
        // Pairs that cannot occur in a path-C round (AL, LL, HA, HH) emit 0.
        const uint32_t idx = threadIdx.x - 16;
        uint32_t lo = 0, hi = 0, nb = 0;
        switch (idx) {
        case 0: lo = 0x0040u; nb = 2; break;             // A A
        case 8: lo = 0x6540u; hi = 0x7u; nb = 5; break;  // A H
        case 1: lo = 0x0004u; nb = 1; break;             // L A
        case 9: lo = 0x7654u; nb = 4; break;             // L H
        case 6: lo = 0x3210u; nb = 4; break;             // H L
        default: break;
        }
        sel[16 + idx].s01 = lo;
        sel[16 + idx].s23 = hi | (nb << 16);
    } else if (threadIdx.x < 40) {
        // K2 path A: entry (odd << 2 | big1 << 1 | big0) for a word pair of
        // 1- or 2-byte words (big = 2-byte); F / S = planes of the first /
        // second bytes of 4 words (bytes 0-3 / 4-7 of prmt), the pair being
        // words 0, 1 (odd = 0) or 2, 3 (odd = 1) of the planes
        const uint32_t idx = threadIdx.x - 32;
        const uint32_t o = 2u * (idx >> 2), b0 = idx & 1u, b1 = (idx >> 1) & 1u;
        uint32_t sel_v = 0, j = 0;
        const uint32_t bytes[4] = {o, 4u + o, o + 1u, 5u + o}; // F0 S0 F1 S1
        for (uint32_t t = 0; t < 4; ++t) {
            if ((t == 1 && !b0) || (t == 3 && !b1))
                continue;
            sel_v |= bytes[t] << (4 * j++);
        }
        sel[32 + idx].s01 = sel_v;
        sel[32 + idx].s23 = j; // byte count
    } else if (threadIdx.x < 56) {
        // K2 path D (no surrogate, words of 1, 2 or 3 bytes): entry c0 | c1 << 2
        // with c = bytes - 1 of each word of a pair.  prmt bytes 0-3 =
        // [X0, Y0, X1, Y1] (middle / last byte planes of the pair), bytes 4, 5 =
        // Z0, Z1 (3-byte leads): s01 = selector of the pair's first four
        // bytes, s23 = selector of bytes five and six | byte count << 16
        const uint32_t idx = threadIdx.x - 40;
        const uint32_t c0 = idx & 3u, c1 = idx >> 2;
        uint32_t b[6] = {0, 0, 0, 0, 0, 0}, j = 0;
        if (c0 < 3 && c1 < 3) {
            if (c0 == 2)
                b[j++] = 4;
            if (c0 >= 1)
                b[j++] = 0;
            b[j++] = 1;
            if (c1 == 2)
                b[j++] = 5;
            if (c1 >= 1)
                b[j++] = 2;
            b[j++] = 3;
        }
        sel[40 + idx].s01 = b[0] | b[1] << 4 | b[2] << 8 | b[3] << 12;
        sel[40 + idx].s23 = b[4] | b[5] << 4 | j << 16;
    }
}

// ====================================================== pipelined transcode
//
// Persistent CTAs (grid = resident capacity + 1).  CTA 0 runs the central
// scanner (scan_windows) on all its warps.  Every other CTA holds two
// independent tile groups of 4 warps (8 KiB tiles).  Each group claims tiles
// from a ticket counter (tiles finish roughly in ticket order), computes a
// tile into one of its two shared staging buffers and publishes the tile
// aggregate; it copies a buffer out when it is about to reuse it, two tiles
// later, by which time the scanner has normally published that tile's
// exclusive prefix.  The two groups run unsynchronised, so one group's
// HBM-bound copy-out overlaps the other's ALU-bound compute.  Every CTA is
// resident and a tile publishes its aggregate before its group waits on
// anything, and the scanner's partial-window fallback makes every prefix
// depend only on earlier tiles, so progress is guaranteed.
//
// Named barriers per group g (kGroupThreads threads): 1+3g ticket broadcast,
// 2+3g tile computed, 3+3g prefix broadcast.

#ifndef LU_GROUP_WARPS
#define LU_GROUP_WARPS 4
#endif
constexpr int kGroupWarps = LU_GROUP_WARPS;
constexpr int kGroupsPerCta = 8 / kGroupWarps;
constexpr int kGroupThreads = 32 * kGroupWarps;
constexpr int kPipeTile = kGroupWarps * kChunkBytes; // 8 KiB
constexpr int kPipeThreads = kGroupsPerCta * kGroupThreads;
static_assert(kPipeThreads / 32 == kScanWarps, "CTA 0's warps are the scanner warps");

constexpr int kMaxBufs = 3;
// When a group takes its next tile ticket: 0 right after the tile-done
// barrier (the atomic overlaps the combine), 1 at the top of the next
// iteration after the resolve (default: a group never holds an unprocessed
// tile while it waits on a prefix; K1 -1..-2%), 2 at the top before the
// resolve (atomic and status poll overlap; neutral), 3 one iteration ahead
// (K1 +6-24%: tiles held through resolve waits delay every later prefix).
#ifndef LU_CLAIM_AT
#define LU_CLAIM_AT 1
#endif
#ifndef LU_RESOLVE_SLEEP
#define LU_RESOLVE_SLEEP 32 // ns between polls of a tile's status word
#endif

struct GroupShared {
    WarpResult wres[kMaxBufs][kGroupWarps];
    uint32_t warp_excl[kMaxBufs][kGroupWarps];
    uint64_t excl[kMaxBufs];
    uint32_t first_err[kMaxBufs];
    uint32_t tile_of[kMaxBufs];
    uint32_t units[kMaxBufs]; // tile output units before its first error (or all)
    uint32_t claim;
    uint32_t skip; // the claimed tile lies after a tile known to hold an error
    uint32_t hint_s[kGroupWarps]; // a direction's per-warp hint when it is kept in shared memory (kHintInSmem)
};

__device__ __forceinline__ void bar_sync(uint32_t id, uint32_t n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Direction traits: UTF-8 -> UTF-16 (K1) and UTF-16 -> UTF-8 (K2); BE = the
// UTF-16 side is big-endian (byte swap fused into K1's compaction / K2's load).
template <bool BE>
struct DirU8U16T {
    using OutT = uint16_t;
    static constexpr int kStride = kOutStrideU16;
    static constexpr int kBufs = kBufsK1;
    static constexpr int kUnitShift = 0; // input positions are bytes
    static constexpr int kScanPerLane = LU_SCAN_PER_LANE; // 96-tile scanner windows
    static constexpr bool kHintInSmem = false;
    using In = ChunkIn;
    template <bool B>
    __device__ static void load(const uint8_t *base, int64_t tile_off, int64_t lo_b, int64_t hi_b, uint32_t wit,
                                In &in)
    {
        load_chunk<B>(base, tile_off + (int64_t)wit * kChunkBytes, lo_b, hi_b, in);
    }
    template <bool B>
    __device__ static void compute(const uint8_t *base, int64_t tile_off, int64_t lo_b, int64_t hi_b, OutT *out_w,
                                   const SelPair *sel, WarpResult &wr, uint32_t wit, const In &in, uint32_t &hint)
    {
        u8u16_warp<B, BE>(base, tile_off, lo_b, hi_b, out_w, sel, wr, wit, in, hint);
    }
    __device__ static void copy_out(const OutT *src, uint32_t cnt, OutT *out_a, uint64_t g0)
    {
        copy_out_u16(src, cnt, out_a, g0);
    }
};

template <bool BE>
struct DirU16U8T {
    using OutT = uint8_t;
    static constexpr int kStride = kOutStrideU8;
    static constexpr int kBufs = kBufsK2;
    static constexpr int kUnitShift = 1; // input positions are 16-bit words
    static constexpr int kScanPerLane = LU_K2_SCAN_PER_LANE; // 128-tile windows
    static constexpr bool kHintInSmem = false;
    using In = ChunkIn;
    template <bool B>
    __device__ static void load(const uint8_t *base, int64_t tile_off, int64_t lo_b, int64_t hi_b, uint32_t wit,
                                In &in)
    {
        load_chunk<B, BE>(base, tile_off + (int64_t)wit * kChunkBytes, lo_b, hi_b, in);
    }
    template <bool B>
    __device__ static void compute(const uint8_t *base, int64_t tile_off, int64_t lo_b, int64_t hi_b, OutT *out_w,
                                   const SelPair *sel, WarpResult &wr, uint32_t wit, const In &in, uint32_t &hint)
    {
        // ASCII chunks: a warp whose previous chunk was all ASCII (hint 4)
        // first tries the narrow-only path.  Kept outside the warp body
        // (inside it, even out of line, it cost K2 1.5% on every profile).
        if (LU_K2_ASCII && !B && hint == 4u &&
            u16u8_ascii_chunk(in.q[0], in.q[1], in.q[2], in.q[3], (uint32_t)__cvta_generic_to_shared(out_w))) {
            if (lane_id() == 0) {
                wr.err = 0;
                wr.pos = 0;
                wr.units = kChunkBytes / 2;
            }
            return;
        }
        u16u8_warp_r<B>(base, tile_off, lo_b, hi_b, out_w, sel + 16, wr, wit, in);
        if (LU_K2_ASCII && !B) {
            // one byte per word and no error: the chunk was all ASCII
            __syncwarp();
            const bool ascii = wr.err == 0 && wr.units == (uint32_t)(kChunkBytes / 2);
            __syncwarp();
            hint = ascii ? 4u : 2u;
        }
    }
    __device__ static void copy_out(const OutT *src, uint32_t cnt, OutT *out_a, uint64_t g0)
    {
        copy_out_u8(src, cnt, out_a, g0);
    }
};

using DirU8U16 = DirU8U16T<false>;
using DirU16U8 = DirU16U8T<false>;

// Group thread 0: wait for the scanner's exclusive prefix of the tile held in
// buffer b, and write the result record if this is the first-error tile or
// the last tile.
template <class Dir>
__device__ __forceinline__ void pipe_resolve(GroupShared &ps, uint32_t b, uint64_t *status, Outcome *res,
                                             uint32_t ntiles, int64_t lo_b, uint64_t n_units, uint64_t st)
{
    const uint32_t tile = ps.tile_of[b];
    if ((st >> kFlagShift) != 2)
        st = ld_acquire(&status[tile]);
    uint32_t spins = 0;
    const uint64_t t0 = (st >> kFlagShift) != 2 ? gtimer() : 0;
    while ((st >> kFlagShift) != 2) {
        __nanosleep(LU_RESOLVE_SLEEP);
        st = ld_acquire(&status[tile]);
        ++spins;
        hang_check(spins, t0);
    }
    LU_CNT(9, spins);
    LU_CNT(10, spins ? 1 : 0);
    const uint64_t ex = st & (kErrBit | kValMask);
    ps.excl[b] = ex;
    if (!(ex & kErrBit)) {
        const uint32_t first = ps.first_err[b];
        const uint64_t written = ex + ps.units[b];
        const int64_t tile_off = (int64_t)tile * kPipeTile;
        if (first < kGroupWarps) {
            res->status = kStatusMalformed;
            res->pad = 0;
            res->consumed = (uint64_t)((tile_off + ps.wres[b][first].pos - lo_b) >> Dir::kUnitShift);
            res->written = written;
        } else if (tile == ntiles - 1) {
            res->status = kStatusOk;
            res->pad = 0;
            res->consumed = n_units;
            res->written = written;
        }
    }
}

// Every warp of the group: copy its staged region of buffer b out (prefix known).
template <class Dir>
__device__ __forceinline__ void pipe_copy(GroupShared &ps, uint32_t b, uint32_t wit, typename Dir::OutT *out_g,
                                          typename Dir::OutT *out_a, uint64_t out_lead)
{
    const uint64_t ex = ps.excl[b];
    if (!(ex & kErrBit) && wit <= ps.first_err[b])
        Dir::copy_out(out_g + (b * kGroupWarps + wit) * Dir::kStride, ps.wres[b][wit].units, out_a,
                      ex + ps.warp_excl[b][wit] + out_lead);
}

// Warp 0 of a group, after the tile-done barrier: combine the 4 warp
// results of buffer buf on lanes 0..3 (shallow dependency chain: this is on
// the group's critical path) and publish the tile aggregate.
__device__ __forceinline__ void group_combine(GroupShared &ps, uint32_t buf, uint32_t tile, uint64_t *status,
                                              unsigned int *err_tile, uint32_t ntiles)
{
    const uint32_t lane = lane_id();
    const WarpResult r = ps.wres[buf][lane & (kGroupWarps - 1)];
    const uint32_t errm = __ballot_sync(0xffffffffu, lane < kGroupWarps && r.err);
    const uint32_t first = errm ? (uint32_t)__ffs(errm) - 1 : kGroupWarps;
    const uint32_t u = (lane < kGroupWarps && lane <= first) ? r.units : 0u;
    uint32_t inc = u;
#pragma unroll
    for (int d = 1; d < kGroupWarps; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= (uint32_t)d)
            inc += o;
    }
    if (lane < kGroupWarps)
        ps.warp_excl[buf][lane] = inc - u;
    const uint32_t units = __shfl_sync(0xffffffffu, inc, kGroupWarps - 1);
    if (lane == 0) {
        ps.first_err[buf] = first;
        ps.tile_of[buf] = tile;
        ps.units[buf] = units;
        // atomicMax: never overwrites a prefix (flag 2 > flag 1) that the
        // scanner already published for a tile behind an error
        atomicMax(reinterpret_cast<unsigned long long *>(&status[tile]),
                  (unsigned long long)(kFlagAgg | (first < kGroupWarps ? kErrBit : 0ull) | (uint64_t)units));
        if (first < kGroupWarps)
            atomicMax(err_tile, ntiles - tile);
    }
}

// Small inputs (ntiles <= 2 x resident CTAs, e.g. config 1's 4 MiB): every
// group owns exactly one tile -- the CTA with role r (the r-th CTA to start)
// takes tiles 2r and 2r+1 -- so there is no ticket, no scanner and no
// deferred copy-out.  After publishing its aggregate the group sums the
// aggregates of all earlier tiles itself (its 128 threads load them in
// parallel; they belong to CTAs that started earlier, so the wait always
// ends), then copies out.  Latency of a call drops from the persistent
// pipeline's fill/drain chain to compute + one look-back.
template <class Dir>
__device__ __forceinline__ void small_tile(GroupShared &ps, uint32_t tile, uint32_t g, uint32_t wit, uint32_t gtid,
                                           const uint8_t *__restrict__ base, int64_t lo_b, int64_t hi_b,
                                           uint64_t n_units, typename Dir::OutT *out_g, typename Dir::OutT *out_a,
                                           uint64_t out_lead, uint64_t *status, unsigned int *err_tile,
                                           Outcome *res, uint32_t ntiles, const SelPair *sel,
                                           unsigned long long *lb_sum, uint32_t *lb_err)
{
    const uint32_t bar_done = 2 + 3 * g, bar_prefix = 3 + 3 * g;
    const int64_t tile_off = (int64_t)tile * kPipeTile;
    const bool interior = (tile_off - 4 >= lo_b) && (tile_off + kPipeTile + 4 <= hi_b);
    typename Dir::In in;
    uint32_t hint = 2;
    typename Dir::OutT *out_w = out_g + wit * Dir::kStride; // buffer 0
    if (interior) {
        Dir::template load<false>(base, tile_off, lo_b, hi_b, wit, in);
        Dir::template compute<false>(base, tile_off, lo_b, hi_b, out_w, sel, ps.wres[0][wit], wit, in, hint);
    } else {
        Dir::template load<true>(base, tile_off, lo_b, hi_b, wit, in);
        Dir::template compute<true>(base, tile_off, lo_b, hi_b, out_w, sel, ps.wres[0][wit], wit, in, hint);
    }
    bar_sync(bar_done, kGroupThreads);
    if (wit == 0)
        group_combine(ps, 0, tile, status, err_tile, ntiles);
    // look-back: thread t of the group sums the aggregates of tiles j < tile
    // with j = t (mod 128), loads issued 4 at a time
    unsigned long long acc = 0;
    uint32_t err = 0;
    for (uint32_t j0 = gtid; j0 < tile; j0 += 4 * kGroupThreads) {
        uint64_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t j = j0 + k * kGroupThreads;
            v[k] = j < tile ? ld_acquire(&status[j]) : kFlagAgg;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t j = j0 + k * kGroupThreads;
            uint32_t spins = 0;
            uint64_t t0 = 0;
            while ((v[k] >> kFlagShift) == 0) {
                if (spins++ == 0)
                    t0 = gtimer();
                hang_check(spins, t0);
                __nanosleep(32);
                v[k] = ld_acquire(&status[j]);
            }
            acc += v[k] & kValMask;
            err |= (v[k] & kErrBit) ? 1u : 0u;
        }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1)
        acc += __shfl_xor_sync(0xffffffffu, acc, d);
    err = __any_sync(0xffffffffu, err != 0);
    if ((gtid & 31) == 0) {
        lb_sum[wit] = acc;
        lb_err[wit] = err;
    }
    bar_sync(bar_prefix, kGroupThreads);
    if (gtid == 0) {
        unsigned long long sum = 0;
        uint32_t eor = 0;
#pragma unroll
        for (int k = 0; k < kGroupWarps; ++k) {
            sum += lb_sum[k];
            eor |= lb_err[k];
        }
        const bool e = eor != 0;
        const uint64_t ex = (sum & kValMask) | (e ? kErrBit : 0ull);
        ps.excl[0] = ex;
        if (!e) {
            const uint32_t first = ps.first_err[0];
            const uint64_t written = sum + ps.units[0];
            if (first < kGroupWarps) {
                res->status = kStatusMalformed;
                res->pad = 0;
                res->consumed = (uint64_t)((tile_off + ps.wres[0][first].pos - lo_b) >> Dir::kUnitShift);
                res->written = written;
            } else if (tile == ntiles - 1) {
                res->status = kStatusOk;
                res->pad = 0;
                res->consumed = n_units;
                res->written = written;
            }
        }
    }
    bar_sync(bar_prefix, kGroupThreads);
    pipe_copy<Dir>(ps, 0, wit, out_g, out_a, out_lead);
}

template <class Dir>
__global__ void __launch_bounds__(kPipeThreads, 3)
    k_transcode(const uint8_t *__restrict__ base, uint32_t lead, uint64_t n_units, uint64_t n_bytes,
                typename Dir::OutT *__restrict__ out_a, uint32_t out_lead, uint64_t *__restrict__ status,
                Outcome *__restrict__ res, uint32_t ntiles, uint32_t small)
{
    using OutT = typename Dir::OutT;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ SelPair sel[56]; // K1 compaction selectors, then K2 path-C, path-A and path-D selectors
    __shared__ GroupShared gshared[kGroupsPerCta];
    __shared__ ScanShared scan_s;
    __shared__ uint32_t role_s;
    __shared__ unsigned long long lb_sum[kGroupsPerCta][kGroupWarps];
    __shared__ uint32_t lb_err[kGroupsPerCta][kGroupWarps];

    const int64_t lo_b = lead, hi_b = (int64_t)lead + (int64_t)n_bytes;
    unsigned int *ticket = reinterpret_cast<unsigned int *>(status + ntiles);
    unsigned int *err_tile = ticket + 1;  // zeroed with the status words
    unsigned int *role_ctr = ticket + 2;  // idem
    sel_table_init(sel);
    scan_init(scan_s);
    // The scanner is the first CTA to start, not blockIdx 0: CUDA does not
    // promise to dispatch blocks in index order, and other kernels (user
    // streams, MPS, NCCL) may hold SMs, so a fixed scanner CTA could still be
    // waiting for a slot while the workers that depend on it spin.  The
    // first CTA to take a role ticket is running by construction; every
    // other wait is on tiles claimed by running CTAs, so the kernel makes
    // progress whatever subset of its CTAs is resident.
    if (threadIdx.x == 0)
        role_s = atomicAdd(role_ctr, 1u);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    LU_PROF_INIT();
    if (small) {
        const uint32_t g = warp / kGroupWarps, wit = warp % kGroupWarps;
        const uint32_t tile = role_s * kGroupsPerCta + g;
        if (tile < ntiles)
            small_tile<Dir>(gshared[g], tile, g, wit, threadIdx.x - g * kGroupThreads, base, lo_b, hi_b, n_units,
                            reinterpret_cast<OutT *>(smem_raw) + g * (Dir::kBufs * kGroupWarps * Dir::kStride), out_a,
                            out_lead, status, err_tile, res, ntiles, sel, lb_sum[g], lb_err[g]);
        return;
    }
    if (role_s == 0) {
        scan_windows<Dir::kScanPerLane>(status, ntiles, warp, scan_s);
        LU_PROF_FLUSH();
        return;
    }
    const uint32_t g = warp / kGroupWarps, wit = warp % kGroupWarps;
    const uint32_t gtid = threadIdx.x - g * kGroupThreads;
    const uint32_t bar_claim = 1 + 3 * g, bar_done = 2 + 3 * g, bar_prefix = 3 + 3 * g;
    GroupShared &ps = gshared[g];
    if (Dir::kHintInSmem) {
        ps.hint_s[wit] = 2; // every lane writes the same value; only this warp reads it
        __syncwarp();
    }
    constexpr uint32_t kBufs = Dir::kBufs;
    OutT *out_g = reinterpret_cast<OutT *>(smem_raw) + g * (kBufs * kGroupWarps * Dir::kStride);

    uint32_t i = 0;
    uint32_t hint = 2; // K1: the warp's class-path prediction (u8_round_detect_spec)
    uint64_t st_pre = 0; // group thread 0: early poll of the next status word to resolve
    uint32_t et_pre = 0; // group thread 0: err_tile as read before the last tile-done barrier
    // group thread 0: the next tile; the ticket is taken right after the
    // tile-done barrier so its latency overlaps the combine + publish
    uint32_t next_claim = 0;
#if LU_CLAIM_AT == 0 || LU_CLAIM_AT == 3
    if (gtid == 0)
        next_claim = atomicAdd(ticket, 1u);
#endif
#if LU_CLAIM_AT == 3
    uint32_t pending_claim = 0;
#endif
    for (;; ++i) {
        const uint32_t buf = i % kBufs;
        // Group thread 0 claims the next tile (atomic in flight) and resolves
        // the buffer about to be reused; one barrier publishes both.  The
        // tile's input loads are then issued before the copy-out of that
        // buffer, so the copy-out hides their latency.
        LU_T0();
        if (gtid == 0) {
#if LU_CLAIM_AT == 2
            next_claim = atomicAdd(ticket, 1u);
#elif LU_CLAIM_AT == 3
            if (i > 0)
                next_claim = pending_claim;
            pending_claim = atomicAdd(ticket, 1u); // consumed one iteration later
#endif
            if (i >= kBufs)
                pipe_resolve<Dir>(ps, buf, status, res, ntiles, lo_b, n_units, st_pre);
            LU_T(12); // resolve
#if LU_CLAIM_AT == 1
            next_claim = atomicAdd(ticket, 1u);
#endif
            ps.claim = next_claim;
            // a tile after one that holds an error is never copied out and its
            // count is never used: skip its work (the reference stops at the
            // first error too).  err_tile: max(ntiles - t) over error tiles t.
            // (et_pre was read before the last tile-done barrier: no extra L2
            // round trip here; a stale value only means less skipping)
            ps.skip = et_pre != 0 && ntiles - et_pre < next_claim;
            LU_T(13); // ticket wait
        }
        LU_T(0); // claim + resolve (warp 0) / nothing
        bar_sync(bar_claim, kGroupThreads); // publishes ps.claim and, for i >= kBufs, ps.excl[buf]
        LU_T(3); // claim barrier wait
        const uint32_t tile = ps.claim;
        const bool skip = ps.skip;
        const int64_t tile_off = (int64_t)tile * kPipeTile;
        const bool interior = (tile_off - 4 >= lo_b) && (tile_off + kPipeTile + 4 <= hi_b);
        typename Dir::In in;
        if (tile < ntiles && !skip) {
            if (interior)
                Dir::template load<false>(base, tile_off, lo_b, hi_b, wit, in);
            else
                Dir::template load<true>(base, tile_off, lo_b, hi_b, wit, in);
        }
        if (i >= kBufs)
            pipe_copy<Dir>(ps, buf, wit, out_g, out_a, out_lead);
        LU_T(2); // copy-out
        // past the end, or behind a known error: stop claiming (the scanner
        // publishes everything behind an error without waiting for it); the
        // drain below still copies out the last computed tile
        if (tile >= ntiles || skip)
            break;
        OutT *out_w = out_g + (buf * kGroupWarps + wit) * Dir::kStride;
        if constexpr (Dir::kHintInSmem) {
            if (interior)
                Dir::template compute<false>(base, tile_off, lo_b, hi_b, out_w, sel, ps.wres[buf][wit], wit, in,
                                             ps.hint_s[wit]);
            else
                Dir::template compute<true>(base, tile_off, lo_b, hi_b, out_w, sel, ps.wres[buf][wit], wit, in,
                                            ps.hint_s[wit]);
        } else {
            if (interior)
                Dir::template compute<false>(base, tile_off, lo_b, hi_b, out_w, sel, ps.wres[buf][wit], wit, in, hint);
            else
                Dir::template compute<true>(base, tile_off, lo_b, hi_b, out_w, sel, ps.wres[buf][wit], wit, in, hint);
        }
        LU_T(4); // compute
        // poll the status word resolved at the top of the next iteration now:
        // its L2 round trip overlaps the other warps' compute
        if (gtid == 0 && i + 1 >= kBufs)
            st_pre = ld_acquire(&status[ps.tile_of[(i + 1) % kBufs]]);
        if (gtid == 0)
            et_pre = *reinterpret_cast<volatile uint32_t *>(err_tile);
        bar_sync(bar_done, kGroupThreads);
        LU_T(5); // tile-done barrier wait
        LU_CNT(6, 1);
        if (wit == 0) {
#if LU_CLAIM_AT == 0
            if (gtid == 0)
                next_claim = atomicAdd(ticket, 1u);
#endif
            group_combine(ps, buf, tile, status, err_tile, ntiles);
        }
        LU_T(7); // combine + publish
    }
    // drain the tiles computed in the last kBufs - 1 iterations, oldest first
    for (uint32_t d = kBufs - 1; d >= 1; --d) {
        if (i >= d) {
            const uint32_t b = (i - d) % kBufs;
            if (gtid == 0)
                pipe_resolve<Dir>(ps, b, status, res, ntiles, lo_b, n_units, 0);
            bar_sync(bar_prefix, kGroupThreads);
            pipe_copy<Dir>(ps, b, wit, out_g, out_a, out_lead);
        }
    }
    LU_PROF_FLUSH();
}

// ================================================================= K3 / K4
//
// Persistent validators fed by a TMA ring.  The input is cut into 32 KiB
// stages (two consecutive 2 KiB chunks per warp); CTA b takes stages b,
// b + grid, ...  Thread 0 keeps kValStages stages in flight per CTA with cp.async.bulk (TMA bulk
// copies, completion counted on an mbarrier per ring slot), each stage copied
// with 16 bytes of look-behind and look-ahead so every warp finds its halo
// quads in shared memory; warps read their chunk with LDS.128.  This keeps
// ~200 KB of loads in flight per SM without prefetch registers (a register
// double buffer cost occupancy; cp.async per warp measured slower).  The first
// and last stages (whose +-16-byte window leaves [lo, hi)) are loaded
// directly with masked loads.
//
// A warp that finds an error publishes atomicMax(n - pos); the CTA stops after
// the stage in which one of its warps found an error, or once a published
// error lies before its next stage (the reference stops at the first error).
// The last warp to finish writes the result record.
// ws layout: [u64 max(n - bad_pos)][u32 warps done][u32 pad][u64 count].

#ifndef LU_LC_CTAS
#define LU_LC_CTAS 3 // resident CTAs per SM the lane-contiguous validator is compiled for
#endif
#ifndef LU_K3_LC
#define LU_K3_LC 1 // UTF-8 validation / length through k_validate8_lc
#endif

constexpr int kValStages = 2;
constexpr int kValCPW = 2;                                   // chunks per warp per stage
constexpr int kStageBytes = kWarps * kValCPW * kChunkBytes; // 32 KiB
constexpr int kStageAlloc = kStageBytes + 32;      // + 16 B halo on each side
constexpr size_t kSmemVal = (size_t)kValStages * kStageAlloc;

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred P;\n\tLU_W%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra LU_W%=;\n\t}" ::"r"(bar),
                 "r"(parity)
                 : "memory");
}

template <bool Utf16, bool Count = false, bool Swap16 = false>
__global__ void __launch_bounds__(kThreads, 3) k_validate_w(const uint8_t *__restrict__ base, uint32_t lead,
                                                            uint64_t n, uint64_t *__restrict__ ws,
                                                            Outcome *__restrict__ res, uint64_t nstages)
{
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ __align__(8) uint64_t bar[kValStages];
    __shared__ WarpResult wr_s[kWarps];
    const uint32_t tid = threadIdx.x;
    const uint32_t warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint64_t total_warps = (uint64_t)gridDim.x * kWarps;
    const uint64_t n_bytes = Utf16 ? 2 * n : n;
    const int64_t lo_b = lead, hi_b = (int64_t)lead + (int64_t)n_bytes;
    auto tma_ok = [&](uint64_t j) {
        const int64_t s0 = (int64_t)j * kStageBytes;
        return s0 - 16 >= lo_b && s0 + kStageBytes + 16 <= hi_b;
    };
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring);
    auto issue = [&](uint64_t j, uint32_t slot) {
        const uint32_t b = bar0 + 8 * slot;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kStageAlloc) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ring0 + slot * kStageAlloc),
                     "l"(base + (int64_t)j * kStageBytes - 16), "r"(kStageAlloc), "r"(b)
                     : "memory");
    };
    if (tid == 0) {
        for (int k = 0; k < kValStages; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * k));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (uint32_t k = 0; k < (uint32_t)kValStages; ++k) {
            const uint64_t j = blockIdx.x + (uint64_t)k * gridDim.x;
            if (j < nstages && tma_ok(j))
                issue(j, k);
        }
    uint32_t hint = 2;    // K3: the warp's class-path prediction (u8_round_detect_spec)
    uint32_t count = 0;   // Count: this lane's output units over the warp's chunks
    uint32_t parity = 0;  // bit k: mbarrier phase of ring slot k
    uint64_t i = 0, j = blockIdx.x;
    for (; j < nstages; ++i, j += gridDim.x) {
        const uint32_t slot = (uint32_t)(i % kValStages);
        const bool fast = tma_ok(j);
        if (fast) {
            mbar_wait(bar0 + 8 * slot, (parity >> slot) & 1);
            parity ^= 1u << slot;
        }
        uint32_t err = 0;
        // the warp's kValCPW consecutive chunks of the stage
#pragma unroll 1
        for (int ci = 0; ci < kValCPW && !err; ++ci) {
            const int64_t off = (int64_t)j * kStageBytes + (int64_t)(warp * kValCPW + ci) * kChunkBytes;
            if (off >= hi_b)
                break;
            ChunkIn in;
            if (fast) {
                const uint8_t *sb = ring + slot * kStageAlloc + 16 + (warp * kValCPW + ci) * kChunkBytes;
#pragma unroll
                for (int r = 0; r < kChunkBytes / 512; ++r) {
                    in.q[r] = *reinterpret_cast<const uint4 *>(sb + r * 512 + 16 * lane);
                    if (Swap16)
                        in.q[r] = make_uint4(swap16x2(in.q[r].x), swap16x2(in.q[r].y), swap16x2(in.q[r].z),
                                             swap16x2(in.q[r].w));
                }
                in.halo_p = *reinterpret_cast<const uint32_t *>(sb - 4);
                in.halo_n = *reinterpret_cast<const uint32_t *>(sb + kChunkBytes);
                if (Swap16) {
                    in.halo_p = swap16x2(in.halo_p);
                    in.halo_n = swap16x2(in.halo_n);
                }
            } else {
                load_chunk<true, Swap16>(base, off, lo_b, hi_b, in);
            }
            uint32_t pos = 0, cc = 0;
            if (Utf16) {
                if (fast)
                    u16val_warp_in<false, Count>(off, lo_b, hi_b, in, err, pos, &cc);
                else
                    u16val_warp_in<true, Count>(off, lo_b, hi_b, in, err, pos, &cc);
            } else {
                if (fast)
                    u8val_warp_in<false, Count>(base, off, lo_b, hi_b, in, wr_s[warp], 0, hint, &cc);
                else
                    u8val_warp_in<true, Count>(base, off, lo_b, hi_b, in, wr_s[warp], 0, hint, &cc);
                __syncwarp();
                err = wr_s[warp].err;
                pos = wr_s[warp].pos;
            }
            count += cc;
            if (err && lane == 0) {
                const int64_t pb = off + pos - lo_b;
                const uint64_t pu = Utf16 ? (uint64_t)(pb >> 1) : (uint64_t)pb;
                atomicMax(reinterpret_cast<unsigned long long *>(ws), (unsigned long long)(n - pu));
            }
        }
        // stop after this stage if an error is known before the next one
        bool stop_me = err != 0;
        if (tid == 0) {
            const uint64_t best = *reinterpret_cast<volatile uint64_t *>(ws);
            const int64_t next0 = (int64_t)(j + gridDim.x) * kStageBytes;
            stop_me |= best != 0 && lo_b + (Utf16 ? 2 : 1) * (int64_t)(n - best) < next0;
        }
        const bool stop = __syncthreads_or(stop_me); // also: every warp is done with the slot
        if (stop)
            break;
        if (tid == 0) {
            const uint64_t jn = j + (uint64_t)kValStages * gridDim.x;
            if (jn < nstages && tma_ok(jn))
                issue(jn, slot);
        }
    }
    // an early stop leaves up to kValStages - 1 stages in flight: let them land
    // before the CTA (and its shared memory) goes away
    if (tid == 0 && j < nstages) {
        for (uint32_t d = 1; d < (uint32_t)kValStages; ++d) {
            const uint64_t jd = j + (uint64_t)d * gridDim.x;
            const uint32_t slot = (uint32_t)((i + d) % kValStages);
            if (jd < nstages && tma_ok(jd)) {
                mbar_wait(bar0 + 8 * slot, (parity >> slot) & 1);
                parity ^= 1u << slot;
            }
        }
    }
    if (Count) {
        const uint32_t wsum = __reduce_add_sync(0xffffffffu, count);
        if (lane == 0 && wsum)
            atomicAdd(reinterpret_cast<unsigned long long *>(ws + 2), (unsigned long long)wsum);
    }
    if (lane == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(reinterpret_cast<unsigned int *>(ws + 1), 1u);
        if (prev == total_warps - 1) {
            __threadfence();
            const uint64_t b = atomicAdd(reinterpret_cast<unsigned long long *>(ws), 0ull);
            res->status = b ? kStatusMalformed : kStatusOk;
            res->pad = 0;
            res->consumed = n - b;
            res->written = (Count && !b) ? atomicAdd(reinterpret_cast<unsigned long long *>(ws + 2), 0ull) : 0;
        }
    }
}

// ============================================== K3 (lane-contiguous layout)
//
// validate_utf8 / utf16_length_from_utf8 with the lane-contiguous detectors of
// lu_utf8_lc.cuh.  No CTA-wide step: every warp owns a private ring of
// kLcSlots slots (one 2 KiB chunk plus 16 bytes of look-behind / look-ahead
// each) that its lane 0 keeps filled with TMA bulk copies (one mbarrier per
// slot); warp g of G takes chunks g, g + G, ...  Lane l reads its 64 bytes
// with four LDS.128 and runs the detector of the warp's predicted class over
// its 16 quads in a straight line; one vote per chunk.  A miss falls to the
// exact general detector on the same registers; only a chunk that detector
// flags (a real error) or a chunk at the ends of the input goes through the
// round-layout code (u8val_warp_in), which owns the error offsets.
// ws layout and result protocol as k_validate_w.

#ifndef LU_LC_SUB
#define LU_LC_SUB 2 // chunks per ring slot (one TMA bulk copy, one stop check, one refill per slot)
#endif
#ifndef LU_LC_SLOTS
#define LU_LC_SLOTS 2
#endif
constexpr int kLcSub = LU_LC_SUB;
constexpr int kLcSlots = LU_LC_SLOTS;
constexpr int kLcHalo = 16;
constexpr int kLcSuper = kLcSub * kChunkBytes;           // input bytes per slot
constexpr int kLcSlotBytes = kLcSuper + 2 * kLcHalo;
constexpr size_t kSmemLc = (size_t)kWarps * kLcSlots * kLcSlotBytes;

__device__ __forceinline__ uint4 lds128(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Round-layout fallback for one chunk: from the ring slot (sa = shared address
// of the chunk's first byte) when the chunk is interior, else masked global
// loads.  Out of line: it is rare and must not shape the fast path's registers.
// Returns the new class hint << 32 | this lane's share of the chunk's count.
template <bool Count>
__device__ __noinline__ uint64_t lc_slow_chunk(const uint8_t *__restrict__ base, int64_t off, int64_t lo_b,
                                               int64_t hi_b, uint32_t sa, bool interior, WarpResult *wr, uint32_t hint)
{
    const uint32_t lane = lane_id();
    ChunkIn in;
    uint32_t c = 0;
    if (interior) {
#pragma unroll
        for (int r = 0; r < kChunkBytes / 512; ++r)
            in.q[r] = lds128(sa + r * 512 + 16 * lane);
        in.halo_p = lds32(sa - 4);
        in.halo_n = lds32(sa + kChunkBytes);
        u8val_warp_in<false, Count>(base, off, lo_b, hi_b, in, *wr, 0, hint, &c);
    } else {
        load_chunk<true>(base, off, lo_b, hi_b, in);
        u8val_warp_in<true, Count>(base, off, lo_b, hi_b, in, *wr, 0, hint, &c);
    }
    return ((uint64_t)hint << 32) | c;
}

// Lane l's 64 bytes of the chunk at shared address sa, plus the quads before /
// after them (previous / next lane, or the slot's halo for lanes 0 / 31).
__device__ __forceinline__ void lc_load(uint32_t sa, uint32_t lane, uint32_t (&x)[kLcQuads], uint32_t &xp,
                                        uint32_t &xn)
{
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 v = lds128(sa + 64 * lane + 16 * j);
        x[4 * j] = v.x;
        x[4 * j + 1] = v.y;
        x[4 * j + 2] = v.z;
        x[4 * j + 3] = v.w;
    }
    const uint32_t hp = lds32(sa - 4), hn = lds32(sa + kChunkBytes);
    xp = __shfl_up_sync(0xffffffffu, x[kLcQuads - 1], 1);
    xn = __shfl_down_sync(0xffffffffu, x[0], 1);
    xp = lane == 0 ? hp : xp;
    xn = lane == 31 ? hn : xn;
}

template <bool Count>
__global__ void __launch_bounds__(kThreads, LU_LC_CTAS) k_validate8_lc(const uint8_t *__restrict__ base, uint32_t lead,
                                                                       uint64_t n, uint64_t *__restrict__ ws,
                                                                       Outcome *__restrict__ res, uint32_t nsuper)
{
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ __align__(8) uint64_t bar[kWarps * kLcSlots];
    __shared__ WarpResult wr_s[kWarps];
    __shared__ __align__(16) uint64_t best_s[2]; // the CTA's copy of the ws header's first 16 bytes
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const uint32_t total_warps = gridDim.x * kWarps;
    const uint32_t gw = blockIdx.x * kWarps + warp;
    const uint32_t best_a = (uint32_t)__cvta_generic_to_shared(&best_s[0]);
    const int64_t lo_b = lead, hi_b = (int64_t)lead + (int64_t)n;
    // slots (kLcSub consecutive chunks) whose +-16-byte window lies inside
    // [lo, hi) come through the ring: [1, s_hi) (lead < 16: slot 0 never does)
    const uint32_t s_hi = hi_b >= kLcSuper + kLcHalo ? (uint32_t)((hi_b - kLcHalo) / kLcSuper) : 0u;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bar[warp * kLcSlots]);
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring) + warp * (kLcSlots * kLcSlotBytes);
    auto issue = [&](uint32_t sc, uint32_t slot) {
        const uint32_t b = bar0 + 8 * slot;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kLcSlotBytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ring0 + slot * kLcSlotBytes),
                     "l"(base + (int64_t)sc * kLcSuper - kLcHalo), "r"(kLcSlotBytes), "r"(b)
                     : "memory");
    };
    if (threadIdx.x == 0)
        best_s[0] = 0;
    if (lane == 0) {
        for (int k = 0; k < kLcSlots; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * k));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (lane == 0)
        for (uint32_t k = 0; k < (uint32_t)kLcSlots; ++k) {
            const uint32_t sc = gw + k * total_warps;
            if (sc >= 1 && sc < s_hi)
                issue(sc, k);
        }
    uint32_t hint = 2;   // the warp's class prediction (0, 1, 3; 2 = general)
    uint32_t units = 0;  // Count: this lane's output units over the warp's chunks
    uint32_t parity = 0; // bit k: mbarrier phase of ring slot k
    uint32_t slot = 0;
    uint32_t sc = gw;
    bool stopped = false;
    for (; sc < nsuper; sc += total_warps) {
        const bool fast = sc >= 1 && sc < s_hi;
        // Published first-error position: warp 0 of the CTA refreshes a copy in
        // shared memory every iteration (cp.async: no register held across the
        // chunks; .cg: through L2 -- an L1-cached copy would never see another
        // SM's update); every warp reads that copy after its chunks.  One
        // poller per CTA: every warp polling the same L2 line cost K3 9%.
        if (warp == 0 && lane == 0)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;" ::"r"(best_a), "l"(ws)
                         : "memory");
        const uint32_t sa0 = ring0 + slot * kLcSlotBytes + kLcHalo;
        if (fast) {
            mbar_wait(bar0 + 8 * slot, (parity >> slot) & 1);
            parity ^= 1u << slot;
        }
        uint32_t err = 0;
#pragma unroll 1
        for (int h = 0; h < kLcSub; ++h) {
            const int64_t off = (int64_t)sc * kLcSuper + h * kChunkBytes;
            if (off >= hi_b)
                break;
            const uint32_t sa = sa0 + h * kChunkBytes;
            bool slow = !fast;
            if (fast) {
                uint32_t x[kLcQuads], xp, xn;
                lc_load(sa, lane, x, xp, xn);
                uint32_t fd = 1, c_nc = 0, c_nf = 0;
                if (hint == 0)
                    fd = lc_detect<0, Count>(x, xp, xn, c_nc, c_nf);
                else if (hint == 1)
                    fd = lc_detect<1, Count>(x, xp, xn, c_nc, c_nf);
                else if (hint == 3)
                    fd = lc_detect<3, Count>(x, xp, xn, c_nc, c_nf);
                else if (hint == (uint32_t)kLcBmp)
                    fd = lc_detect<kLcBmp, Count>(x, xp, xn, c_nc, c_nf);
                if (__any_sync(0xffffffffu, fd != 0)) {
                    // class miss: the exact general detector on the same registers
                    uint32_t cls = 0;
                    c_nc = 0;
                    c_nf = 0;
                    fd = lc_detect_general<Count>(x, xp, xn, c_nc, c_nf, cls);
                    hint = lc_path_of(__reduce_or_sync(0xffffffffu, cls));
                    slow = __any_sync(0xffffffffu, fd != 0);
                }
                // 64 bytes per lane minus continuations plus 4-byte leads
                if (Count && !slow)
                    units += 64u - (c_nc >> 7) + (c_nf >> 7);
            }
            if (slow) {
                const uint64_t hc = lc_slow_chunk<Count>(base, off, lo_b, hi_b, sa, fast, &wr_s[warp], hint);
                hint = (uint32_t)(hc >> 32);
                __syncwarp();
                err = wr_s[warp].err;
                const uint32_t pos = wr_s[warp].pos;
                __syncwarp();
                if (Count)
                    units += (uint32_t)hc; // this lane's share of the chunk's count (u8val_warp_in)
                if (err) {
                    if (lane == 0) {
                        const uint64_t pu = (uint64_t)(off + pos - lo_b);
                        atomicMax(reinterpret_cast<unsigned long long *>(ws), (unsigned long long)(n - pu));
                    }
                    break;
                }
            }
        }
        __syncwarp(); // every lane is done with the slot
        // stop once an error is known before this warp's next slot
        uint32_t stop = err;
        if (lane == 0) {
            if (warp == 0)
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            uint64_t best;
            asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(best) : "r"(best_a) : "memory");
            if (best != 0)
                stop |= (uint64_t)(hi_b - (int64_t)best) < (uint64_t)(sc + total_warps) * kLcSuper ? 1u : 0u;
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) {
            stopped = true;
            break;
        }
        if (lane == 0) {
            const uint32_t sn = sc + kLcSlots * total_warps;
            if (sn < s_hi && sn >= 1)
                issue(sn, slot);
        }
        slot = slot == kLcSlots - 1 ? 0u : slot + 1;
    }
    // an early stop leaves up to kLcSlots - 1 slots in flight: let them land
    // before the CTA (and its shared memory) goes away
    if (stopped) {
        for (uint32_t d = 1; d < (uint32_t)kLcSlots; ++d) {
            const uint64_t sd = (uint64_t)sc + (uint64_t)d * total_warps;
            slot = slot == kLcSlots - 1 ? 0u : slot + 1;
            if (sd >= 1 && sd < s_hi) {
                mbar_wait(bar0 + 8 * slot, (parity >> slot) & 1);
                parity ^= 1u << slot;
            }
        }
    }
    if (Count) {
        const uint32_t wsum = __reduce_add_sync(0xffffffffu, units);
        if (lane == 0 && wsum)
            atomicAdd(reinterpret_cast<unsigned long long *>(ws + 2), (unsigned long long)wsum);
    }
    if (lane == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(reinterpret_cast<unsigned int *>(ws + 1), 1u);
        if (prev == total_warps - 1) {
            __threadfence();
            const uint64_t b = atomicAdd(reinterpret_cast<unsigned long long *>(ws), 0ull);
            res->status = b ? kStatusMalformed : kStatusOk;
            res->pad = 0;
            res->consumed = n - b;
            res->written = (Count && !b) ? atomicAdd(reinterpret_cast<unsigned long long *>(ws + 2), 0ull) : 0;
        }
    }
}

// ================================================================== batched
//
// Many small independent cases in one launch (the reference's differential
// campaign and byte-triple sweep, difftest.py:90-104): case i is
// units [offs[i], offs[i+1]) of one buffer.  One warp per case walks the
// case's 2 KiB chunks in order through the same warp bodies as K1-K4
// (boundary variants, the case bounds as [lo, hi)), carrying its running
// output count -- no cross-warp ordering, no scanner.  Case i's output goes to
// its worst-case slot (word offs[i] for UTF-8 -> UTF-16, byte 3 * offs[i] for
// UTF-16 -> UTF-8); res[i] is its own lu_outcome.
// Op: 0 utf8 -> utf16le, 1 utf16le -> utf8, 2 validate utf8, 3 validate utf16le.
template <int Op>
__global__ void __launch_bounds__(kThreads) k_batch(const uint8_t *__restrict__ base, uint32_t lead,
                                                    const uint64_t *__restrict__ offs, uint32_t ncases,
                                                    void *__restrict__ out_a, uint32_t out_lead,
                                                    Outcome *__restrict__ res)
{
    constexpr bool kUtf16 = (Op == 1 || Op == 3);
    constexpr int kShift = kUtf16 ? 1 : 0;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ SelPair sel[56];
    __shared__ WarpResult wres[kWarps];
    sel_table_init(sel);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const uint32_t total_warps = gridDim.x * kWarps;
    for (uint32_t c = blockIdx.x * kWarps + warp; c < ncases; c += total_warps) {
        const uint64_t u0 = offs[c], u1 = offs[c + 1];
        const int64_t lo_b = (int64_t)lead + ((int64_t)u0 << kShift);
        const int64_t hi_b = (int64_t)lead + ((int64_t)u1 << kShift);
        uint64_t running = 0, consumed = u1 - u0;
        uint32_t hint = 2;
        uint32_t status = kStatusOk;
        for (int64_t chunk = lo_b & ~(int64_t)15; chunk < hi_b; chunk += kChunkBytes) {
            uint32_t err, pos, units = 0;
            if (Op == 0 || Op == 1) {
                ChunkIn in;
                load_chunk<true>(base, chunk, lo_b, hi_b, in);
                if (Op == 0) {
                    uint16_t *stage = reinterpret_cast<uint16_t *>(smem_raw) + warp * kOutStrideU16;
                    u8u16_warp<true>(base, chunk, lo_b, hi_b, stage, sel, wres[warp], 0, in, hint);
                    __syncwarp();
                    units = wres[warp].units;
                    copy_out_u16(stage, units, reinterpret_cast<uint16_t *>(out_a), out_lead + u0 + running);
                } else {
                    uint8_t *stage = smem_raw + warp * kOutStrideU8;
                    u16u8_warp_r<true>(base, chunk, lo_b, hi_b, stage, sel + 16, wres[warp], 0, in);
                    __syncwarp();
                    units = wres[warp].units;
                    copy_out_u8(stage, units, reinterpret_cast<uint8_t *>(out_a), out_lead + 3 * u0 + running);
                }
                err = wres[warp].err;
                pos = wres[warp].pos;
            } else if (Op == 2) {
                {
                    ChunkIn in;
                    load_chunk<true>(base, chunk, lo_b, hi_b, in);
                    u8val_warp_in<true>(base, chunk, lo_b, hi_b, in, wres[warp], 0, hint);
                }
                __syncwarp();
                err = wres[warp].err;
                pos = wres[warp].pos;
            } else {
                u16val_warp_r<true>(base, chunk, lo_b, hi_b, err, pos);
            }
            __syncwarp(); // the staging region / result slot is reused next chunk
            running += units;
            if (err) {
                status = kStatusMalformed;
                consumed = (uint64_t)((chunk + pos - lo_b) >> kShift);
                break;
            }
        }
        if (lane == 0) {
            res[c].status = status;
            res[c].pad = 0;
            res[c].consumed = consumed;
            res[c].written = running;
        }
    }
}

// ============================================================ char counts
//
// utf8_char_count / utf16le_char_count (scalar.py:246-257): bytes that are
// not continuations, or words minus low surrogates.  No validation.  A plain
// HBM-bound reduction: 16 bytes per thread per step, one atomic per warp.
// ws layout: [u64 sum][u32 warps done][u32 pad].
#ifndef LU_CHARS_UNROLL
#define LU_CHARS_UNROLL 8
#endif
constexpr int kCharsUnroll = LU_CHARS_UNROLL; // 16-byte loads in flight per thread

template <bool Utf16>
__global__ void __launch_bounds__(kThreads) k_chars(const uint8_t *__restrict__ base, uint32_t lead, uint64_t n,
                                                    uint64_t *__restrict__ ws, uint64_t *__restrict__ out,
                                                    uint64_t nvec)
{
    const int64_t lo_b = lead, hi_b = (int64_t)lead + (int64_t)(Utf16 ? 2 * n : n);
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    uint64_t acc = 0;
    uint64_t v = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    // full vectors [vf0, vf1): kCharsUnroll independent 16-byte loads in flight per
    // thread (64 B/thread reads ~7 TB/s where 16 B/thread stops at ~4.8,
    // tools/probe/read_probe.cu); the ends go through the masked loop below
    const uint64_t vf0 = (uint64_t)(lo_b + 15) / 16, vf1 = (uint64_t)hi_b / 16;
    if (v >= vf0) {
        for (; v + (kCharsUnroll - 1) * stride < vf1; v += kCharsUnroll * stride) {
            uint4 q[kCharsUnroll];
#pragma unroll
            for (int j = 0; j < kCharsUnroll; ++j)
                q[j] = __ldcs(reinterpret_cast<const uint4 *>(base + (int64_t)(v + j * stride) * 16));
            // 128 x (continuation bytes | low surrogates) by dp4a, no POPC
            uint32_t c = 0;
#pragma unroll
            for (int j = 0; j < kCharsUnroll; ++j) {
                if (Utf16) {
                    // high bytes of the vector's 8 words, 4 per register (as K4)
                    uint32_t nhs, ls;
                    u16_sur4(hi_bytes(q[j].x, q[j].y), nhs, ls);
                    c = __dp4a(ls & H8, 0x01010101u, c);
                    u16_sur4(hi_bytes(q[j].z, q[j].w), nhs, ls);
                    c = __dp4a(ls & H8, 0x01010101u, c);
                } else {
                    const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        c = __dp4a(w4[k] & ~(w4[k] << 1) & H8, 0x01010101u, c);
                }
            }
            // u8: count the bytes that are NOT continuations; u16: the low surrogates
            acc += Utf16 ? (c >> 7) : 16u * kCharsUnroll - (c >> 7);
        }
    }
    for (; v < nvec; v += stride) {
        const int64_t a = (int64_t)v * 16;
        const bool full = a >= lo_b && a + 16 <= hi_b;
        const uint4 q =
            full ? __ldcs(reinterpret_cast<const uint4 *>(base + a)) : load_u128_masked(base, a, lo_b, hi_b);
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = w4[k];
            if (Utf16) {
                uint32_t hs, ls;
                u16_sur_masks(x, hs, ls);
                if (!full) {
                    const uint32_t vw = valid_words(a + 4 * k, lo_b, hi_b);
                    ls &= ((vw & 1) ? 0x8000u : 0u) | ((vw & 2) ? 0x80000000u : 0u);
                }
                c += __popc(ls);
            } else {
                uint32_t nc = ~(x & ~(x << 1)) & H8; // not a continuation byte
                if (!full)
                    nc &= valid_mask(a + 4 * k, lo_b, hi_b);
                c += __popc(nc);
            }
        }
        acc += c;
    }
    const uint32_t lane = lane_id();
    unsigned long long wsum = acc;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1)
        wsum += __shfl_down_sync(0xffffffffu, wsum, d);
    if (lane == 0) {
        if (wsum)
            atomicAdd(reinterpret_cast<unsigned long long *>(ws), wsum);
        __threadfence();
        const unsigned int prev = atomicAdd(reinterpret_cast<unsigned int *>(ws + 1), 1u);
        if (prev == (uint64_t)gridDim.x * kWarps - 1) {
            __threadfence();
            const uint64_t t = atomicAdd(reinterpret_cast<unsigned long long *>(ws), 0ull);
            *out = Utf16 ? n - t : t;
        }
    }
}

// =============================================================== host side

static thread_local std::string g_err;

static int fail(int code, const char *msg)
{
    g_err = msg;
    return code;
}

static int cuda_fail(cudaError_t e, const char *what)
{
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return LU_ERR_CUDA;
}

static uint64_t n_tiles(uint64_t bytes, uint32_t lead, uint64_t tile = kTileBytes)
{
    uint64_t t = (bytes + lead + tile - 1) / tile;
    return t ? t : 1;
}

// cudaFuncSetAttribute is per device: remember, per device, which kernels
// already have their dynamic shared memory limit raised (a process may drive
// several GPUs).  Bit k of g_attr_done[dev] = attribute group k is set.
static std::mutex g_attr_mu;
static uint64_t g_attr_done[64];

static int ensure_smem_attr(int group, const void *const *fns, const int *bytes, int nfns)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= 64)
        return fail(LU_ERR_INVALID, "device index out of range");
    std::lock_guard<std::mutex> lock(g_attr_mu);
    if (g_attr_done[dev] & (1ull << group))
        return 0;
    for (int k = 0; k < nfns; ++k) {
        e = cudaFuncSetAttribute(fns[k], cudaFuncAttributeMaxDynamicSharedMemorySize, bytes[k]);
        if (e != cudaSuccess)
            return cuda_fail(e, "cudaFuncSetAttribute");
    }
    g_attr_done[dev] |= 1ull << group;
    return 0;
}

static int set_smem_attrs()
{
    const void *fns[4] = {(const void *)k_transcode<DirU8U16>, (const void *)k_transcode<DirU16U8>,
                          (const void *)k_transcode<DirU8U16T<true>>, (const void *)k_transcode<DirU16U8T<true>>};
    const int bytes[4] = {(int)kSmemK1, (int)kSmemK2, (int)kSmemK1, (int)kSmemK2};
    return ensure_smem_attr(0, fns, bytes, 4);
}

// Grid of a persistent pipelined kernel: every CTA must be resident (tiles
// wait on smaller tiles held by other CTAs), so never exceed the occupancy.
// Resident capacity (SMs x CTAs per SM) of a kernel configuration, cached per
// device: the occupancy query costs several microseconds of host time per
// call, which dominated small calls (config 1).
struct CapEntry {
    int dev;
    const void *fn;
    int threads;
    size_t smem;
    uint64_t cap;
};
static std::mutex g_cap_mu;
static CapEntry g_cap[64];
static int g_ncap = 0;

static int resident_capacity(const void *fn, int threads, size_t smem, uint64_t *cap)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaGetDevice");
    {
        std::lock_guard<std::mutex> lock(g_cap_mu);
        for (int k = 0; k < g_ncap; ++k)
            if (g_cap[k].dev == dev && g_cap[k].fn == fn && g_cap[k].threads == threads && g_cap[k].smem == smem) {
                *cap = g_cap[k].cap;
                return 0;
            }
    }
    int sms = 0, per_sm = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    if (e != cudaSuccess)
        return cuda_fail(e, "occupancy query");
    *cap = (uint64_t)sms * (uint64_t)per_sm;
    std::lock_guard<std::mutex> lock(g_cap_mu);
    if (g_ncap < 64)
        g_cap[g_ncap++] = CapEntry{dev, fn, threads, smem, *cap};
    return 0;
}

// Grid of a persistent kernel: never more CTAs than are resident at once.
static int persistent_grid(const void *fn, int threads, size_t smem, uint64_t ntiles, unsigned *grid,
                           unsigned extra = 0)
{
    uint64_t cap = 0;
    if (int rc = resident_capacity(fn, threads, smem, &cap))
        return rc;
    if (cap < 1 + extra)
        return fail(LU_ERR_CUDA, "persistent kernel cannot be resident on this device");
    // extra: CTAs that process no tiles (the transcode kernels' scanner CTA)
    *grid = (unsigned)(ntiles + extra < cap ? ntiles + extra : cap);
    return 0;
}

} // namespace lu

using namespace lu;

template <bool Count>
static int launch_validate8_lc(const uint8_t *base, uint32_t lead, uint64_t n_units, void *ws, lu_outcome *res,
                               uint64_t nbytes_frame, cudaStream_t stream)
{
    const void *fn = (const void *)k_validate8_lc<Count>;
    const int sb = (int)kSmemLc;
    if (int rc = ensure_smem_attr(24 + Count, &fn, &sb, 1))
        return rc;
    const uint64_t nsuper = (nbytes_frame + kLcSuper - 1) / kLcSuper;
    if (nsuper > 0x3fffffffull) // 32-bit slot indices (with head room for sc + slots * warps)
        return fail(LU_ERR_INVALID, "input too large");
    const uint64_t nblocks = (nsuper + kWarps - 1) / kWarps;
    unsigned grid = 0;
    // at least one CTA: its last warp writes the result (also for empty input)
    int rc = persistent_grid(fn, kThreads, kSmemLc, nblocks ? nblocks : 1, &grid);
    if (rc)
        return rc;
    k_validate8_lc<Count><<<grid, kThreads, kSmemLc, stream>>>(base, lead, n_units, reinterpret_cast<uint64_t *>(ws),
                                                               reinterpret_cast<Outcome *>(res), (uint32_t)nsuper);
    return 0;
}

template <bool Utf16, bool Count, bool Swap16 = false>
static int launch_validate(const uint8_t *base, uint32_t lead, uint64_t n_units, void *ws, lu_outcome *res,
                           uint64_t nbytes_frame, cudaStream_t stream)
{
    const void *fn = (const void *)k_validate_w<Utf16, Count, Swap16>;
    const int sb = (int)kSmemVal;
    if (int rc = ensure_smem_attr(8 + 4 * Utf16 + 2 * Count + Swap16, &fn, &sb, 1))
        return rc;
    const uint64_t nstages = (nbytes_frame + kStageBytes - 1) / kStageBytes;
    unsigned grid = 0;
    // at least one CTA: its last warp writes the result (also for empty input)
    int rc = persistent_grid(fn, kThreads, kSmemVal, nstages ? nstages : 1, &grid);
    if (rc)
        return rc;
    k_validate_w<Utf16, Count, Swap16><<<grid, kThreads, kSmemVal, stream>>>(
        base, lead, n_units, reinterpret_cast<uint64_t *>(ws), reinterpret_cast<Outcome *>(res), nstages);
    return 0;
}

// Validators (count = false) and the validate+count length functions.
static int validate_impl(bool utf16, bool count, const uint8_t *inb, uint64_t n_units, void *ws, uint64_t ws_bytes,
                         lu_outcome *res, cudaStream_t stream, bool be = false)
{
    if ((!inb && n_units) || !res || !ws)
        return fail(LU_ERR_INVALID, "null pointer");
    if ((utf16 && ((uintptr_t)inb & 1)) || ((uintptr_t)ws & 7) || ((uintptr_t)res & 7))
        return fail(LU_ERR_INVALID, "misaligned in/ws/res pointer");
    // the kernels' 24-byte header starts at the first 16-byte boundary of ws
    // (k_validate8_lc fetches it with a 16-byte cp.async)
    const uint64_t ws_skip = (16 - ((uintptr_t)ws & 15)) & 15;
    if (ws_bytes < 24 + ws_skip)
        return fail(LU_ERR_WORKSPACE, "workspace too small (see lu_workspace_bytes)");
    ws = reinterpret_cast<uint8_t *>(ws) + ws_skip;
    const uint32_t lead = (uint32_t)((uintptr_t)inb & 15);
    const uint64_t nt = n_tiles(utf16 ? 2 * n_units : n_units, lead);
    if (nt > 0x7fffffffull)
        return fail(LU_ERR_INVALID, "input too large");
    cudaError_t e = cudaMemsetAsync(ws, 0, 24, stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync");
    const uint8_t *base = inb ? inb - lead : reinterpret_cast<const uint8_t *>(16);
    const uint64_t frame = lead + (utf16 ? 2 * n_units : n_units);
    int rc;
    if (utf16 && be)
        rc = launch_validate<true, false, true>(base, lead, n_units, ws, res, frame, stream);
    else if (utf16)
        rc = count ? launch_validate<true, true>(base, lead, n_units, ws, res, frame, stream)
                   : launch_validate<true, false>(base, lead, n_units, ws, res, frame, stream);
    else if (LU_K3_LC)
        rc = count ? launch_validate8_lc<true>(base, lead, n_units, ws, res, frame, stream)
                   : launch_validate8_lc<false>(base, lead, n_units, ws, res, frame, stream);
    else
        rc = count ? launch_validate<false, true>(base, lead, n_units, ws, res, frame, stream)
                   : launch_validate<false, false>(base, lead, n_units, ws, res, frame, stream);
    if (rc)
        return rc;
    e = cudaGetLastError();
    if (e != cudaSuccess)
        return cuda_fail(e, "k_validate launch");
    return 0;
}

static int chars_impl(bool utf16, const uint8_t *inb, uint64_t n_units, void *ws, uint64_t ws_bytes, uint64_t *count,
                      cudaStream_t stream)
{
    if ((!inb && n_units) || !count || !ws)
        return fail(LU_ERR_INVALID, "null pointer");
    if ((utf16 && ((uintptr_t)inb & 1)) || ((uintptr_t)ws & 7) || ((uintptr_t)count & 7))
        return fail(LU_ERR_INVALID, "misaligned in/ws/count pointer");
    if (ws_bytes < 16)
        return fail(LU_ERR_WORKSPACE, "workspace too small (see lu_workspace_bytes)");
    const uint32_t lead = (uint32_t)((uintptr_t)inb & 15);
    const uint64_t nbytes = utf16 ? 2 * n_units : n_units;
    cudaError_t e = cudaMemsetAsync(ws, 0, 16, stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync");
    const uint8_t *base = inb ? inb - lead : reinterpret_cast<const uint8_t *>(16);
    const uint64_t nvec = (lead + nbytes + 15) / 16;
    unsigned grid = 0;
    const void *fn = utf16 ? (const void *)k_chars<true> : (const void *)k_chars<false>;
    // at least one CTA: its last warp writes the result (0 for empty input)
    int rc = persistent_grid(fn, kThreads, 0, nvec ? (nvec + kThreads - 1) / kThreads : 1, &grid);
    if (rc)
        return rc;
    if (utf16)
        k_chars<true><<<grid, kThreads, 0, stream>>>(base, lead, n_units, reinterpret_cast<uint64_t *>(ws), count,
                                                     nvec);
    else
        k_chars<false><<<grid, kThreads, 0, stream>>>(base, lead, n_units, reinterpret_cast<uint64_t *>(ws), count,
                                                      nvec);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        return cuda_fail(e, "k_chars launch");
    return 0;
}

template <class Dir>
static int u8u16_impl(const uint8_t *in, uint64_t n_bytes, uint16_t *out, uint64_t out_cap_words, void *ws,
                      uint64_t ws_bytes, lu_outcome *res, cudaStream_t stream)
{
    if ((!in && n_bytes) || !res || !ws)
        return fail(LU_ERR_INVALID, "null pointer");
    if (((uintptr_t)out & 1) || ((uintptr_t)ws & 7) || ((uintptr_t)res & 7))
        return fail(LU_ERR_INVALID, "misaligned out/ws/res pointer");
    if (out_cap_words < n_bytes)
        return fail(LU_ERR_CAPACITY, "output capacity below the worst case (1 word per input byte)");
    if (!out && n_bytes)
        return fail(LU_ERR_INVALID, "null output");
    const uint32_t lead = (uint32_t)((uintptr_t)in & 15);
    const uint64_t nt = n_tiles(n_bytes, lead, kPipeTile);
    if (ws_bytes < 8 * (nt + 2)) // tile status words + ticket / error-tile / role counters
        return fail(LU_ERR_WORKSPACE, "workspace too small (see lu_workspace_bytes)");
    if (nt > 0x7fffffffull)
        return fail(LU_ERR_INVALID, "input too large");
    int rc = set_smem_attrs();
    if (rc)
        return rc;
    cudaError_t e = cudaMemsetAsync(ws, 0, 8 * (nt + 2), stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync");
    const uint8_t *base = in ? in - lead : reinterpret_cast<const uint8_t *>(16);
    uint16_t *out_safe = out ? out : reinterpret_cast<uint16_t *>(16);
    const uint32_t out_lead = (uint32_t)(((uintptr_t)out_safe & 15) >> 1);
    uint16_t *out_a = out_safe - out_lead;
    unsigned grid = 0;
    uint64_t cap = 0;
    rc = resident_capacity((const void *)k_transcode<Dir>, kPipeThreads, kSmemK1, &cap);
    if (rc)
        return rc;
    const uint32_t small = nt <= kGroupsPerCta * cap ? 1u : 0u; // one tile per group: no scanner
    grid = small ? (unsigned)((nt + kGroupsPerCta - 1) / kGroupsPerCta) : (unsigned)(nt + 1 < cap ? nt + 1 : cap);
    if (!small && cap < 2)
        return fail(LU_ERR_CUDA, "persistent kernel cannot be resident on this device");
    k_transcode<Dir><<<grid, kPipeThreads, kSmemK1, stream>>>(base, lead, n_bytes, n_bytes, out_a, out_lead,
                                                                   reinterpret_cast<uint64_t *>(ws),
                                                                   reinterpret_cast<Outcome *>(res), (uint32_t)nt,
                                                                   small);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        return cuda_fail(e, "k_utf8_to_utf16le launch");
    return 0;
}

template <class Dir>
static int u16u8_impl(const uint16_t *in, uint64_t n_words, uint8_t *out, uint64_t out_cap_bytes, void *ws,
                      uint64_t ws_bytes, lu_outcome *res, cudaStream_t stream)
{
    if ((!in && n_words) || !res || !ws)
        return fail(LU_ERR_INVALID, "null pointer");
    if (((uintptr_t)in & 1) || ((uintptr_t)ws & 7) || ((uintptr_t)res & 7))
        return fail(LU_ERR_INVALID, "misaligned in/ws/res pointer");
    if (out_cap_bytes < 3 * n_words)
        return fail(LU_ERR_CAPACITY, "output capacity below the worst case (3 bytes per input word)");
    if (!out && n_words)
        return fail(LU_ERR_INVALID, "null output");
    const uint8_t *inb = reinterpret_cast<const uint8_t *>(in);
    const uint32_t lead = (uint32_t)((uintptr_t)inb & 15);
    const uint64_t nt = n_tiles(2 * n_words, lead, kPipeTile);
    if (ws_bytes < 8 * (nt + 2)) // tile status words + ticket / error-tile / role counters
        return fail(LU_ERR_WORKSPACE, "workspace too small (see lu_workspace_bytes)");
    if (nt > 0x7fffffffull)
        return fail(LU_ERR_INVALID, "input too large");
    int rc = set_smem_attrs();
    if (rc)
        return rc;
    cudaError_t e = cudaMemsetAsync(ws, 0, 8 * (nt + 2), stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync");
    const uint8_t *base = inb ? inb - lead : reinterpret_cast<const uint8_t *>(16);
    uint8_t *out_safe = out ? out : reinterpret_cast<uint8_t *>(16);
    const uint32_t out_lead = (uint32_t)((uintptr_t)out_safe & 15);
    unsigned grid = 0;
    uint64_t cap = 0;
    rc = resident_capacity((const void *)k_transcode<Dir>, kPipeThreads, kSmemK2, &cap);
    if (rc)
        return rc;
    const uint32_t small = nt <= kGroupsPerCta * cap ? 1u : 0u; // one tile per group: no scanner
    grid = small ? (unsigned)((nt + kGroupsPerCta - 1) / kGroupsPerCta) : (unsigned)(nt + 1 < cap ? nt + 1 : cap);
    if (!small && cap < 2)
        return fail(LU_ERR_CUDA, "persistent kernel cannot be resident on this device");
    k_transcode<Dir><<<grid, kPipeThreads, kSmemK2, stream>>>(
        base, lead, n_words, 2 * n_words, out_safe - out_lead, out_lead, reinterpret_cast<uint64_t *>(ws),
        reinterpret_cast<Outcome *>(res), (uint32_t)nt, small);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        return cuda_fail(e, "k_utf16le_to_utf8 launch");
    return 0;
}

template <int Op>
static int batch_impl(const uint8_t *inb, const uint64_t *offs, uint32_t ncases, void *out, lu_outcome *res,
                      cudaStream_t stream)
{
    constexpr bool kUtf16 = (Op == 1 || Op == 3);
    if (!offs || (!res && ncases))
        return fail(LU_ERR_INVALID, "null pointer");
    if ((kUtf16 && ((uintptr_t)inb & 1)) || ((uintptr_t)offs & 7) || ((uintptr_t)res & 7) ||
        (Op == 0 && ((uintptr_t)out & 1)))
        return fail(LU_ERR_INVALID, "misaligned pointer");
    if ((Op == 0 || Op == 1) && !out && ncases)
        return fail(LU_ERR_INVALID, "null output");
    if (ncases == 0)
        return 0;
    const size_t smem = Op == 0 ? sizeof(uint16_t) * kOutStrideU16 * kWarps : (Op == 1 ? kOutStrideU8 * kWarps : 0);
    const void *fn = (const void *)k_batch<Op>;
    const int sb = (int)smem;
    if (int rc = ensure_smem_attr(1 + Op, &fn, &sb, 1))
        return rc;
    const uint32_t lead = (uint32_t)((uintptr_t)inb & 15);
    const uint8_t *base = inb ? inb - lead : reinterpret_cast<const uint8_t *>(16);
    uint32_t out_lead = 0;
    void *out_a = out;
    if (Op == 0 && out) {
        out_lead = (uint32_t)(((uintptr_t)out & 15) >> 1);
        out_a = reinterpret_cast<uint16_t *>(out) - out_lead;
    } else if (Op == 1 && out) {
        out_lead = (uint32_t)((uintptr_t)out & 15);
        out_a = reinterpret_cast<uint8_t *>(out) - out_lead;
    }
    unsigned grid = 0;
    int rc = persistent_grid((const void *)k_batch<Op>, kThreads, smem, (ncases + kWarps - 1) / kWarps, &grid);
    if (rc)
        return rc;
    k_batch<Op><<<grid, kThreads, smem, stream>>>(base, lead, offs, ncases, out_a, out_lead,
                                                   reinterpret_cast<Outcome *>(res));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return cuda_fail(e, "k_batch launch");
    return 0;
}

extern "C" {

const char *lu_last_error(void) { return g_err.c_str(); }

#ifdef LU_PROF
int lu_prof_read(unsigned long long *out32, int reset)
{
    cudaError_t e = cudaMemcpyFromSymbol(out32, g_prof, sizeof(g_prof));
    if (e == cudaSuccess && reset) {
        static const unsigned long long z[48] = {};
        e = cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    }
    return e == cudaSuccess ? 0 : -1;
}
#endif

const char *lu_version(void) { return "laneutf_b200 0.1.0 (sm_100a)"; }

uint64_t lu_workspace_bytes(int op, uint64_t n_units)
{
    switch (op) {
    case LU_OP_UTF8_TO_UTF16LE:
    case LU_OP_UTF8_TO_UTF16BE:
        return 8 * (n_tiles(n_units, 15, kPipeTile) + 2) + 64;
    case LU_OP_UTF16LE_TO_UTF8:
    case LU_OP_UTF16BE_TO_UTF8:
        return 8 * (n_tiles(2 * n_units, 15, kPipeTile) + 2) + 64;
    case LU_OP_VALIDATE_UTF8:
    case LU_OP_VALIDATE_UTF16LE:
    case LU_OP_UTF16_LENGTH_FROM_UTF8:
    case LU_OP_UTF8_LENGTH_FROM_UTF16LE:
    case LU_OP_UTF8_CHAR_COUNT:
    case LU_OP_UTF16LE_CHAR_COUNT:
    case LU_OP_VALIDATE_UTF16BE:
        return 64;
    default:
        return 0;
    }
}

int lu_device_supported(int dev)
{
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess)
        return 0;
    return p.major == 10 && p.minor == 0;
}

int lu_tile_bytes(void) { return kPipeTile; }

int lu_utf8_to_utf16le(const uint8_t *in, uint64_t n_bytes, uint16_t *out, uint64_t out_cap_words, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, cudaStream_t stream)
{
    return u8u16_impl<DirU8U16>(in, n_bytes, out, out_cap_words, ws, ws_bytes, res, stream);
}

int lu_utf8_to_utf16be(const uint8_t *in, uint64_t n_bytes, uint16_t *out, uint64_t out_cap_words, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, cudaStream_t stream)
{
    return u8u16_impl<DirU8U16T<true>>(in, n_bytes, out, out_cap_words, ws, ws_bytes, res, stream);
}

int lu_utf16le_to_utf8(const uint16_t *in, uint64_t n_words, uint8_t *out, uint64_t out_cap_bytes, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, cudaStream_t stream)
{
    return u16u8_impl<DirU16U8>(in, n_words, out, out_cap_bytes, ws, ws_bytes, res, stream);
}

int lu_utf16be_to_utf8(const uint16_t *in, uint64_t n_words, uint8_t *out, uint64_t out_cap_bytes, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, cudaStream_t stream)
{
    return u16u8_impl<DirU16U8T<true>>(in, n_words, out, out_cap_bytes, ws, ws_bytes, res, stream);
}

int lu_validate_utf8(const uint8_t *in, uint64_t n_bytes, void *ws, uint64_t ws_bytes, lu_outcome *res,
                     cudaStream_t stream)
{
    return validate_impl(false, false, in, n_bytes, ws, ws_bytes, res, stream);
}

int lu_validate_utf16le(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, lu_outcome *res,
                        cudaStream_t stream)
{
    return validate_impl(true, false, reinterpret_cast<const uint8_t *>(in), n_words, ws, ws_bytes, res, stream);
}

int lu_validate_utf16be(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, lu_outcome *res,
                        cudaStream_t stream)
{
    return validate_impl(true, false, reinterpret_cast<const uint8_t *>(in), n_words, ws, ws_bytes, res, stream, true);
}

int lu_utf16_length_from_utf8(const uint8_t *in, uint64_t n_bytes, void *ws, uint64_t ws_bytes, lu_outcome *res,
                              cudaStream_t stream)
{
    return validate_impl(false, true, in, n_bytes, ws, ws_bytes, res, stream);
}

int lu_utf8_length_from_utf16le(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, lu_outcome *res,
                                cudaStream_t stream)
{
    return validate_impl(true, true, reinterpret_cast<const uint8_t *>(in), n_words, ws, ws_bytes, res, stream);
}

int lu_utf8_char_count(const uint8_t *in, uint64_t n_bytes, void *ws, uint64_t ws_bytes, uint64_t *count,
                       cudaStream_t stream)
{
    return chars_impl(false, in, n_bytes, ws, ws_bytes, count, stream);
}

int lu_utf16le_char_count(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, uint64_t *count,
                          cudaStream_t stream)
{
    return chars_impl(true, reinterpret_cast<const uint8_t *>(in), n_words, ws, ws_bytes, count, stream);
}

int lu_batch_utf8_to_utf16le(const uint8_t *data, const uint64_t *offsets, uint32_t n_cases, uint16_t *out,
                             lu_outcome *res, cudaStream_t stream)
{
    return batch_impl<0>(data, offsets, n_cases, out, res, stream);
}

int lu_batch_utf16le_to_utf8(const uint16_t *data, const uint64_t *offsets, uint32_t n_cases, uint8_t *out,
                             lu_outcome *res, cudaStream_t stream)
{
    return batch_impl<1>(reinterpret_cast<const uint8_t *>(data), offsets, n_cases, out, res, stream);
}

int lu_batch_validate_utf8(const uint8_t *data, const uint64_t *offsets, uint32_t n_cases, lu_outcome *res,
                           cudaStream_t stream)
{
    return batch_impl<2>(data, offsets, n_cases, nullptr, res, stream);
}

int lu_batch_validate_utf16le(const uint16_t *data, const uint64_t *offsets, uint32_t n_cases, lu_outcome *res,
                              cudaStream_t stream)
{
    return batch_impl<3>(reinterpret_cast<const uint8_t *>(data), offsets, n_cases, nullptr, res, stream);
}

} // extern "C"
