// lu_common.cuh -- shared pieces of the sm_100a transcode/validate kernels.
//
// Geometry (all kernels): a warp owns a contiguous 2 KiB chunk of input and
// walks it in 4 rounds of 512 B, lane l holding bytes [16l, 16l+16) of the
// round in registers (neighbours by shuffle).  The transcode kernels group 4
// chunks into an 8 KiB tile; tiles are ordered by the central scanner
// (scan_windows, the warps of the first CTA to start) rather than a per-tile
// look-back; inputs of at most two tiles per resident CTA use one tile per
// group and an in-group look-back instead (small_tile).
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
constexpr int kChunkBytes = 2048;                     // input bytes per warp chunk
constexpr int kTileBytes = kWarps * kChunkBytes;      // 16 KiB: a CTA's chunks (validators' tile count)

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

// Inclusive warp sum scan: five shfl.up steps whose in-range predicate
// guards the add (no lane-index compares).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v)
{
    asm volatile("{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 t|p, %0, 1, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 2, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 4, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 8, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 16, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t}"
        : "+r"(v));
    return v;
}

// Hang guard: a spin-wait that sees no progress for kHangNs of GPU time
// traps (a launch error the caller sees) instead of hanging the device.  No
// valid schedule waits that long: every wait is on work of CTAs that are
// already running (see k_transcode).
constexpr uint64_t kHangNs = 10ull * 1000000000ull;
__device__ __forceinline__ uint64_t gtimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void hang_check(uint32_t spins, uint64_t t0)
{
    if ((spins & 1023u) == 1023u && gtimer() - t0 > kHangNs)
        __trap();
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

// Optional phase profiler (make prof -> liblaneutf_b200_prof.so; never the
// shipped library): per-phase SM clock cycles summed over groups.
#ifdef LU_PROF
__device__ unsigned long long g_prof[48];
__shared__ unsigned long long s_prof[10][24]; // [warp][counter], lane 0 only
#define LU_T0() long long _t0 = clock64()
#define LU_T(k)                                                                       \
    do {                                                                              \
        const long long _t1 = clock64();                                              \
        if ((threadIdx.x & 31) == 0)                                                  \
            s_prof[threadIdx.x >> 5][k] += (unsigned long long)(_t1 - _t0);           \
        _t0 = _t1;                                                                    \
    } while (0)
#define LU_CNT(k, v)                                                                  \
    do {                                                                              \
        if ((threadIdx.x & 31) == 0)                                                  \
            s_prof[threadIdx.x >> 5][k] += (unsigned long long)(v);                   \
    } while (0)
#define LU_PROF_INIT()                                                                \
    do {                                                                              \
        if ((threadIdx.x & 31) == 0)                                                  \
            for (int _k = 0; _k < 24; ++_k)                                           \
                s_prof[threadIdx.x >> 5][_k] = 0;                                     \
    } while (0)
#define LU_PROF_FLUSH()                                                               \
    do {                                                                              \
        if ((threadIdx.x & 31) == 0)                                                  \
            for (int _k = 0; _k < 24; ++_k)                                           \
                atomicAdd(&g_prof[_k + ((threadIdx.x >> 5) % 4 ? 24 : 0)], s_prof[threadIdx.x >> 5][_k]);                 \
    } while (0)
#else
#define LU_T0()
#define LU_T(k)
#define LU_CNT(k, v)
#define LU_PROF_INIT()
#define LU_PROF_FLUSH()
#endif

// Central scanner: the kScanWarps warps of the first CTA to start (which
// computes no tiles).
// Tiles publish only their aggregate (flag 1).  Scanner warp k owns the
// fixed windows k, k + kScanWarps, ... of kScanWindow tiles (lane l holds
// tiles [4l, 4l+4) of a window).  It takes the window base from the previous
// window's warp through shared memory, then repeatedly polls the window and
// replaces every newly published entry of the window's leading published run
// by flag 2 | EXCLUSIVE prefix; once the whole window is done it hands its end
// value on.  Only the base hand-off is serial; kScanWarps windows are polled
// and scanned in parallel (one warp sweeping serially was the throughput
// limit: ~3 us per pass).  A tile's owner just polls its own status word.
//
// A window is normally published in one shot once all its tiles are in.
// Progress: a group may hold a claimed, unpublished tile while it waits for
// the prefix of an older tile in the same window, so waiting for the whole
// window could deadlock.  If a window stays incomplete kPartialAfter cycles
// after its first tile was published, its leading published run is published
// on every poll from then on; a tile's prefix then depends only on tiles
// before it, which guarantees progress.  (Publishing the run on every poll
// from the start is correct too but cost K1 ~50%: scanner throughput.)
//
// Errors: the count of a tile at or after the first malformed tile is never
// used (nothing there is copied out), so a prefix is the plain sum of the
// preceding counts, with the error bit set iff some preceding tile is
// malformed.
constexpr int kScanWarps = 8;
#ifndef LU_SCAN_PER_LANE
#define LU_SCAN_PER_LANE 3
#endif
constexpr int kScanPerLane = LU_SCAN_PER_LANE;
constexpr uint32_t kScanWindow = 32 * kScanPerLane; // 96 tiles (K1)
// K2 scans 128-tile windows (re-swept after the early base hand-off; was 192):
// where the per-window hand-off is the limit
#ifndef LU_K2_SCAN_PER_LANE
#define LU_K2_SCAN_PER_LANE 4
#endif
#ifndef LU_PARTIAL_AFTER
#define LU_PARTIAL_AFTER 40000
#endif
constexpr long long kPartialAfter = LU_PARTIAL_AFTER;           // SM cycles (~20 us)

struct ScanShared {
    unsigned long long base[kScanWarps]; // end value of the window in the slot
    uint32_t tag[kScanWarps];            // window index + 1 once base is valid
    uint32_t errw;                       // smallest window known to lie behind an error (~0: none)
};

__device__ __forceinline__ void scan_init(ScanShared &ss)
{
    if (threadIdx.x < kScanWarps)
        ss.tag[threadIdx.x] = 0;
    if (threadIdx.x == 0)
        ss.errw = 0xffffffffu;
}

template <int kPL = kScanPerLane>
__device__ __forceinline__ void scan_windows(uint64_t *status, uint32_t ntiles, uint32_t sw, ScanShared &ss)
{
    constexpr uint32_t kWin = 32 * kPL; // tiles per window
    const uint32_t lane = lane_id();
    const uint32_t nwin = (ntiles + kWin - 1) / kWin;
    volatile unsigned long long *vbase = ss.base;
    volatile uint32_t *vtag = ss.tag;
    volatile uint32_t *verrw = &ss.errw;
    for (uint32_t w = sw; w < nwin; w += kScanWarps) {
        const uint32_t t0 = w * kWin + lane * kPL;
        unsigned long long base = 0;
        bool have_base = w == 0; // the base is taken only when first needed
        uint64_t s[kPL];
        uint32_t have = 0; // bit j: s[j] holds a published aggregate
        uint32_t done = 0; // entries of the window already replaced by prefixes
        long long t_first = 0; // clock when the first tile of the window was seen
        bool partial = false;
        const uint64_t t_win = gtimer();
        for (uint32_t polls = 0;; ++polls) {
            hang_check(polls, t_win);
            // Everything in a window behind an error is "error before": publish
            // it at once without waiting for the tiles (whose owners skip their
            // work, see k_transcode) -- groups then never wait on them.  (The
            // non-blocking look at the previous window's base costs nothing
            // measurable on valid input.)
            // Windows behind a window known to follow an error (errw) need no
            // base either: the serial base hand-off would otherwise pace the
            // publication of every remaining window.
            if (!have_base) {
                uint32_t ready = 0;
                if (lane == 0)
                    ready = (vtag[(w - 1) % kScanWarps] == w) ? 1u : (*verrw < w ? 2u : 0u);
                ready = __shfl_sync(0xffffffffu, ready, 0);
                if (ready) {
                    base = ready == 1 ? vbase[(w - 1) % kScanWarps] : kErrBit;
                    have_base = true;
                }
            }
            if (have_base && (base & kErrBit)) {
#pragma unroll
                for (int j = 0; j < kPL; ++j)
                    if (lane * kPL + j >= done && t0 + j < ntiles)
                        st_release(&status[t0 + j], kFlagInc | kErrBit | (base & kValMask));
                if (lane == 0) {
                    atomicMin(&ss.errw, w);
                    vbase[w % kScanWarps] = base;
                    __threadfence_block();
                    vtag[w % kScanWarps] = w + 1;
                }
                break;
            }
#pragma unroll
            for (int j = 0; j < kPL; ++j)
                if (!(have & (1u << j))) {
                    const uint32_t t = t0 + j;
                    s[j] = t < ntiles ? ld_acquire(&status[t]) : kFlagAgg;
                    if (s[j] >> kFlagShift)
                        have |= 1u << j;
                }
            // leading published run of the window: lanes before the first
            // lane with a gap are full; that lane contributes its own run
            const uint32_t lrun = (uint32_t)__ffs(~have) - 1; // 0..kPL
            const uint32_t notfull = __ballot_sync(0xffffffffu, lrun < kPL);
            const uint32_t fl = notfull ? (uint32_t)__ffs(notfull) - 1 : 32u;
            const uint32_t myr = lane < fl ? kPL : (lane == fl ? lrun : 0u);
            const uint32_t run = kPL * fl + (fl < 32 ? __shfl_sync(0xffffffffu, lrun, fl & 31) : 0u);
            if (!partial && run != kWin) {
                if (__any_sync(0xffffffffu, have != 0)) {
                    const long long now = clock64();
                    if (t_first == 0)
                        t_first = now;
                    partial = now - t_first > kPartialAfter;
                }
                partial = __shfl_sync(0xffffffffu, partial, 0);
            }
            if (run > done && (partial || run == kWin)) {
                LU_CNT(11, 1);
                // Window-local scan first: it does not need the base, so it
                // runs while the base is still on its way, and the serial
                // part of the hand-off chain shrinks to wait + add + store.
                uint32_t lsum = 0, errj = kPL;
#pragma unroll
                for (int j = kPL - 1; j >= 0; --j)
                    if ((uint32_t)j < myr) {
                        lsum += (uint32_t)s[j]; // aggregate counts are < 2^15
                        if (s[j] & kErrBit)
                            errj = (uint32_t)j;
                    }
                uint32_t incl = lsum;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= (uint32_t)d)
                        incl += o;
                }
                const uint32_t errball = __ballot_sync(0xffffffffu, errj < kPL);
                const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
                if (!have_base) {
                    // Wait for the previous window's base, or for a window
                    // before this one to be known to hold an error.  The
                    // second exit is needed: once errw < w the previous
                    // window's warp can publish it AND its next window
                    // (w + 7, same slot) without waiting for anyone, so the
                    // tag w may already be overwritten by w + 8.
                    const uint32_t slot = (w - 1) % kScanWarps;
                    uint32_t ready = 0;
                    if (lane == 0) {
                        const uint64_t t_wait = gtimer();
                        for (uint32_t spins = 0;; ++spins) {
                            hang_check(spins, t_wait);
                            if (vtag[slot] == w) {
                                ready = 1;
                                break;
                            }
                            if (*verrw < w) {
                                ready = 2;
                                break;
                            }
                        }
                    }
                    ready = __shfl_sync(0xffffffffu, ready, 0);
                    base = ready == 1 ? vbase[slot] : kErrBit;
                    have_base = true;
                }
                // a complete window hands its end value on before it
                // publishes its tiles' prefixes (the next window only needs
                // the base)
                if (run == kWin && lane == 0) {
                    if (errball || (base & kErrBit))
                        atomicMin(&ss.errw, w);
                    vbase[w % kScanWarps] = (base + wtot) | (errball ? kErrBit : 0ull);
                    __threadfence_block();
                    vtag[w % kScanWarps] = w + 1;
                }
                const bool err_before = (base & kErrBit) || (errball & ((1u << lane) - 1u));
                uint64_t ex = (base & kValMask) + (incl - lsum);
#pragma unroll
                for (int j = 0; j < kPL; ++j) {
                    const uint32_t idx = lane * kPL + j;
                    if ((uint32_t)j < myr && idx >= done && t0 + j < ntiles)
                        st_release(&status[t0 + j],
                                   kFlagInc | ((err_before || errj < (uint32_t)j) ? kErrBit : 0ull) | ex);
                    ex += (uint32_t)s[j];
                }
                done = run;
                if (run == kWin)
                    break;
                if (errball) {
                    // the rest of the window lies behind an error: publish it now
#pragma unroll
                    for (int j = 0; j < kPL; ++j)
                        if (lane * kPL + j >= run && t0 + j < ntiles)
                            st_release(&status[t0 + j], kFlagInc | kErrBit | (base & kValMask));
                    if (lane == 0) {
                        atomicMin(&ss.errw, w);
                        vbase[w % kScanWarps] = base | kErrBit;
                        __threadfence_block();
                        vtag[w % kScanWarps] = w + 1;
                    }
                    break;
                }
            }
            __nanosleep(64);
        }
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

// ------------------------------------------------------ warp chunk loads

__device__ __forceinline__ uint4 ld16(const uint8_t *base, int64_t a, int64_t lo, int64_t hi, bool boundary)
{
    if (!boundary)
        return __ldcs(reinterpret_cast<const uint4 *>(base + a));
    if (a + 16 <= lo || a >= hi)
        return make_uint4(0, 0, 0, 0);
    return load_u128_masked(base, a, lo, hi);
}

__device__ __forceinline__ uint32_t ld4(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    if (a + 4 <= lo || a >= hi)
        return 0u;
    if (a >= lo && a + 4 <= hi)
        return __ldg(reinterpret_cast<const uint32_t *>(base + a));
    return load_u32_masked(base, a, lo, hi);
}

// 4-byte halo word; interior tiles are known to be in bounds
template <bool Boundary>
__device__ __forceinline__ uint32_t halo4(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    if (!Boundary)
        return __ldg(reinterpret_cast<const uint32_t *>(base + a));
    return ld4(base, a, lo, hi);
}

// A warp's 2 KiB input chunk in registers (16 B per lane per round) plus the
// 4-byte halos; loaded separately so a caller can issue the loads early and
// overlap their latency with other work (the pipelined copy-out).
struct ChunkIn {
    uint4 q[kChunkBytes / 512];
    uint32_t halo_p; // lane 0: the 4 bytes before the chunk
    uint32_t halo_n; // lane 31: the 4 bytes after it
};

// byte-swap both 16-bit units of a quad (UTF-16BE <-> LE)
__device__ __forceinline__ uint32_t swap16x2(uint32_t x) { return prmt(x, 0u, 0x2301u); }

// Swap16: the input is UTF-16BE; every word is byte-swapped on load so the
// UTF-16 kernels see LE words (swap_utf16_byte_order fused into the load,
// SURVEY 8f(1); the reference swaps the whole buffer first, cli.py:90-94).
template <bool Boundary, bool Swap16 = false>
__device__ __forceinline__ void load_chunk(const uint8_t *__restrict__ base, int64_t chunk, int64_t lo_b, int64_t hi_b,
                                           ChunkIn &in)
{
    const uint32_t lane = lane_id();
#pragma unroll
    for (int r = 0; r < kChunkBytes / 512; ++r) {
        in.q[r] = ld16(base, chunk + r * 512 + 16 * (int64_t)lane, lo_b, hi_b, Boundary);
        if (Swap16)
            in.q[r] = make_uint4(swap16x2(in.q[r].x), swap16x2(in.q[r].y), swap16x2(in.q[r].z), swap16x2(in.q[r].w));
    }
    in.halo_p = (lane == 0) ? halo4<Boundary>(base, chunk - 4, lo_b, hi_b) : 0u;
    in.halo_n = (lane == 31) ? halo4<Boundary>(base, chunk + kChunkBytes, lo_b, hi_b) : 0u;
    if (Swap16) {
        in.halo_p = swap16x2(in.halo_p);
        in.halo_n = swap16x2(in.halo_n);
    }
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
