// Experiment harness (not part of the product): times K1 building blocks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/kexp tools/kexp.cu
// Modes of a one-CTA-per-tile K1: 0 full (decoupled look-back), 1 prefix
// precomputed (no look-back wait), 2 look-back but no copy-out, 3 compute
// only; plus a plain copy kernel moving the same bytes (roofline check).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include "../paper_2212_05098_b200/csrc/lu_common.cuh"
#include "../paper_2212_05098_b200/csrc/lu_utf8.cuh"

using namespace lu;
constexpr int kOutStrideU16 = kChunkBytes + 16;

__device__ void copy_out_u16(const uint16_t *src, uint32_t cnt, uint16_t *out_a, uint64_t g0)
{
    if (cnt == 0) return;
    const uint32_t lane = lane_id();
    const uint32_t shift = (uint32_t)(g0 & 7);
    uint16_t *dst = out_a + (g0 - shift);
    const uint32_t total = shift + cnt;
    const uint32_t full_lo = shift ? 1u : 0u, full_hi = total >> 3;
    const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src);
    if (shift == 0) {
        const uint4 *s128 = reinterpret_cast<const uint4 *>(src);
        for (uint32_t c = full_lo + lane; c < full_hi; c += 32) __stcs(reinterpret_cast<uint4 *>(dst) + c, s128[c]);
    } else if ((shift & 1) == 0) {
        for (uint32_t c = full_lo + lane; c < full_hi; c += 32) {
            const uint32_t m = (8 * c - shift) >> 1;
            __stcs(reinterpret_cast<uint4 *>(dst) + c, make_uint4(s32[m], s32[m + 1], s32[m + 2], s32[m + 3]));
        }
    } else {
        for (uint32_t c = full_lo + lane; c < full_hi; c += 32) {
            const uint32_t m = (8 * c - shift - 1) >> 1;
            const uint32_t w0 = s32[m], w1 = s32[m + 1], w2 = s32[m + 2], w3 = s32[m + 3], w4 = s32[m + 4];
            __stcs(reinterpret_cast<uint4 *>(dst) + c, make_uint4(prmt(w0, w1, 0x5432), prmt(w1, w2, 0x5432), prmt(w2, w3, 0x5432), prmt(w3, w4, 0x5432)));
        }
    }
    if (lane < 16) {
        uint32_t chunk = lane < 8 ? (shift ? 0u : 0xffffffffu) : ((total & 7) && !(shift && full_hi == 0) ? full_hi : 0xffffffffu);
        if (chunk != 0xffffffffu) { const uint32_t i = 8 * chunk + (lane & 7); if (i >= shift && i < total) dst[i] = src[i - shift]; }
    }
}

__device__ void sel_init(SelPair *sel)
{
    if (threadIdx.x < 16) {
        uint32_t idx = threadIdx.x, s[2] = {0, 0}, j = 0;
        for (uint32_t p = 0; p < 4; ++p) if (idx & (1u << p)) { s[j >> 1] |= (p | ((4 + p) << 4)) << (8 * (j & 1)); ++j; }
        sel[idx].s01 = s[0]; sel[idx].s23 = s[1];
    }
}

struct TS { WarpResult wres[kWarps]; uint32_t wex[kWarps]; uint64_t excl; uint32_t units; };

template <int Mode>
__global__ void __launch_bounds__(kThreads, 4) k1(const uint8_t *base, uint64_t n, uint16_t *out, uint64_t *status, const uint64_t *prefix, uint32_t *units_out)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint16_t *out_s = reinterpret_cast<uint16_t *>(smem_raw);
    __shared__ SelPair sel[16];
    __shared__ TS ts;
    const int64_t tile_off = (int64_t)blockIdx.x * kTileBytes;
    sel_init(sel);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    uint16_t *out_w = out_s + warp * kOutStrideU16;
    const bool interior = (tile_off - 4 >= 0) && (tile_off + kTileBytes + 4 <= (int64_t)n);
    if (interior) u8u16_warp<false>(base, tile_off, 0, n, out_w, sel, ts.wres[warp]);
    else u8u16_warp<true>(base, tile_off, 0, n, out_w, sel, ts.wres[warp]);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int w = 0; w < kWarps; ++w) { ts.wex[w] = acc; acc += ts.wres[w].units; }
        ts.units = acc;
        if (units_out) units_out[blockIdx.x] = acc;
    }
    __syncthreads();
    if (Mode == 0 || Mode == 2) {
        if (threadIdx.x < 32) { uint64_t ex = lookback(status, blockIdx.x, ts.units); if (threadIdx.x == 0) ts.excl = ex; }
    } else if (threadIdx.x == 0) {
        ts.excl = prefix[blockIdx.x];
    }
    __syncthreads();
    if (Mode == 0 || Mode == 1)
        copy_out_u16(out_w, ts.wres[warp].units, out, ts.excl + ts.wex[warp]);
}

template <int PerLane>
__device__ uint64_t lookback_w(uint64_t *status, uint32_t tile, uint64_t agg)
{
    const uint32_t lane = lane_id();
    if (tile == 0) { if (lane == 0) st_release(&status[0], kFlagInc | agg); return 0; }
    if (lane == 0) st_release(&status[tile], kFlagAgg | agg);
    uint64_t excl = 0; int64_t pred = (int64_t)tile - 1;
    while (true) {
        uint64_t s[PerLane];
#pragma unroll
        for (int j = 0; j < PerLane; ++j) { const int64_t t = pred - (int64_t)(PerLane * lane + j); s[j] = (t >= 0) ? ld_acquire(&status[t]) : kFlagInc; }
#pragma unroll
        for (int j = 0; j < PerLane; ++j) { const int64_t t = pred - (int64_t)(PerLane * lane + j); while ((s[j] >> kFlagShift) == 0) s[j] = ld_acquire(&status[t]); }
        int jinc = PerLane;
#pragma unroll
        for (int j = PerLane - 1; j >= 0; --j) if ((s[j] >> kFlagShift) == 2) jinc = j;
        uint64_t v = 0;
#pragma unroll
        for (int j = PerLane - 1; j >= 0; --j) if (j <= jinc) v = seq_combine(v, s[j] & (kErrBit | kValMask));
        const uint32_t inc = __ballot_sync(0xffffffffu, jinc < PerLane);
        const uint32_t stop = inc ? (uint32_t)(__ffs(inc) - 1) : 31u;
        if (lane > stop) v = 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) { uint64_t o = __shfl_down_sync(0xffffffffu, v, d); if (lane + d < 32) v = seq_combine(o, v); }
        v = __shfl_sync(0xffffffffu, v, 0);
        excl = seq_combine(v, excl);
        if (inc) break;
        pred -= 32 * PerLane;
    }
    if (lane == 0) st_release(&status[tile], kFlagInc | seq_combine(excl, agg));
    return excl;
}

// pure look-back throughput: each CTA (one warp) publishes 1 and looks back
template <int PerLane>
__global__ void klb(uint64_t *status, uint64_t *out)
{
    uint64_t ex = lookback_w<PerLane>(status, blockIdx.x, 1);
    if (lane_id() == 0 && ex != blockIdx.x) out[0] = 1;
}

template <int W, int Mode>
__global__ void __launch_bounds__(W * 32) k1w(const uint8_t *base, uint64_t n, uint16_t *out, uint64_t *status, const uint64_t *prefix, uint32_t *units_out)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint16_t *out_s = reinterpret_cast<uint16_t *>(smem_raw);
    __shared__ SelPair sel[16];
    __shared__ WarpResult wres[W];
    __shared__ uint64_t excl_s;
    __shared__ uint32_t wex[W], units_s;
    const int64_t tile_off = (int64_t)blockIdx.x * W * kChunkBytes;
    sel_init(sel);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    uint16_t *out_w = out_s + warp * kOutStrideU16;
    const bool interior = (tile_off - 4 >= 0) && (tile_off + W * kChunkBytes + 4 <= (int64_t)n);
    // u8u16_warp derives the chunk from threadIdx; tile_off is per CTA
    if (interior) u8u16_warp<false>(base, tile_off, 0, n, out_w, sel, wres[warp]);
    else u8u16_warp<true>(base, tile_off, 0, n, out_w, sel, wres[warp]);
    __syncthreads();
    if (threadIdx.x == 0) { uint32_t acc = 0; for (int w = 0; w < W; ++w) { wex[w] = acc; acc += wres[w].units; } units_s = acc; }
    __syncthreads();
    if (Mode == 0) { if (threadIdx.x < 32) { uint64_t ex = lookback(status, blockIdx.x, units_s); if (threadIdx.x == 0) excl_s = ex; } }
    else if (threadIdx.x == 0) excl_s = 0;
    __syncthreads();
    if (Mode == 0) copy_out_u16(out_w, wres[warp].units, out, excl_s + wex[warp]);
}

// copy-out reading aligned 16-byte smem vectors (conflict-free), uniform word shift
__device__ void copy_out_u16_v2(const uint16_t *src, uint32_t cnt, uint16_t *out_a, uint64_t g0)
{
    if (cnt == 0) return;
    const uint32_t lane = lane_id();
    const uint32_t shift = (uint32_t)(g0 & 7);
    uint16_t *dst = out_a + (g0 - shift);
    const uint32_t total = shift + cnt;
    const uint32_t full_lo = shift ? 1u : 0u, full_hi = total >> 3;
    const uint4 *s128 = reinterpret_cast<const uint4 *>(src);
    const uint32_t r = (8u - shift) & 7u; // word offset of chunk data inside the aligned smem vector
    for (uint32_t c = full_lo + lane; c < full_hi; c += 32) {
        const uint32_t v = (8 * c - shift) >> 3;
        const uint4 a = s128[v];
        uint4 o;
        if (r == 0) {
            o = a;
        } else {
            const uint4 b = s128[v + 1];
            const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            switch (r) {
            case 1: o = make_uint4(prmt(w[0], w[1], 0x5432), prmt(w[1], w[2], 0x5432), prmt(w[2], w[3], 0x5432), prmt(w[3], w[4], 0x5432)); break;
            case 2: o = make_uint4(w[1], w[2], w[3], w[4]); break;
            case 3: o = make_uint4(prmt(w[1], w[2], 0x5432), prmt(w[2], w[3], 0x5432), prmt(w[3], w[4], 0x5432), prmt(w[4], w[5], 0x5432)); break;
            case 4: o = make_uint4(w[2], w[3], w[4], w[5]); break;
            case 5: o = make_uint4(prmt(w[2], w[3], 0x5432), prmt(w[3], w[4], 0x5432), prmt(w[4], w[5], 0x5432), prmt(w[5], w[6], 0x5432)); break;
            case 6: o = make_uint4(w[3], w[4], w[5], w[6]); break;
            default: o = make_uint4(prmt(w[3], w[4], 0x5432), prmt(w[4], w[5], 0x5432), prmt(w[5], w[6], 0x5432), prmt(w[6], w[7], 0x5432)); break;
            }
        }
        __stcs(reinterpret_cast<uint4 *>(dst) + c, o);
    }
    if (lane < 16) {
        uint32_t chunk = lane < 8 ? (shift ? 0u : 0xffffffffu) : ((total & 7) && !(shift && full_hi == 0) ? full_hi : 0xffffffffu);
        if (chunk != 0xffffffffu) { const uint32_t i = 8 * chunk + (lane & 7); if (i >= shift && i < total) dst[i] = src[i - shift]; }
    }
}

__device__ __forceinline__ void nbar(uint32_t id, uint32_t n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// central scanner: publishes EXCLUSIVE prefixes (flag 2) in tile order
template <int K>
__device__ void scanner(uint64_t *status, uint32_t ntiles)
{
    const uint32_t lane = lane_id();
    uint32_t next = 0;
    uint64_t acc = 0;
    while (next < ntiles) {
        uint64_t s[K];
#pragma unroll
        for (int j = 0; j < K; ++j) { const uint32_t t = next + lane * K + j; s[j] = t < ntiles ? ld_acquire(&status[t]) : 0ull; }
        uint32_t r = K;
#pragma unroll
        for (int j = K - 1; j >= 0; --j) if ((s[j] >> kFlagShift) == 0) r = j;
        const uint32_t full = __ballot_sync(0xffffffffu, r == K);
        const uint32_t f = full == 0xffffffffu ? 32u : (uint32_t)__ffs(~full) - 1;
        const uint32_t myr = lane < f ? K : (lane == f ? r : 0u);
        const uint32_t total = __reduce_add_sync(0xffffffffu, myr);
        if (total == 0) { __nanosleep(64); continue; }
        uint64_t S = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) if ((uint32_t)j < myr) S = seq_combine(S, s[j] & (kErrBit | kValMask));
        uint64_t inc = S;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const uint64_t o = __shfl_up_sync(0xffffffffu, inc, d); if (lane >= (uint32_t)d) inc = seq_combine(o, inc); }
        uint64_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) ex = 0;
        uint64_t run = seq_combine(acc, ex);
#pragma unroll
        for (int j = 0; j < K; ++j) if ((uint32_t)j < myr) { st_release(&status[next + lane * K + j], kFlagInc | run); run = seq_combine(run, s[j] & (kErrBit | kValMask)); }
        acc = seq_combine(acc, __shfl_sync(0xffffffffu, inc, 31));
        next += total;
    }
}

template <int K, bool V2>
__global__ void __launch_bounds__(288, 3) kpipe(const uint8_t *base, uint64_t n, uint16_t *out, uint64_t *status, uint32_t ntiles)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint16_t *out_s = reinterpret_cast<uint16_t *>(smem_raw); // [2][8][stride]
    __shared__ SelPair sel[16];
    __shared__ WarpResult wres[2][8];
    __shared__ uint32_t wex[2][8], s_tile[2], s_claim;
    __shared__ uint64_t s_excl[2];
    unsigned int *ticket = reinterpret_cast<unsigned int *>(status + ntiles);
    sel_init(sel);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 8) { if (blockIdx.x == 0) scanner<K>(status, ntiles); return; }
    auto copy_buf = [&](uint32_t b) {
        if (threadIdx.x == 0) {
            uint64_t st = ld_acquire(&status[s_tile[b]]);
            while ((st >> kFlagShift) != 2) { __nanosleep(32); st = ld_acquire(&status[s_tile[b]]); }
            s_excl[b] = st & (kErrBit | kValMask);
        }
        nbar(5, 256);
        const uint64_t ex = s_excl[b];
        if (!(ex & kErrBit)) {
            if (V2) copy_out_u16_v2(out_s + (b * 8 + warp) * kOutStrideU16, wres[b][warp].units, out, ex + wex[b][warp]);
            else copy_out_u16(out_s + (b * 8 + warp) * kOutStrideU16, wres[b][warp].units, out, ex + wex[b][warp]);
        }
    };
    uint32_t i = 0;
    for (;; ++i) {
        const uint32_t buf = i & 1;
        if (i >= 2) copy_buf(buf);
        if (threadIdx.x == 0) s_claim = atomicAdd(ticket, 1u);
        nbar(6, 256);
        const uint32_t tile = s_claim;
        if (tile >= ntiles) break;
        const int64_t tile_off = (int64_t)tile * kTileBytes;
        uint16_t *out_w = out_s + (buf * 8 + warp) * kOutStrideU16;
        const bool interior = (tile_off - 4 >= 0) && (tile_off + kTileBytes + 4 <= (int64_t)n);
        if (interior) u8u16_warp<false>(base, tile_off, 0, n, out_w, sel, wres[buf][warp]);
        else u8u16_warp<true>(base, tile_off, 0, n, out_w, sel, wres[buf][warp]);
        nbar(7, 256);
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int w = 0; w < 8; ++w) { wex[buf][w] = acc; acc += wres[buf][w].units; }
            s_tile[buf] = tile;
            st_release(&status[tile], kFlagAgg | acc);
        }
    }
    if (i >= 1) { nbar(6, 256); copy_buf((i - 1) & 1); }
}

template <int K, bool V2>
__global__ void __launch_bounds__(288, 3) kpipe_t(const uint8_t *base, uint64_t n, uint16_t *out, uint64_t *status, uint32_t ntiles, unsigned long long *tm)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint16_t *out_s = reinterpret_cast<uint16_t *>(smem_raw); // [2][8][stride]
    __shared__ SelPair sel[16];
    __shared__ WarpResult wres[2][8];
    __shared__ uint32_t wex[2][8], s_tile[2], s_claim;
    __shared__ uint64_t s_excl[2];
    unsigned int *ticket = reinterpret_cast<unsigned int *>(status + ntiles);
    sel_init(sel);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 8) { if (blockIdx.x == 0) scanner<K>(status, ntiles); return; }
    auto copy_buf = [&](uint32_t b) {
        if (threadIdx.x == 0) {
            uint64_t st = ld_acquire(&status[s_tile[b]]);
            while ((st >> kFlagShift) != 2) { __nanosleep(32); st = ld_acquire(&status[s_tile[b]]); }
            s_excl[b] = st & (kErrBit | kValMask);
        }
        nbar(5, 256);
        long long tc = clock64();
        const uint64_t ex = s_excl[b];
        if (!(ex & kErrBit)) {
            if (V2) copy_out_u16_v2(out_s + (b * 8 + warp) * kOutStrideU16, wres[b][warp].units, out, ex + wex[b][warp]);
            else copy_out_u16(out_s + (b * 8 + warp) * kOutStrideU16, wres[b][warp].units, out, ex + wex[b][warp]);
        }
        if (lane_id() == 0) atomicAdd(&tm[1], (unsigned long long)(clock64() - tc));
    };
    uint32_t i = 0;
    for (;; ++i) {
        const uint32_t buf = i & 1;
        long long t0 = clock64();
        if (i >= 2) copy_buf(buf);
        long long t1 = clock64();
        if (threadIdx.x == 0) s_claim = atomicAdd(ticket, 1u);
        nbar(6, 256);
        long long t2 = clock64();
        const uint32_t tile = s_claim;
        if (tile >= ntiles) break;
        const int64_t tile_off = (int64_t)tile * kTileBytes;
        uint16_t *out_w = out_s + (buf * 8 + warp) * kOutStrideU16;
        const bool interior = (tile_off - 4 >= 0) && (tile_off + kTileBytes + 4 <= (int64_t)n);
        if (interior) u8u16_warp<false>(base, tile_off, 0, n, out_w, sel, wres[buf][warp]);
        else u8u16_warp<true>(base, tile_off, 0, n, out_w, sel, wres[buf][warp]);
        long long t3 = clock64();
        nbar(7, 256);
        long long t4 = clock64();
        if (lane_id() == 0) {
            atomicAdd(&tm[0], (unsigned long long)(t1 - t0)); // copy phase incl. prefix wait
            atomicAdd(&tm[2], (unsigned long long)(t2 - t1)); // claim
            atomicAdd(&tm[3], (unsigned long long)(t3 - t2)); // compute
            atomicAdd(&tm[4], (unsigned long long)(t4 - t3)); // barrier after compute
            atomicAdd(&tm[5], 1ull);
        }
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int w = 0; w < 8; ++w) { wex[buf][w] = acc; acc += wres[buf][w].units; }
            s_tile[buf] = tile;
            st_release(&status[tile], kFlagAgg | acc);
        }
    }
    if (i >= 1) { nbar(6, 256); copy_buf((i - 1) & 1); }
}

// warp-specialized: 8 compute warps, 4 copy-out warps, 1 scanner warp (CTA 0)
template <int K>
__global__ void __launch_bounds__(416, 2) kpipe2(const uint8_t *base, uint64_t n, uint16_t *out, uint64_t *status, uint32_t ntiles)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint16_t *out_s = reinterpret_cast<uint16_t *>(smem_raw); // [2][8][stride]
    __shared__ SelPair sel[16];
    __shared__ WarpResult wres[2][8];
    __shared__ uint32_t wex[2][8], s_tile[2], s_claim;
    __shared__ uint64_t s_excl[2];
    unsigned int *ticket = reinterpret_cast<unsigned int *>(status + ntiles);
    sel_init(sel);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 12) { if (blockIdx.x == 0) scanner<K>(status, ntiles); return; }
    if (warp >= 8) {
        // copy-out warps: drain staging buffers in iteration order
        const uint32_t cw = warp - 8;
        for (uint32_t i = 0;; ++i) {
            const uint32_t b = i & 1;
            nbar(1 + b, 384); // staging b full (or sentinel)
            const uint32_t tile = s_tile[b];
            if (tile == 0xffffffffu) break;
            if (threadIdx.x == 256) {
                uint64_t st = ld_acquire(&status[tile]);
                while ((st >> kFlagShift) != 2) { __nanosleep(32); st = ld_acquire(&status[tile]); }
                s_excl[b] = st & (kErrBit | kValMask);
            }
            nbar(7, 128);
            const uint64_t ex = s_excl[b];
            if (!(ex & kErrBit)) {
                for (uint32_t w = cw; w < 8; w += 4)
                    copy_out_u16_v2(out_s + (b * 8 + w) * kOutStrideU16, wres[b][w].units, out, ex + wex[b][w]);
            }
            asm volatile("bar.arrive %0, %1;" ::"r"(3 + b), "r"(384) : "memory"); // staging b free
        }
        return;
    }
    uint32_t i = 0;
    for (;; ++i) {
        const uint32_t buf = i & 1;
        if (threadIdx.x == 0) s_claim = atomicAdd(ticket, 1u);
        nbar(5, 256);
        const uint32_t tile = s_claim;
        if (i >= 2) nbar(3 + buf, 384); // wait until the copy warps drained buf
        if (tile >= ntiles) {
            if (threadIdx.x == 0) s_tile[buf] = 0xffffffffu;
            __syncwarp();
            asm volatile("bar.arrive %0, %1;" ::"r"(1 + buf), "r"(384) : "memory");
            break;
        }
        const int64_t tile_off = (int64_t)tile * kTileBytes;
        uint16_t *out_w = out_s + (buf * 8 + warp) * kOutStrideU16;
        const bool interior = (tile_off - 4 >= 0) && (tile_off + kTileBytes + 4 <= (int64_t)n);
        if (interior) u8u16_warp<false>(base, tile_off, 0, n, out_w, sel, wres[buf][warp]);
        else u8u16_warp<true>(base, tile_off, 0, n, out_w, sel, wres[buf][warp]);
        nbar(6, 256);
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int w = 0; w < 8; ++w) { wex[buf][w] = acc; acc += wres[buf][w].units; }
            s_tile[buf] = tile;
            st_release(&status[tile], kFlagAgg | acc);
        }
        __syncwarp();
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + buf), "r"(384) : "memory");
    }
}

__global__ void kcopy(const uint4 *in, uint64_t n16, uint4 *out, uint64_t m16)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m16; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(in + (i % n16));
        __stcs(out + i, v);
    }
}

int main(int argc, char **argv)
{
    const int prof = argc > 1 ? atoi(argv[1]) : 0; // 0 latin-like, 1 cjk-like
    const uint64_t n = 256ull << 20;
    std::vector<uint8_t> h(n);
    std::mt19937_64 rng(1);
    uint64_t i = 0;
    while (i + 4 < n) {
        uint32_t r = rng();
        if (r % 7 == 0) { h[i++] = ' '; continue; }
        if (prof == 0) {
            if (r % 20 == 1) { uint32_t cp = 0xC0 + (r >> 8) % 0xC0; h[i++] = 0xC0 | (cp >> 6); h[i++] = 0x80 | (cp & 0x3F); }
            else h[i++] = 'a' + (r >> 8) % 26;
        } else {
            if (r % 10 == 1) h[i++] = 'a' + (r >> 8) % 26;
            else { uint32_t cp = 0x4E00 + (r >> 8) % 0x5200; h[i++] = 0xE0 | (cp >> 12); h[i++] = 0x80 | ((cp >> 6) & 0x3F); h[i++] = 0x80 | (cp & 0x3F); }
        }
    }
    while (i < n) h[i++] = ' ';
    uint8_t *d_in; uint16_t *d_out; uint64_t *d_status, *d_prefix; uint32_t *d_units;
    const uint32_t nt = n / kTileBytes;
    cudaMalloc(&d_in, n); cudaMalloc(&d_out, 2 * n); cudaMalloc(&d_status, 8 * (nt + 1)); cudaMalloc(&d_prefix, 8 * nt); cudaMalloc(&d_units, 4 * nt);
    cudaMemcpy(d_in, h.data(), n, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(uint16_t) * kOutStrideU16 * kWarps;
    cudaFuncSetAttribute(k1<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k1<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k1<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k1<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // exact prefix for mode 1
    cudaMemset(d_status, 0, 8 * (nt + 1));
    k1<3><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, d_units);
    std::vector<uint32_t> units(nt); std::vector<uint64_t> pre(nt);
    cudaMemcpy(units.data(), d_units, 4 * nt, cudaMemcpyDeviceToHost);
    uint64_t acc = 0; for (uint32_t t = 0; t < nt; ++t) { pre[t] = acc; acc += units[t]; }
    cudaMemcpy(d_prefix, pre.data(), 8 * nt, cudaMemcpyHostToDevice);
    printf("profile %d: output words %llu\n", prof, (unsigned long long)acc);
    if (argc > 2) { // profiling mode: one more compute-only launch, then exit
        k1<3><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, nullptr);
        cudaDeviceSynchronize();
        return 0;
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        double alg = (double)n + 2.0 * acc;
        printf("%-28s %8.1f us  input %7.1f GiB/s  alg %7.1f GB/s\n", name, ms * 1e3, n / (ms * 1e-3) / (1 << 30), alg / (ms * 1e-3) / 1e9);
    };
    run("mode0 full", [&] { cudaMemsetAsync(d_status, 0, 8 * (nt + 1)); k1<0><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, nullptr); });
    run("mode1 no-lookback", [&] { k1<1><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, nullptr); });
    run("mode2 lookback, no copy", [&] { cudaMemsetAsync(d_status, 0, 8 * (nt + 1)); k1<2><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, nullptr); });
    run("mode3 compute only", [&] { k1<3><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, nullptr); });
    run("copy in->out (same bytes)", [&] { kcopy<<<148 * 8, 512>>>((const uint4 *)d_in, n / 16, (uint4 *)d_out, 2 * acc / 16); });
    auto runw = [&](const char *name, auto kern, int W) {
        const size_t sm = sizeof(uint16_t) * kOutStrideU16 * W;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const uint32_t ntw = n / (W * kChunkBytes);
        run(name, [&] { cudaMemsetAsync(d_status, 0, 8 * (ntw + 1)); kern<<<ntw, W * 32, sm>>>(d_in, n, d_out, d_status, d_prefix, nullptr); });
    };
    cudaFree(d_status); cudaMalloc(&d_status, 8 * (n / 2048 + 1));
    {
        const size_t sm = 2 * sizeof(uint16_t) * kOutStrideU16 * 8;
        auto rp = [&](const char *name, auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 288, sm);
            run(name, [&] { cudaMemsetAsync(d_status, 0, 8 * (nt + 1)); kern<<<148 * per, 288, sm>>>(d_in, n, d_out, d_status, nt); });
            printf("   (blocks/SM %d)\n", per);
        };
        rp("pipe scanner K8 copy-v1", kpipe<8, false>);
        rp("pipe scanner K16 copy-v1", kpipe<16, false>);
        rp("pipe scanner K16 copy-v2", kpipe<16, true>);
        {
            auto kern = kpipe_t<16, true>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 288, sm);
            unsigned long long *d_tm; cudaMalloc(&d_tm, 64); cudaMemset(d_tm, 0, 64);
            cudaMemsetAsync(d_status, 0, 8 * (nt + 1));
            kern<<<148 * per, 288, sm>>>(d_in, n, d_out, d_status, nt, d_tm);
            unsigned long long tm[8]; cudaMemcpy(tm, d_tm, 64, cudaMemcpyDeviceToHost);
            double c = (double)tm[5];
            printf("   per warp-tile cycles: copy-phase %.0f (of which copy %.0f), claim %.0f, compute %.0f, post-compute barrier %.0f  (warp-tiles %llu)\n",
                   tm[0] / c, tm[1] / c, tm[2] / c, tm[3] / c, tm[4] / c, tm[5]);
        }
        {
            auto kern = kpipe2<16>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 416, sm);
            run("pipe2 warp-specialized", [&] { cudaMemsetAsync(d_status, 0, 8 * (nt + 1)); kern<<<148 * per, 416, sm>>>(d_in, n, d_out, d_status, nt); });
            printf("   (blocks/SM %d)\n", per);
        }
        // correctness check of the last run against mode-1 output
        std::vector<uint16_t> o1(acc), o2(acc);
        cudaMemcpy(o2.data(), d_out, 2 * acc, cudaMemcpyDeviceToHost);
        k1<1><<<nt, kThreads, smem>>>(d_in, n, d_out, d_status, d_prefix, nullptr);
        cudaMemcpy(o1.data(), d_out, 2 * acc, cudaMemcpyDeviceToHost);
        printf("pipe output matches: %s\n", o1 == o2 ? "yes" : "NO");
    }
    runw("W4 full", k1w<4, 0>, 4);
    runw("W4 compute only", k1w<4, 3>, 4);
    runw("W2 full", k1w<2, 0>, 2);
    runw("W2 compute only", k1w<2, 3>, 2);
    runw("W1 full", k1w<1, 0>, 1);
    runw("W1 compute only", k1w<1, 3>, 1);
    const uint32_t nlb = 16384;
    auto lb = [&](const char *name, auto kern) {
        for (int w = 0; w < 3; ++w) { cudaMemsetAsync(d_status, 0, 8 * (nlb + 1)); kern<<<nlb, 32>>>(d_status, d_prefix); }
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) { cudaMemsetAsync(d_status, 0, 8 * (nlb + 1)); kern<<<nlb, 32>>>(d_status, d_prefix); }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        printf("%-28s %8.1f us for %u tiles -> %.1f tiles/us\n", name, ms * 1e3, nlb, nlb / (ms * 1e3));
    };
    lb("lookback-only perlane=1", klb<1>);
    lb("lookback-only perlane=2", klb<2>);
    lb("lookback-only perlane=4", klb<4>);
    lb("lookback-only perlane=8", klb<8>);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
