// lu_utf8.cuh -- UTF-8 side: K1 utf8 -> utf16le transcode, K3 utf8 validate.
//
// Semantics = laneutf.scalar.transcode_utf8_to_utf16le / validate_utf8
// (/root/reference/pkg/src/laneutf/scalar.py:46-105, 150-197): output is the
// transcoding of the longest valid prefix, ``consumed`` is the index of the
// first invalid byte.  That index is the minimum position of a LOCAL predicate
// (exhaustively checked against scalar on all byte
// triples), so no sequential decoder state is needed:
//
//   byte i is bad iff
//     * it is C0, C1 or F5..FF, or
//     * it is a continuation (80..BF) not claimed by the nearest
//       non-continuation among i-1..i-3, or
//     * it is a lead C2..F4 whose continuations are missing / truncated or
//       whose second byte is out of range (E0 A0.., ED ..9F, F0 90.., F4 ..8F).
//
// Per 4-byte quad the kernels compute SWAR byte masks (bit 7 of each byte):
// C = continuation, L = >=C0, E = >=E0, F = >=F0.  A cheap detector flags any
// step that may contain a bad byte ("must be continuation" xor C, plus the
// special second-byte / overlong / range checks); a flagged step is resolved
// by the exact predicate above (u8_bad_at), which is the only place error
// offsets come from.
#pragma once

#include "lu_common.cuh"

namespace lu {

struct U8Masks {
    uint32_t C, L, E, F;
};

__device__ __forceinline__ U8Masks u8_classify(uint32_t x)
{
    const uint32_t t1 = x << 1;
    U8Masks m;
    m.C = x & ~t1 & H8;
    m.L = x & t1 & H8;
    m.E = m.L & (x << 2);
    m.F = m.E & (x << 3);
    return m;
}

// bit 7 set in each byte that is zero
__device__ __forceinline__ uint32_t zero8(uint32_t v)
{
    return ~(((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v) & H8;
}

// Detector: nonzero if a bad byte may lie in this quad (or the first three
// bytes of the following quad belong to a lead of this quad with a missing
// continuation, which the next quad's "must ^ C" reports).  Never misses the
// first bad byte of the input ("detector completeness").
__device__ __forceinline__ uint32_t u8_detect(uint32_t x, uint32_t xn, const U8Masks &m, const U8Masks &p,
                                              bool any_f)
{
    const uint32_t must = fsl(p.L, m.L, 8) | fsl(p.E, m.E, 16) | fsl(p.F, m.F, 24);
    uint32_t d = must ^ m.C;
    // C0 / C1: 2-byte leads whose payload bits 4..1 are zero
    d |= m.L & ~m.E & ~((x & 0x1E1E1E1Eu) + 0x7F7F7F7Fu);
    // E0 80..9F (overlong) / ED A0..BF (surrogate): hi byte of the decoded
    // word & 0xF8 is 0x00 or 0xD8
    const uint32_t n1 = fsr(x, xn, 8);
    const uint32_t h = ((x << 4) & 0xF0F0F0F0u) | ((n1 >> 2) & 0x08080808u);
    d |= m.E & ~m.F & (zero8(h) | zero8(h ^ 0xD8D8D8D8u));
    if (any_f) {
        // F0 80..8F (overlong), F4 90.. / F5..F7 (> U+10FFFF), F8..FF
        const uint32_t key = ((x & 0x07070707u) << 2) | ((n1 >> 4) & 0x03030303u);
        d |= m.F & (~(key + 0x7F7F7F7Fu) | (key + 0x6F6F6F6Fu) | (x << 4));
    }
    return d;
}

// Exact reference predicate for the byte at p (bytes p[-3..3] readable).
__device__ __forceinline__ bool u8_bad_at(const uint8_t *p)
{
    const uint32_t c = p[0];
    if (c < 0x80)
        return false;
    if (c < 0xC0) {
        int d = 1;
        while (d <= 3 && (p[-d] & 0xC0) == 0x80)
            ++d;
        if (d > 3)
            return true;
        const uint32_t lb = p[-d];
        const int len = lb >= 0xF0 ? 4 : lb >= 0xE0 ? 3 : lb >= 0xC0 ? 2 : 1;
        return !(d < len);
    }
    if (c < 0xC2 || c > 0xF4)
        return true;
    const int len = c >= 0xF0 ? 4 : c >= 0xE0 ? 3 : 2;
    for (int t = 1; t < len; ++t)
        if ((p[t] & 0xC0) != 0x80)
            return true;
    const uint32_t c1 = p[1];
    if (c == 0xE0 && c1 < 0xA0)
        return true;
    if (c == 0xED && c1 > 0x9F)
        return true;
    if (c == 0xF0 && c1 < 0x90)
        return true;
    if (c == 0xF4 && c1 > 0x8F)
        return true;
    return false;
}

// first bad byte (0..3) of the quad at in_s[q], 4 if none
__device__ __forceinline__ uint32_t u8_first_bad_quad(const uint32_t *in_s, int q)
{
    const uint8_t *b = reinterpret_cast<const uint8_t *>(in_s + q);
    for (uint32_t k = 0; k < 4; ++k)
        if (u8_bad_at(b + k))
            return k;
    return 4;
}

struct WarpResult {
    uint32_t err;   // 1 if the warp's chunk holds the first bad unit of the tile
    uint32_t pos;   // tile-relative byte offset (aligned frame) of that unit
    uint32_t units; // output units before it (or all of the chunk's units)
    uint32_t pad;
};

// ============================================================ K1: utf8->utf16

struct alignas(8) SelPair {
    uint32_t s01, s23;
};

// words of a quad: lo/hi byte planes -> up to four packed UTF-16 words
__device__ __forceinline__ void u8_decode_quad(uint32_t x, uint32_t xn, const U8Masks &m, uint32_t fi1, bool any4,
                                               uint32_t &lo, uint32_t &hi)
{
    const uint32_t n1 = fsr(x, xn, 8);
    const uint32_t n2 = fsr(x, xn, 16);
    const uint32_t lo3 = ((n1 << 6) & 0xC0C0C0C0u) | (n2 & 0x3F3F3F3Fu);
    const uint32_t hi3 = ((x << 4) & 0xF0F0F0F0u) | ((n1 >> 2) & 0x0F0F0F0Fu);
    const uint32_t lo2 = ((x << 6) & 0xC0C0C0C0u) | (n1 & 0x3F3F3F3Fu);
    const uint32_t hi2 = (x >> 2) & 0x07070707u;
    const uint32_t sA = sgn8(x);
    const uint32_t sL = sgn8(m.L);
    const uint32_t sE = sgn8(m.E);
    const uint32_t sF = sgn8(m.F);
    const uint32_t sS = sgn8(m.C & fi1); // first continuation after an F lead: low surrogate
    const uint32_t s2 = sL & ~sE;
    const uint32_t s3 = sE & ~sF;
    lo = (x & ~sA) | (lo2 & s2) | (lo3 & (s3 | sS));
    hi = (hi2 & s2) | (hi3 & s3);
    if (any4) {
        // high surrogate at the lead: 0xD7C0 + (cp >> 10)
        const uint32_t mm = ((n1 << 2) & 0xFCFCFCFCu) | ((n2 >> 4) & 0x03030303u);
        const uint32_t lo4 = ((mm | H8) - 0x40404040u) ^ (~mm & H8); // bytewise mm - 0x40
        const uint32_t carry = ((n1 >> 4) | (n1 >> 5)) & 0x01010101u;
        const uint32_t hi4 = (x & 0x07070707u) + carry + 0xD7D7D7D7u;
        // low surrogate at the first continuation: 0xDC00 | cp & 0x3FF
        const uint32_t hiS = 0xDCDCDCDCu | ((n1 >> 2) & 0x03030303u);
        lo |= lo4 & sF;
        hi |= (hi4 & sF) | (hiS & sS);
    }
}

template <bool Boundary>
__device__ __forceinline__ void u8u16_warp(const uint32_t *in_s, uint16_t *out_w, const SelPair *sel,
                                           int64_t tile_off, int64_t lo_b, int64_t hi_b, WarpResult &wr)
{
    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const int q0 = kInHead + (int)warp * kChunkQuads;
    uint32_t running = 0;
    uint32_t err = 0, err_pos = 0, units = 0;

#pragma unroll 1
    for (int g = 0; g < kGroups; ++g) {
        uint32_t x[kGroup], xn[kGroup], fi1[kGroup], e[kGroup];
        U8Masks mk[kGroup];
        uint32_t det = 0, pk = 0;
        const int qg = q0 + g * kGroup * 32;
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
            const int q = qg + j * 32 + (int)lane;
            x[j] = in_s[q];
            const uint32_t xp = in_s[q - 1];
            xn[j] = in_s[q + 1];
            mk[j] = u8_classify(x[j]);
            const U8Masks mp = u8_classify(xp);
            fi1[j] = fsl(mp.F, mk[j].F, 8);
            e[j] = (~mk[j].C | fi1[j]) & H8;
            if (Boundary)
                e[j] &= valid_mask(tile_off + 4 * (int64_t)(q - kInHead), lo_b, hi_b);
            const bool any_f = __any_sync(0xffffffffu, (mk[j].F | mp.F) != 0);
            det |= u8_detect(x[j], xn[j], mk[j], mp, any_f);
            pk |= (uint32_t)__popc(e[j]) << (8 * j);
        }
        if (g == kGroups - 1 && lane == 31) {
            // chunk end: leads of the last quad whose continuations lie past the chunk
            const uint32_t cn = u8_classify(xn[kGroup - 1]).C;
            const U8Masks &m = mk[kGroup - 1];
            const uint32_t c = m.C;
            det |= (m.L & ~fsr(c, cn, 8)) | (m.E & ~fsr(c, cn, 16)) | (m.F & ~fsr(c, cn, 24));
        }
        const uint32_t incl = warp_scan_packed(pk);
        const uint32_t excl = incl - pk;
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);

        if (__any_sync(0xffffffffu, det != 0)) {
            // exact resolution, in stream order
            bool found = false;
            if (g > 0) {
                // the three bytes before the group (a lead there may miss a
                // continuation that only this group's detector saw)
                uint32_t tb = 3;
                if (lane == 0) {
                    const uint8_t *b = reinterpret_cast<const uint8_t *>(in_s + qg);
                    for (uint32_t k = 0; k < 3; ++k)
                        if (u8_bad_at(b - 3 + (int)k)) {
                            tb = k;
                            break;
                        }
                }
                tb = __shfl_sync(0xffffffffu, tb, 0);
                if (tb < 3) {
                    uint32_t drop = 0;
                    if (lane == 0) {
                        const uint32_t xq = in_s[qg - 1];
                        const U8Masks mq = u8_classify(xq);
                        const U8Masks mqq = u8_classify(in_s[qg - 2]);
                        uint32_t eq = (~mq.C | fsl(mqq.F, mq.F, 8)) & H8;
                        if (Boundary)
                            eq &= valid_mask(tile_off + 4 * (int64_t)(qg - 1 - kInHead), lo_b, hi_b);
                        // bytes 1+tb .. 3 of that quad are at or after the error
                        eq &= ~((1u << (8 * (1 + tb))) - 1u);
                        drop = (uint32_t)__popc(eq);
                    }
                    drop = __shfl_sync(0xffffffffu, drop, 0);
                    err = 1;
                    err_pos = 4u * (uint32_t)(qg - kInHead) - 3u + tb;
                    units = running - drop;
                    found = true;
                }
            }
            uint32_t before = running;
#pragma unroll
            for (int j = 0; j < kGroup; ++j) {
                if (!found) {
                    const int q = qg + j * 32 + (int)lane;
                    const uint32_t kb = u8_first_bad_quad(in_s, q);
                    const uint32_t bm = __ballot_sync(0xffffffffu, kb < 4);
                    if (bm) {
                        const uint32_t fl = (uint32_t)__ffs(bm) - 1;
                        const uint32_t within = (uint32_t)__popc(e[j] & ((1u << (8 * (kb & 3))) - 1u)) +
                                                ((excl >> (8 * j)) & 0xFFu);
                        const uint32_t kbf = __shfl_sync(0xffffffffu, kb, fl);
                        const uint32_t wf = __shfl_sync(0xffffffffu, within, fl);
                        err = 1;
                        err_pos = 4u * (uint32_t)(qg + j * 32 + (int)fl - kInHead) + kbf;
                        units = before + wf;
                        found = true;
                    }
                }
                before += (tot >> (8 * j)) & 0xFFu;
            }
        }

        // decode + compact into the warp's staging region
        uint32_t base = running;
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
            const bool any4 = __any_sync(0xffffffffu, (mk[j].F | (mk[j].C & fi1[j])) != 0);
            uint32_t lo, hi;
            u8_decode_quad(x[j], xn[j], mk[j], fi1[j], any4, lo, hi);
            const uint32_t idx = (e[j] * 0x00204081u) >> 28;
            const SelPair sp = sel[idx];
            const uint32_t w01 = prmt(lo, hi, sp.s01);
            const uint32_t w23 = prmt(lo, hi, sp.s23);
            const uint32_t c = (uint32_t)__popc(e[j]);
            uint16_t *dst = out_w + base + ((excl >> (8 * j)) & 0xFFu);
            if (c > 0)
                dst[0] = (uint16_t)w01;
            if (c > 1)
                dst[1] = (uint16_t)(w01 >> 16);
            if (c > 2)
                dst[2] = (uint16_t)w23;
            if (c > 3)
                dst[3] = (uint16_t)(w23 >> 16);
            base += (tot >> (8 * j)) & 0xFFu;
        }
        running = base;
        if (err)
            break;
    }
    if (!err)
        units = running;
    if (lane == 0) {
        wr.err = err;
        wr.pos = err_pos;
        wr.units = units;
    }
}

// ============================================================ K3: validate

template <bool Boundary>
__device__ __forceinline__ void u8val_warp(const uint32_t *in_s, int64_t tile_off, int64_t lo_b, int64_t hi_b,
                                           WarpResult &wr)
{
    (void)tile_off;
    (void)lo_b;
    (void)hi_b;
    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const int q0 = kInHead + (int)warp * kChunkQuads;
    uint32_t err = 0, err_pos = 0;
#pragma unroll 4
    for (int s = 0; s < kSteps; ++s) {
        const int q = q0 + s * 32 + (int)lane;
        const uint32_t x = in_s[q];
        const uint32_t xp = in_s[q - 1];
        const uint32_t xn = in_s[q + 1];
        const U8Masks m = u8_classify(x);
        const U8Masks mp = u8_classify(xp);
        const bool any_f = __any_sync(0xffffffffu, (m.F | mp.F) != 0);
        uint32_t det = u8_detect(x, xn, m, mp, any_f);
        if (s == kSteps - 1 && lane == 31) {
            const uint32_t cn = u8_classify(xn).C;
            det |= (m.L & ~fsr(m.C, cn, 8)) | (m.E & ~fsr(m.C, cn, 16)) | (m.F & ~fsr(m.C, cn, 24));
        }
        if (__any_sync(0xffffffffu, det != 0)) {
            const int qs = q0 + s * 32;
            uint32_t tb = 3;
            if (s > 0 && lane == 0) {
                const uint8_t *b = reinterpret_cast<const uint8_t *>(in_s + qs);
                for (uint32_t k = 0; k < 3; ++k)
                    if (u8_bad_at(b - 3 + (int)k)) {
                        tb = k;
                        break;
                    }
            }
            tb = __shfl_sync(0xffffffffu, tb, 0);
            if (tb < 3) {
                err = 1;
                err_pos = 4u * (uint32_t)(qs - kInHead) - 3u + tb;
                break;
            }
            const uint32_t kb = u8_first_bad_quad(in_s, q);
            const uint32_t bm = __ballot_sync(0xffffffffu, kb < 4);
            if (bm) {
                const uint32_t fl = (uint32_t)__ffs(bm) - 1;
                err = 1;
                err_pos = 4u * (uint32_t)(qs + (int)fl - kInHead) + __shfl_sync(0xffffffffu, kb, fl);
                break;
            }
        }
    }
    if (lane == 0) {
        wr.err = err;
        wr.pos = err_pos;
        wr.units = 0;
    }
}

} // namespace lu
