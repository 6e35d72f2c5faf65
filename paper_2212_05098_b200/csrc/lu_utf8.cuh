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
// Work layout: a warp owns a contiguous 2 KiB chunk of its CTA's 16 KiB tile
// and walks it in 4 rounds of 512 B; in a round lane l holds bytes
// [16l, 16l+16) in registers (one coalesced 16-byte load), i.e. four 32-bit
// "quads".  Neighbour quads come from warp shuffles.  Per quad the kernels
// build SWAR byte masks (bit 7 of each byte): C = continuation, L = >=C0,
// E = >=E0, F = >=F0.  A cheap detector ("must be a continuation" xor C, the
// C0/C1 test, and second-byte range tests behind a warp-uniform prefilter)
// flags any round that may hold a bad byte; a flagged round is resolved by
// the exact predicate (u8_bad_at), the only source of error offsets.
#pragma once

#include "lu_common.cuh"

#include <type_traits>

#ifndef LU_ONE_VOTE
#define LU_ONE_VOTE 1
#endif
#ifndef LU_K1_CHUNK5
#define LU_K1_CHUNK5 1 // ... and for the BMP class
#endif
#ifndef LU_K1_CHUNK3
#define LU_K1_CHUNK3 1 // K1: straight-line chunks for class 3 (ASCII + 4-byte) too
#endif
#ifndef LU_MERGED_TERMS
#define LU_MERGED_TERMS 1
#endif

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

// byte at aligned-frame offset a, 0 outside [lo, hi) (rare paths only)
__device__ __forceinline__ uint32_t gbyte(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    return (a >= lo && a < hi) ? (uint32_t)base[a] : 0u;
}

__device__ __forceinline__ bool u8_bad_global(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    uint8_t w[7];
#pragma unroll
    for (int k = 0; k < 7; ++k)
        w[k] = (uint8_t)gbyte(base, a - 3 + k, lo, hi);
    return u8_bad_at(w + 3);
}

// emit mask of the quad at aligned offset a (rare path: error fix-ups)
__device__ __forceinline__ uint32_t u8_emit_global(const uint8_t *base, int64_t a, int64_t lo, int64_t hi)
{
    uint32_t x = 0, xp = 0, vm = 0;
    for (int k = 0; k < 4; ++k) {
        x |= gbyte(base, a + k, lo, hi) << (8 * k);
        xp |= gbyte(base, a - 4 + k, lo, hi) << (8 * k);
        if (a + k >= lo && a + k < hi)
            vm |= 0x80u << (8 * k);
    }
    const U8Masks m = u8_classify(x), p = u8_classify(xp);
    return (~m.C | fsl(p.F, m.F, 8)) & H8 & vm;
}

struct WarpResult {
    uint32_t err;   // 1 if the warp's chunk holds the first bad unit of the tile
    uint32_t pos;   // tile-relative byte offset (aligned frame) of that unit
    uint32_t units; // output units before it (or all of the chunk's units)
    uint32_t pad;
};

// One round's detector + masks, shared by K1 and K3.
//
// Like the paper's engines (ASCII and 1/2-byte fast paths,
// /root/reference/pkg/src/laneutf/utf8_to_utf16.py:245-276), a warp round
// picks the cheapest exact path its bytes allow (warp-uniform votes):
//   path 0  no byte >= E0 in the round or its look-behind: ASCII + 2-byte
//           leads only, "must be continuation" = L(i-1);
//   path 1  no F-class byte and no 2-byte lead: ASCII + 3-byte leads;
//   path 3  no 2-byte and no 3-byte lead: ASCII + 4-byte leads (text
//           outside the BMP, e.g. emoji); only the F0/F4/F5+ range check;
//   path 2  everything else (general detector and decoder).
// Every path flags every bad byte its class mix can contain.
struct U8Round {
    uint32_t w[6];   // xp, q0..q3, xn
    U8Masks m[5];    // masks of w[0..4] (F only computed off path 0)
    uint32_t key[5]; // path 3 (fast): per byte plane - 1 of a 4-byte lead (u8_plane_m1), quads 1..4
    uint32_t det;    // nonzero: a bad byte may lie in this lane's 16 bytes
    int path;
    uint32_t next;   // u8_round_detect: the class hint for the warp's next round (path, or kHintBmp)
};

// Class hint beyond the paths 0..3: ASCII + 2-byte + 3-byte leads, no F-class
// byte and no E0 / ED lead (BMP text of mixed scripts, e.g. accented Latin with
// typographic punctuation or currency signs): u8_fast01 / u8u16_round<kHintBmp>.
constexpr uint32_t kHintBmp = 5;

// E0 80..9F (overlong) / ED A0..BF (surrogate): u = (b&0xF)<<1 | bit5(c1) in {0, 27}
__device__ __forceinline__ uint32_t u8_check_e(uint32_t x, uint32_t n1, const U8Masks &c)
{
    const uint32_t u = ((x & 0x0F0F0F0Fu) << 1) | ((n1 >> 5) & 0x01010101u);
    return c.E & ~c.F & ~((u + 0x7F7F7F7Fu) & ((u ^ 0x1B1B1B1Bu) + 0x7F7F7F7Fu));
}
// Per byte (a 4-byte lead x with second byte n1): plane - 1 in bits 0..4,
// where plane = (x & 7) << 2 | (n1 >> 4) & 3 is the code point >> 16.  Valid
// planes are 1..16, so bit 4 is set exactly for plane 0 (F0 80..8F, overlong)
// and planes 17..31 (F4 90.. / F5..F7, > U+10FFFF); bit 5 keeps the
// subtraction from borrowing across bytes.  The path-3 decoder reuses the
// value (high surrogate = D800 | (plane - 1) << 6 | ...).
__device__ __forceinline__ uint32_t u8_plane_m1(uint32_t x, uint32_t n1)
{
    return (((x & 0x07070707u) << 2) | ((n1 >> 4) & 0x03030303u) | 0x20202020u) - 0x01010101u;
}
// F0 80..8F (overlong), F4 90.. / F5..F7 (> U+10FFFF), F8..FF
__device__ __forceinline__ uint32_t u8_check_f(uint32_t x, uint32_t n1, const U8Masks &c)
{
    return c.F & ((u8_plane_m1(x, n1) << 3) | (x << 4));
}
// E-class bytes whose low nibble is 0, D, E or F (E0 / ED candidates)
__device__ __forceinline__ uint32_t u8_prefilter_e(uint32_t x, const U8Masks &c)
{
    const uint32_t v = x + 0x03030303u;
    return c.E & ~(v << 4) & ~(v << 5);
}

__device__ __forceinline__ void u8_round_detect(U8Round &R)
{
    uint32_t anye = 0;
#pragma unroll
    for (int k = 0; k <= 4; ++k) {
        const uint32_t x = R.w[k];
        const uint32_t t1 = x << 1;
        R.m[k].C = x & ~t1 & H8;
        R.m[k].L = x & t1 & H8;
        R.m[k].E = R.m[k].L & (x << 2);
        R.m[k].F = 0;
        anye |= R.m[k].E;
    }
    uint32_t det = 0;
    if (!__any_sync(0xffffffffu, anye != 0)) {
        R.path = 0;
        R.next = 0;
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            const U8Masks &c = R.m[k];
            det |= fsl(R.m[k - 1].L, c.L, 8) ^ c.C;
            det |= c.L & ~((R.w[k] & 0x1E1E1E1Eu) + 0x7F7F7F7Fu); // C0 / C1
        }
        R.det = det;
        return;
    }
    uint32_t anyf = 0, any2 = 0;
#pragma unroll
    for (int k = 0; k <= 4; ++k) {
        R.m[k].F = R.m[k].E & (R.w[k] << 3);
        anyf |= R.m[k].F;
        if (k > 0)
            any2 |= R.m[k].L & ~R.m[k].E;
    }
    if (!__any_sync(0xffffffffu, (anyf | any2) != 0)) {
        R.path = 1;
        R.next = 1;
        uint32_t pe = 0;
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            const U8Masks &c = R.m[k], &p = R.m[k - 1];
            det |= (fsl(p.L, c.L, 8) | fsl(p.E, c.E, 16)) ^ c.C;
            pe |= u8_prefilter_e(R.w[k], c);
        }
        if (__any_sync(0xffffffffu, pe != 0)) {
#pragma unroll
            for (int k = 1; k <= 4; ++k)
                det |= u8_check_e(R.w[k], fsr(R.w[k], R.w[k + 1], 8), R.m[k]);
        }
        R.det = det;
        return;
    }
    uint32_t any3 = 0; // 3-byte leads (only needed once path 1 is ruled out)
#pragma unroll
    for (int k = 1; k <= 4; ++k)
        any3 |= R.m[k].E & ~R.m[k].F;
    if (!__any_sync(0xffffffffu, (any2 | any3) != 0)) {
        R.path = 3;
        R.next = 3;
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            const U8Masks &c = R.m[k], &p = R.m[k - 1];
            det |= (fsl(p.L, c.L, 8) | fsl(p.E, c.E, 16) | fsl(p.F, c.F, 24)) ^ c.C;
            det |= u8_check_f(R.w[k], fsr(R.w[k], R.w[k + 1], 8), c);
        }
        R.det = det;
        return;
    }
    R.path = 2;
    uint32_t pe = 0;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
        const U8Masks &c = R.m[k], &p = R.m[k - 1];
        const uint32_t x = R.w[k];
        det |= (fsl(p.L, c.L, 8) | fsl(p.E, c.E, 16) | fsl(p.F, c.F, 24)) ^ c.C;
        det |= c.L & ~c.E & ~((x & 0x1E1E1E1Eu) + 0x7F7F7F7Fu); // C0 / C1
        pe |= u8_prefilter_e(x, c);
    }
    R.next = kHintBmp; // no F-class byte and no E0 / ED lead in the round: the BMP class next time
    if (__any_sync(0xffffffffu, (pe | anyf) != 0)) {
        R.next = 2;
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            const uint32_t n1 = fsr(R.w[k], R.w[k + 1], 8);
            det |= u8_check_e(R.w[k], n1, R.m[k]) | u8_check_f(R.w[k], n1, R.m[k]);
        }
    }
    R.det = det;
}

// chunk end (lane 31, last round): leads of the last quad whose
// continuations would lie past the chunk, checked against the halo quad
__device__ __forceinline__ uint32_t u8_chunk_end_check(const U8Round &R)
{
    const uint32_t cn = u8_classify(R.w[5]).C;
    const U8Masks &m = R.m[4];
    return (m.L & ~fsr(m.C, cn, 8)) | (m.E & ~fsr(m.C, cn, 16)) | (m.F & ~fsr(m.C, cn, 24));
}

// Speculative per-class detectors.  A warp predicts that a round has the same
// class mix as its previous one (the path `hint`) and runs only that path's
// detector, which flags every bad byte the path's class can contain AND every
// byte outside the class (a lead of another length, a continuation the class
// cannot claim).  If nothing is flagged anywhere in the warp the prediction
// holds and the round takes that path with det = 0, so one vote replaces the
// general detector's two to four class votes; otherwise the general detector
// (u8_round_detect) runs and its path becomes the next hint.  The masks are
// filled as the path's decoder and chunk-end check expect (exact when the
// prediction holds).
//
// "Must be a continuation" is computed arithmetically on the FMA pipe where
// the class allows it: for path 1 it is E(i-1) | E(i-2) = E * 0x10100 (low
// word) plus the previous quad's spill (high word of the same product); for
// path 3, F * 0x01010100.  Terms overlap only where a lead follows a lead
// that needed a continuation, which is flagged one byte earlier, so the sum
// (carries fall outside bit 7 or onto already-flagged bytes) is as good as
// the OR.  Returns a value whose bit 7 bytes flag; other bits are garbage.

// path 0: ASCII and 2-byte leads only
__device__ __forceinline__ uint32_t u8_fast0(U8Round &R)
{
    uint32_t Lp;
    {
        const uint32_t x = R.w[0];
        Lp = x & (x << 1) & H8;
    }
    uint32_t det = 0;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
        const uint32_t x = R.w[k];
        const uint32_t t1 = x << 1;
        const uint32_t C = x & ~t1 & H8, L = x & t1 & H8;
        det |= fsl(Lp, L, 8) ^ C;                          // continuation structure
#if LU_MERGED_TERMS
        // a lead >= E0 (not this class) or C0 / C1: one LOP3 per term pair
        det |= L & ((x << 2) | ~((x & 0x1E1E1E1Eu) + 0x7F7F7F7Fu));
#else
        det |= L & (x << 2);                               // a lead >= E0: not this class
        det |= L & ~((x & 0x1E1E1E1Eu) + 0x7F7F7F7Fu);      // C0 / C1
#endif
        R.m[k].C = C;
        R.m[k].L = L;
        R.m[k].E = 0;
        R.m[k].F = 0;
        Lp = L;
    }
    return det & H8;
}

// path 1: ASCII and 3-byte leads only
__device__ __forceinline__ uint32_t u8_fast1(U8Round &R)
{
    uint32_t Ep;
    {
        const uint32_t x = R.w[0];
        Ep = x & (x << 1) & (x << 2) & H8;
    }
    uint32_t spill = __umulhi(Ep, 0x10100u);
    uint32_t det = 0;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
        const uint32_t x = R.w[k];
        const uint32_t t1 = x << 1, t2 = x << 2;
        const uint32_t C = x & ~t1 & H8, L = x & t1 & H8;
        const uint32_t E = L & t2;
        const uint32_t need = E * 0x10100u + spill;        // E(i-1) | E(i-2)
        spill = __umulhi(E, 0x10100u);
        det |= need ^ C;
        const uint32_t v = x + 0x03030303u;                // E0 / ED candidates (u8_prefilter_e)
#if LU_MERGED_TERMS
        // a 2-byte lead, an F-class byte, or an E0 / ED candidate: with
        // E = L & t2, L & ~t2 | E & (x3 | ~v4 & ~v5) = L & (~t2 | x3 | ~(v4 | v5))
        det |= L & (~t2 | (x << 3) | ~((v << 4) | (v << 5)));
#else
        det |= L & ~t2;                                    // a 2-byte lead: not this class
        det |= E & (x << 3);                               // an F-class byte: not this class
        det |= E & ~(v << 4) & ~(v << 5);
#endif
        R.m[k].C = C;
        R.m[k].L = E;
        R.m[k].E = E;
        R.m[k].F = 0;
    }
    return det & H8;
}

// path 3: ASCII and 4-byte leads only (text outside the BMP, e.g. emoji)
__device__ __forceinline__ uint32_t u8_fast3(U8Round &R)
{
    {
        const uint32_t x = R.w[0];
        R.m[0].F = x & (x << 1) & (x << 2) & (x << 3) & H8;
    }
    uint32_t spill = __umulhi(R.m[0].F, 0x01010100u);
    uint32_t det = 0;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
        const uint32_t x = R.w[k];
        const uint32_t t1 = x << 1;
        const uint32_t C = x & ~t1 & H8, L = x & t1 & H8;
        const uint32_t F = L & (x << 2) & (x << 3);
        const uint32_t need = F * 0x01010100u + spill;     // F(i-1) | F(i-2) | F(i-3)
        spill = __umulhi(F, 0x01010100u);
        det |= need ^ C;
        det |= L & ~F;                                     // a 2- or 3-byte lead: not this class
        // F0 80..8F, F4 90.., F5..FF (u8_check_f); plane - 1 is kept for the decoder
        const uint32_t key = u8_plane_m1(x, fsr(x, R.w[k + 1], 8));
        det |= F & ((key << 3) | (x << 4));
        R.key[k] = key;
        R.m[k].C = C;
        R.m[k].L = F;
        R.m[k].E = F;
        R.m[k].F = F;
    }
    return det & H8;
}

// BMP class (kHintBmp): ASCII, 2-byte and 3-byte leads; flags F-class bytes and
// E0 / ED candidates (so no second-byte range check is needed), C0 / C1 and
// every continuation the leads do not claim
__device__ __forceinline__ uint32_t u8_fast01(U8Round &R)
{
    uint32_t Lp, Ep;
    {
        const uint32_t x = R.w[0];
        Lp = x & (x << 1) & H8;
        Ep = Lp & (x << 2);
    }
    uint32_t det = 0;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
        const uint32_t x = R.w[k];
        const uint32_t t1 = x << 1, t2 = x << 2;
        const uint32_t C = x & ~t1 & H8, L = x & t1 & H8;
        const uint32_t E = L & t2;
        det |= (fsl(Lp, L, 8) | fsl(Ep, E, 16)) ^ C;
        det |= L & ~t2 & ~((x & 0x1E1E1E1Eu) + 0x7F7F7F7Fu); // C0 / C1
        const uint32_t u = x + 0x03030303u;                   // E0 / ED candidates (u8_prefilter_e)
        det |= E & ((x << 3) | ~((u << 4) | (u << 5)));       // an F-class byte or a candidate
        R.m[k].C = C;
        R.m[k].L = L;
        R.m[k].E = E;
        R.m[k].F = 0;
        Lp = L;
        Ep = E;
    }
    return det & H8;
}

// Round detection with the warp's path prediction (see above); hint is
// warp-uniform, updated to the round's actual path on a miss.
// Returns true when the prediction held (R.det = 0).  check_end (lane 31 in
// the chunk's last round): the chunk-end check joins the prediction vote, so a
// predicted round never needs the resolution vote; on a miss the caller adds
// it to R.det.
__device__ __forceinline__ bool u8_round_detect_spec(U8Round &R, uint32_t &hint, bool check_end = false)
{
    uint32_t fd;
    switch (hint) {
    case 0:
        fd = u8_fast0(R);
        break;
    case 1:
        fd = u8_fast1(R);
        break;
    case 3:
        fd = u8_fast3(R);
        break;
    default:
        fd = 1;
        break;
    }
    if (check_end)
        fd |= u8_chunk_end_check(R);
    if (__any_sync(0xffffffffu, fd != 0)) {
        u8_round_detect(R);
        hint = (uint32_t)R.path;
        return false;
    }
    R.path = (int)hint;
    R.det = 0;
    return true;
}

// ============================================================ K1: utf8->utf16

struct alignas(8) SelPair {
    uint32_t s01, s23;
};

// lo/hi byte planes of the UTF-16 word emitted at each byte position
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
    const uint32_t s2 = sgn8(m.L & ~m.E);
    const uint32_t s3 = sgn8(m.E & ~m.F);
    lo = (x & ~sA) | (lo2 & s2) | (lo3 & s3);
    hi = (hi2 & s2) | (hi3 & s3);
    if (any4) {
        const uint32_t sF = sgn8(m.F);
        const uint32_t sS = sgn8(m.C & fi1); // first continuation after an F lead: low surrogate
        // high surrogate at the lead: 0xD7C0 + (cp >> 10)
        const uint32_t mm = ((n1 << 2) & 0xFCFCFCFCu) | ((n2 >> 4) & 0x03030303u);
        const uint32_t lo4 = ((mm | H8) - 0x40404040u) ^ (~mm & H8); // bytewise mm - 0x40
        const uint32_t carry = ((n1 >> 4) | (n1 >> 5)) & 0x01010101u;
        const uint32_t hi4 = (x & 0x07070707u) + carry + 0xD7D7D7D7u;
        // low surrogate at the first continuation: 0xDC00 | cp & 0x3FF
        const uint32_t hiS = 0xDCDCDCDCu | ((n1 >> 2) & 0x03030303u);
        lo |= (lo4 & sF) | (lo3 & sS);
        hi |= (hi4 & sF) | (hiS & sS);
    }
}

// path 3: ASCII and 4-byte leads only.  Non-ASCII bytes are F leads (high
// surrogate) or continuations; every continuation gets the low-surrogate
// form, which is right for the first one after a lead and never emitted for
// the others.
__device__ __forceinline__ void u8_decode4(uint32_t x, uint32_t xn, const U8Masks &m, uint32_t key, uint32_t &lo,
                                           uint32_t &hi)
{
    const uint32_t n1 = fsr(x, xn, 8);
    const uint32_t n2 = fsr(x, xn, 16);
    // low surrogate at the first continuation: DC00 | (b1 & 0xF) << 6 | b2 & 0x3F
    const uint32_t lo3 = ((n1 << 6) & 0xC0C0C0C0u) | (n2 & 0x3F3F3F3Fu);
    const uint32_t hiS = 0xDCDCDCDCu | ((n1 >> 2) & 0x03030303u);
    // high surrogate at the lead: (cp >> 10) - 0x40 = (plane - 1) << 6 | (b1 & 0xF) << 2 | b2 >> 4 & 3;
    // key = plane - 1 in bits 0..4 (u8_plane_m1, computed by the detector)
    const uint32_t km1 = key;
    const uint32_t hi4 = ((km1 >> 2) & 0x07070707u) | 0xD8D8D8D8u;
    const uint32_t lo4 = ((km1 << 6) & 0xC0C0C0C0u) | ((n1 << 2) & 0x3C3C3C3Cu) | ((n2 >> 4) & 0x03030303u);
    const uint32_t sA = sgn8(x);
    const uint32_t sF = sgn8(m.F);
    lo = (x & ~sA) | (((lo4 & sF) | (lo3 & ~sF)) & sA);
    hi = ((hi4 & sF) | (hiS & ~sF)) & sA;
}

// path 0: ASCII and 2-byte leads only
__device__ __forceinline__ void u8_decode2(uint32_t x, uint32_t xn, uint32_t &lo, uint32_t &hi)
{
    const uint32_t n1 = fsr(x, xn, 8);
    const uint32_t lo2 = ((x << 6) & 0xC0C0C0C0u) | (n1 & 0x3F3F3F3Fu);
    const uint32_t sA = sgn8(x);
    lo = (x & ~sA) | (lo2 & sA);
    hi = (x >> 2) & 0x07070707u & sA;
}

// path 1: ASCII and 3-byte leads only
__device__ __forceinline__ void u8_decode3(uint32_t x, uint32_t xn, uint32_t &lo, uint32_t &hi)
{
    const uint32_t n1 = fsr(x, xn, 8);
    const uint32_t n2 = fsr(x, xn, 16);
    const uint32_t lo3 = ((n1 << 6) & 0xC0C0C0C0u) | (n2 & 0x3F3F3F3Fu);
    const uint32_t hi3 = ((x << 4) & 0xF0F0F0F0u) | ((n1 >> 2) & 0x0F0F0F0Fu);
    const uint32_t sA = sgn8(x);
    lo = (x & ~sA) | (lo3 & sA);
    hi = hi3 & sA;
}

// class hint of a warp whose last chunk was all ASCII (hints 0..3 are the class paths)
constexpr uint32_t kHintAscii = 4;

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void sts16_if(uint32_t addr, uint32_t v, uint32_t room, uint32_t j)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.gt.u32 p, %2, %3;\n\t@p st.shared.u16 [%0], %1;\n\t}" ::"r"(addr),
                 "h"((unsigned short)v), "r"(room), "r"(j)
                 : "memory");
}

// One round's emit masks, scan, exact error resolution, decode and
// compaction for a statically known class path P (0, 1, 3; 2 = general), so
// each path's live ranges stay separate.
template <int P, bool Boundary, bool BE>
__device__ __forceinline__ void u8u16_round(const U8Round &R, int r, const uint8_t *__restrict__ base, int64_t tile_off,
                                            int64_t chunk, int64_t lane_off, int64_t lo_b, int64_t hi_b,
                                            uint32_t sbase, const SelPair *sel, uint32_t &running, uint32_t &err,
                                            uint32_t &err_pos, uint32_t &units)
{
    const uint32_t lane = lane_id();
    uint32_t e[4], fi1[4], c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (P == 2 || P == 3) {
            fi1[k] = fsl(R.m[k].F, R.m[k + 1].F, 8);
            e[k] = (~R.m[k + 1].C | fi1[k]) & H8;
        } else {
            fi1[k] = 0;
            e[k] = ~R.m[k + 1].C & H8;
        }
        if (Boundary)
            e[k] &= valid_mask(lane_off + 4 * k, lo_b, hi_b);
        c[k] = (uint32_t)__popc(e[k]);
    }
    const uint32_t cnt = c[0] + c[1] + c[2] + c[3];
    const uint32_t incl = warp_incl_scan(cnt);
    const uint32_t excl = incl - cnt;
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);

    // a predicted (fast) round has det = 0 (lane 31's chunk-end check joined
    // the prediction vote): no resolution vote
    if (P == 2 && __any_sync(0xffffffffu, R.det != 0)) {
        // exact resolution in stream order: tail of the previous round first
        const int64_t rstart = chunk + r * 512;
        bool found = false;
        if (r > 0) {
            uint32_t tb = 3;
            if (lane == 0) {
                for (uint32_t t = 0; t < 3; ++t)
                    if (u8_bad_global(base, rstart - 3 + t, lo_b, hi_b)) {
                        tb = t;
                        break;
                    }
            }
            tb = __shfl_sync(0xffffffffu, tb, 0);
            if (tb < 3) {
                uint32_t drop = 0;
                if (lane == 0) {
                    // emits of the previous round's last quad at or after the error
                    const uint32_t eq = u8_emit_global(base, rstart - 4, lo_b, hi_b);
                    drop = (uint32_t)__popc(eq & ~((1u << (8 * (1 + tb))) - 1u));
                }
                drop = __shfl_sync(0xffffffffu, drop, 0);
                err = 1;
                err_pos = (uint32_t)(rstart - 3 + tb - tile_off);
                units = running - drop;
                found = true;
            }
        }
        if (!found) {
            // a lead missing a continuation is flagged at the continuation
            // slot, possibly in the next lane: scan when either lane flagged
            const uint32_t scan = R.det | __shfl_down_sync(0xffffffffu, R.det, 1);
            uint32_t kb = 16;
            if (scan != 0) {
                for (uint32_t t = 0; t < 16; ++t)
                    if (u8_bad_global(base, lane_off + t, lo_b, hi_b)) {
                        kb = t;
                        break;
                    }
            }
            const uint32_t bm = __ballot_sync(0xffffffffu, kb < 16);
            if (bm) {
                const uint32_t fl = (uint32_t)__ffs(bm) - 1;
                uint32_t em = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    em |= ((e[k] * 0x00204081u) >> 28) << (4 * k);
                const uint32_t within = excl + (uint32_t)__popc(em & ((1u << (kb & 15)) - 1u));
                const uint32_t kbf = __shfl_sync(0xffffffffu, kb, fl);
                const uint32_t wf = __shfl_sync(0xffffffffu, within, fl);
                err = 1;
                err_pos = (uint32_t)(rstart - tile_off) + 16 * fl + kbf;
                units = running + wf;
            }
        }
    }

    // decode + compact into the warp's staging region
    bool any4 = false;
    if (P == 2) {
        uint32_t f4 = R.m[0].F;
#pragma unroll
        for (int k = 1; k <= 4; ++k)
            f4 |= R.m[k].F;
        any4 = __any_sync(0xffffffffu, f4 != 0);
    }
    uint32_t lop[4], hip[4];
    if (P == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            u8_decode2(R.w[k + 1], R.w[k + 2], lop[k], hip[k]);
    } else if (P == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            u8_decode3(R.w[k + 1], R.w[k + 2], lop[k], hip[k]);
    } else if (P == 3) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            u8_decode4(R.w[k + 1], R.w[k + 2], R.m[k + 1], R.key[k + 1], lop[k], hip[k]);
    } else if (P == (int)kHintBmp) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            u8_decode_quad(R.w[k + 1], R.w[k + 2], R.m[k + 1], 0u, false, lop[k], hip[k]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            u8_decode_quad(R.w[k + 1], R.w[k + 2], R.m[k + 1], fi1[k], any4, lop[k], hip[k]);
    }
    uint32_t off = running + excl;
    const uint32_t lane_end = off + cnt;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t lo = lop[k], hi = hip[k];
        const uint32_t idx = (e[k] * 0x00204081u) >> 28;
        const SelPair sp = sel[idx];
        const uint32_t w01 = BE ? prmt(hi, lo, sp.s01) : prmt(lo, hi, sp.s01);
        const uint32_t w23 = BE ? prmt(hi, lo, sp.s23) : prmt(lo, hi, sp.s23);
        const uint32_t a = sbase + 2 * off;
        const uint32_t room = lane_end - off;
        // Stores past this quad's words are overwritten by the next
        // quad's stores (program order); only slots that valid input
        // could push into the next lane's region are predicated.
        if (Boundary) {
            sts16_if(a, w01, room, 0);
            sts16_if(a + 2, w01 >> 16, room, 1);
            sts16_if(a + 4, w23, room, 2);
            sts16_if(a + 6, w23 >> 16, room, 3);
        } else {
            sts16(a, w01);
            if (k < 3)
                sts16(a + 2, w01 >> 16);
            else
                sts16_if(a + 2, w01 >> 16, room, 1);
            if (k < 2)
                sts16(a + 4, w23);
            else
                sts16_if(a + 4, w23, room, 2);
            if (k < 1)
                sts16(a + 6, w23 >> 16);
            else
                sts16_if(a + 6, w23 >> 16, room, 3);
        }
        off += c[k];
    }
    running += tot;
}

// BE: emit UTF-16BE (the word's high byte first): the compaction prmt takes
// its two byte planes in the other order, at no cost.
// Straight-line chunk for an interior warp whose prediction is the fast
// class P: all four rounds take P's detector and tail with no branch between
// them (each round's prediction vote is only OR-ed into the result), so the
// compiler can overlap the rounds.  Returns nonzero if some round left the
// class (or lane 31's chunk-end check fired): the caller then redoes the chunk
// with the adaptive per-round path, which overwrites the staging region.
template <int P, bool BE>
__device__ __forceinline__ uint32_t u8u16_chunk_fast(const uint8_t *__restrict__ base, int64_t tile_off,
                                                     int64_t chunk, int64_t lo_b, int64_t hi_b, uint32_t sbase,
                                                     const SelPair *sel, const ChunkIn &in, const uint32_t *rn,
                                                     uint32_t &running)
{
    const uint32_t lane = lane_id();
    constexpr int kRounds = kChunkBytes / 512;
    const uint4 *q = in.q;
    uint32_t carry = in.halo_p;
    uint32_t miss = 0, err = 0, err_pos = 0, units = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t lane_off = chunk + r * 512 + 16 * (int64_t)lane;
        const uint32_t rp = __shfl_sync(0xffffffffu, q[r].w, (lane + 31) & 31);
        U8Round R;
        R.w[0] = (lane == 0) ? carry : rp;
        carry = rp;
        R.w[1] = q[r].x;
        R.w[2] = q[r].y;
        R.w[3] = q[r].z;
        R.w[4] = q[r].w;
        R.w[5] = (lane == 31) ? (r + 1 < kRounds ? rn[r + 1 < kRounds ? r + 1 : r] : in.halo_n) : rn[r];
        uint32_t fd = P == 0 ? u8_fast0(R) : P == 1 ? u8_fast1(R) : P == 3 ? u8_fast3(R) : u8_fast01(R);
        if (r == kRounds - 1 && lane == 31)
            fd |= u8_chunk_end_check(R);
#if LU_ONE_VOTE
        miss |= fd; // one vote for the chunk, below
#else
        miss |= __any_sync(0xffffffffu, fd != 0) ? 1u : 0u;
#endif
        R.path = P;
        R.det = 0;
        u8u16_round<P, false, BE>(R, r, base, tile_off, chunk, lane_off, lo_b, hi_b, sbase, sel, running, err,
                                  err_pos, units);
    }
#if LU_ONE_VOTE
    return __any_sync(0xffffffffu, miss != 0) ? 1u : 0u;
#else
    return miss;
#endif
}

template <bool Boundary, bool BE = false>
__device__ __forceinline__ void u8u16_warp(const uint8_t *__restrict__ base, int64_t tile_off, int64_t lo_b,
                                           int64_t hi_b, uint16_t *out_w, const SelPair *sel, WarpResult &wr,
                                           uint32_t warp /* warp index inside the tile */, const ChunkIn &in,
                                           uint32_t &hint)
{
    const uint32_t lane = lane_id();
    const int64_t chunk = tile_off + (int64_t)warp * kChunkBytes;
    constexpr int kRounds = kChunkBytes / 512;
    const uint4 *q = in.q;
    uint32_t carry = in.halo_p;
    const uint32_t halo_n = in.halo_n;
    uint32_t rn[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
        rn[r] = __shfl_sync(0xffffffffu, q[r].x, (lane + 1) & 31);

    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(out_w);
    uint32_t running = 0, err = 0, err_pos = 0, units = 0;

    // ASCII chunks (the paper's ASCII fast path, utf8_to_utf16.py:245-251):
    // a warp whose previous chunk was all ASCII (kHintAscii) tests the chunk's
    // bytes with one vote and, if none is >= 0x80, widens them straight into
    // the staging region with two 16-byte stores per round -- no detector, no
    // scan, no compaction.
    if (!Boundary && hint == kHintAscii) {
        uint32_t na = 0;
#pragma unroll
        for (int r = 0; r < kRounds; ++r)
            na |= q[r].x | q[r].y | q[r].z | q[r].w;
        if (!__any_sync(0xffffffffu, (na & H8) != 0)) {
            constexpr uint32_t s01 = BE ? 0x1404u : 0x4140u, s23 = BE ? 0x3424u : 0x4342u;
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const uint32_t a = sbase + 1024u * r + 32u * lane;
                sts128(a, prmt(q[r].x, 0u, s01), prmt(q[r].x, 0u, s23), prmt(q[r].y, 0u, s01), prmt(q[r].y, 0u, s23));
                sts128(a + 16, prmt(q[r].z, 0u, s01), prmt(q[r].z, 0u, s23), prmt(q[r].w, 0u, s01),
                       prmt(q[r].w, 0u, s23));
            }
            if (lane == 0) {
                wr.err = 0;
                wr.pos = 0;
                wr.units = kChunkBytes;
            }
            return;
        }
        hint = 0;
    }

    if (!Boundary && (hint < 2 || (LU_K1_CHUNK3 && hint == 3) || (LU_K1_CHUNK5 && hint == kHintBmp))) {
        uint32_t miss;
        if (hint == 0)
            miss = u8u16_chunk_fast<0, BE>(base, tile_off, chunk, lo_b, hi_b, sbase, sel, in, rn, running);
        else if (LU_K1_CHUNK3 && hint == 3)
            miss = u8u16_chunk_fast<3, BE>(base, tile_off, chunk, lo_b, hi_b, sbase, sel, in, rn, running);
        else if (LU_K1_CHUNK5 && hint == kHintBmp)
            miss = u8u16_chunk_fast<(int)kHintBmp, BE>(base, tile_off, chunk, lo_b, hi_b, sbase, sel, in, rn, running);
        else
            miss = u8u16_chunk_fast<1, BE>(base, tile_off, chunk, lo_b, hi_b, sbase, sel, in, rn, running);
        if (!miss) {
            // a class-0 chunk that emitted one word per byte is all ASCII
            if (hint == 0 && running == (uint32_t)kChunkBytes)
                hint = kHintAscii;
            if (lane == 0) {
                wr.err = 0;
                wr.pos = 0;
                wr.units = running;
            }
            return;
        }
        running = 0; // redo the chunk round by round
    }

#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t lane_off = chunk + r * 512 + 16 * (int64_t)lane;
        const uint32_t rp = __shfl_sync(0xffffffffu, q[r].w, (lane + 31) & 31);
        U8Round R;
        R.w[0] = (lane == 0) ? carry : rp;
        carry = rp;
        R.w[1] = q[r].x;
        R.w[2] = q[r].y;
        R.w[3] = q[r].z;
        R.w[4] = q[r].w;
        R.w[5] = (lane == 31) ? (r + 1 < kRounds ? rn[r + 1 < kRounds ? r + 1 : r] : halo_n) : rn[r];
        // predicted class path first (u8_round_detect_spec); the general
        // detector and decoder only when the prediction misses
        bool fast = false;
#define LU_FAST_ROUND(PP, FN)                                                                                          \
    if (hint == PP) {                                                                                                  \
        uint32_t fd = FN(R);                                                                                           \
        if (r == kRounds - 1 && lane == 31)                                                                            \
            fd |= u8_chunk_end_check(R); /* joins the prediction vote: det = 0 below */                                \
        if (!__any_sync(0xffffffffu, fd != 0)) {                                                                       \
            fast = true;                                                                                               \
            R.path = PP;                                                                                               \
            R.det = 0u;                                                                                                \
            u8u16_round<PP, Boundary, BE>(R, r, base, tile_off, chunk, lane_off, lo_b, hi_b, sbase, sel, running, err, \
                                          err_pos, units);                                                             \
        }                                                                                                              \
    }
        LU_FAST_ROUND(0, u8_fast0)
        else LU_FAST_ROUND(1, u8_fast1) else LU_FAST_ROUND(3, u8_fast3) else LU_FAST_ROUND(kHintBmp, u8_fast01)
#undef LU_FAST_ROUND
        if (!fast) {
            u8_round_detect(R);
            hint = R.next;
            if (r == kRounds - 1 && lane == 31)
                R.det |= u8_chunk_end_check(R);
            u8u16_round<2, Boundary, BE>(R, r, base, tile_off, chunk, lane_off, lo_b, hi_b, sbase, sel, running, err,
                                         err_pos, units);
            if (err) // only a general round can find an error
                break;
        }
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

// Count = true also returns, in `count`, the UTF-16 length of the chunk
// (one word per non-continuation byte plus one per 4-byte lead; exact when the
// input is valid) -- utf16_length_from_utf8.
// `in` holds the chunk at tile_off + warp * kChunkBytes (load_chunk<Boundary>),
// loaded by the caller so it can be prefetched a chunk ahead.
template <bool Boundary, bool Count = false>
__device__ __forceinline__ void u8val_warp_in(const uint8_t *__restrict__ base, int64_t tile_off, int64_t lo_b,
                                              int64_t hi_b, const ChunkIn &in, WarpResult &wr,
                                              uint32_t warp /* warp index in tile */, uint32_t &hint,
                                              uint32_t *count = nullptr)
{
    uint32_t cnt = 0, cacc = 0; // Count: exact total / per-byte counters (interior chunks)
    const uint32_t lane = lane_id();
    const int64_t chunk = tile_off + (int64_t)warp * kChunkBytes;
    constexpr int kRounds = kChunkBytes / 512;
    const uint4 *q = in.q;
    uint32_t carry = in.halo_p;
    const uint32_t halo_n = in.halo_n;
    uint32_t rn[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
        rn[r] = __shfl_sync(0xffffffffu, q[r].x, (lane + 1) & 31);
    uint32_t err = 0, err_pos = 0;
    // straight-line chunk when the prediction is path 0, 1 or 3 (as K1's
    // u8u16_chunk_fast): four detector rounds, votes OR-ed, no branches
    // between them; redo round by round if a round left the class.  Path 3
    // has its own copy so the path 0 / 1 code stays as it was.
    auto chunk_fast = [&](auto pc) -> bool {
        constexpr int P = decltype(pc)::value;
        uint32_t miss = 0, cf = 0, cy = in.halo_p;
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const uint32_t rp = __shfl_sync(0xffffffffu, q[r].w, (lane + 31) & 31);
            U8Round R;
            R.w[0] = (lane == 0) ? cy : rp;
            cy = rp;
            R.w[1] = q[r].x;
            R.w[2] = q[r].y;
            R.w[3] = q[r].z;
            R.w[4] = q[r].w;
            R.w[5] = (lane == 31) ? (r + 1 < kRounds ? rn[r + 1 < kRounds ? r + 1 : r] : halo_n) : rn[r];
            uint32_t fd = P == 3 ? u8_fast3(R) : (hint == 0 ? u8_fast0(R) : u8_fast1(R));
            if (r == kRounds - 1 && lane == 31)
                fd |= u8_chunk_end_check(R);
#if LU_ONE_VOTE
            miss |= fd;
#else
            miss |= __any_sync(0xffffffffu, fd != 0) ? 1u : 0u;
#endif
            if (Count) {
#pragma unroll
                for (int k = 1; k <= 4; ++k)
                    cf += P == 3 ? ((~R.m[k].C & H8) >> 7) + (R.m[k].F >> 7)
                                 : (~R.m[k].C & H8) >> 7; // no F bytes in paths 0 / 1
            }
        }
#if LU_ONE_VOTE
        if (__any_sync(0xffffffffu, miss != 0))
#else
        if (miss)
#endif
            return false;
        if (lane == 0) {
            wr.err = 0;
            wr.pos = 0;
            wr.units = 0;
        }
        if (Count)
            *count = (cf * 0x01010101u) >> 24;
        return true;
    };
    if (!Boundary && hint < 2) {
        if (chunk_fast(std::integral_constant<int, 0>{}))
            return;
    } else if (!Boundary && !Count && hint == 3) {
        if (chunk_fast(std::integral_constant<int, 3>{}))
            return;
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const uint32_t rp = __shfl_sync(0xffffffffu, q[r].w, (lane + 31) & 31);
        U8Round R;
        R.w[0] = (lane == 0) ? carry : rp;
        carry = rp;
        R.w[1] = q[r].x;
        R.w[2] = q[r].y;
        R.w[3] = q[r].z;
        R.w[4] = q[r].w;
        R.w[5] = (lane == 31) ? (r + 1 < kRounds ? rn[r + 1 < kRounds ? r + 1 : r] : halo_n) : rn[r];
        const bool last31 = r == kRounds - 1 && lane == 31;
        const bool predicted = u8_round_detect_spec(R, hint, last31);
        if (!predicted && last31)
            R.det |= u8_chunk_end_check(R);
        if (Count) {
#pragma unroll
            for (int k = 1; k <= 4; ++k) {
                if (Boundary) {
                    const uint32_t vm = valid_mask(chunk + r * 512 + 16 * (int64_t)lane + 4 * (k - 1), lo_b, hi_b);
                    cnt += __popc(~R.m[k].C & vm) + __popc(R.m[k].F & vm);
                } else {
                    // per-byte counters (<= 2 per quad, <= 32 per chunk): no POPC
                    cacc += ((~R.m[k].C & H8) >> 7) + (R.m[k].F >> 7);
                }
            }
        }
        // a predicted round has det = 0 (its chunk-end check joined the prediction vote)
        if (!predicted && __any_sync(0xffffffffu, R.det != 0)) {
            const int64_t rstart = chunk + r * 512;
            uint32_t tb = 3;
            if (r > 0 && lane == 0) {
                for (uint32_t t = 0; t < 3; ++t)
                    if (u8_bad_global(base, rstart - 3 + t, lo_b, hi_b)) {
                        tb = t;
                        break;
                    }
            }
            tb = __shfl_sync(0xffffffffu, tb, 0);
            if (tb < 3) {
                err = 1;
                err_pos = (uint32_t)(rstart - 3 + tb - tile_off);
                break;
            }
            uint32_t kb = 16;
            const uint32_t scan = R.det | __shfl_down_sync(0xffffffffu, R.det, 1);
            if (scan != 0) {
                const int64_t lane_off = rstart + 16 * (int64_t)lane;
                for (uint32_t t = 0; t < 16; ++t)
                    if (u8_bad_global(base, lane_off + t, lo_b, hi_b)) {
                        kb = t;
                        break;
                    }
            }
            const uint32_t bm = __ballot_sync(0xffffffffu, kb < 16);
            if (bm) {
                const uint32_t fl = (uint32_t)__ffs(bm) - 1;
                err = 1;
                err_pos = (uint32_t)(rstart - tile_off) + 16 * fl + __shfl_sync(0xffffffffu, kb, fl);
                break;
            }
        }
    }
    if (lane == 0) {
        wr.err = err;
        wr.pos = err_pos;
        wr.units = 0;
    }
    if (Count)
        *count = cnt + ((cacc * 0x01010101u) >> 24);
}

template <bool Boundary, bool Count = false>
__device__ __forceinline__ void u8val_warp(const uint8_t *__restrict__ base, int64_t tile_off, int64_t lo_b,
                                           int64_t hi_b, WarpResult &wr, uint32_t warp /* warp index in tile */,
                                           uint32_t *count = nullptr)
{
    ChunkIn in;
    load_chunk<Boundary>(base, tile_off + (int64_t)warp * kChunkBytes, lo_b, hi_b, in);
    uint32_t hint = 2;
    u8val_warp_in<Boundary, Count>(base, tile_off, lo_b, hi_b, in, wr, warp, hint, count);
}

} // namespace lu
