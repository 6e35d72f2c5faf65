// lu_utf8_lc.cuh -- lane-contiguous UTF-8 detectors (K3 validate_utf8 /
// utf16_length_from_utf8, scalar.py:150-197, 220-232).
//
// Layout: a warp owns a 2 KiB chunk and lane l holds its bytes [64l, 64l+64)
// -- sixteen 32-bit quads in stream order -- so the look-behind / look-ahead
// quads of 15 of a lane's 16 quads are its own registers: one shuffle pair,
// one vote and no per-round bookkeeping per chunk (the round layout of
// lu_utf8.cuh pays two shuffles, two lane selects and a vote per 512 bytes).
//
// The per-quad tests are those of u8_fast0 / u8_fast1 / u8_fast3 and of the
// general detector u8_round_detect (lu_utf8.cuh): each class detector flags
// every bad byte its class can contain and every byte outside the class; the
// general detector (class 2) flags exactly the chunks that hold a bad byte
// (or whose first / last sequence straddles the chunk edge badly).  A flagged
// chunk is resolved by the round-layout code (exact predicate u8_bad_at), the
// only source of error offsets.
#pragma once

#include "lu_utf8.cuh"

namespace lu {

#ifndef LU_LC_MAD
#define LU_LC_MAD 0
#endif

constexpr int kLcQuads = kChunkBytes / 128; // quads per lane (16)
// class hint beyond the class paths 0..3: ASCII + 2-byte + 3-byte leads, no
// F-class byte (kHintBmp, lu_utf8.cuh)
constexpr int kLcBmp = (int)kHintBmp;

// a * b + c as one integer multiply-add (IMAD: the FMA pipe, which these
// ALU-bound detectors leave half idle); opaque to the optimiser so it is not
// turned back into shift + add
__device__ __forceinline__ uint32_t mad32(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Leads of the lane's last quad whose continuations fall into the next quad
// (next lane's first quad, or the 4 bytes after the chunk for lane 31).  For
// lanes < 31 the next lane flags the same bytes at the continuation slot; the
// test is cheap enough to run on every lane without a branch.
__device__ __forceinline__ uint32_t lc_end_check(uint32_t C, uint32_t L, uint32_t E, uint32_t F, uint32_t xn)
{
    const uint32_t cn = xn & ~(xn << 1) & H8;
    return (L & ~fsr(C, cn, 8)) | (E & ~fsr(C, cn, 16)) | (F & ~fsr(C, cn, 24));
}

// Class detectors over a lane's 16 quads.  x[0..15] the lane's bytes, xp / xn
// the quads before / after them.  Returns nonzero (bit 7 of a byte) iff the
// lane saw a byte that is bad or outside class P.  Count: nc += 128 x the
// lane's continuation bytes, nf += 128 x its F-class leads (dp4a on the FMA
// pipe); the lane's UTF-16 length is 64 - nc / 128 + nf / 128 when the chunk
// is valid (one word per non-continuation byte plus one per 4-byte lead).
template <int P, bool Count>
__device__ __forceinline__ uint32_t lc_detect(const uint32_t (&x)[kLcQuads], uint32_t xp, uint32_t xn, uint32_t &nc,
                                              uint32_t &nf)
{
    uint32_t det = 0;
    if (P == 0) {
        // ASCII and 2-byte leads only
        uint32_t Lp = xp & (xp << 1) & H8, C = 0, L = 0;
#pragma unroll
        for (int k = 0; k < kLcQuads; ++k) {
            const uint32_t v = x[k];
            const uint32_t t1 = v << 1;
            C = v & ~t1 & H8;
            L = v & t1 & H8;
            det |= fsl(Lp, L, 8) ^ C;
            det |= L & ((v << 2) | ~((v & 0x1E1E1E1Eu) + 0x7F7F7F7Fu)); // a lead >= E0, or C0 / C1
            if (Count)
                nc = __dp4a(C, 0x01010101u, nc);
            Lp = L;
        }
        det |= lc_end_check(C, L, 0u, 0u, xn);
    } else if (P == 1) {
        // ASCII and 3-byte leads only; "must be a continuation" = E * 0x10100 + spill (u8_fast1)
        const uint32_t Ep = xp & (xp << 1) & (xp << 2) & H8;
        uint32_t spill = __umulhi(Ep, 0x10100u), C = 0, E = 0;
#pragma unroll
        for (int k = 0; k < kLcQuads; ++k) {
            const uint32_t v = x[k];
            const uint32_t t1 = v << 1, t2 = v << 2;
            C = v & ~t1 & H8;
            const uint32_t L = v & t1 & H8;
            E = L & t2;
            const uint32_t need = E * 0x10100u + spill;
            spill = __umulhi(E, 0x10100u);
            det |= need ^ C;
            // E0 / ED candidates (u8_prefilter_e): u = v + 0x03030303, bits 3 / 2 of
            // u as u << 4, u << 5 -- one multiply-add each, on the FMA pipe
#if LU_LC_MAD
            const uint32_t u4 = mad32(v, 16u, 0x30303030u), u5 = mad32(v, 32u, 0x60606060u);
            det |= L & (~t2 | (v << 3) | ~(u4 | u5));
#else
            const uint32_t u = v + 0x03030303u;
            det |= L & (~t2 | (v << 3) | ~((u << 4) | (u << 5)));
#endif
            if (Count)
                nc = __dp4a(C, 0x01010101u, nc);
        }
        det |= lc_end_check(C, E, E, 0u, xn);
    } else if (P == 3) {
        // ASCII and 4-byte leads only (u8_fast3)
        const uint32_t Fp = xp & (xp << 1) & (xp << 2) & (xp << 3) & H8;
        uint32_t spill = __umulhi(Fp, 0x01010100u), C = 0, F = 0;
#pragma unroll
        for (int k = 0; k < kLcQuads; ++k) {
            const uint32_t v = x[k];
            const uint32_t vn = k + 1 < kLcQuads ? x[k + 1 < kLcQuads ? k + 1 : k] : xn;
            const uint32_t t1 = v << 1;
            C = v & ~t1 & H8;
            const uint32_t L = v & t1 & H8;
            F = L & (v << 2) & (v << 3);
            const uint32_t need = F * 0x01010100u + spill;
            spill = __umulhi(F, 0x01010100u);
            det |= need ^ C;
            det |= L & ~F; // a 2- or 3-byte lead: not this class
            det |= F & ((u8_plane_m1(v, fsr(v, vn, 8)) << 3) | (v << 4));
            if (Count) {
                nc = __dp4a(C, 0x01010101u, nc);
                nf = __dp4a(F, 0x01010101u, nf);
            }
        }
        det |= lc_end_check(C, F, F, F, xn);
    } else if (P == kLcBmp) {
        // ASCII, 2-byte and 3-byte leads (BMP text of mixed scripts, e.g.
        // accented Latin with typographic punctuation): flags F-class bytes and
        // E0 / ED candidates, so no second-byte range check is needed
        uint32_t Lp = xp & (xp << 1) & H8, Ep = Lp & (xp << 2), C = 0, L = 0, E = 0;
#pragma unroll
        for (int k = 0; k < kLcQuads; ++k) {
            const uint32_t v = x[k];
            const uint32_t t1 = v << 1, t2 = v << 2;
            C = v & ~t1 & H8;
            L = v & t1 & H8;
            E = L & t2;
            det |= (fsl(Lp, L, 8) | fsl(Ep, E, 16)) ^ C;
            det |= L & ~t2 & ~((v & 0x1E1E1E1Eu) + 0x7F7F7F7Fu); // C0 / C1
            const uint32_t u = v + 0x03030303u;                   // E0 / ED candidates (u8_prefilter_e)
            det |= E & ((v << 3) | ~((u << 4) | (u << 5)));       // an F-class byte or a candidate
            if (Count)
                nc = __dp4a(C, 0x01010101u, nc);
            Lp = L;
            Ep = E;
        }
        det |= lc_end_check(C, L, E, 0u, xn);
    }
    return det & H8;
}

// General detector (every class): exact, no prefilter votes.  cls: bit 0 a
// 2-byte lead, bit 1 a 3-byte lead, bit 2 an F-class byte was seen by this
// lane (the caller votes the chunk's class from them for the next chunk).
template <bool Count>
__device__ __forceinline__ uint32_t lc_detect_general(const uint32_t (&x)[kLcQuads], uint32_t xp, uint32_t xn,
                                                      uint32_t &nc, uint32_t &nf, uint32_t &cls)
{
    U8Masks p = u8_classify(xp), c = p;
    uint32_t det = 0, o2 = 0, o3 = 0, o4 = 0;
#pragma unroll
    for (int k = 0; k < kLcQuads; ++k) {
        const uint32_t v = x[k];
        const uint32_t vn = k + 1 < kLcQuads ? x[k + 1 < kLcQuads ? k + 1 : k] : xn;
        c = u8_classify(v);
        det |= (fsl(p.L, c.L, 8) | fsl(p.E, c.E, 16) | fsl(p.F, c.F, 24)) ^ c.C;
        det |= c.L & ~c.E & ~((v & 0x1E1E1E1Eu) + 0x7F7F7F7Fu); // C0 / C1
        const uint32_t n1 = fsr(v, vn, 8);
        det |= u8_check_e(v, n1, c) | u8_check_f(v, n1, c);
        o2 |= c.L & ~c.E;
        o3 |= c.E & ~c.F;
        o4 |= c.F;
        if (Count) {
            nc = __dp4a(c.C, 0x01010101u, nc);
            nf = __dp4a(c.F, 0x01010101u, nf);
        }
        p = c;
    }
    det |= lc_end_check(c.C, c.L, c.E, c.F, xn);
    cls = (o2 ? 1u : 0u) | (o3 ? 2u : 0u) | (o4 ? 4u : 0u);
    return det & H8;
}

// class path of a chunk from the OR of its lanes' cls bits (u8_round_detect's rule)
__device__ __forceinline__ uint32_t lc_path_of(uint32_t cls)
{
    if (!(cls & 6u))
        return 0; // no byte >= E0
    if (cls == 2u)
        return 1; // 3-byte leads only
    if (cls == 4u)
        return 3; // 4-byte leads only
    if (cls == 3u)
        return kLcBmp; // 2- and 3-byte leads, no F-class byte
    return 2;
}

} // namespace lu
