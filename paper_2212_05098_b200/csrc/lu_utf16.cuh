// lu_utf16.cuh -- UTF-16LE side: K2 utf16le -> utf8 transcode, K4 validate.
//
// Semantics = laneutf.scalar.transcode_utf16le_to_utf8 / validate_utf16le
// (/root/reference/pkg/src/laneutf/scalar.py:108-147, 200-217).  Word i is bad
// iff it is a high surrogate not followed by a low one, or a low surrogate not
// preceded by a high one -- an exact local predicate, so
// the detector IS the exact check here.  Output bytes per word: 1 (< 0x80),
// 2 (< 0x800), 3 (other non-surrogates), 4 for a high surrogate that starts a
// pair, 0 for the low surrogate that ends one.  Work layout as on the UTF-8
// side: a warp walks its 2 KiB chunk in 512-byte rounds, lane l holding 16
// bytes (8 words, four 32-bit quads of two words each) per round.
#pragma once

#include "lu_common.cuh"
#include "lu_utf8.cuh" // WarpResult

namespace lu {

__device__ __forceinline__ bool is_hs(uint32_t w) { return (w & 0xFC00u) == 0xD800u; }
__device__ __forceinline__ bool is_ls(uint32_t w) { return (w & 0xFC00u) == 0xDC00u; }

// UTF-8 bytes of one word (pair-aware), little-endian packed, and their count.
// Bad words get a bounded garbage encoding (<= 3 bytes): nothing at or after
// the first bad word is ever copied out.
__device__ __forceinline__ void u16_encode(uint32_t w, uint32_t wprev, uint32_t wnext, uint32_t &u, uint32_t &len)
{
    const bool hs = is_hs(w), ls = is_ls(w);
    if (hs && is_ls(wnext)) {
        const uint32_t cp = 0x10000u + (((w - 0xD800u) << 10) | (wnext - 0xDC00u));
        u = (0xF0u | (cp >> 18)) | ((0x80u | ((cp >> 12) & 0x3Fu)) << 8) | ((0x80u | ((cp >> 6) & 0x3Fu)) << 16) |
            ((0x80u | (cp & 0x3Fu)) << 24);
        len = 4;
    } else if (ls && is_hs(wprev)) {
        u = 0;
        len = 0;
    } else if (w < 0x80u) {
        u = w;
        len = 1;
    } else if (w < 0x800u) {
        u = (0xC0u | (w >> 6)) | ((0x80u | (w & 0x3Fu)) << 8);
        len = 2;
    } else {
        u = (0xE0u | (w >> 12)) | ((0x80u | ((w >> 6) & 0x3Fu)) << 8) | ((0x80u | (w & 0x3Fu)) << 16);
        len = 3;
    }
}

// bad bits for the two words of a quad: bit 0 = low word, bit 1 = high word
__device__ __forceinline__ uint32_t u16_bad2(uint32_t w0, uint32_t w1, uint32_t wp, uint32_t wn)
{
    const uint32_t b0 = (is_hs(w0) && !is_ls(w1)) || (is_ls(w0) && !is_hs(wp));
    const uint32_t b1 = (is_hs(w1) && !is_ls(wn)) || (is_ls(w1) && !is_hs(w0));
    return b0 | (b1 << 1);
}

// fast any-surrogate test for a quad
__device__ __forceinline__ bool u16_any_sur(uint32_t x)
{
    const uint32_t t = (x & 0xF800F800u) ^ 0xD800D800u; // zero half iff surrogate
    return ((t & 0xFFFFu) == 0) || ((t >> 16) == 0);
}

// valid-word bits (bit 0 low word, bit 1 high word) for boundary tiles
__device__ __forceinline__ uint32_t valid_words(int64_t a, int64_t lo, int64_t hi)
{
    return (uint32_t)(a >= lo && a + 2 <= hi) | ((uint32_t)(a + 2 >= lo && a + 4 <= hi) << 1);
}

// SWAR surrogate masks of a quad (two words): bit 15 / 31 set for a high
// (resp. low) surrogate.
__device__ __forceinline__ void u16_sur_masks(uint32_t x, uint32_t &hs, uint32_t &ls)
{
    // one zero test for "surrogate" ((w & 0xF800) == 0xD800, exact per half:
    // no carry between halves), then bit 10 (moved to bit 15) splits high
    // from low
    const uint32_t c = (x & 0xF800F800u) ^ 0xD800D800u;
    const uint32_t sur = ~(((c & 0x7FFF7FFFu) + 0x7FFF7FFFu) | c) & 0x80008000u;
    const uint32_t lowbit = x << 5; // bit 10 -> 15, bit 26 -> 31
    hs = sur & ~lowbit;
    ls = sur & lowbit;
}

// High / low bytes of the four 16-bit words of two quads, one word per byte
// (byte j of the result = word j of the pair a, b).
__device__ __forceinline__ uint32_t hi_bytes(uint32_t a, uint32_t b) { return prmt(a, b, 0x7531u); }
__device__ __forceinline__ uint32_t lo_bytes(uint32_t a, uint32_t b) { return prmt(a, b, 0x6420u); }

// Surrogate masks of four words from their gathered high bytes: bit 7 of
// byte j of ls is set iff word j is a low surrogate, and bit 7 of byte j of
// nhs is CLEAR iff word j is a high surrogate (complemented: saves a NOT).
// The other bits are garbage; callers only test bit 7 of each byte.  4 words
// per 32-bit op instead of 2 (u16_sur_masks): high byte in D8..DF <=>
// surrogate, bit 2 of it tells low from high.
__device__ __forceinline__ void u16_sur4(uint32_t hb, uint32_t &nhs, uint32_t &ls)
{
    const uint32_t c = hb ^ 0xD8D8D8D8u;                 // zero top 5 bits <=> surrogate
    const uint32_t u = (c & 0x78787878u) + 0x7F7F7F7Fu;  // bit 7: some of bits 3..6 set (no carry out)
    const uint32_t b5 = hb << 5;                         // bit 2 -> bit 7
    nhs = u | c | b5;
    ls = ~(u | c) & b5;
}

__device__ __forceinline__ void sts8(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void sts8_if(uint32_t addr, uint32_t v, uint32_t n, uint32_t j)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.gt.u32 p, %2, %3;\n\t@p st.shared.u8 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"(n), "r"(j)
                 : "memory");
}

// 16-bit stores of two UTF-8 bytes (low half of v) at an even address
__device__ __forceinline__ void sts16b(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}

__device__ __forceinline__ void sts16b_if(uint32_t addr, uint32_t v, uint32_t n, uint32_t j)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.gt.u32 p, %2, %3;\n\t@p st.shared.u16 [%0], %1;\n\t}" ::"r"(addr),
                 "h"((unsigned short)v), "r"(n), "r"(j)
                 : "memory");
}

#ifndef LU_K2_ASCII
#define LU_K2_ASCII 1
#endif
#ifndef LU_K2_PATH_D
#define LU_K2_PATH_D 1 // SWAR path for rounds without surrogates that mix 1-, 2- and 3-byte words
#endif

// ASCII chunk (every word < 0x80): one vote, then the words' low bytes are
// packed straight into the staging region (one 8-byte store per round) -- no
// class votes, no scan, no compaction.  Returns false (nothing stored) if the
// chunk holds a word >= 0x80.  Out of line so the general body keeps its
// register allocation (inlined it cost K2 1-2% on every other profile).
__device__ __noinline__ bool u16u8_ascii_chunk(uint4 q0, uint4 q1, uint4 q2, uint4 q3, uint32_t sbase)
{
    const uint32_t lane = lane_id();
    const uint32_t na = q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w | q2.x | q2.y | q2.z | q2.w | q3.x |
                        q3.y | q3.z | q3.w;
    if (__any_sync(0xffffffffu, (na & 0xFF80FF80u) != 0))
        return false;
    const uint4 q[4] = {q0, q1, q2, q3};
#pragma unroll
    for (int r = 0; r < 4; ++r)
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(sbase + 256u * r + 8u * lane),
                     "r"(prmt(q[r].x, q[r].y, 0x6420u)), "r"(prmt(q[r].z, q[r].w, 0x6420u))
                     : "memory");
    return true;
}

// General round of the K2 warp body, out of line (keeps the unrolled round
// loop small: interior chunks only come here for rounds with surrogates that
// are not path C, i.e. malformed or mixed with BMP words; boundary chunks for
// every round): per-word pair-aware encode (u16_encode), exact local error
// predicate (u16_bad2), seven predicated byte stores per word pair.  w0..w5 =
// the quad before, the lane's four quads, the quad after (by value: an array
// argument would pin the caller's quads in local memory).  Returns {running
// after the round, err, round-relative err_pos, units before the error}.
template <bool Boundary>
__device__ __noinline__ uint4 u16u8_round_general(uint32_t w0_, uint32_t w1_, uint32_t w2_, uint32_t w3_, uint32_t w4_,
                                                  uint32_t w5_, bool sur, int64_t lane_off, int64_t lo_b, int64_t hi_b,
                                                  uint32_t sbase, uint32_t running)
{
    const uint32_t w[6] = {w0_, w1_, w2_, w3_, w4_, w5_};
    uint32_t err = 0, err_pos = 0, units = 0;
        uint32_t lo[4], hi[4], n[4], bad[4];
        uint32_t cnt = 0, anybad = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = w[k + 1];
            const uint32_t w0 = x & 0xFFFFu, w1 = x >> 16, wp = w[k] >> 16, wn = w[k + 2] & 0xFFFFu;
            uint32_t u0, l0, u1, l1;
            // (interior chunks: rounds without surrogates took path A, B or D above)
            if ((LU_K2_PATH_D && !Boundary) || sur) {
                u16_encode(w0, wp, w1, u0, l0);
                u16_encode(w1, w0, wn, u1, l1);
                bad[k] = u16_bad2(w0, w1, wp, wn);
            } else {
                // no surrogates in the round: 1-3 bytes per word, never an error
                u0 = w0 < 0x80u ? w0
                     : w0 < 0x800u ? (0xC0u | (w0 >> 6)) | ((0x80u | (w0 & 0x3Fu)) << 8)
                                   : (0xE0u | (w0 >> 12)) | ((0x80u | ((w0 >> 6) & 0x3Fu)) << 8) |
                                         ((0x80u | (w0 & 0x3Fu)) << 16);
                l0 = 1u + (w0 >= 0x80u) + (w0 >= 0x800u);
                u1 = w1 < 0x80u ? w1
                     : w1 < 0x800u ? (0xC0u | (w1 >> 6)) | ((0x80u | (w1 & 0x3Fu)) << 8)
                                   : (0xE0u | (w1 >> 12)) | ((0x80u | ((w1 >> 6) & 0x3Fu)) << 8) |
                                         ((0x80u | (w1 & 0x3Fu)) << 16);
                l1 = 1u + (w1 >= 0x80u) + (w1 >= 0x800u);
                bad[k] = 0;
            }
            if (Boundary) {
                const uint32_t v = valid_words(lane_off + 4 * k, lo_b, hi_b);
                if (!(v & 1))
                    l0 = 0;
                if (!(v & 2))
                    l1 = 0;
                bad[k] &= v;
            }
            // l0 <= 4 and u1 < 2^32, so the pair packs into 64 bits
            const uint64_t p = (uint64_t)u0 | ((uint64_t)u1 << (8 * l0));
            lo[k] = (uint32_t)p;
            hi[k] = (uint32_t)(p >> 32);
            n[k] = (l0 + l1) | (l0 << 8); // total bytes | bytes of the low word
            cnt += l0 + l1;
            anybad |= bad[k];
        }
        const uint32_t incl = warp_incl_scan(cnt);
        const uint32_t excl = incl - cnt;
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        if (((LU_K2_PATH_D && !Boundary) || sur) && __any_sync(0xffffffffu, anybad != 0)) {
            uint32_t kb = 8, within = excl;
#pragma unroll
            for (int k = 3; k >= 0; --k)
                if (bad[k]) {
                    const uint32_t which = (bad[k] & 1) ? 0u : 1u;
                    kb = 2 * k + which;
                }
            // bytes emitted before the first bad word of this lane
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t nk = n[k] & 0xFFu, l0k = n[k] >> 8;
                if ((uint32_t)(2 * k + 1) < kb)
                    within += nk;
                else if ((uint32_t)(2 * k) < kb)
                    within += l0k;
            }
            const uint32_t bm = __ballot_sync(0xffffffffu, kb < 8);
            const uint32_t fl = (uint32_t)__ffs(bm) - 1;
            const uint32_t kbf = __shfl_sync(0xffffffffu, kb, fl);
            const uint32_t wf = __shfl_sync(0xffffffffu, within, fl);
            err = 1;
            err_pos = 16 * fl + 2 * kbf; // round-relative; the caller adds the round's offset
            units = running + wf;
        }
        uint32_t off = running + excl;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t a = sbase + off;
            const uint32_t nk = n[k] & 0xFFu;
            sts8_if(a, lo[k], nk, 0);
            sts8_if(a + 1, lo[k] >> 8, nk, 1);
            sts8_if(a + 2, lo[k] >> 16, nk, 2);
            sts8_if(a + 3, lo[k] >> 24, nk, 3);
            sts8_if(a + 4, hi[k], nk, 4);
            sts8_if(a + 5, hi[k] >> 8, nk, 5);
            sts8_if(a + 6, hi[k] >> 16, nk, 6);
            off += nk;
        }
        return make_uint4(running + tot, err, err_pos, units);
}

// Path D of the K2 warp body, out of line (the round loop is unrolled four
// times; inlined, this path cost the single-class profiles 1-3%): one round
// without surrogates whose words mix 1, 2 and 3 bytes.  w1..w4 the lane's four
// quads; returns the warp's running byte offset after the round.
__device__ __noinline__ uint32_t u16u8_round_d(uint32_t w1, uint32_t w2, uint32_t w3, uint32_t w4, uint32_t sbase,
                                               uint32_t running, const SelPair *sel)
{
    const uint32_t w[5] = {0u, w1, w2, w3, w4};
            // path D (warp-uniform, interior chunks): no surrogate, words of
            // 1, 2 and 3 bytes mixed (BMP text of mixed scripts).  Per word
            // the UTF-8 string is the last len bytes of (Z', X', Y'):
            //   Z' = E0 | w >> 12,  X' = (80 or C0) | (w >> 6) & 3F,  Y' = 80 | w & 3F (ASCII: w)
            // built as byte planes on the gathered high / low bytes (4 words
            // per op); per word pair two prmt through a 9-entry selector table
            uint32_t T[4], Z[2], cl[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t hb = hi_bytes(w[2 * j + 1], w[2 * j + 2]), lb = lo_bytes(w[2 * j + 1], w[2 * j + 2]);
                const uint32_t z = hb | (lb & H8);
                const uint32_t big = (((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & H8;  // word >= 0x80
                const uint32_t mid = (((hb & 0x78787878u) + 0x7F7F7F7Fu) | hb) & H8; // word >= 0x800
                const uint32_t m = sgn8(big);
                const uint32_t X = ((hb << 2) & 0x3C3C3C3Cu) | ((lb >> 6) & 0x03030303u) | H8 | ((~mid & H8) >> 1);
                const uint32_t Y = (lb & ~m) | (((lb & 0x3F3F3F3Fu) | H8) & m);
                Z[j] = ((hb >> 4) & 0x0F0F0F0Fu) | 0xE0E0E0E0u;
                T[2 * j] = prmt(X, Y, 0x5140u);     // [X0, Y0, X1, Y1]
                T[2 * j + 1] = prmt(X, Y, 0x7362u); // [X2, Y2, X3, Y3]
                cl[j] = (big >> 7) + (mid >> 7);     // bytes - 1 per word (0..2)
            }
            const char *selb = reinterpret_cast<const char *>(sel) + 192;
            uint32_t pl[4], ph[4], nb[4], cnt = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t c = cl[k >> 1] >> (16 * (k & 1));
                // byte offset (idx * 8) of idx = c0 | c1 << 2 (c in bytes 0 and 1)
                const uint32_t bo = ((c & 0x3u) | ((c >> 6) & 0xCu)) << 3;
                const SelPair sp = *reinterpret_cast<const SelPair *>(selb + bo);
                const uint32_t zz = Z[k >> 1] >> (16 * (k & 1));
                pl[k] = prmt(T[k], zz, sp.s01);
                ph[k] = prmt(T[k], zz, sp.s23);
                nb[k] = sp.s23 >> 16;
                cnt += nb[k];
            }
            const uint32_t incl = warp_incl_scan(cnt);
            uint32_t off = running + incl - cnt;
            // 2..6 bytes per quad
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t a = sbase + off;
                sts8(a, pl[k]);
                sts8(a + 1, pl[k] >> 8);
                sts8_if(a + 2, pl[k] >> 16, nb[k], 2);
                sts8_if(a + 3, pl[k] >> 24, nb[k], 3);
                sts8_if(a + 4, ph[k], nb[k], 4);
                sts8_if(a + 5, ph[k] >> 8, nb[k], 5);
                off += nb[k];
            }
            return running + __shfl_sync(0xffffffffu, incl, 31);
}

// K2 warp body for the pipelined kernel: the warp's 2 KiB chunk (1024 words)
// in 4 rounds of 512 B, lane l holding words [8l, 8l+8) of the round in
// registers; neighbour words by shuffle.  Per word: pair-aware UTF-8 encode
// (u16_encode) and the exact local error predicate (u16_bad2); a warp-uniform
// fast path skips the surrogate logic when a round has no surrogate.
template <bool Boundary>
__device__ __forceinline__ void u16u8_warp_r(const uint8_t *__restrict__ base, int64_t tile_off, int64_t lo_b,
                                             int64_t hi_b, uint8_t *out_w, const SelPair *sel, WarpResult &wr,
                                             uint32_t warp, const ChunkIn &in)
{
    const uint32_t lane = lane_id();
    const int64_t chunk = tile_off + (int64_t)warp * kChunkBytes;
    constexpr int kRounds = kChunkBytes / 512;
    const uint4 *q = in.q;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(out_w);
    uint32_t running = 0, err = 0, err_pos = 0, units = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t lane_off = chunk + r * 512 + 16 * (int64_t)lane;
        uint32_t w[6];
        w[0] = 0;
        w[1] = q[r].x;
        w[2] = q[r].y;
        w[3] = q[r].z;
        w[4] = q[r].w;
        w[5] = 0;
        // any surrogate among the lane's words: high bytes gathered 4 words
        // per register, D8..DF.  (A low surrogate right after the lane's
        // words belongs to the next lane / round, which sees it itself.)
        uint32_t any;
        {
            const uint32_t c0 = hi_bytes(w[1], w[2]) ^ 0xD8D8D8D8u, c1 = hi_bytes(w[3], w[4]) ^ 0xD8D8D8D8u;
            const uint32_t u0 = (c0 & 0x78787878u) + 0x7F7F7F7Fu, u1 = (c1 & 0x78787878u) + 0x7F7F7F7Fu;
            any = (~(u0 | c0) | ~(u1 | c1)) & H8;
        }
        const bool sur = __any_sync(0xffffffffu, any != 0);
        if (sur) {
            // only rounds with surrogates look at the words around a lane's
            // quads (pairs that straddle lanes, rounds or the chunk)
            const uint32_t rp = __shfl_sync(0xffffffffu, q[r].w, (lane + 31) & 31);
            const uint32_t pr = r > 0 ? __shfl_sync(0xffffffffu, q[r > 0 ? r - 1 : 0].w, 31) : in.halo_p;
            const uint32_t rx = __shfl_sync(0xffffffffu, q[r].x, (lane + 1) & 31);
            const uint32_t nr = r + 1 < kRounds ? __shfl_sync(0xffffffffu, q[r + 1 < kRounds ? r + 1 : r].x, 0) : in.halo_n;
            w[0] = lane == 0 ? pr : rp;
            w[5] = lane == 31 ? nr : rx;
        }
        // path C (warp-uniform, interior chunks): surrogates present, but every
        // word is ASCII or a surrogate and every pair is well formed (so no
        // error): a quad is at most 5 bytes -- the 4-byte forms of both
        // halves come from SWAR byte planes, then two byte-string selects
        if (!Boundary && sur) {
            // high / low bytes of the lane's 8 words gathered 4 per register
            // (as K4): the class check and the 4-byte forms cover 4 words per op
            const uint32_t hb0 = hi_bytes(w[1], w[2]), hb1 = hi_bytes(w[3], w[4]);
            const uint32_t lb0 = lo_bytes(w[1], w[2]), lb1 = lo_bytes(w[3], w[4]);
            uint32_t nhs0, ls0, nhs1, ls1, nhsp, lsp, nhsn, lsn;
            u16_sur4(hb0, nhs0, ls0);
            u16_sur4(hb1, nhs1, ls1);
            u16_sur4(w[0] & 0xFF000000u, nhsp, lsp); // the word before the lane's words, at byte 3
            u16_sur4(w[5] >> 8, nhsn, lsn);           // the word after them, at byte 0
            // a BMP word >= U+0080 that is not a surrogate: (>= 0x80) & (not hs) & (not ls)
            const uint32_t big0 = (((hb0 | (lb0 & H8)) & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | hb0 | lb0;
            const uint32_t big1 = (((hb1 | (lb1 & H8)) & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | hb1 | lb1;
            const uint32_t other = (big0 & nhs0 & ~ls0) | (big1 & nhs1 & ~ls1);
            // pairs: ls == hs of the previous word (hs complemented)
            const uint32_t ok = (ls0 ^ fsl(nhsp, nhs0, 8)) & (ls1 ^ fsl(nhs0, nhs1, 8)) &
                                ((lsn ^ (nhs1 >> 24)) | 0xFFFFFF00u);
            if (!__any_sync(0xffffffffu, ((other | ~ok) & H8) != 0)) {
                // UTF-8 bytes of a pair led by each word (only used at high
                // surrogates): U = (hs & 0x3FF) + 0x40 = cp >> 10, L = low 10 bits
                //   F0 | U >> 8,  80 | (U >> 2) & 3F,  80 | (U & 3) << 4 | L >> 6,  80 | L & 3F
                uint32_t S[8];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t hb = j ? hb1 : hb0, lb = j ? lb1 : lb0;
                    const uint32_t hbn = j ? fsr(hb1, (w[5] >> 8) & 0xFFu, 8) : fsr(hb0, hb1, 8);
                    const uint32_t lbn = j ? fsr(lb1, w[5] & 0xFFu, 8) : fsr(lb0, lb1, 8);
                    const uint32_t sl = ((lb & 0x7F7F7F7Fu) + 0x40404040u) ^ (lb & H8); // low byte of U
                    const uint32_t cy = (lb & (lb << 1) & H8) >> 7;                     // its carry (lb >= C0)
                    // byte 0 of a non-high-surrogate word's string: its low
                    // byte (the ASCII character; unused for a low surrogate)
                    const uint32_t nm = sgn8(j ? nhs1 : nhs0);
                    const uint32_t B0 = (lb & nm) | ((((hb & 0x03030303u) + cy) | 0xF0F0F0F0u) & ~nm);
                    const uint32_t B1 = ((sl >> 2) & 0x3F3F3F3Fu) | H8;
                    const uint32_t B2 = ((sl << 4) & 0x30303030u) | ((hbn << 2) & 0x0C0C0C0Cu) |
                                        ((lbn >> 6) & 0x03030303u) | H8;
                    const uint32_t B3 = (lbn & 0x3F3F3F3Fu) | H8;
                    // transpose the four planes into one 4-byte string per word
                    const uint32_t t01a = prmt(B0, B1, 0x5140u), t01b = prmt(B0, B1, 0x7362u);
                    const uint32_t t23a = prmt(B2, B3, 0x5140u), t23b = prmt(B2, B3, 0x7362u);
                    S[4 * j + 0] = prmt(t01a, t23a, 0x5410u);
                    S[4 * j + 1] = prmt(t01a, t23a, 0x7632u);
                    S[4 * j + 2] = prmt(t01b, t23b, 0x5410u);
                    S[4 * j + 3] = prmt(t01b, t23b, 0x7632u);
                }
                // per word pair: class index (bit 7 of a byte = high
                // surrogate, bit 6 = low surrogate; c = 2 H, 1 L, 0 ASCII) ->
                // selector table: the pair's bytes are one prmt of the two
                // 4-byte strings, plus a fifth byte (A H) and the count
                const uint32_t cl0 = (~nhs0 & H8) | ((ls0 & H8) >> 1);
                const uint32_t cl1 = (~nhs1 & H8) | ((ls1 & H8) >> 1);
                const char *selb = reinterpret_cast<const char *>(sel);
                uint32_t pl[4], ph[4], nb[4], cnt = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t cl = k < 2 ? cl0 : cl1;
                    // byte offset (idx * 8) of idx = c0 | c1 << 2: bits 6, 7, 14, 15
                    // (or 22, 23, 30, 31) of cl moved to bits 3..6 by a multiply
                    const uint32_t bo = (k & 1) ? (__umulhi(cl & 0xC0C00000u, 0x2080u) & 0x78u)
                                                : (__umulhi(cl & 0x0000C0C0u, 0x20800000u) & 0x78u);
                    const SelPair sp = *reinterpret_cast<const SelPair *>(selb + bo);
                    pl[k] = prmt(S[2 * k], S[2 * k + 1], sp.s01);
                    ph[k] = prmt(S[2 * k], S[2 * k + 1], sp.s23);
                    nb[k] = sp.s23 >> 16;
                    cnt += nb[k];
                }
                const uint32_t incl = warp_incl_scan(cnt);
                uint32_t off = running + incl - cnt;
                // 1..5 bytes per quad (valid pairs: AA 2, AH 5, HL 4, LA 1, LH 4)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t a = sbase + off;
                    sts8(a, pl[k]);
                    sts8_if(a + 1, pl[k] >> 8, nb[k], 1);
                    sts8_if(a + 2, pl[k] >> 16, nb[k], 2);
                    sts8_if(a + 3, pl[k] >> 24, nb[k], 3);
                    sts8_if(a + 4, ph[k], nb[k], 4);
                    off += nb[k];
                }
                running += __shfl_sync(0xffffffffu, incl, 31);
                continue;
            }
        }
        // path A (warp-uniform, interior chunks): no surrogate and every word
        // < U+0800, so each word is 1 or 2 bytes -- both words of a quad are
        // encoded in SWAR and packed into one 32-bit byte string
        bool path_a = false, path_b = false;
        if (!Boundary && !sur) {
            uint32_t any800 = 0;
#pragma unroll
            for (int k = 1; k <= 4; ++k)
                any800 |= w[k] & 0xF800F800u;
            path_a = !__any_sync(0xffffffffu, any800 != 0);
            if (!path_a) {
                // path B: no 2-byte word (every word ASCII or >= U+0800)
                // (gathered bytes, 4 words per op: >= 0x80 and not >= 0x800)
                uint32_t two = 0;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t hb = hi_bytes(w[2 * j + 1], w[2 * j + 2]), lb = lo_bytes(w[2 * j + 1], w[2 * j + 2]);
                    const uint32_t z = hb | (lb & H8);
                    const uint32_t big = ((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z;
                    const uint32_t mid = ((hb & 0x78787878u) + 0x7F7F7F7Fu) | hb;
                    two |= big & ~mid;
                }
                path_b = !__any_sync(0xffffffffu, (two & H8) != 0);
            }
        }
        if (path_b) {
            // every word 1 or 3 bytes: the three byte planes of the 3-byte
            // form are built on the gathered high / low bytes (4 words per
            // op); per quad two prmt pick [A0 B1_0 B2_0 A1 | B1_1 B2_1] (word 0
            // three bytes) or [A0 A1 B1_1 B2_1]; 2, 4 or 6 bytes per quad
            uint32_t F[2], P1[2], P2[2], big[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t hb = hi_bytes(w[2 * j + 1], w[2 * j + 2]), lb = lo_bytes(w[2 * j + 1], w[2 * j + 2]);
                const uint32_t z = hb | (lb & H8);
                big[j] = (((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & H8; // word >= 0x80: 3 bytes here
                const uint32_t m = sgn8(big[j]);
                const uint32_t P0 = ((hb >> 4) & 0x0F0F0F0Fu) | 0xE0E0E0E0u;                  // 1110xxxx
                P1[j] = ((hb << 2) & 0x3C3C3C3Cu) | ((lb >> 6) & 0x03030303u) | H8;          // 10xxxxxx
                P2[j] = (lb & 0x3F3F3F3Fu) | H8;                                            // 10xxxxxx
                F[j] = (P0 & m) | (lb & ~m);                                                // first byte
            }
            uint32_t pl[4], ph[4], nb[4], cnt = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = k >> 1, i0 = 2 * (k & 1);
                const uint32_t pp = prmt(F[j], P1[j], (k & 1) ? 0x7362u : 0x5140u); // [A0, B1_0, A1, B1_1]
                const uint32_t b0 = (big[j] >> (8 * i0 + 7)) & 1u, b1 = (big[j] >> (8 * i0 + 15)) & 1u;
                pl[k] = prmt(pp, P2[j], b0 ? (0x2010u | ((4u + i0) << 8)) : (0x0320u | ((5u + i0) << 12)));
                ph[k] = prmt(pp, P2[j], 0x0003u | ((5u + i0) << 4));
                nb[k] = 2u + 2u * (b0 + b1);
                cnt += nb[k];
            }
            const uint32_t incl = warp_incl_scan(cnt);
            uint32_t off = running + incl - cnt;
            // every quad is 2, 4 or 6 bytes, so all stores of the round share
            // the parity of the warp's running offset (warp-uniform): even --
            // three exact 16-bit stores; odd -- the first and last byte alone,
            // the pairs between them 16-bit (was six 8-bit stores per quad)
            if (!(running & 1u)) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t a = sbase + off;
                    sts16b(a, pl[k]);
                    sts16b_if(a + 2, pl[k] >> 16, nb[k], 2);
                    sts16b_if(a + 4, ph[k], nb[k], 4);
                    off += nb[k];
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t a = sbase + off;
                    sts8(a, pl[k]);
                    sts16b_if(a + 1, pl[k] >> 8, nb[k], 3);
                    sts16b_if(a + 3, fsr(pl[k], ph[k], 24), nb[k], 5);
                    sts8(a + nb[k] - 1, prmt(pl[k], ph[k], nb[k] - 1));
                    off += nb[k];
                }
            }
            running += __shfl_sync(0xffffffffu, incl, 31);
            continue;
        }
        if (path_a) {
            // self-contained (own scan and stores): its live ranges do not
            // overlap the general path's, which otherwise spills
            // first / second byte planes of 4 words per op on the gathered
            // high / low bytes (high byte <= 7 here): F = lb (ASCII) or
            // 110 hhh ll, S = 10 llllll; per word pair one prmt selected by
            // the pair's 2-byte flags (table after path C's, K2 sel + 16)
            uint32_t F[2], S[2], big[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t hb = hi_bytes(w[2 * j + 1], w[2 * j + 2]), lb = lo_bytes(w[2 * j + 1], w[2 * j + 2]);
                const uint32_t z = hb | (lb & H8);
                big[j] = (((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & H8; // word >= 0x80
                const uint32_t m = sgn8(big[j]);
                const uint32_t f2 = (hb << 2) | ((lb >> 6) & 0x03030303u) | 0xC0C0C0C0u;
                F[j] = (f2 & m) | (lb & ~m);
                S[j] = (lb & 0x3F3F3F3Fu) | H8;
            }
            const char *selb = reinterpret_cast<const char *>(sel) + 128;
            uint32_t pk[4], nb[4], cnt = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t bg = big[k >> 1];
                // byte offset (idx * 8) of idx = big0 | big1 << 1: bits 7, 15 (or
                // 23, 31) of the plane moved to bits 3, 4 by a multiply
                const uint32_t bo = (k & 1) ? 32u + (__umulhi(bg & 0x80800000u, 0x1020u) & 0x18u)
                                            : (__umulhi(bg & 0x00008080u, 0x10200000u) & 0x18u);
                const SelPair sp = *reinterpret_cast<const SelPair *>(selb + bo);
                pk[k] = prmt(F[k >> 1], S[k >> 1], sp.s01);
                nb[k] = sp.s23;
                cnt += nb[k];
            }
            const uint32_t incl = warp_incl_scan(cnt);
            uint32_t off = running + incl - cnt;
            // 2..4 bytes per quad: two unconditional, two predicated stores
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t a = sbase + off;
                sts8(a, pk[k]);
                sts8(a + 1, pk[k] >> 8);
                sts8_if(a + 2, pk[k] >> 16, nb[k], 2);
                sts8_if(a + 3, pk[k] >> 24, nb[k], 3);
                off += nb[k];
            }
            running += __shfl_sync(0xffffffffu, incl, 31);
            continue;
        }
        if (LU_K2_PATH_D && !Boundary && !sur) {
            // path D (warp-uniform, interior chunks): no surrogate, words of 1,
            // 2 and 3 bytes mixed (BMP text of mixed scripts) -- u16u8_round_d
            running = u16u8_round_d(w[1], w[2], w[3], w[4], sbase, running, sel);
            continue;
        }
        {
            const uint4 g = u16u8_round_general<Boundary>(w[0], w[1], w[2], w[3], w[4], w[5], sur, lane_off, lo_b, hi_b,
                                                          sbase, running);
            if (g.y) {
                err = 1;
                err_pos = (uint32_t)(chunk + r * 512 - tile_off) + g.z;
                units = g.w;
            }
            running = g.x;
        }
        if (err)
            break;
    }
    if (!err)
        units = running;
    // one byte per word: the chunk was all ASCII
    if (lane == 0) {
        wr.err = err;
        wr.pos = err_pos;
        wr.units = units;
    }
}


// K4 warp body: validate one 2 KiB chunk (1024 words) in 4 rounds of 512 B,
// lane l holding words [8l, 8l+8) in registers.  A low surrogate must sit
// exactly where the previous word is a high surrogate, so the round is clean
// iff ls == hs shifted by one word.  The high bytes of a lane's 8 words are
// gathered into two registers (one prmt each), so the masks and the shifted
// compare cover 4 words per op; a flagged round is resolved with the exact
// predicate u16_bad2.
// Count = true also returns, in `count`, the UTF-8 length of the chunk's
// words (1/2/3 bytes per BMP word, 4 per high surrogate, 0 per low one; exact
// when the input is valid) -- utf8_length_from_utf16le.
// `in` holds the chunk (load_chunk<Boundary, Swap16>), loaded by the caller so
// it can be prefetched a chunk ahead.
template <bool Boundary, bool Count = false>
__device__ __forceinline__ void u16val_warp_in(int64_t tile_off, int64_t lo_b, int64_t hi_b, const ChunkIn &in,
                                               uint32_t &err, uint32_t &err_pos, uint32_t *count = nullptr)
{
    const uint32_t lane = lane_id();
    const int64_t chunk = tile_off;
    constexpr int kRounds = kChunkBytes / 512;
    const uint4 *q = in.q;
    // hs of the word before the round, at byte 3 (lane 0: carried across rounds)
    uint32_t hcarry;
    {
        uint32_t hsh, lsh;
        u16_sur4(hi_bytes(in.halo_p, in.halo_p), hsh, lsh);
        hcarry = hsh;
    }
    uint32_t cnt = 0;
    uint32_t accp = 0, accl = 0; // Count, interior chunks: 128 x (class hits), 128 x (low surrogates), by dp4a
    err = 0;
    err_pos = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const uint32_t hbA = hi_bytes(q[r].x, q[r].y), hbB = hi_bytes(q[r].z, q[r].w);
        uint32_t hsA, lsA, hsB, lsB;
        u16_sur4(hbA, hsA, lsA);
        u16_sur4(hbB, hsB, lsB);
        const uint32_t rp = __shfl_sync(0xffffffffu, hsB, (lane + 31) & 31);
        const uint32_t hsp = (lane == 0) ? hcarry : rp;
        hcarry = rp;
        // (hs complemented) bit 7 of ok is set where ls == hs of the previous word
        uint32_t ok = (lsA ^ fsl(hsp, hsA, 8)) & (lsB ^ fsl(hsA, hsB, 8));
        if (r == kRounds - 1 && lane == 31) {
            // chunk end: the word after the chunk must match the last hs
            uint32_t hsN, lsN;
            u16_sur4(in.halo_n >> 8, hsN, lsN);
            ok &= (lsN ^ (hsB >> 24)) | 0xFFFFFF00u;
        }
        const uint32_t det = ~ok & H8;
        if (Count) {
            const uint32_t lbA = lo_bytes(q[r].x, q[r].y), lbB = lo_bytes(q[r].z, q[r].w);
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const uint32_t hb = g ? hbB : hbA, lb = g ? lbB : lbA;
                const uint32_t z = hb | (lb & H8);
                const uint32_t big = (((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & H8;  // word >= 0x80
                const uint32_t mid = (((hb & 0x78787878u) + 0x7F7F7F7Fu) | hb) & H8; // word >= 0x800
                uint32_t one = H8;
                if (Boundary) {
                    const int64_t a = chunk + r * 512 + 16 * (int64_t)lane + 8 * g;
                    const uint32_t v = valid_words(a, lo_b, hi_b) | (valid_words(a + 4, lo_b, hi_b) << 2);
                    one = ((v & 1) ? 0x80u : 0u) | ((v & 2) ? 0x8000u : 0u) | ((v & 4) ? 0x800000u : 0u) |
                          ((v & 8) ? 0x80000000u : 0u);
                }
                const uint32_t hs = ~(g ? hsB : hsA) & H8, ls = (g ? lsB : lsA) & H8;
                // out-of-range words read as 0: no big/mid/surrogate bits
                if (Boundary) {
                    cnt += __popc(one) + __popc(big) + __popc(mid) + __popc(hs) - 3 * __popc(ls);
                } else {
                    // interior: every word counts 1 (added at the end); the class
                    // bits are summed by dp4a (one multiply-add each, no POPC)
                    accp = __dp4a(big, 0x01010101u, accp);
                    accp = __dp4a(mid, 0x01010101u, accp);
                    accp = __dp4a(hs, 0x01010101u, accp);
                    accl = __dp4a(ls, 0x01010101u, accl);
                }
            }
        }
        if (__any_sync(0xffffffffu, det != 0)) {
            // rare: exact predicate on the raw words (neighbour quads by shuffle)
            const uint32_t prevw = __shfl_sync(0xffffffffu, r > 0 ? q[r > 0 ? r - 1 : 0].w : 0u, 31);
            const uint32_t nextw = __shfl_sync(0xffffffffu, r + 1 < kRounds ? q[r + 1 < kRounds ? r + 1 : r].x : 0u, 0);
            const uint32_t rpw = __shfl_sync(0xffffffffu, q[r].w, (lane + 31) & 31);
            const uint32_t rnw = __shfl_sync(0xffffffffu, q[r].x, (lane + 1) & 31);
            uint32_t w[6];
            w[0] = (lane == 0) ? (r == 0 ? in.halo_p : prevw) : rpw;
            w[1] = q[r].x;
            w[2] = q[r].y;
            w[3] = q[r].z;
            w[4] = q[r].w;
            w[5] = (lane == 31) ? (r + 1 < kRounds ? nextw : in.halo_n) : rnw;
            if (r > 0) {
                // the pair (last word of the previous round, first word of
                // this one) is only compared here: a high surrogate ending
                // the previous round without its low surrogate comes first
                uint32_t tb = (lane == 0 && is_hs(w[0] >> 16) && !is_ls(w[1] & 0xFFFFu)) ? 1u : 0u;
                if (Boundary && tb)
                    tb = valid_words(chunk + r * 512 - 4, lo_b, hi_b) >> 1;
                if (__shfl_sync(0xffffffffu, tb, 0)) {
                    err = 1;
                    err_pos = (uint32_t)(r * 512) - 2;
                    return;
                }
            }
            const int64_t lane_off = chunk + r * 512 + 16 * (int64_t)lane;
            uint32_t kb = 8;
#pragma unroll
            for (int k = 3; k >= 0; --k) {
                uint32_t b = u16_bad2(w[k + 1] & 0xFFFFu, w[k + 1] >> 16, w[k] >> 16, w[k + 2] & 0xFFFFu);
                if (Boundary)
                    b &= valid_words(lane_off + 4 * k, lo_b, hi_b);
                if (b)
                    kb = 2 * k + ((b & 1) ? 0u : 1u);
            }
            const uint32_t bm = __ballot_sync(0xffffffffu, kb < 8);
            if (bm) {
                const uint32_t fl = (uint32_t)__ffs(bm) - 1;
                err = 1;
                err_pos = (uint32_t)(r * 512) + 16 * fl + 2 * __shfl_sync(0xffffffffu, kb, fl);
                return;
            }
        }
    }
    if (Count)
        *count = Boundary ? cnt : (uint32_t)(kChunkBytes / 64) + (accp >> 7) - 3 * (accl >> 7);
}

template <bool Boundary, bool Count = false, bool Swap16 = false>
__device__ __forceinline__ void u16val_warp_r(const uint8_t *__restrict__ base, int64_t tile_off, int64_t lo_b,
                                              int64_t hi_b, uint32_t &err, uint32_t &err_pos,
                                              uint32_t *count = nullptr)
{
    ChunkIn in;
    load_chunk<Boundary, Swap16>(base, tile_off, lo_b, hi_b, in);
    u16val_warp_in<Boundary, Count>(tile_off, lo_b, hi_b, in, err, err_pos, count);
}

} // namespace lu
