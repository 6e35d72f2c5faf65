"""Seeded synthetic workloads of BASELINE.json's five configs (host or device).

The paper measured on lipsum files that are not in this container; these
seeded profiles stand in for them ("Workloads").  Everything is a
pure function of (profile, size, seed), computed with integer torch ops so the
same code generates bit-identical buffers on the CPU (tests) and directly in
HBM on the GPU (bench; no host round trip for 256 MiB - 16 GiB inputs).

Random stream: SplitMix64 in counter form, output k (k >= 1) =
mix64(seed + k * 0x9E3779B97F4A7C15 mod 2**64) -- bit-identical to the
reference's sequential ``laneutf.corpus.SplitMix64`` (corpus.py:65-82; pinned
against its stream in tests/test_corpus.py).  Bounded draws use the high 32
bits: ``(hi32 * bound) >> 32``.

Character model.  Slot j (j = 0, 1, ...) is one in-word character drawn from
outputs 2j+1 and 2j+2: the low 32 bits of the first pick the class, its high
32 bits end the word with probability 1/6 (geometric word length, mean 6,
followed by U+0020), the second picks the code point uniformly in the class
range.  Config 1 ("mix") has no word structure.  A buffer of exactly N bytes
(UTF-8) or N words (UTF-16) takes whole slots while they fit and pads the
remainder (< one slot) with U+0020, so it never ends mid-character.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = [
    "GOLDEN",
    "PROFILES",
    "splitmix64",
    "generate",
    "inject_errors",
    "UTF8_ERROR_KINDS",
    "UTF16_ERROR_KINDS",
    "config5_segments",
    "config5_generate",
]

GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= 1 << 63 else v


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(seed: int, k: torch.Tensor) -> torch.Tensor:
    """Output number k (>= 1) of SplitMix64(seed), as int64 bit patterns."""
    z = k * _s64(GOLDEN) + _s64(seed)
    z = (z ^ _lsr(z, 30)) * _s64(_M1)
    z = (z ^ _lsr(z, 27)) * _s64(_M2)
    return z ^ _lsr(z, 31)


def _hi32(r: torch.Tensor) -> torch.Tensor:
    return _lsr(r, 32)


def _lo32(r: torch.Tensor) -> torch.Tensor:
    return r & 0xFFFFFFFF


def _below(r: torch.Tensor, bound: int) -> torch.Tensor:
    return (_hi32(r) * bound) >> 32


@dataclass(frozen=True)
class _Class:
    prob: float
    lo: int = 0
    hi: int = 0  # inclusive code point range (used when pool is None)
    pool: tuple[int, ...] | None = None
    skip_surrogates: bool = False


_LETTERS = tuple(range(0x61, 0x7B)) + tuple(range(0x41, 0x5B))
_PUNCT = tuple(ord(c) for c in ".,;:!?'-()\"")
_DIGITS = tuple(range(0x30, 0x3A))


@dataclass(frozen=True)
class Profile:
    name: str
    classes: tuple[_Class, ...]
    words: bool = True


PROFILES = {
    # config 2/3 profiles (in-word class mix; one U+0020 ends each word)
    "latin": Profile("latin", (_Class(0.95, pool=_LETTERS + _PUNCT), _Class(0.05, 0x00C0, 0x017F))),
    "cyrillic": Profile("cyrillic", (_Class(0.20, pool=_PUNCT), _Class(0.80, 0x0400, 0x04FF))),
    "cjk": Profile("cjk", (_Class(0.10, pool=_LETTERS + _DIGITS), _Class(0.90, 0x4E00, 0x9FFF))),
    "emoji": Profile("emoji", (_Class(0.50, pool=_LETTERS), _Class(0.50, 0x1F300, 0x1FAFF))),
    # accented Latin with typographic punctuation / currency signs: ASCII + 2-byte + 3-byte
    # in every 2 KiB chunk (no single class path; the validators' BMP class)
    "typo": Profile("typo", (_Class(0.85, pool=_LETTERS + _PUNCT), _Class(0.10, 0x00C0, 0x017F),
                             _Class(0.05, 0x2010, 0x20AC))),
    # plain ASCII text (the paper's ASCII fast path; exercises the kernels' ASCII chunk path)
    "ascii": Profile("ascii", (_Class(1.0, pool=_LETTERS + _PUNCT + _DIGITS),)),
    # config 1: uniform within each UTF-8 length class, no word structure
    "mix": Profile(
        "mix",
        (
            _Class(0.60, 0x0000, 0x007F),
            _Class(0.20, 0x0080, 0x07FF),
            _Class(0.15, 0x0800, 0xFFFF, skip_surrogates=True),
            _Class(0.05, 0x10000, 0x10FFFF),
        ),
        words=False,
    ),
}
PROFILE_ALIASES = {"a": "latin", "b": "cyrillic", "c": "cjk", "d": "emoji", "1": "mix"}


def _profile(name: str) -> Profile:
    return PROFILES[PROFILE_ALIASES.get(name, name)]


def _code_points(prof: Profile, r1: torch.Tensor, r2: torch.Tensor) -> torch.Tensor:
    u = _lo32(r1)
    cp = torch.zeros_like(u)
    acc = 0.0
    done = torch.zeros_like(u, dtype=torch.bool)
    for i, cls in enumerate(prof.classes):
        acc += cls.prob
        thr = (1 << 32) if i == len(prof.classes) - 1 else int(round(acc * (1 << 32)))
        sel = (~done) & (u < thr)
        if cls.pool is not None:
            pool = torch.tensor(cls.pool, dtype=torch.int64, device=u.device)
            v = pool[_below(r2, len(cls.pool))]
        elif cls.skip_surrogates:
            span = (cls.hi - cls.lo + 1) - 0x800
            v = cls.lo + _below(r2, span)
            v = v + (v >= 0xD800).to(torch.int64) * 0x800
        else:
            v = cls.lo + _below(r2, cls.hi - cls.lo + 1)
        cp = torch.where(sel, v, cp)
        done |= sel
    return cp


def _utf8_units(cp: torch.Tensor):
    """(bytes [n,4] int64, length [n]) of each code point."""
    n1 = cp < 0x80
    n2 = (cp >= 0x80) & (cp < 0x800)
    n3 = (cp >= 0x800) & (cp < 0x10000)
    length = torch.where(n1, 1, torch.where(n2, 2, torch.where(n3, 3, 4)))
    b = torch.zeros(cp.shape[0], 4, dtype=torch.int64, device=cp.device)
    c0 = _lsr(cp, 0) & 0x3F
    c1 = (cp >> 6) & 0x3F
    c2 = (cp >> 12) & 0x3F
    b[:, 0] = torch.where(n1, cp, torch.where(n2, 0xC0 | (cp >> 6), torch.where(n3, 0xE0 | (cp >> 12), 0xF0 | (cp >> 18))))
    b[:, 1] = torch.where(n2, 0x80 | c0, torch.where(n3, 0x80 | c1, 0x80 | c2))
    b[:, 2] = torch.where(n3, 0x80 | c0, 0x80 | c1)
    b[:, 3] = 0x80 | c0
    return b, length


def _utf16_units(cp: torch.Tensor):
    big = cp >= 0x10000
    v = cp - 0x10000
    w = torch.zeros(cp.shape[0], 2, dtype=torch.int64, device=cp.device)
    w[:, 0] = torch.where(big, 0xD800 + (v >> 10), cp)
    w[:, 1] = 0xDC00 + (v & 0x3FF)
    return w, torch.where(big, 2, 1)


def generate(profile: str, size: int, seed: int, *, utf16: bool = False, device="cpu",
             batch_slots: int = 1 << 24) -> torch.Tensor:
    """A valid buffer of exactly ``size`` bytes (UTF-8, uint8) or ``size``
    words (UTF-16LE, returned as uint8 of 2*size bytes)."""
    prof = _profile(profile)
    device = torch.device(device)
    unit_dtype = torch.int16 if utf16 else torch.uint8
    out = torch.full((size,), 0x20, dtype=unit_dtype, device=device)
    pos = 0
    slot0 = 0
    max_unit = 3 if utf16 else 5
    while size - pos >= max_unit:
        nb = min(batch_slots, max(1024, (size - pos) + 16))
        j = torch.arange(slot0, slot0 + nb, dtype=torch.int64, device=device)
        r1 = splitmix64(seed, 2 * j + 1)
        r2 = splitmix64(seed, 2 * j + 2)
        cp = _code_points(prof, r1, r2)
        if utf16:
            units, length = _utf16_units(cp)
        else:
            units, length = _utf8_units(cp)
        width = units.shape[1]
        if prof.words:
            space = (_below(r1, 6) == 0)  # word ends after this char
            units = torch.cat([units, torch.full((nb, 1), 0x20, dtype=torch.int64, device=device)], dim=1)
            # put the space right after the character
            k = torch.arange(width + 1, device=device).unsqueeze(0)
            units = torch.where((k == length.unsqueeze(1)) & space.unsqueeze(1), 0x20, units)
            length = length + space.to(torch.int64)
            width += 1
        end = torch.cumsum(length, 0) + pos
        fits = end <= size
        take = int(fits.sum().item())
        if take == 0:
            break
        end = end[:take]
        length = length[:take]
        units = units[:take]
        start = end - length
        k = torch.arange(width, device=device).unsqueeze(0)
        mask = k < length.unsqueeze(1)
        idx = (start.unsqueeze(1) + k)[mask]
        vals = units[mask]
        if utf16:
            vals = torch.where(vals >= 0x8000, vals - 0x10000, vals)
        out[idx] = vals.to(unit_dtype)
        pos = int(end[-1].item())
        slot0 += take
        if take < nb:
            break
    return out.view(torch.uint8) if utf16 else out


UTF8_ERROR_KINDS = (
    "overlong-2",
    "overlong-3",
    "overlong-4",
    "lone-continuation",
    "truncated",
    "encoded-surrogate",
    "above-10ffff",
    "byte-f8-ff",
)
UTF16_ERROR_KINDS = ("unpaired-high", "unpaired-low")


def _utf8_len(b: int) -> int:
    if b < 0x80:
        return 1
    if b < 0xC0:
        return 0
    return 2 if b < 0xE0 else 3 if b < 0xF0 else 4


def inject_errors(buf: torch.Tensor, *, utf16: bool, rate: float, seed: int,
                  kinds: tuple[str, ...] | None = None) -> list[tuple[int, str]]:
    """Plant length-preserving errors in a VALID buffer, in place.

    ``round(units * rate)`` (at least 1) positions uniform over the buffer
    (SplitMix64 stream ``seed``); each is snapped forward to a character
    start suitable for its kind, kinds cycle through ``kinds``.  Returns the
    (unit offset, kind) list.  The expected first-error offset is NOT
    computed here -- tests and the bench take it from the oracle, as the
    reference's corpus.mutate does (corpus.py:276-285).
    """
    units = buf.numel() // 2 if utf16 else buf.numel()
    kinds = kinds or (UTF16_ERROR_KINDS if utf16 else UTF8_ERROR_KINDS)
    count = max(1, int(round(units * rate)))
    ks = torch.arange(1, 2 * count + 1, dtype=torch.int64)
    draws = splitmix64(seed, ks)
    planted = []
    view = buf.view(torch.int16) if utf16 else buf
    for e in range(count):
        r_pos, r_val = draws[2 * e], draws[2 * e + 1]
        p = int(_below(r_pos.view(1), max(units - 8, 1))[0])
        v = int(_hi32(r_val.view(1))[0])
        kind = kinds[e % len(kinds)]
        lo = max(p - 4, 0)
        win = view[lo : min(lo + 64, units)].cpu().tolist()
        if utf16:
            win = [w & 0xFFFF for w in win]
            i = p - lo
            # next non-surrogate word whose neighbours keep the error unpaired
            while i < len(win) - 1 and (0xD800 <= win[i] < 0xE000 or (i > 0 and 0xD800 <= win[i - 1] < 0xDC00)):
                i += 1
            if i >= len(win) - 1:
                continue
            new = (0xD800 + v % 0x400) if kind == "unpaired-high" else (0xDC00 + v % 0x400)
            view[lo + i] = new - 0x10000
            planted.append((lo + i, kind))
            continue
        i = p - lo
        need3 = kind in ("overlong-3", "overlong-4", "encoded-surrogate", "above-10ffff")
        need_multi = kind == "truncated"
        while i < len(win) - 5:
            L = _utf8_len(win[i])
            if L == 0:
                i += 1
                continue
            if need3 and L != 3:
                i += L
                continue
            if need_multi and L < 2:
                i += 1
                continue
            break
        if i >= len(win) - 5:
            continue
        L = _utf8_len(win[i])
        if kind == "overlong-2":
            new = [0xC0 | (v & 1)]
        elif kind == "overlong-3":
            new = [0xE0, 0x80 + v % 0x20, 0x80 + (v >> 8) % 0x40]
        elif kind == "overlong-4":
            new = [0xF0, 0x80 + v % 0x10, 0x80 + (v >> 8) % 0x40, 0x80 + (v >> 16) % 0x40]
        elif kind == "lone-continuation":
            new = [0x80 + v % 0x40]
        elif kind == "truncated":
            new = win[i : i + L - 1] + [0x23]
        elif kind == "encoded-surrogate":
            new = [0xED, 0xA0 + v % 0x20, 0x80 + (v >> 8) % 0x40]
        elif kind == "above-10ffff":
            new = [0xF4, 0x90 + v % 0x30, 0x80, 0x80] if v & 1 else [0xF5 + (v >> 1) % 3, 0x80, 0x80, 0x80]
        else:  # byte-f8-ff
            new = [0xF8 + v % 8]
        view[lo + i : lo + i + len(new)] = torch.tensor(new, dtype=torch.uint8)
        planted.append((lo + i, kind))
    return planted


def config5_segments(total_units: int, seed: int = 5, segment_units: int = 64 << 20,
                     utf16: bool = False) -> list[tuple[str, int, int]]:
    """Config 5 layout: (profile, seed, units) per 64 MiB segment.

    Segment k draws its profile from SplitMix64(seed) output k+1 (uniform over
    latin / cyrillic / cjk / emoji) and is generated with seed 1000*seed + k.
    For UTF-16 a segment is 32 Mi words (64 MiB).
    """
    seg = segment_units // 2 if utf16 else segment_units
    n = (total_units + seg - 1) // seg
    draws = splitmix64(seed, torch.arange(1, n + 1, dtype=torch.int64))
    names = ("latin", "cyrillic", "cjk", "emoji")
    out = []
    for k in range(n):
        units = min(seg, total_units - k * seg)
        out.append((names[int(_below(draws[k].view(1), 4)[0])], 1000 * seed + k, units))
    return out


def config5_generate(total_units: int, *, seed: int = 5, utf16: bool = False, device="cuda",
                     segment_units: int = 64 << 20) -> torch.Tensor:
    """Config 5 buffer (the concatenated seeded 64 MiB segments of
    ``config5_segments``), generated segment by segment on ``device``; uint8
    (UTF-8 bytes, or UTF-16LE words as 2 * total_units bytes).  Segments end
    on character boundaries, so the buffer is valid text."""
    unit = 2 if utf16 else 1
    out = torch.empty(unit * total_units, dtype=torch.uint8, device=device)
    pos = 0
    for name, sseed, units in config5_segments(total_units, seed, segment_units, utf16):
        out[unit * pos: unit * (pos + units)] = generate(name, units, sseed, utf16=utf16, device=device)
        pos += units
    return out


def config5_range(total_units: int, begin: int, end: int, *, seed: int = 5, utf16: bool = False, device="cuda",
                  segment_units: int = 64 << 20) -> torch.Tensor:
    """Units [begin, end) of the config-5 buffer (``config5_generate``)
    without materialising the rest: only the segments overlapping the range
    are generated.  Used by the multi-GPU driver, where each rank builds just
    its shard (plus a few units of look-ahead for its end cut)."""
    unit = 2 if utf16 else 1
    begin, end = max(0, begin), min(end, total_units)
    out = torch.empty(unit * max(end - begin, 0), dtype=torch.uint8, device=device)
    pos = 0
    for name, sseed, units in config5_segments(total_units, seed, segment_units, utf16):
        lo, hi = max(pos, begin), min(pos + units, end)
        if lo < hi:
            seg = generate(name, units, sseed, utf16=utf16, device=device)
            out[unit * (lo - begin): unit * (hi - begin)] = seg[unit * (lo - pos): unit * (hi - pos)]
            del seg
        pos += units
        if pos >= end:
            break
    return out
