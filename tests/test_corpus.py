"""Seeded workload generators (BASELINE.json configs) and error injection."""

import collections

import numpy as np
import pytest
import torch

import oracle
from paper_2212_05098_b200 import corpus


@pytest.mark.parametrize("profile", ["latin", "cyrillic", "cjk", "emoji", "mix"])
@pytest.mark.parametrize("utf16", [False, True])
def test_valid_exact_size_deterministic(profile, utf16):
    n = 100_003
    a = corpus.generate(profile, n, seed=5, utf16=utf16)
    b = corpus.generate(profile, n, seed=5, utf16=utf16)
    assert torch.equal(a, b)
    assert a.numel() == (2 * n if utf16 else n)
    data = a.numpy().tobytes()
    v = oracle.validate_utf16le(data) if utf16 else oracle.validate_utf8(data)
    assert v == ("ok", n, 0)
    c = corpus.generate(profile, n, seed=6, utf16=utf16)
    assert not torch.equal(a, c)


def test_same_text_in_both_encodings():
    for profile in ("latin", "cjk", "emoji", "mix"):
        u8 = corpus.generate(profile, 20_000, seed=3).numpy().tobytes().decode("utf-8")
        u16 = corpus.generate(profile, 20_000, seed=3, utf16=True).numpy().tobytes().decode("utf-16-le")
        k = min(len(u8), len(u16)) - 8
        assert u8[:k] == u16[:k]


def test_profile_mix_statistics():
    """In-word class mix and mean word length (BASELINE.json configs 1-2)."""
    expect = {"latin": {1: 0.95, 2: 0.05}, "cyrillic": {1: 0.2, 2: 0.8}, "cjk": {1: 0.1, 3: 0.9},
              "emoji": {1: 0.5, 4: 0.5}, "mix": {1: 0.6, 2: 0.2, 3: 0.15, 4: 0.05}}
    for profile, mix in expect.items():
        text = corpus.generate(profile, 400_000, seed=1).numpy().tobytes().decode("utf-8")
        words = text.split(" ") if profile != "mix" else [text]
        chars = "".join(words)
        lens = collections.Counter(len(ch.encode("utf-8")) for ch in chars)
        total = sum(lens.values())
        for k, p in mix.items():
            assert abs(lens[k] / total - p) < 0.01, (profile, k, lens[k] / total)
        if profile != "mix":
            mean_len = np.mean([len(w) for w in words[:-1] if w])
            assert 5.7 < mean_len < 6.3, (profile, mean_len)


def test_code_point_ranges():
    ranges = {"latin": (0xC0, 0x17F), "cyrillic": (0x400, 0x4FF), "cjk": (0x4E00, 0x9FFF), "emoji": (0x1F300, 0x1FAFF)}
    for profile, (lo, hi) in ranges.items():
        text = corpus.generate(profile, 100_000, seed=2).numpy().tobytes().decode("utf-8")
        wide = [ord(c) for c in text if ord(c) >= 0x80]
        assert wide and min(wide) >= lo and max(wide) <= hi
    mix = corpus.generate("mix", 300_000, seed=0).numpy().tobytes().decode("utf-8")
    assert not any(0xD800 <= ord(c) < 0xE000 for c in mix)
    assert max(ord(c) for c in mix) > 0xF0000


@pytest.mark.parametrize("kind", corpus.UTF8_ERROR_KINDS)
def test_utf8_error_injection(kind):
    base = corpus.generate("cjk", 50_000, seed=4)
    for s in range(5):
        buf = base.clone()
        planted = corpus.inject_errors(buf, utf16=False, rate=1e-4, seed=s, kinds=(kind,))
        assert planted and all(k == kind for _, k in planted)
        st, consumed, _ = oracle.validate_utf8(buf.numpy().tobytes())
        assert st == "malformed-input"
        assert consumed == min(p for p, _ in planted)


@pytest.mark.parametrize("kind", corpus.UTF16_ERROR_KINDS)
def test_utf16_error_injection(kind):
    base = corpus.generate("emoji", 50_000, seed=4, utf16=True)
    for s in range(5):
        buf = base.clone()
        planted = corpus.inject_errors(buf, utf16=True, rate=1e-4, seed=s, kinds=(kind,))
        st, consumed, _ = oracle.validate_utf16le(buf.numpy().tobytes())
        assert st == "malformed-input"
        assert consumed == min(p for p, _ in planted)


def test_config5_layout():
    segs = corpus.config5_segments(16 << 30)
    assert len(segs) == 256 and all(u == 64 << 20 for _, _, u in segs)
    names = collections.Counter(p for p, _, _ in segs)
    assert set(names) == {"latin", "cyrillic", "cjk", "emoji"}
    assert corpus.config5_segments(16 << 30) == segs
    segs16 = corpus.config5_segments(8 << 30, utf16=True)
    assert len(segs16) == 256 and all(u == 32 << 20 for _, _, u in segs16)
