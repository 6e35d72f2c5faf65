"""Row 8f(4): utf16_length_from_utf8 / utf8_length_from_utf16le (validate +
count in one pass) and utf8_char_count / utf16le_char_count (reductions),
against the oracle (oracle/ restates scalar.py:220-257)."""

import random

import numpy as np
import pytest
import torch

import oracle
import paper_2212_05098_b200 as lu
from paper_2212_05098_b200 import corpus

pytestmark = pytest.mark.gpu


def ref_len_u8(data: bytes):
    st, consumed, written = oracle.utf8_to_utf16le(data)[0]
    return written if st == "ok" else ValueError(f"invalid UTF-8 at byte {consumed}")


def ref_len_u16(data: bytes):
    st, consumed, written = oracle.utf16le_to_utf8(data)[0]
    return written if st == "ok" else ValueError(f"invalid UTF-16 at word {consumed}")


def check_u8(data: bytes, dev_data=None):
    """dev_data: the same bytes as a (possibly misaligned) CUDA tensor slice."""
    arg = data if dev_data is None else dev_data
    want = ref_len_u8(data)
    if isinstance(want, ValueError):
        with pytest.raises(ValueError) as ei:
            lu.utf16_length_from_utf8(arg)
        assert str(ei.value) == str(want)
    else:
        assert lu.utf16_length_from_utf8(arg) == want
    assert lu.utf8_char_count(arg) == oracle.char_count_utf8(data)


def check_u16(data: bytes, dev_data=None):
    arg = data if dev_data is None else dev_data
    want = ref_len_u16(data)
    if isinstance(want, ValueError):
        with pytest.raises(ValueError) as ei:
            lu.utf8_length_from_utf16le(arg)
        assert str(ei.value) == str(want)
    else:
        assert lu.utf8_length_from_utf16le(arg) == want
    assert lu.utf16le_char_count(arg) == oracle.char_count_utf16le(data)


def test_empty_and_odd(cuda_ok):
    assert lu.utf16_length_from_utf8(b"") == 0
    assert lu.utf8_length_from_utf16le(b"") == 0
    assert lu.utf8_char_count(b"") == 0
    assert lu.utf16le_char_count(b"") == 0
    for fn in (lu.utf8_length_from_utf16le, lu.utf16le_char_count):
        with pytest.raises(ValueError, match="even number of bytes"):
            fn(b"\x41\x00\x42")


def test_known_answers(cuda_ok):
    s = "aµ∇𝒪 漢字 🙂"
    assert lu.utf16_length_from_utf8(s.encode()) == len(s.encode("utf-16-le")) // 2
    assert lu.utf8_length_from_utf16le(s.encode("utf-16-le")) == len(s.encode())
    assert lu.utf8_char_count(s.encode()) == len(s)
    assert lu.utf16le_char_count(s.encode("utf-16-le")) == len(s)
    with pytest.raises(ValueError, match=r"^invalid UTF-8 at byte 2$"):
        lu.utf16_length_from_utf8(b"ab\xc0\xafcd")
    with pytest.raises(ValueError, match=r"^invalid UTF-16 at word 1$"):
        lu.utf8_length_from_utf16le(b"a\x00\x00\xdcb\x00")


@pytest.mark.parametrize("profile", ["mix", "latin", "cyrillic", "cjk", "emoji"])
def test_profiles_every_alignment_and_tail(cuda_ok, profile):
    t8 = corpus.generate(profile, 70_000, seed=31)
    t16 = corpus.generate(profile, 35_000, seed=32, utf16=True).view(torch.uint8).reshape(-1)
    base8, base16 = t8.numpy().tobytes(), t16.numpy().tobytes()
    d8, d16 = t8.cuda(), t16.cuda()
    for lead in range(0, 17):
        for tail in (0, 1, 2, 3, 7, 15):
            check_u8(base8[lead: len(base8) - tail], d8[lead: len(base8) - tail])
            check_u16(base16[2 * lead: len(base16) - 2 * tail], d16[2 * lead: len(base16) - 2 * tail])


def test_random_and_mutated(cuda_ok):
    rng = random.Random(5)
    for _ in range(60):
        n = rng.randrange(0, 9000)
        check_u8(bytes(rng.randrange(256) for _ in range(n)))
        check_u16(bytes(rng.randrange(256) for _ in range(2 * (n // 2))))
    base = corpus.generate("mix", 50_000, seed=33)
    for s in range(20):
        d = base.clone()
        corpus.inject_errors(d, utf16=False, rate=3e-5, seed=900 + s)
        check_u8(d.numpy().tobytes())
    base = corpus.generate("emoji", 25_000, seed=34, utf16=True)
    for s in range(20):
        d = base.clone()
        corpus.inject_errors(d, utf16=True, rate=3e-5, seed=950 + s)
        check_u16(d.numpy().tobytes())


@pytest.mark.parametrize("profile,seed", [("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4), ("typo", 6),
                                          ("ascii", 5), ("mix", 0)])
def test_full_size_lengths_equal_transcode(cuda_ok, profile, seed):
    """256 MiB: the one-pass length equals the transcode's written count, and
    the char counts equal the oracle's."""
    dev = torch.device("cuda", 0)
    u8 = corpus.generate(profile, 256 << 20, seed, device=dev)
    res, _ = lu.transcode_device(lu.UTF8_TO_UTF16, u8)
    written = lu.outcome_from_tensor(res.cpu()).written
    assert lu.utf16_length_from_utf8(u8) == written
    host8 = u8.cpu().numpy()
    assert lu.utf8_char_count(u8) == oracle.char_count_utf8(host8)
    u16 = corpus.generate(profile, 128 << 20, seed, utf16=True, device=dev)
    res, _ = lu.transcode_device(lu.UTF16_TO_UTF8, u16)
    written = lu.outcome_from_tensor(res.cpu()).written
    assert lu.utf8_length_from_utf16le(u16) == written
    assert lu.utf16le_char_count(u16) == oracle.char_count_utf16le(u16.cpu().numpy())
