"""Parity of the B200 engine (through the C ABI) with the oracle.

Every comparison is bit-exact: status, consumed (= error offset), written and
the payload bytes.  The oracle (oracle/) is pinned against the reference by
tests/test_oracle.py.
"""

import random

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from paper_2212_05098_b200 import (
    UTF8_TO_UTF16,
    UTF16_TO_UTF8,
    TranscodeStatus,
    corpus,
    outcome_from_tensor,
    transcode,
    transcode_device,
    transcode_to_bytes,
    validate,
    validate_device,
)

from .helpers import payload_matches, words_to_bytes

pytestmark = pytest.mark.gpu

TILE = 16384


def check_u8(data: bytes):
    ref, ref_payload = oracle.utf8_to_utf16le(data)
    got, payload = transcode_to_bytes(UTF8_TO_UTF16, data, engine="native")
    assert got.as_tuple() == ref, (len(data), got, ref)
    assert payload == ref_payload
    v = validate(UTF8_TO_UTF16, data, engine="native")
    assert v.as_tuple() == oracle.validate_utf8(data), (len(data), v)


def check_u16(data: bytes):
    ref, ref_payload = oracle.utf16le_to_utf8(data)
    got, payload = transcode_to_bytes(UTF16_TO_UTF8, data, engine="native")
    assert got.as_tuple() == ref, (len(data), got, ref)
    assert payload == ref_payload
    v = validate(UTF16_TO_UTF8, data, engine="native")
    assert v.as_tuple() == oracle.validate_utf16le(data), (len(data), v)


# ----------------------------------------------------------------- golden


def test_golden_utf8_to_utf16(cuda_ok, golden):
    for case in golden["utf8_to_utf16"]:
        got, payload = transcode_to_bytes(UTF8_TO_UTF16, case["input_bytes"], engine="native")
        assert list(got.as_tuple()) == case["outcome"], case["name"]
        assert payload_matches(case["payload"], payload), case["name"]
        v = validate(UTF8_TO_UTF16, case["input_bytes"], engine="native")
        assert list(v.as_tuple()) == case["validate"], case["name"]


def test_golden_utf16_to_utf8(cuda_ok, golden):
    for case in golden["utf16_to_utf8"]:
        got, payload = transcode_to_bytes(UTF16_TO_UTF8, case["input_bytes"], engine="native")
        assert list(got.as_tuple()) == case["outcome"], case["name"]
        assert payload_matches(case["payload"], payload), case["name"]
        v = validate(UTF16_TO_UTF8, case["input_bytes"], engine="native")
        assert list(v.as_tuple()) == case["validate"], case["name"]


def test_empty_and_odd(cuda_ok):
    for d in (UTF8_TO_UTF16, UTF16_TO_UTF8):
        got, payload = transcode_to_bytes(d, b"", engine="native")
        assert got.as_tuple() == ("ok", 0, 0) and payload == b""
        assert validate(d, b"", engine="native").as_tuple() == ("ok", 0, 0)
    with pytest.raises(ValueError):
        transcode_to_bytes(UTF16_TO_UTF8, b"\x41", engine="native")
    with pytest.raises(ValueError):
        validate(UTF16_TO_UTF8, b"\x00\x41\xff", engine="native")


# --------------------------------------------------------------- fuzzing

INTERESTING = list(range(0x80, 0x100)) + [0x00, 0x20, 0x41, 0x7F]


def test_random_short_buffers(cuda_ok):
    rng = random.Random(1234)
    for k in range(1500):
        n = rng.randrange(0, 200)
        pool = INTERESTING if k % 2 else range(256)
        check_u8(bytes(rng.choice(pool) for _ in range(n)))
    soup = [0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xD835, 0xDCAA, 0x41, 0xE9, 0x4E2D, 0xFFFF, 0x7F, 0x80, 0x7FF, 0x800]
    for k in range(1500):
        n = rng.randrange(0, 150)
        words = [rng.choice(soup) if k % 2 else rng.randrange(0x10000) for _ in range(n)]
        check_u16(words_to_bytes(words))


@given(st.binary(max_size=300))
@settings(max_examples=300, deadline=None)
def test_hypothesis_utf8(cuda_ok, data):
    check_u8(data)


@given(st.lists(st.integers(0, 0xFFFF), max_size=200))
@settings(max_examples=300, deadline=None)
def test_hypothesis_utf16(cuda_ok, words):
    check_u16(words_to_bytes(words))


@given(st.text(max_size=400))
@settings(max_examples=300, deadline=None)
def test_hypothesis_valid_text_round_trip(cuda_ok, text):
    u8 = text.encode("utf-8")
    got, u16 = transcode_to_bytes(UTF8_TO_UTF16, u8, engine="native")
    assert got.ok and u16 == text.encode("utf-16-le")
    got, back = transcode_to_bytes(UTF16_TO_UTF8, u16, engine="native")
    assert got.ok and back == u8


# ------------------------------------------------ tile / warp boundaries


def _boundary_positions(n):
    pos = set()
    for b in list(range(0, n, 2048)) + list(range(0, min(n, 4096), 128)):
        for d in range(-5, 6):
            if 0 <= b + d < n:
                pos.add(b + d)
    return sorted(pos)


@pytest.mark.parametrize("profile", ["mix", "latin", "cjk", "emoji"])  # detector paths 2, 0, 1, 3
def test_utf8_errors_at_boundaries(cuda_ok, profile):
    base = corpus.generate(profile, 3 * TILE + 777, seed=21).numpy()
    rng = random.Random(7)
    patterns = [b"\x80", b"\xc0", b"\xc1\xbf", b"\xe0\x80\x80", b"\xed\xa0\x80", b"\xf0\x8f\xbf\xbf",
                b"\xf4\x90\x80\x80", b"\xf5", b"\xff", b"\xe2\x28", b"\xc2", b"\xf0\x9f\x98"]
    for p in _boundary_positions(len(base)):
        pat = rng.choice(patterns)
        data = base.copy()
        data[p : p + len(pat)] = np.frombuffer(pat, dtype=np.uint8)[: len(data) - p]
        check_u8(data.tobytes())
    # truncation exactly at the end of the input, every tail length
    for cut in range(1, 40):
        check_u8(base[: len(base) - cut].tobytes())


def test_utf16_errors_at_boundaries(cuda_ok):
    base = corpus.generate("emoji", (3 * TILE + 778) // 2, seed=22, utf16=True).numpy()
    words = base.view(np.uint16)
    for p in _boundary_positions(len(words)):
        for w in (0xD800, 0xDC00, 0xDBFF):
            data = words.copy()
            data[p] = w
            check_u16(data.tobytes())
    for cut in range(1, 10):
        check_u16(words[: len(words) - cut].tobytes())


def test_every_lead_and_misalignment(cuda_ok):
    """Input / output pointers at every offset inside a 16-byte granule."""
    dev = torch.device("cuda", 0)
    text = corpus.generate("mix", 3 * TILE + 100, seed=23).numpy().tobytes()
    ref, ref_payload = oracle.utf8_to_utf16le(text)
    big = torch.zeros(len(text) + 64, dtype=torch.uint8, device=dev)
    for lead in range(16):
        big[lead : lead + len(text)] = torch.frombuffer(bytearray(text), dtype=torch.uint8).to(dev)
        src = big[lead : lead + len(text)]
        out_big = torch.full((2 * len(text) + 64,), 0xEE, dtype=torch.uint8, device=dev)
        for olead in (0, 2, 6, 14):
            out = out_big[olead : olead + 2 * len(text)].view(torch.uint16)
            res, _ = transcode_device(UTF8_TO_UTF16, src, out)
            got = outcome_from_tensor(res.cpu())
            assert got.as_tuple() == ref, (lead, olead)
            assert out.view(torch.uint8)[: 2 * got.written].cpu().numpy().tobytes() == ref_payload
        v = outcome_from_tensor(validate_device(UTF8_TO_UTF16, src).cpu())
        assert v.as_tuple() == oracle.validate_utf8(text)
    # UTF-16 input at every even lead
    u16 = text.decode("utf-8").encode("utf-16-le")
    ref16, ref16_payload = oracle.utf16le_to_utf8(u16)
    big = torch.zeros(len(u16) + 64, dtype=torch.uint8, device=dev)
    for lead in range(0, 16, 2):
        big[lead : lead + len(u16)] = torch.frombuffer(bytearray(u16), dtype=torch.uint8).to(dev)
        src = big[lead : lead + len(u16)]
        for olead in (0, 1, 5, 15):
            out_big = torch.full((3 * len(u16) // 2 + 64,), 0xEE, dtype=torch.uint8, device=dev)
            out = out_big[olead : olead + 3 * len(u16) // 2]
            res, _ = transcode_device(UTF16_TO_UTF8, src, out)
            got = outcome_from_tensor(res.cpu())
            assert got.as_tuple() == ref16, (lead, olead)
            assert out[: got.written].cpu().numpy().tobytes() == ref16_payload


def test_canary_no_write_past_written(cuda_ok):
    dev = torch.device("cuda", 0)
    base = corpus.generate("mix", 2 * TILE + 300, seed=24).numpy()
    for p in (0, 1, 100, TILE - 1, TILE + 3, 2 * TILE + 200):
        data = base.copy()
        data[p] = 0xFF
        src = torch.from_numpy(data).to(dev)
        out = torch.full((2 * len(data) + 32,), 0xA5, dtype=torch.uint8, device=dev)
        res, _ = transcode_device(UTF8_TO_UTF16, src, out[: 2 * len(data)].view(torch.uint16))
        got = outcome_from_tensor(res.cpu())
        ref, ref_payload = oracle.utf8_to_utf16le(data.tobytes())
        assert got.as_tuple() == ref
        host = out.cpu().numpy()
        assert host[: 2 * got.written].tobytes() == ref_payload
        assert (host[2 * got.written :] == 0xA5).all(), p
    # host bytearray out: only the prefix is written
    data = base.copy()
    data[5000] = 0xFF
    buf = bytearray(b"\xee" * (2 * len(data)))
    got = transcode(UTF8_TO_UTF16, data.tobytes(), buf, engine="native")
    ref, ref_payload = oracle.utf8_to_utf16le(data.tobytes())
    assert got.status is TranscodeStatus.MALFORMED_INPUT and got.as_tuple() == ref
    assert got.consumed in (4997, 4998, 4999, 5000)
    assert bytes(buf[: 2 * got.written]) == ref_payload
    assert set(buf[2 * got.written :]) == {0xEE}


@pytest.mark.parametrize("utf16", [False, True])
@pytest.mark.parametrize("be", [False, True])
def test_guard_bytes_around_misaligned_outputs(cuda_ok, utf16, be):
    """Output placed at every misaligned device offset inside a guarded
    buffer: bytes before the output and past ``written`` keep their guard
    value (own bounds check in place of a sanitizer), for valid and malformed
    inputs, LE and BE."""
    from paper_2212_05098_b200 import swap_utf16_byte_order

    dev = torch.device("cuda", 0)
    unit_out = 1 if utf16 else 2
    base = corpus.generate("emoji" if utf16 else "mix", 3 * TILE // (2 if utf16 else 1) + 77, seed=25,
                           utf16=utf16).numpy().view(np.uint8)
    for err_at in (None, 2 * 700, 2 * (TILE // 2 + 5)):
        data = base.copy()
        if err_at is not None:
            data[err_at: err_at + 2] = [0x00, 0xDC] if utf16 else [0xC1, 0x80]
        ref, ref_payload = (oracle.utf16le_to_utf8 if utf16 else oracle.utf8_to_utf16le)(data.tobytes())
        src_bytes = swap_utf16_byte_order(data.tobytes()) if (utf16 and be) else data.tobytes()
        if be and not utf16:
            ref_payload = swap_utf16_byte_order(ref_payload)
        src = torch.frombuffer(bytearray(src_bytes), dtype=torch.uint8).to(dev)
        cap = 3 * (len(data) // 2) if utf16 else 2 * len(data)
        for shift in range(0, 16, 1 if utf16 else 2):
            guard = torch.full((cap + 64,), 0x5A, dtype=torch.uint8, device=dev)
            out = guard[16 + shift: 16 + shift + cap]
            direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
            res, _ = transcode_device(direction, src, out if utf16 else out.view(torch.uint16),
                                      utf16_byte_order="be" if be else "le")
            got = outcome_from_tensor(res.cpu())
            assert got.as_tuple() == ref, (shift, err_at)
            host = guard.cpu().numpy()
            w = unit_out * got.written
            assert (host[: 16 + shift] == 0x5A).all(), ("before", shift, err_at)
            assert host[16 + shift: 16 + shift + w].tobytes() == ref_payload, (shift, err_at)
            assert (host[16 + shift + w:] == 0x5A).all(), ("after", shift, err_at)


# ------------------------------------------------------ full-size configs


@pytest.mark.parametrize("profile", ["latin", "cyrillic", "cjk", "emoji", "typo", "ascii", "mix"])
def test_config2_config3_full_size(cuda_ok, profile):
    """256 MiB buffers of each profile, both directions, against the oracle
    (configs 2 / 3, plus the mixed-BMP, plain-ASCII and all-lengths profiles
    that exercise the BMP class / path D, the ASCII chunk paths and the
    general paths at full size)."""
    dev = torch.device("cuda", 0)
    n = 256 << 20
    seed = {"latin": 1, "cyrillic": 2, "cjk": 3, "emoji": 4, "typo": 6, "ascii": 5, "mix": 0}[profile]
    src = corpus.generate(profile, n, seed, device=dev)
    res, out = transcode_device(UTF8_TO_UTF16, src)
    got = outcome_from_tensor(res.cpu())
    host = src.cpu().numpy()
    ref_words = np.empty(n, dtype=np.uint16)
    ref = oracle.run_mt(oracle.OP_U8_U16, host, nthreads=16, out=ref_words)
    assert got.as_tuple() == ref == ("ok", n, ref[2])
    assert torch.equal(out[: got.written].cpu().view(torch.int16),
                       torch.from_numpy(ref_words[: got.written].view(np.int16)))
    # UTF-16 buffer of the same profile, back to UTF-8
    src16 = corpus.generate(profile, n // 2, seed, utf16=True, device=dev)
    res, out8 = transcode_device(UTF16_TO_UTF8, src16)
    got = outcome_from_tensor(res.cpu())
    host16 = src16.cpu().numpy()
    ref_bytes = np.empty(3 * (n // 2), dtype=np.uint8)
    ref = oracle.run_mt(oracle.OP_U16_U8, host16, nthreads=16, out=ref_bytes)
    assert got.as_tuple() == ref
    assert torch.equal(out8[: got.written].cpu(), torch.from_numpy(ref_bytes[: got.written]))


def test_config1_round_trip(cuda_ok):
    dev = torch.device("cuda", 0)
    src = corpus.generate("mix", 4 << 20, 0, device=dev)
    res, words = transcode_device(UTF8_TO_UTF16, src)
    got = outcome_from_tensor(res.cpu())
    ref, ref_payload = oracle.utf8_to_utf16le(src.cpu().numpy())
    assert got.as_tuple() == ref and got.ok
    assert words[: got.written].cpu().numpy().tobytes() == ref_payload
    res, back = transcode_device(UTF16_TO_UTF8, words[: got.written])
    got2 = outcome_from_tensor(res.cpu())
    assert got2.as_tuple() == ("ok", got.written, 4 << 20)
    assert torch.equal(back[: 4 << 20], src)


@pytest.mark.parametrize("utf16", [False, True])
def test_config4_error_injection(cuda_ok, utf16):
    """256 MiB, errors at 1e-6/unit: validate + transcode vs the oracle, plus
    a zero-error control buffer."""
    dev = torch.device("cuda", 0)
    profile = "emoji" if utf16 else "cjk"
    units = (256 << 20) // 2 if utf16 else 256 << 20
    src = corpus.generate(profile, units, 3 if not utf16 else 4, utf16=utf16, device=dev)
    direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
    # control
    v = outcome_from_tensor(validate_device(direction, src).cpu())
    assert v.as_tuple() == ("ok", units, 0)
    planted = corpus.inject_errors(src, utf16=utf16, rate=1e-6, seed=101 + int(utf16))
    assert len(planted) > 10
    host = src.cpu().numpy()
    ref_v = oracle.run_mt(oracle.OP_VAL_U16 if utf16 else oracle.OP_VAL_U8, host, nthreads=16)
    v = outcome_from_tensor(validate_device(direction, src).cpu())
    assert v.as_tuple() == ref_v and ref_v[0] == "malformed-input"
    assert ref_v[1] == min(p for p, _ in planted) or ref_v[1] <= min(p for p, _ in planted)
    res, out = transcode_device(direction, src)
    got = outcome_from_tensor(res.cpu())
    if utf16:
        ref_out = np.empty(3 * units, dtype=np.uint8)
        ref = oracle.run_mt(oracle.OP_U16_U8, host, nthreads=16, out=ref_out)
        assert got.as_tuple() == ref
        assert out[: got.written].cpu().numpy().tobytes() == ref_out[: got.written].tobytes()
    else:
        ref_out = np.empty(units, dtype=np.uint16)
        ref = oracle.run_mt(oracle.OP_U8_U16, host, nthreads=16, out=ref_out)
        assert got.as_tuple() == ref
        assert out[: got.written].cpu().numpy().tobytes() == ref_out[: got.written].tobytes()


@pytest.mark.parametrize("profile", ["latin", "cyrillic", "cjk", "emoji"])
@pytest.mark.parametrize("kind", corpus.UTF8_ERROR_KINDS)
def test_each_utf8_error_kind(cuda_ok, kind, profile):
    base = corpus.generate(profile, 200_000, seed=9).numpy()
    for s in range(20):
        data = torch.from_numpy(base.copy())
        corpus.inject_errors(data, utf16=False, rate=2e-5, seed=500 + s, kinds=(kind,))
        check_u8(data.numpy().tobytes())


@pytest.mark.parametrize("kind", corpus.UTF16_ERROR_KINDS)
def test_each_utf16_error_kind(cuda_ok, kind):
    base = corpus.generate("emoji", 100_000, seed=9, utf16=True).numpy()
    for s in range(20):
        data = torch.from_numpy(base.copy())
        corpus.inject_errors(data, utf16=True, rate=2e-5, seed=600 + s, kinds=(kind,))
        check_u16(data.numpy().tobytes())


# ------------------------------------------------ host-buffer pipeline (8f row 2)


@pytest.mark.parametrize("utf16", [False, True])
def test_pipelined_host_path(cuda_ok, utf16):
    """Pinned host in/out through the chunked pipeline, small chunks, errors
    placed in the middle chunk and right at chunk cuts; canary past written."""
    from paper_2212_05098_b200 import hostpipe

    units = 3_000_000
    base = corpus.generate("mix", units, seed=31, utf16=utf16)
    chunk = 256 << 10
    cases = [None, 5, chunk - 1, chunk, 3 * chunk + 1, units // 2, units - 1]
    for pos in cases:
        data = base.clone()
        if pos is not None:
            if utf16:
                data.view(torch.int16)[pos] = 0xDC00 - 0x10000
            else:
                data[pos] = 0xFF
        host_in = data.pin_memory()
        cap = 2 * units if not utf16 else 3 * units
        host_out = torch.full((cap + 64,), 0xA5, dtype=torch.uint8).pin_memory()
        got = hostpipe.pipelined_transcode(not utf16, host_in, host_out, chunk_bytes=chunk)
        raw = data.numpy().tobytes()
        ref, payload = oracle.utf16le_to_utf8(raw) if utf16 else oracle.utf8_to_utf16le(raw)
        assert got.as_tuple() == ref, (pos, got, ref)
        out = host_out.numpy()
        assert out[: len(payload)].tobytes() == payload
        assert (out[len(payload):] == 0xA5).all()


def test_facade_routes_pinned_host_buffers(cuda_ok):
    data = corpus.generate("cjk", 20 << 20, seed=32).pin_memory()
    out = torch.empty(40 << 20, dtype=torch.uint8).pin_memory()
    got = transcode(UTF8_TO_UTF16, data, out, engine="native")
    ref, payload = oracle.utf8_to_utf16le(data.numpy())
    assert got.as_tuple() == ref
    assert out[: len(payload)].numpy().tobytes() == payload


# ------------------------------------------------ scanner progress (no deadlock)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("utf16", [False, True])
def test_kernels_on_pinned_host_buffers(cuda_ok, utf16):
    """The kernels read/write pinned host memory directly (zero-copy PCIe).
    Slow, uneven tile loads made a group wait on a window holding its own
    claimed tile; the scanner's partial-window fallback must keep progressing
    (this hung before it).  Results must equal the device-memory run."""
    from paper_2212_05098_b200 import _native

    dev = torch.device("cuda", 0)
    op = _native.OP_UTF16LE_TO_UTF8 if utf16 else _native.OP_UTF8_TO_UTF16LE
    for profile, seed in (("latin", 1), ("emoji", 4), ("cjk", 3)):
        nbytes = 48 << 20
        n_units = nbytes // 2 if utf16 else nbytes
        d_src = corpus.generate(profile, n_units, seed, utf16=utf16, device=dev)
        h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        h_src.copy_(d_src.view(torch.uint8).cpu())
        cap = 3 * n_units if utf16 else n_units
        out_bytes = cap if utf16 else 2 * cap
        h_out = torch.empty(out_bytes, dtype=torch.uint8).pin_memory()
        d_out = torch.empty(out_bytes, dtype=torch.uint8, device=dev)
        ws = torch.empty(_native.workspace_bytes(op, n_units) // 8 + 1, dtype=torch.int64, device=dev)
        res_h = torch.empty(3, dtype=torch.int64, device=dev)
        res_d = torch.empty(3, dtype=torch.int64, device=dev)
        s = torch.cuda.current_stream(dev)
        view = (lambda t: t) if utf16 else (lambda t: t.view(torch.int16))
        src_view = (lambda t: t.view(torch.int16)) if utf16 else (lambda t: t)
        _native.launch(op, src_view(d_src.view(torch.uint8)), n_units, view(d_out), cap, ws, res_d, s)
        for _ in range(3):
            _native.launch(op, src_view(h_src), n_units, view(h_out), cap, ws, res_h, s)
            torch.cuda.synchronize()
            assert res_h.cpu().tolist() == res_d.cpu().tolist()
        w = int(res_d[2]) * (1 if utf16 else 2)
        assert torch.equal(h_out[:w], d_out[:w].cpu())


# ------------------------------------------------ config 5 (16 GiB, sharded)


@pytest.mark.slow
@pytest.mark.parametrize("utf16", [False, True])
def test_config5_full_size_single_gpu(cuda_ok, utf16):
    """16 GiB of config-5 text (mixed profiles in seeded 64 MiB segments) on
    one GPU: the output equals the oracle's (segment by segment), the
    UTF-8 <-> UTF-16 round trip is exact, and cutting the input
    at character boundaries into P = 2, 4, 8 shards, transcoding each shard
    separately and combining the per-shard records (the multi-GPU rule,
    shard.combine_records) reproduces the whole-buffer outcome and output."""
    from paper_2212_05098_b200 import shard

    dev = torch.device("cuda", 0)
    units = (16 << 30) // (2 if utf16 else 1)
    src = corpus.config5_generate(units, utf16=utf16, device=dev)
    direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
    back_dir = UTF8_TO_UTF16 if utf16 else UTF16_TO_UTF8
    res, out = transcode_device(direction, src)
    whole = outcome_from_tensor(res.cpu())
    assert whole.ok and whole.consumed == units
    unit_out = 1 if utf16 else 2
    payload = out.view(torch.uint8)[: unit_out * whole.written]
    res2, back = transcode_device(back_dir, payload)
    o2 = outcome_from_tensor(res2.cpu())
    assert o2.ok and torch.equal(back.view(torch.uint8)[: src.numel()], src)
    del back, res2
    # bit-exact against the oracle, segment by segment: segments end on
    # character boundaries, so the whole-buffer output is the concatenation
    # of the per-segment outputs (oracle.run_mt: all host threads)
    import os

    unit_in = 2 if utf16 else 1
    op = oracle.OP_U16_U8 if utf16 else oracle.OP_U8_U16
    pos = off = 0
    for _name, _seed, seg_units in corpus.config5_segments(units, utf16=utf16):
        seg = src[unit_in * pos: unit_in * (pos + seg_units)].cpu().numpy()
        ref_out = np.empty(3 * seg_units if utf16 else seg_units, dtype=np.uint8 if utf16 else np.uint16)
        st, consumed, wr = oracle.run_mt(op, seg, os.cpu_count() or 1, ref_out)
        assert (st, consumed) == ("ok", seg_units)
        got = payload[unit_out * off: unit_out * (off + wr)].cpu().numpy()
        assert np.array_equal(got, ref_out.view(np.uint8)[: unit_out * wr]), (pos, off)
        pos += seg_units
        off += wr
    assert (pos, off) == (units, whole.written)
    words = src.view(torch.int16) if utf16 else src

    def unit_at(i):
        return int(words[i].item()) & 0xFFFF

    for world in (2, 4, 8):
        cuts = shard.plan_cuts(units, world, unit_at, utf16)
        records = []
        off = 0
        for r in range(world):
            a, b = cuts[r], cuts[r + 1]
            piece = src[a * (2 if utf16 else 1): b * (2 if utf16 else 1)]
            rr, oo = transcode_device(direction, piece)
            rec = outcome_from_tensor(rr.cpu())
            records.append((0 if rec.ok else 1, rec.consumed, rec.written))
            # the shard's payload is the whole payload's slice at its offset
            got = oo.view(torch.uint8)[: unit_out * rec.written]
            assert torch.equal(got, payload[unit_out * off: unit_out * (off + rec.written)])
            off += rec.written
            del rr, oo, got
        status, consumed, written, offsets = shard.combine_records(records, cuts[:-1])
        assert (status, consumed, written) == (0, units, whole.written)


# ------------------------------------------------ class-path prediction


def _class_switching_buffer(seed: int, utf16: bool, total: int = 3 << 20) -> bytes:
    """Valid text whose class mix changes every few hundred bytes, so the
    kernels' per-warp class-path prediction (u8_round_detect_spec) misses and
    recovers at round, chunk and tile boundaries all the time."""
    rng = random.Random(seed)
    parts, n = [], 0
    names = ["latin", "cyrillic", "cjk", "emoji", "mix"]
    while n < total:
        size = rng.choice([rng.randint(4, 64), rng.randint(100, 700), rng.randint(1500, 5000)])
        if utf16:
            size = max(2, size // 2)
        t = corpus.generate(rng.choice(names), size, rng.randint(0, 1 << 30), utf16=utf16)
        b = t.numpy().tobytes()
        parts.append(b)
        n += len(b)
    return b"".join(parts)


@pytest.mark.parametrize("utf16", [False, True])
def test_class_switching_text(cuda_ok, utf16):
    data = _class_switching_buffer(11 + utf16, utf16)
    check = check_u16 if utf16 else check_u8
    check(data)
    rng = random.Random(5 + utf16)
    unit = 2 if utf16 else 1
    for _ in range(12):
        b = bytearray(data)
        pos = rng.randrange(0, len(b) // unit) * unit
        if utf16:
            b[pos:pos + 2] = rng.choice([0xD800, 0xDC00, 0xDBFF, 0xDFFF]).to_bytes(2, "little")
        else:
            b[pos] = rng.choice([0x80, 0xBF, 0xC0, 0xC1, 0xE0, 0xED, 0xF0, 0xF4, 0xF5, 0xFF, rng.randrange(256)])
        check(bytes(b))


@pytest.mark.parametrize("utf16", [False, True])
def test_ascii_chunk_fast_path(cuda_ok, utf16):
    """Large ASCII buffers run through the persistent pipeline, where a warp
    whose previous chunk was all ASCII takes the ASCII chunk path (widen /
    narrow straight into staging).  Pure ASCII, ASCII with isolated multi-unit
    characters (the warp must leave and re-enter the path), and single errors."""
    unit = 2 if utf16 else 1
    n_units = (24 << 20) // unit
    data = corpus.generate("ascii", n_units, 21, utf16=utf16).numpy().tobytes()
    assert max(data) < 0x80
    check = check_u16 if utf16 else check_u8
    check(data)
    rng = random.Random(77 + utf16)
    b = bytearray(data)
    for _ in range(60):
        cp = rng.choice([0xE9, 0x416, 0x4E2D, 0xFFFD, 0x1F600, 0x10FFFF])
        enc = chr(cp).encode("utf-16-le" if utf16 else "utf-8")
        pos = rng.randrange(0, n_units - 8) * unit
        b[pos:pos + len(enc)] = enc
    check(bytes(b))
    for _ in range(6):
        e = bytearray(b)
        pos = rng.randrange(0, n_units) * unit
        if utf16:
            e[pos:pos + 2] = rng.choice([0xD800, 0xDC00]).to_bytes(2, "little")
        else:
            e[pos] = rng.choice([0x80, 0xC0, 0xE0, 0xF0, 0xFF])
        check(bytes(e))


@pytest.mark.timeout(600)
def test_error_path_progress_stress(cuda_ok):
    """Repeated transcodes/validations of buffers with errors injected at
    several rates never hang and always report the validator's offset
    (tools/stress_kernels.py watches every launch).  Regression test for the
    scanner's base hand-off behind an error (the previous window's tag slot can
    be reused by window w + 8 before it is seen; lu_common.cuh scan_windows)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "stress_kernels.py"), "--iters", "40",
                        "--mib", "64", "--limit-s", "20"], capture_output=True, text=True, timeout=540)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "stress ok" in r.stdout
