"""Row 8f(3): the differential campaign and the byte-triple sweep through the
GPU in batched form (reference harness: difftest.check_case,
difftest.py:90-104; the 2^24-triple check of SURVEY App. A.6).  Every case is
independent; each result and payload must equal the oracle's exactly."""

import numpy as np
import pytest
import torch

import oracle
from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, batch_device, corpus, transcode_batch, validate_batch

pytestmark = pytest.mark.gpu

OPS = {  # (direction, validate_only) -> oracle op
    (UTF8_TO_UTF16, False): oracle.OP_U8_U16,
    (UTF16_TO_UTF8, False): oracle.OP_U16_U8,
    (UTF8_TO_UTF16, True): oracle.OP_VAL_U8,
    (UTF16_TO_UTF8, True): oracle.OP_VAL_U16,
}


def make_cases(n: int, seed: int, utf16: bool):
    """Seeded mix of case kinds: random units, text slices (starting anywhere),
    mutated slices, and long slices crossing several 2 KiB warp chunks."""
    rng = np.random.default_rng(seed)
    unit = 2 if utf16 else 1
    pool = corpus.generate("mix", 1 << 21, seed, utf16=utf16).numpy().view(np.uint8)
    pool_units = len(pool) // unit
    kinds = rng.integers(0, 8, size=n)
    lens = np.where(kinds < 2, rng.integers(0, 40, size=n),
                    np.where(kinds < 7, rng.integers(0, 700, size=n), rng.integers(2000, 9000, size=n)))
    starts = rng.integers(0, pool_units - 9000, size=n)
    parts = []
    for k, L, s in zip(kinds.tolist(), lens.tolist(), starts.tolist()):
        if k == 0:
            parts.append(rng.integers(0, 256, size=L * unit, dtype=np.uint8))
            continue
        c = pool[s * unit: (s + L) * unit].copy()
        if k in (2, 3, 4) and L:
            for _ in range(int(rng.integers(1, 4))):
                c[int(rng.integers(0, len(c)))] = rng.integers(0, 256)
        if k == 1 and utf16 and L:  # plant surrogates
            w = c.view(np.uint16)
            w[int(rng.integers(0, len(w)))] = rng.choice([0xD800, 0xDBFF, 0xDC00, 0xDFFF])
        parts.append(c)
    data = np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    return data, offs


def run_and_check(direction: str, validate_only: bool, data: np.ndarray, offs: np.ndarray):
    utf16 = direction == UTF16_TO_UTF8
    dev = torch.device("cuda", 0)
    d = torch.from_numpy(data).to(dev) if len(data) else torch.zeros(0, dtype=torch.uint8, device=dev)
    res, out = batch_device(direction, d, torch.from_numpy(offs).to(dev), validate_only=validate_only)
    got = res.cpu().numpy()
    ref, ref_out = oracle.batch(OPS[(direction, validate_only)], data, offs.astype(np.uint64))
    if not validate_only:
        ref[:, 2] = ref[:, 2]
    else:
        ref[:, 2] = 0
    bad = np.nonzero((got != ref).any(axis=1))[0]
    assert len(bad) == 0, (direction, validate_only, bad[:5], got[bad[:5]], ref[bad[:5]])
    if validate_only:
        return
    # payloads: compare every written unit at its worst-case slot
    out_h = out.cpu().numpy()
    written = ref[:, 2]
    slot = (offs[:-1] if not utf16 else 3 * offs[:-1])
    mask = np.zeros(len(out_h), dtype=bool)
    # mark [slot, slot + written) for all cases (vectorised with a difference array)
    diff = np.zeros(len(out_h) + 1, dtype=np.int64)
    np.add.at(diff, slot, 1)
    np.add.at(diff, slot + written, -1)
    mask = np.cumsum(diff[:-1]) > 0
    assert np.array_equal(out_h[mask], ref_out[: len(out_h)][mask])


@pytest.mark.parametrize("direction", [UTF8_TO_UTF16, UTF16_TO_UTF8])
@pytest.mark.parametrize("validate_only", [False, True])
def test_campaign_1e5(cuda_ok, direction, validate_only):
    data, offs = make_cases(100_000, seed=1234 + (direction == UTF16_TO_UTF8), utf16=direction == UTF16_TO_UTF8)
    run_and_check(direction, validate_only, data, offs)


def test_list_facade(cuda_ok):
    cases = [b"", b"abc", b"\xc3\xa9t\xc3\xa9", b"ab\xc0cd", "🙂x".encode(), b"\xe2\x82"]
    for (o, p), c in zip(transcode_batch(UTF8_TO_UTF16, cases), cases):
        ref, ref_p = oracle.utf8_to_utf16le(c)
        assert o.as_tuple() == ref and p == ref_p
    for o, c in zip(validate_batch(UTF8_TO_UTF16, cases), cases):
        assert o.as_tuple() == oracle.validate_utf8(c)
    cases16 = [b"", "héllo🙂".encode("utf-16-le"), b"\x00\xd8a\x00", b"\x00\xdc"]
    for (o, p), c in zip(transcode_batch(UTF16_TO_UTF8, cases16), cases16):
        ref, ref_p = oracle.utf16le_to_utf8(c)
        assert o.as_tuple() == ref and p == ref_p
    with pytest.raises(ValueError, match="even number"):
        validate_batch(UTF16_TO_UTF8, [b"abc"])


@pytest.mark.slow
@pytest.mark.parametrize("direction", [UTF8_TO_UTF16, UTF16_TO_UTF8])
def test_campaign_1e6(cuda_ok, direction):
    """The reference's 10^6-case differential campaign size, both ops."""
    data, offs = make_cases(1_000_000, seed=99 + (direction == UTF16_TO_UTF8), utf16=direction == UTF16_TO_UTF8)
    run_and_check(direction, False, data, offs)
    run_and_check(direction, True, data, offs)


@pytest.mark.slow
def test_all_byte_triples(cuda_ok):
    """Every 3-byte input (2^24 cases): consumed/written/payload == oracle,
    through the production warp bodies (detector paths, exact predicate)."""
    i = np.arange(1 << 24, dtype=np.uint32)
    data = np.stack([(i >> 16) & 255, (i >> 8) & 255, i & 255], axis=1).astype(np.uint8).reshape(-1)
    offs = 3 * np.arange((1 << 24) + 1, dtype=np.int64)
    run_and_check(UTF8_TO_UTF16, True, data, offs)
    run_and_check(UTF8_TO_UTF16, False, data, offs)
