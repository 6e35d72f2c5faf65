"""Row 8f(1): UTF-16BE with the byte swap fused into the kernels.  The
reference reaches BE only through its CLI (swap the input / output with
swap_utf16_byte_order around the LE call, cli.py:90-94, 113-114; tests
test_cli.py:56-80), so the contract is: BE outcome == LE outcome of the
swapped buffer, BE payload == swapped LE payload."""

import random

import numpy as np
import pytest
import torch

import oracle
from paper_2212_05098_b200 import (
    UTF8_TO_UTF16,
    UTF16_TO_UTF8,
    corpus,
    outcome_from_tensor,
    swap_utf16_byte_order,
    transcode,
    transcode_device,
    transcode_to_bytes,
    validate,
)

pytestmark = pytest.mark.gpu

SAMPLE = "laneutf: aµ∇𝒪 — 漢字かな 🙂 Ünïcödé\n" * 3


def check_u8_be(data: bytes):
    ref, ref_payload = oracle.utf8_to_utf16le(data)
    got, payload = transcode_to_bytes(UTF8_TO_UTF16, data, engine="native", utf16_byte_order="be")
    assert got.as_tuple() == ref
    assert payload == swap_utf16_byte_order(ref_payload)


def check_u16_be(data_le: bytes):
    ref, ref_payload = oracle.utf16le_to_utf8(data_le)
    be = swap_utf16_byte_order(data_le)
    got, payload = transcode_to_bytes(UTF16_TO_UTF8, be, engine="native", utf16_byte_order="be")
    assert got.as_tuple() == ref
    assert payload == ref_payload
    v = validate(UTF16_TO_UTF8, be, engine="native", utf16_byte_order="be")
    assert v.as_tuple() == oracle.validate_utf16le(data_le)


def test_known_answers(cuda_ok):
    o, p = transcode_to_bytes(UTF8_TO_UTF16, SAMPLE.encode(), utf16_byte_order="be")
    assert o.ok and p == SAMPLE.encode("utf-16-be")
    o, p = transcode_to_bytes(UTF16_TO_UTF8, SAMPLE.encode("utf-16-be"), utf16_byte_order="be")
    assert o.ok and p == SAMPLE.encode()
    with pytest.raises(ValueError, match="utf16_byte_order"):
        transcode_to_bytes(UTF8_TO_UTF16, b"a", utf16_byte_order="BE")


def test_random_mutated_and_errors(cuda_ok):
    rng = random.Random(11)
    for _ in range(40):
        n = rng.randrange(0, 6000)
        check_u8_be(bytes(rng.randrange(256) for _ in range(n)))
        check_u16_be(bytes(rng.randrange(256) for _ in range(2 * (n // 2))))
    base = corpus.generate("emoji", 40_000, seed=41, utf16=True)
    for s in range(15):
        d = base.clone()
        corpus.inject_errors(d, utf16=True, rate=3e-5, seed=700 + s)
        check_u16_be(d.numpy().tobytes())
    base8 = corpus.generate("mix", 80_000, seed=42)
    for s in range(15):
        d = base8.clone()
        corpus.inject_errors(d, utf16=False, rate=3e-5, seed=750 + s)
        check_u8_be(d.numpy().tobytes())


def test_device_misalignment(cuda_ok):
    le = corpus.generate("emoji", 30_000, seed=43, utf16=True).view(torch.uint8).reshape(-1)
    le[2 * 12345: 2 * 12346] = torch.tensor([0x00, 0xDC], dtype=torch.uint8)  # lone low surrogate
    be_host = swap_utf16_byte_order(le.numpy().tobytes())
    d_be = torch.frombuffer(bytearray(be_host), dtype=torch.uint8).cuda()
    for lead in range(0, 9):
        for tail in (0, 1, 5):
            sl = slice(2 * lead, len(be_host) - 2 * tail)
            ref, ref_payload = oracle.utf16le_to_utf8(le.numpy().tobytes()[sl])
            res, out = transcode_device(UTF16_TO_UTF8, d_be[sl], utf16_byte_order="be")
            got = outcome_from_tensor(res.cpu())
            assert got.as_tuple() == ref
            assert out[: got.written].cpu().numpy().tobytes() == ref_payload


@pytest.mark.parametrize("profile,seed", [("latin", 1), ("cjk", 3), ("emoji", 4), ("ascii", 7)])
def test_full_size_be_equals_swapped_le(cuda_ok, profile, seed):
    dev = torch.device("cuda", 0)
    u8 = corpus.generate(profile, 256 << 20, seed, device=dev)
    r_le, o_le = transcode_device(UTF8_TO_UTF16, u8)
    r_be, o_be = transcode_device(UTF8_TO_UTF16, u8, utf16_byte_order="be")
    a, b = outcome_from_tensor(r_le.cpu()), outcome_from_tensor(r_be.cpu())
    assert a == b and a.ok
    w = a.written
    le_bytes = o_le.view(torch.uint8)[: 2 * w].view(-1, 2)
    assert torch.equal(le_bytes.flip(1), o_be.view(torch.uint8)[: 2 * w].view(-1, 2))
    # and back: BE input
    r2, o2 = transcode_device(UTF16_TO_UTF8, o_be.view(torch.uint8)[: 2 * w], utf16_byte_order="be")
    c = outcome_from_tensor(r2.cpu())
    assert c.ok and c.written == u8.numel() and torch.equal(o2[: c.written], u8)


def test_pinned_host_pipeline_be(cuda_ok):
    le = corpus.generate("emoji", 20 << 20, seed=44, utf16=True).view(torch.uint8).reshape(-1)
    le[2 * (9 << 20): 2 * (9 << 20) + 2] = torch.tensor([0x3D, 0xD8], dtype=torch.uint8)  # dangling high
    be = torch.from_numpy(np.frombuffer(swap_utf16_byte_order(le.numpy().tobytes()), dtype=np.uint8).copy())
    src = be.pin_memory()
    dst = torch.empty(3 * (src.numel() // 2), dtype=torch.uint8).pin_memory()
    ref, ref_payload = oracle.utf16le_to_utf8(le.numpy().tobytes())
    got = transcode(UTF16_TO_UTF8, src, dst, utf16_byte_order="be")
    assert got.as_tuple() == ref
    assert dst[: got.written].numpy().tobytes() == ref_payload
    # UTF-8 -> UTF-16BE through the pipeline
    u8 = corpus.generate("mix", 24 << 20, seed=45)
    src8 = u8.pin_memory()
    dst16 = torch.empty(2 * src8.numel(), dtype=torch.uint8).pin_memory()
    ref, ref_payload = oracle.utf8_to_utf16le(u8.numpy().tobytes())
    got = transcode(UTF8_TO_UTF16, src8, dst16, utf16_byte_order="be")
    assert got.as_tuple() == ref
    assert dst16[: 2 * got.written].numpy().tobytes() == swap_utf16_byte_order(ref_payload)
