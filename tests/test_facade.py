"""Facade behaviour that needs no GPU: engine parsing/routing, argument
errors, sizing, byte-order helper (mirrors pkg/tests/test_engine.py)."""

import pytest
import torch

from paper_2212_05098_b200 import (
    DIRECTIONS,
    ENGINE_ENV_VAR,
    UTF8_TO_UTF16,
    UTF16_TO_UTF8,
    EngineKind,
    TranscodeOutcome,
    TranscodeStatus,
    detect,
    parse_engine,
    resolve_engine,
    swap_utf16_byte_order,
    transcode,
    transcode_to_bytes,
    validate,
    worst_case_output_bytes,
)


class TestEngineKind:
    def test_describe(self):
        assert EngineKind.scalar_kind().describe() == "scalar"
        assert EngineKind.emulated(64).describe() == "emulated(64)"
        assert EngineKind.native().describe() == "native"

    @pytest.mark.parametrize(
        "name,expected",
        [
            ("scalar", EngineKind.scalar_kind()),
            ("native", EngineKind.native()),
            (" NATIVE ", EngineKind.native()),
            ("emulated", EngineKind.emulated(64)),
            ("emulated-8", EngineKind.emulated(8)),
            ("emulated(32)", EngineKind.emulated(32)),
        ],
    )
    def test_parse(self, name, expected):
        assert parse_engine(name) == expected

    @pytest.mark.parametrize("name", ["", "turbo", "emulated-", "emulated()", "emulated-x8"])
    def test_parse_rejects(self, name):
        with pytest.raises(ValueError):
            parse_engine(name)

    def test_kind_invariants(self):
        with pytest.raises(ValueError):
            EngineKind("scalar", 8)
        with pytest.raises(ValueError):
            EngineKind("emulated")


def test_default_engine_is_native(monkeypatch):
    monkeypatch.delenv(ENGINE_ENV_VAR, raising=False)
    assert resolve_engine(None) == EngineKind.native()
    monkeypatch.setenv(ENGINE_ENV_VAR, "native")
    assert resolve_engine(None) == EngineKind.native()
    monkeypatch.setenv(ENGINE_ENV_VAR, "turbo")
    with pytest.raises(ValueError):
        resolve_engine(None)


def test_detect_stable():
    assert detect() is detect()


def test_cpu_engines_are_not_shipped():
    for engine in ("scalar", "emulated-64"):
        with pytest.raises(ValueError, match="engine unavailable"):
            transcode_to_bytes(UTF8_TO_UTF16, b"abc", engine=engine)


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only host behaviour")
def test_native_unavailable_without_gpu_fails_loudly():
    with pytest.raises(ValueError, match="native engine unavailable"):
        transcode_to_bytes(UTF8_TO_UTF16, b"abc", engine="native")
    with pytest.raises(ValueError, match="native engine unavailable"):
        validate(UTF8_TO_UTF16, b"abc")
    with pytest.raises(ValueError, match="native engine unavailable"):
        transcode(UTF8_TO_UTF16, b"abc", bytearray(6))


def test_argument_errors_before_device_work():
    with pytest.raises(ValueError):
        transcode_to_bytes("utf8-to-utf32", b"")
    with pytest.raises(ValueError, match="even"):
        transcode_to_bytes(UTF16_TO_UTF8, b"\x41")
    with pytest.raises(ValueError, match="even"):
        validate(UTF16_TO_UTF8, b"\x00\x41\xff")


def test_worst_case_sizes():
    assert worst_case_output_bytes(UTF8_TO_UTF16, 10) == 20
    assert worst_case_output_bytes(UTF16_TO_UTF8, 10) == 15
    with pytest.raises(ValueError):
        worst_case_output_bytes("x", 1)
    assert DIRECTIONS == (UTF8_TO_UTF16, UTF16_TO_UTF8)


def test_swap_byte_order():
    assert swap_utf16_byte_order(b"\x41\x00\x35\xd8") == b"\x00\x41\xd8\x35"
    with pytest.raises(ValueError):
        swap_utf16_byte_order(b"\x41")


def test_outcome_semantics():
    o = TranscodeOutcome(TranscodeStatus.MALFORMED_INPUT, 3, 2)
    assert not o.ok and o.error_offset == 3 and o.as_tuple() == ("malformed-input", 3, 2)
    with pytest.raises(ValueError):
        TranscodeOutcome(TranscodeStatus.OK, 3, 2).error_offset
