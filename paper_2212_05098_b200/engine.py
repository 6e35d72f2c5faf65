"""Entry points with the reference facade's signatures, backed by the B200 engine.

Mirrors ``laneutf.engine`` (/root/reference/pkg/src/laneutf/engine.py):
``transcode`` (178-209), ``transcode_to_bytes`` (212-223), ``validate``
(226-240), ``EngineKind``/``parse_engine`` (58-103), ``detect`` (141-153),
``resolve_engine`` with the ``LANEUTF_ENGINE`` override (156-163),
``worst_case_output_bytes`` (171-175) and ``swap_utf16_byte_order``
(243-250).  Same argument meaning, return values and error behaviour:
malformed input is a status, never an exception; ``ValueError`` for an
unknown direction, an unparsable or unavailable engine, and odd UTF-16 byte
lengths (raised before any device work).

This build fills the reference's reserved ``native`` slot (engine.py:1-16,
194-200) with the sm_100a engine and is the default engine.  The reference's
CPU engines (``scalar``, ``emulated(n)``) are parsed for compatibility but
are not part of this build: asking for one raises ``ValueError`` exactly like
the reference does for an engine missing from its inventory.  There is no CPU
fallback anywhere on this path.

Beyond the reference signatures, ``data`` / ``out`` may also be torch tensors:
a CUDA tensor stays on the device (zero-copy), a pinned CPU tensor is copied
asynchronously.  ``transcode_device`` is the stream-ordered, device-resident
form used by the benchmark and the multi-GPU driver.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _native, hostpipe
from .outcome import STATUS_BY_CODE, TranscodeOutcome, TranscodeStatus


__all__ = [
    "UTF8_TO_UTF16",
    "UTF16_TO_UTF8",
    "DIRECTIONS",
    "ENGINE_ENV_VAR",
    "EngineKind",
    "EngineInventory",
    "parse_engine",
    "resolve_engine",
    "detect",
    "transcode",
    "transcode_to_bytes",
    "validate",
    "transcode_device",
    "validate_device",
    "outcome_from_tensor",
    "swap_utf16_byte_order",
    "worst_case_output_bytes",
    "utf16_length_from_utf8",
    "utf8_length_from_utf16le",
    "utf8_char_count",
    "utf16le_char_count",
    "count_device",
    "batch_device",
    "transcode_batch",
    "validate_batch",
]

UTF8_TO_UTF16 = "utf8-to-utf16"
UTF16_TO_UTF8 = "utf16-to-utf8"
DIRECTIONS = (UTF8_TO_UTF16, UTF16_TO_UTF8)

ENGINE_ENV_VAR = "LANEUTF_ENGINE"


@dataclass(frozen=True)
class EngineKind:
    """A selectable backend: ``scalar``, ``emulated(n)``, or ``native`` (engine.py:58-86)."""

    family: str
    lane_count: int | None = None

    def __post_init__(self):
        if self.family not in ("scalar", "emulated", "native"):
            raise ValueError(f"unknown engine family {self.family!r}")
        if (self.family == "emulated") != (self.lane_count is not None):
            raise ValueError("lane_count is for emulated engines only")

    @classmethod
    def scalar_kind(cls) -> "EngineKind":
        return cls("scalar")

    @classmethod
    def emulated(cls, lane_count: int) -> "EngineKind":
        return cls("emulated", lane_count)

    @classmethod
    def native(cls) -> "EngineKind":
        return cls("native")

    def describe(self) -> str:
        if self.family == "emulated":
            return f"emulated({self.lane_count})"
        return self.family


def parse_engine(text: str) -> EngineKind:
    """Accepts ``scalar``, ``native``, ``emulated``, ``emulated-N``, ``emulated(N)`` (engine.py:89-103)."""
    name = text.strip().lower()
    if name == "scalar":
        return EngineKind.scalar_kind()
    if name == "native":
        return EngineKind.native()
    if name == "emulated":
        return EngineKind.emulated(64)
    for prefix, suffix in (("emulated-", ""), ("emulated(", ")")):
        if name.startswith(prefix) and name.endswith(suffix) and len(name) > len(prefix) + len(suffix):
            body = name[len(prefix) : len(name) - len(suffix)]
            if body.isdigit():
                return EngineKind.emulated(int(body))
    raise ValueError(f"cannot parse engine name {text!r}")


def _parse_cpu_features(cpuinfo_text: str) -> frozenset[str]:
    """``flags`` / ``Features`` lines of /proc/cpuinfo (engine.py:106-112)."""
    features: set[str] = set()
    for line in cpuinfo_text.splitlines():
        key, _, value = line.partition(":")
        if key.strip().lower() in ("flags", "features"):
            features.update(value.split())
    return frozenset(features)


def _host_features() -> frozenset[str]:
    try:
        with open("/proc/cpuinfo", encoding="ascii", errors="replace") as fh:
            return _parse_cpu_features(fh.read())
    except OSError:
        return frozenset()


@dataclass(frozen=True)
class EngineInventory:
    """Same fields as the reference (engine.py:132-136) -- ``kinds``,
    ``cpu_features``, ``native_capable_host`` -- plus the device name and,
    when the native engine cannot run, the reason.  ``native_capable_host``
    here means "this host can run the native engine" (a B200 is visible and
    the library loads): the B200 engine's prerequisite is the GPU, not a CPU
    feature set."""

    kinds: tuple[EngineKind, ...]
    cpu_features: frozenset[str]
    native_capable_host: bool
    device_name: str | None = None
    reason: str | None = None

    def available(self, kind: EngineKind) -> bool:
        return kind in self.kinds


@lru_cache(maxsize=1)
def detect() -> EngineInventory:
    """Enumerate usable engines; stable for the life of the process (engine.py:141-153)."""
    reason = _native.unavailable_reason()
    name = torch.cuda.get_device_name() if torch.cuda.is_available() else None
    kinds = (EngineKind.native(),) if reason is None else ()
    return EngineInventory(kinds=kinds, cpu_features=_host_features(), native_capable_host=reason is None,
                           device_name=name, reason=reason)


def resolve_engine(engine: EngineKind | str | None = None) -> EngineKind:
    """Engine named by the argument, else the environment, else ``native``."""
    if engine is None:
        named = os.environ.get(ENGINE_ENV_VAR)
        return parse_engine(named) if named else EngineKind.native()
    if isinstance(engine, str):
        return parse_engine(engine)
    return engine


def _check_byte_order(order: str) -> bool:
    """True for UTF-16BE.  The reference offers BE only through its CLI
    (swap before / after the LE call, cli.py:90-94, 113-114); here it is a
    keyword-only extension of the facade, fused into the kernels."""
    if order not in ("le", "be"):
        raise ValueError(f"utf16_byte_order must be 'le' or 'be', not {order!r}")
    return order == "be"


def _check_direction(direction: str) -> None:
    if direction not in DIRECTIONS:
        raise ValueError(f"direction must be one of {DIRECTIONS}")


def _require_native(kind: EngineKind) -> None:
    if kind.family != "native":
        raise ValueError(
            f"{kind.describe()} engine unavailable: this build ships only the native B200 engine "
            "(the CPU engines live in the reference laneutf package)"
        )
    inventory = detect()
    if not inventory.available(kind):
        raise ValueError(f"native engine unavailable: {inventory.reason}")


def worst_case_output_bytes(direction: str, input_length: int) -> int:
    """engine.py:171-175."""
    _check_direction(direction)
    if direction == UTF8_TO_UTF16:
        return 2 * input_length
    return 3 * (input_length // 2)


# ------------------------------------------------------------------ buffers


def _device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def _byte_len(data) -> int:
    if isinstance(data, torch.Tensor):
        return data.numel() * data.element_size()
    if isinstance(data, np.ndarray):
        return data.nbytes
    return memoryview(data).nbytes


def _to_device_bytes(data, device: torch.device) -> torch.Tensor:
    """Input as a contiguous uint8 CUDA tensor (zero-copy when already there)."""
    if (type(data) is torch.Tensor and data.is_cuda and data.dtype == torch.uint8 and data.dim() == 1
            and data.is_contiguous() and data.get_device() == device.index):
        return data  # fast path: nothing to convert (small calls are host-bound)
    if isinstance(data, torch.Tensor):
        t = data.contiguous()
        if t.dtype != torch.uint8:
            t = t.view(torch.uint8) if t.numel() else torch.empty(0, dtype=torch.uint8)
        t = t.reshape(-1)
        if t.is_cuda:
            return t if t.device == device else t.to(device)
        return t.to(device, non_blocking=t.is_pinned())
    if isinstance(data, np.ndarray):
        arr = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    else:
        arr = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)
    if arr.size == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # read-only host buffers are only read
        host = torch.from_numpy(arr)
    return host.to(device)


def outcome_from_tensor(res: torch.Tensor) -> TranscodeOutcome:
    """Decode a device/host lu_outcome (3 x int64: status|pad, consumed, written)."""
    v = res.view(torch.int64)[:3].tolist()
    status = STATUS_BY_CODE[int(v[0]) & 0xFFFFFFFF]
    return TranscodeOutcome(status, int(v[1]), int(v[2]))


def _side_stream(stream: torch.cuda.Stream | None, device: torch.device) -> torch.cuda.Stream | None:
    """The stream to launch on, ordered after the current stream when it differs.

    Inputs made contiguous, outputs, outcome records and workspaces allocated
    here come from the caching allocator on the *current* stream; a launch on
    another stream first waits for that stream (allocation and copies done),
    and ``_keep_alive`` then ties those temporaries to the launch stream so
    their blocks are not reused while the kernel still runs."""
    if stream is None:
        return None
    cur = torch.cuda.current_stream(device)
    if stream == cur:
        return None
    stream.wait_stream(cur)
    return stream


def _keep_alive(side: torch.cuda.Stream | None, *tensors: torch.Tensor | None) -> None:
    if side is None:
        return
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(side)


def _check_out_tensor(out: torch.Tensor, device: torch.device) -> None:
    """The kernels write ``numel * element_size`` contiguous bytes from
    ``data_ptr``: a strided view or a tensor on another GPU would be
    corrupted (or fault) silently."""
    if not out.is_contiguous():
        raise ValueError("output tensor must be contiguous")
    if out.device != device:
        raise ValueError(f"output tensor is on {out.device}, input on {device}")


def transcode_device(
    direction: str,
    src: torch.Tensor,
    out: torch.Tensor | None = None,
    *,
    res: torch.Tensor | None = None,
    ws: torch.Tensor | None = None,
    stream: torch.cuda.Stream | None = None,
    utf16_byte_order: str = "le",
) -> tuple[torch.Tensor, torch.Tensor]:
    """Device-resident transcode, enqueued on ``stream``; no synchronisation.

    ``src`` is a CUDA tensor holding the input bytes (UTF-8 bytes, or UTF-16LE
    as uint8 of even length / int16 / uint16).  Returns ``(res, out)``:
    ``res`` is an int64[3] CUDA tensor with the lu_outcome (decode with
    ``outcome_from_tensor`` after the stream completes) and ``out`` the
    worst-case output buffer (uint16 words or uint8 bytes).  With a
    ``stream`` other than the current one, the launch is ordered after the
    current stream's work and every temporary allocated here stays alive
    until the launch stream is done with it.
    """
    _check_direction(direction)
    be = _check_byte_order(utf16_byte_order)
    device = src.device
    if out is not None:
        _check_out_tensor(out, device)
    srcb = _to_device_bytes(src, device)
    nbytes = srcb.numel()
    own_out = out is None
    if direction == UTF8_TO_UTF16:
        op, n_units, cap = (_native.OP_UTF8_TO_UTF16BE if be else _native.OP_UTF8_TO_UTF16LE), nbytes, nbytes
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint16, device=device)
        out_cap = out.numel() * out.element_size() // 2
    else:
        if nbytes % 2:
            raise ValueError("UTF-16 input must be an even number of bytes")
        op, n_units = (_native.OP_UTF16BE_TO_UTF8 if be else _native.OP_UTF16LE_TO_UTF8), nbytes // 2
        cap = 3 * n_units
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint8, device=device)
        out_cap = out.numel() * out.element_size()
    own_res, own_ws = res is None, ws is None
    if res is None:
        res = torch.empty(3, dtype=torch.int64, device=device)
    if ws is None:
        ws = torch.empty(_native.workspace_bytes(op, n_units) // 8 + 1, dtype=torch.int64, device=device)
    side = _side_stream(stream, device)
    _native.launch(op, srcb, n_units, out, out_cap, ws, res, stream)
    _keep_alive(side, srcb if srcb.data_ptr() != src.data_ptr() else None, out if own_out else None,
                res if own_res else None, ws if own_ws else None)
    return res, out


def validate_device(
    direction: str,
    src: torch.Tensor,
    *,
    res: torch.Tensor | None = None,
    ws: torch.Tensor | None = None,
    stream: torch.cuda.Stream | None = None,
    utf16_byte_order: str = "le",
) -> torch.Tensor:
    """Device-resident validation; returns the int64[3] outcome tensor
    (stream rules as ``transcode_device``)."""
    _check_direction(direction)
    be = _check_byte_order(utf16_byte_order)
    device = src.device
    srcb = _to_device_bytes(src, device)
    nbytes = srcb.numel()
    if direction == UTF8_TO_UTF16:
        op, n_units = _native.OP_VALIDATE_UTF8, nbytes
    else:
        if nbytes % 2:
            raise ValueError("UTF-16 input must be an even number of bytes")
        op, n_units = (_native.OP_VALIDATE_UTF16BE if be else _native.OP_VALIDATE_UTF16LE), nbytes // 2
    own_res, own_ws = res is None, ws is None
    if res is None:
        res = torch.empty(3, dtype=torch.int64, device=device)
    if ws is None:
        ws = torch.empty(_native.workspace_bytes(op, n_units) // 8 + 1, dtype=torch.int64, device=device)
    side = _side_stream(stream, device)
    _native.launch(op, srcb, n_units, None, 0, ws, res, stream)
    _keep_alive(side, srcb if srcb.data_ptr() != src.data_ptr() else None, res if own_res else None,
                ws if own_ws else None)
    return res


# ------------------------------------------------------------- facade


def _is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def transcode(
    direction: str,
    data,
    out,
    *,
    engine: EngineKind | str | None = None,
    utf16_byte_order: str = "le",
) -> TranscodeOutcome:
    """Route one transcode call to the B200 engine (engine.py:178-209).

    ``consumed`` and ``written`` count code units of the source and
    destination formats.  ``out`` receives exactly the transcoded valid
    prefix (``unit * written`` bytes); nothing past it is touched.
    ``utf16_byte_order="be"`` (keyword-only extension): the UTF-16 side is
    big-endian, byte swap fused into the kernels.

    Host ``data`` and host ``out`` (``bytes`` / ``bytearray`` / memoryview /
    numpy / CPU tensors, the reference callers' case) stream through a
    reusable ring of chunk buffers with H2D, kernels and D2H overlapped
    (hostpipe.py); pinned tensors are read and written in place.  A CUDA
    ``data`` or ``out`` keeps the data on the device.
    """
    _check_direction(direction)
    be = _check_byte_order(utf16_byte_order)
    kind = resolve_engine(engine)
    if direction == UTF16_TO_UTF8 and _byte_len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    _require_native(kind)
    if not _is_device(data) and not _is_device(out):
        if isinstance(out, torch.Tensor) and not out.is_contiguous():
            raise ValueError("output tensor must be contiguous")
        return hostpipe.stream_transcode(direction == UTF8_TO_UTF16, data, out, be=be)
    device = _device()
    src = _to_device_bytes(data, device)
    out_dev = out if _is_device(out) else None
    if out_dev is not None:
        _check_out_tensor(out_dev, device)
    res, buf = transcode_device(direction, src, out_dev, utf16_byte_order=utf16_byte_order)
    outcome = outcome_from_tensor(res.cpu())
    if out_dev is None:
        unit = 2 if direction == UTF8_TO_UTF16 else 1
        sink = hostpipe.host_u8(out, writable=True)
        k = unit * outcome.written
        if sink.size < k:
            raise ValueError("output buffer smaller than the transcoded payload")
        if k:
            hostpipe._t(sink[:k]).copy_(buf.view(torch.uint8)[:k])
    return outcome


def transcode_to_bytes(
    direction: str,
    data,
    *,
    engine: EngineKind | str | None = None,
    utf16_byte_order: str = "le",
) -> tuple[TranscodeOutcome, bytes]:
    """Transcode into a fresh worst-case buffer; returns outcome + payload (engine.py:212-223)."""
    _check_direction(direction)
    be = _check_byte_order(utf16_byte_order)
    kind = resolve_engine(engine)
    if direction == UTF16_TO_UTF8 and _byte_len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    _require_native(kind)
    unit = 2 if direction == UTF8_TO_UTF16 else 1
    if not _is_device(data):
        sink = np.empty(max(worst_case_output_bytes(direction, _byte_len(data)), 1), dtype=np.uint8)
        outcome = hostpipe.stream_transcode(direction == UTF8_TO_UTF16, data, sink, be=be)
        return outcome, sink[: unit * outcome.written].tobytes()
    res, buf = transcode_device(direction, data, utf16_byte_order=utf16_byte_order)
    outcome = outcome_from_tensor(res.cpu())
    payload = buf.view(torch.uint8)[: unit * outcome.written].cpu().numpy().tobytes()
    return outcome, payload


def validate(
    direction: str,
    data,
    *,
    engine: EngineKind | str | None = None,
    utf16_byte_order: str = "le",
) -> TranscodeOutcome:
    """Validation via the B200 read-only kernels; written is always 0 (engine.py:226-240).
    Host data streams through the chunk ring (hostpipe.stream_validate)."""
    _check_direction(direction)
    be = _check_byte_order(utf16_byte_order)
    kind = resolve_engine(engine)
    if direction == UTF16_TO_UTF8 and _byte_len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    _require_native(kind)
    if not _is_device(data):
        return hostpipe.stream_validate(direction == UTF8_TO_UTF16, data, be=be)
    res = validate_device(direction, data, utf16_byte_order=utf16_byte_order)
    outcome = outcome_from_tensor(res.cpu())
    return TranscodeOutcome(outcome.status, outcome.consumed, 0)


# ------------------------------------------- lengths and char counts (8f)


def count_device(op: int, src: torch.Tensor, *, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Enqueue a length (validate + count) or char-count op on a CUDA uint8
    tensor; returns the int64 result tensor (lu_outcome[3] for the length ops,
    [1] count for the char counts).  No synchronisation (stream rules as
    ``transcode_device``)."""
    srcb = _to_device_bytes(src, src.device)
    nbytes = srcb.numel()
    utf16 = op in (_native.OP_UTF8_LENGTH_FROM_UTF16LE, _native.OP_UTF16LE_CHAR_COUNT)
    if utf16 and nbytes % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    n_units = nbytes // 2 if utf16 else nbytes
    chars = op in (_native.OP_UTF8_CHAR_COUNT, _native.OP_UTF16LE_CHAR_COUNT)
    res = torch.empty(1 if chars else 3, dtype=torch.int64, device=srcb.device)
    ws = torch.empty(_native.workspace_bytes(op, n_units) // 8 + 1, dtype=torch.int64, device=srcb.device)
    side = _side_stream(stream, srcb.device)
    _native.launch(op, srcb, n_units, None, 0, ws, res, stream)
    _keep_alive(side, srcb if srcb.data_ptr() != src.data_ptr() else None, res, ws)
    return res


def _length(op: int, data, what: str, unit: str) -> int:
    src = _to_device_bytes(data, _device())
    outcome = outcome_from_tensor(count_device(op, src).cpu())
    if not outcome.ok:
        raise ValueError(f"invalid {what} at {unit} {outcome.consumed}")
    return outcome.written


def utf16_length_from_utf8(data) -> int:
    """Exact UTF-16 length in words; ValueError if the input is invalid
    (scalar.py:220-225).  One read-only pass: the K3 detectors plus a count."""
    return _length(_native.OP_UTF16_LENGTH_FROM_UTF8, data, "UTF-8", "byte")


def utf8_length_from_utf16le(data) -> int:
    """Exact UTF-8 length in bytes; ValueError if the input is invalid
    (scalar.py:228-233)."""
    if _byte_len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    return _length(_native.OP_UTF8_LENGTH_FROM_UTF16LE, data, "UTF-16", "word")


def utf8_char_count(data) -> int:
    """Lead and ASCII bytes, no validation (scalar.py:246-248)."""
    src = _to_device_bytes(data, _device())
    return int(count_device(_native.OP_UTF8_CHAR_COUNT, src).cpu()[0])


def utf16le_char_count(data) -> int:
    """Words minus low surrogates, no validation (scalar.py:251-257)."""
    if _byte_len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    src = _to_device_bytes(data, _device())
    return int(count_device(_native.OP_UTF16LE_CHAR_COUNT, src).cpu()[0])


# ------------------------------------------ batched independent cases (8f)


def batch_device(
    direction: str,
    data: torch.Tensor,
    offsets: torch.Tensor,
    *,
    validate_only: bool = False,
    stream: torch.cuda.Stream | None = None,
) -> tuple[torch.Tensor, torch.Tensor | None]:
    """Many independent cases in one launch (the difftest campaign / triple
    sweep through the GPU).  ``data``: CUDA uint8 tensor;
    ``offsets``: CUDA int64 tensor of n_cases + 1 unit offsets (bytes for
    UTF-8, 16-bit words for UTF-16).  Returns ``(res, out)``: res int64[n, 3]
    (status, consumed, written per case) and the output buffer, where case i's
    payload starts at unit offsets[i] (UTF-8 -> UTF-16, words) or
    3 * offsets[i] (UTF-16 -> UTF-8, bytes).  No synchronisation."""
    _check_direction(direction)
    srcb = _to_device_bytes(data, data.device)
    n = offsets.numel() - 1
    res = torch.empty((max(n, 1), 3), dtype=torch.int64, device=srcb.device)
    out = None
    if direction == UTF8_TO_UTF16:
        op = _native.OP_VALIDATE_UTF8 if validate_only else _native.OP_UTF8_TO_UTF16LE
        if not validate_only:
            out = torch.empty(max(srcb.numel(), 1), dtype=torch.uint16, device=srcb.device)
    else:
        if srcb.numel() % 2:
            raise ValueError("UTF-16 input must be an even number of bytes")
        op = _native.OP_VALIDATE_UTF16LE if validate_only else _native.OP_UTF16LE_TO_UTF8
        if not validate_only:
            out = torch.empty(max(3 * (srcb.numel() // 2), 1), dtype=torch.uint8, device=srcb.device)
    if n > 0:
        _native.launch_batch(op, srcb, offsets, out, res, stream)
    return res[:n], out


def _pack_cases(direction: str, cases) -> tuple[torch.Tensor, torch.Tensor]:
    unit = 1 if direction == UTF8_TO_UTF16 else 2
    lens = [len(c) for c in cases]
    if unit == 2 and any(n % 2 for n in lens):
        raise ValueError("UTF-16 input must be an even number of bytes")
    offs = np.zeros(len(cases) + 1, dtype=np.int64)
    np.cumsum(np.asarray(lens, dtype=np.int64) // unit, out=offs[1:])
    blob = b"".join(bytes(c) for c in cases)
    dev = _device()
    return _to_device_bytes(blob, dev), torch.from_numpy(offs).to(dev)


def transcode_batch(direction: str, cases) -> list[tuple[TranscodeOutcome, bytes]]:
    """``transcode_to_bytes`` for every case of a list, in one launch."""
    data, offs = _pack_cases(direction, cases)
    res, out = batch_device(direction, data, offs)
    rows = res.cpu().tolist()
    offs_h = offs.cpu().tolist()
    outb = out.view(torch.uint8).cpu().numpy() if out is not None else None
    result = []
    for i, (st, consumed, written) in enumerate(rows):
        o = TranscodeOutcome(STATUS_BY_CODE[st & 0xFFFFFFFF], consumed, written)
        if direction == UTF8_TO_UTF16:
            a = 2 * offs_h[i]
            payload = outb[a: a + 2 * written].tobytes()
        else:
            a = 3 * offs_h[i]
            payload = outb[a: a + written].tobytes()
        result.append((o, payload))
    return result


def validate_batch(direction: str, cases) -> list[TranscodeOutcome]:
    """``validate`` for every case of a list, in one launch."""
    data, offs = _pack_cases(direction, cases)
    res, _ = batch_device(direction, data, offs, validate_only=True)
    return [TranscodeOutcome(STATUS_BY_CODE[st & 0xFFFFFFFF], c, 0) for st, c, _ in res.cpu().tolist()]


def swap_utf16_byte_order(data: bytes) -> bytes:
    """Byte-swap every 16-bit unit (LE <-> BE) (engine.py:243-250)."""
    if len(data) % 2:
        raise ValueError("UTF-16 input must have even byte length")
    arr = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint16)
    return arr.byteswap().tobytes()


__all__ += ["TranscodeOutcome", "TranscodeStatus"]
