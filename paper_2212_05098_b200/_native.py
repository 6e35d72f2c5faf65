"""ctypes binding of ``liblaneutf_b200.so`` (C ABI: include/laneutf_b200.h).

Device buffers are torch CUDA tensors owned by Python (torch's caching
allocator); pointers cross the boundary as ``tensor.data_ptr()`` and the
stream as ``torch.cuda.current_stream().cuda_stream``.  ctypes releases the
GIL for the duration of each call.  There is no CPU fallback: if the library
is missing or the device is not sm_100, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

__all__ = [
    "LIB_PATH",
    "NativeUnavailable",
    "lib",
    "available",
    "unavailable_reason",
    "OP_UTF8_TO_UTF16LE",
    "OP_UTF16LE_TO_UTF8",
    "OP_VALIDATE_UTF8",
    "OP_VALIDATE_UTF16LE",
    "OP_UTF16_LENGTH_FROM_UTF8",
    "OP_UTF8_LENGTH_FROM_UTF16LE",
    "OP_UTF8_CHAR_COUNT",
    "OP_UTF16LE_CHAR_COUNT",
    "OP_UTF8_TO_UTF16BE",
    "OP_UTF16BE_TO_UTF8",
    "OP_VALIDATE_UTF16BE",
    "workspace_bytes",
    "launch",
    "launch_batch",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblaneutf_b200.so")

OP_UTF8_TO_UTF16LE = 0
OP_UTF16LE_TO_UTF8 = 1
OP_VALIDATE_UTF8 = 2
OP_VALIDATE_UTF16LE = 3
OP_UTF16_LENGTH_FROM_UTF8 = 4
OP_UTF8_LENGTH_FROM_UTF16LE = 5
OP_UTF8_CHAR_COUNT = 6
OP_UTF16LE_CHAR_COUNT = 7
OP_UTF8_TO_UTF16BE = 8
OP_UTF16BE_TO_UTF8 = 9
OP_VALIDATE_UTF16BE = 10

# C ABI symbols, in header order (tests check the .so exports all of them)
SYMBOLS = (
    "lu_utf8_to_utf16le",
    "lu_utf16le_to_utf8",
    "lu_validate_utf8",
    "lu_validate_utf16le",
    "lu_utf8_to_utf16be",
    "lu_utf16be_to_utf8",
    "lu_validate_utf16be",
    "lu_utf16_length_from_utf8",
    "lu_utf8_length_from_utf16le",
    "lu_utf8_char_count",
    "lu_utf16le_char_count",
    "lu_batch_utf8_to_utf16le",
    "lu_batch_utf16le_to_utf8",
    "lu_batch_validate_utf8",
    "lu_batch_validate_utf16le",
    "lu_workspace_bytes",
    "lu_device_supported",
    "lu_tile_bytes",
    "lu_last_error",
    "lu_version",
)

_ERRORS = {-1: "invalid argument", -2: "workspace too small", -3: "output capacity too small", -4: "CUDA error"}


class NativeUnavailable(ValueError):
    """The native B200 engine cannot run here (no library / no sm_100 GPU)."""


_lock = threading.Lock()
_lib = None
_load_error: str | None = None


def lib():
    """Load (once) and return the ctypes library; raise NativeUnavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                _load_error = f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; g.build()'`)"
                raise NativeUnavailable(_load_error)
            try:
                L = ctypes.CDLL(LIB_PATH)
            except OSError as exc:  # pragma: no cover - depends on the box
                _load_error = f"cannot load {LIB_PATH}: {exc}"
                raise NativeUnavailable(_load_error) from exc
            vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
            for name in ("lu_utf8_to_utf16le", "lu_utf16le_to_utf8", "lu_utf8_to_utf16be", "lu_utf16be_to_utf8"):
                fn = getattr(L, name)
                fn.argtypes = [vp, u64, vp, u64, vp, u64, vp, vp]
                fn.restype = i32
            for name in ("lu_validate_utf8", "lu_validate_utf16le", "lu_validate_utf16be", "lu_utf16_length_from_utf8",
                         "lu_utf8_length_from_utf16le", "lu_utf8_char_count", "lu_utf16le_char_count"):
                fn = getattr(L, name)
                fn.argtypes = [vp, u64, vp, u64, vp, vp]
                fn.restype = i32
            u32 = ctypes.c_uint32
            for name in ("lu_batch_utf8_to_utf16le", "lu_batch_utf16le_to_utf8"):
                fn = getattr(L, name)
                fn.argtypes = [vp, vp, u32, vp, vp, vp]
                fn.restype = i32
            for name in ("lu_batch_validate_utf8", "lu_batch_validate_utf16le"):
                fn = getattr(L, name)
                fn.argtypes = [vp, vp, u32, vp, vp]
                fn.restype = i32
            L.lu_workspace_bytes.argtypes = [i32, u64]
            L.lu_workspace_bytes.restype = u64
            L.lu_device_supported.argtypes = [i32]
            L.lu_device_supported.restype = i32
            L.lu_tile_bytes.argtypes = []
            L.lu_tile_bytes.restype = i32
            L.lu_last_error.argtypes = []
            L.lu_last_error.restype = ctypes.c_char_p
            L.lu_version.argtypes = []
            L.lu_version.restype = ctypes.c_char_p
            _lib = L
    return _lib


def unavailable_reason(device: int | None = None) -> str | None:
    """None if the native engine can run on ``device``, else why not."""
    try:
        L = lib()
    except NativeUnavailable as exc:
        return str(exc)
    if not torch.cuda.is_available():
        return "no CUDA device visible"
    dev = torch.cuda.current_device() if device is None else device
    if not L.lu_device_supported(dev):
        name = torch.cuda.get_device_name(dev)
        return f"device {dev} ({name}) is not sm_100 (B200)"
    return None


def available(device: int | None = None) -> bool:
    return unavailable_reason(device) is None


def workspace_bytes(op: int, n_units: int) -> int:
    return int(lib().lu_workspace_bytes(op, n_units))


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().lu_last_error().decode("utf-8", "replace")
        kind = _ERRORS.get(rc, f"error {rc}")
        if rc == -3:
            raise ValueError(f"output buffer too small: {msg}")
        raise RuntimeError(f"liblaneutf_b200: {kind}: {msg}")


def _ptr(t: torch.Tensor | None) -> int:
    return t.data_ptr() if t is not None and t.numel() else 0


try:  # the raw cudaStream_t of the current stream without building a Stream object
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover - older torch
    _raw_stream = None


def _stream_handle(stream, device: torch.device) -> int:
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None:
        return _raw_stream(device.index if device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


def launch_batch(
    op: int,
    data: torch.Tensor,
    offsets: torch.Tensor,
    out: torch.Tensor | None,
    res: torch.Tensor,
    stream: torch.cuda.Stream | None = None,
) -> None:
    """Enqueue one batched call (op in OP_UTF8_TO_UTF16LE, OP_UTF16LE_TO_UTF8,
    OP_VALIDATE_UTF8, OP_VALIDATE_UTF16LE): ``offsets`` is a CUDA int64 tensor
    of n_cases + 1 unit offsets into ``data``; ``res`` int64[n_cases, 3]."""
    L = lib()
    sp = _stream_handle(stream, data.device)
    n = offsets.numel() - 1
    if op == OP_UTF8_TO_UTF16LE:
        rc = L.lu_batch_utf8_to_utf16le(_ptr(data), _ptr(offsets), n, _ptr(out), _ptr(res), sp)
    elif op == OP_UTF16LE_TO_UTF8:
        rc = L.lu_batch_utf16le_to_utf8(_ptr(data), _ptr(offsets), n, _ptr(out), _ptr(res), sp)
    elif op == OP_VALIDATE_UTF8:
        rc = L.lu_batch_validate_utf8(_ptr(data), _ptr(offsets), n, _ptr(res), sp)
    elif op == OP_VALIDATE_UTF16LE:
        rc = L.lu_batch_validate_utf16le(_ptr(data), _ptr(offsets), n, _ptr(res), sp)
    else:
        raise ValueError(f"unknown batch op {op}")
    _check(rc)


def launch(
    op: int,
    src: torch.Tensor,
    n_units: int,
    out: torch.Tensor | None,
    out_cap_units: int,
    ws: torch.Tensor,
    res: torch.Tensor,
    stream: torch.cuda.Stream | None = None,
) -> None:
    """Enqueue one kernel call on ``stream`` (default: current stream).

    ``src``/``out``/``ws``/``res`` are CUDA tensors; ``res`` holds one
    lu_outcome (>= 24 bytes, 8-byte aligned), or for the char-count ops one
    uint64 count (``out`` unused).  Returns without synchronising.
    """
    L = lib()
    sp = _stream_handle(stream, src.device)
    wsb = ws.numel() * ws.element_size()
    if op == OP_UTF8_TO_UTF16LE:
        rc = L.lu_utf8_to_utf16le(_ptr(src), n_units, _ptr(out), out_cap_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF16LE_TO_UTF8:
        rc = L.lu_utf16le_to_utf8(_ptr(src), n_units, _ptr(out), out_cap_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_VALIDATE_UTF8:
        rc = L.lu_validate_utf8(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_VALIDATE_UTF16LE:
        rc = L.lu_validate_utf16le(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF8_TO_UTF16BE:
        rc = L.lu_utf8_to_utf16be(_ptr(src), n_units, _ptr(out), out_cap_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF16BE_TO_UTF8:
        rc = L.lu_utf16be_to_utf8(_ptr(src), n_units, _ptr(out), out_cap_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_VALIDATE_UTF16BE:
        rc = L.lu_validate_utf16be(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF16_LENGTH_FROM_UTF8:
        rc = L.lu_utf16_length_from_utf8(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF8_LENGTH_FROM_UTF16LE:
        rc = L.lu_utf8_length_from_utf16le(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF8_CHAR_COUNT:
        rc = L.lu_utf8_char_count(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    elif op == OP_UTF16LE_CHAR_COUNT:
        rc = L.lu_utf16le_char_count(_ptr(src), n_units, _ptr(ws), wsb, _ptr(res), sp)
    else:
        raise ValueError(f"unknown op {op}")
    _check(rc)
