"""``laneutf/_b200.py`` -- the module a maintainer adds to the reference package.

This is the reference-side binding of the B200 engine shown in
INTEGRATION.md, as a file that runs: the reference's ``engine.transcode``
raises "native engine unavailable" for ``EngineKind.native()``
(/root/reference/pkg/src/laneutf/engine.py:194-200); the patch in
INTEGRATION.md replaces that branch with a call to ``transcode`` below and
appends ``EngineKind.native()`` to ``detect()``'s kinds when ``available()``
is true.  The module depends only on ``ctypes``, ``torch`` (device buffers)
and the C ABI of ``liblaneutf_b200.so`` (include/laneutf_b200.h); it imports
nothing from ``paper_2212_05098_b200``.

``tests/test_integration.py`` and ``tests/test_gpu_integration.py`` load this
file as a module (without modifying the reference or patching its
``detect()``) and run the reference's own differential-campaign case
generator (difftest.py:139-197) through it against the oracle.
"""

from __future__ import annotations

import ctypes
import os

import torch

_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2212_05098_b200",
                            "liblaneutf_b200.so")
_LIB = ctypes.CDLL(os.environ.get("LANEUTF_B200_LIB", _DEFAULT_LIB))
_vp, _u64 = ctypes.c_void_p, ctypes.c_uint64
for _f in (_LIB.lu_utf8_to_utf16le, _LIB.lu_utf16le_to_utf8):
    _f.argtypes = [_vp, _u64, _vp, _u64, _vp, _u64, _vp, _vp]
    _f.restype = ctypes.c_int
for _f in (_LIB.lu_validate_utf8, _LIB.lu_validate_utf16le):
    _f.argtypes = [_vp, _u64, _vp, _u64, _vp, _vp]
    _f.restype = ctypes.c_int
_LIB.lu_workspace_bytes.argtypes = [ctypes.c_int, _u64]
_LIB.lu_workspace_bytes.restype = _u64
_LIB.lu_device_supported.argtypes = [ctypes.c_int]
_LIB.lu_device_supported.restype = ctypes.c_int
_LIB.lu_last_error.restype = ctypes.c_char_p

UTF8_TO_UTF16 = "utf8-to-utf16"  # engine.py:44-46
OP_UTF8_TO_UTF16LE, OP_UTF16LE_TO_UTF8, OP_VALIDATE_UTF8, OP_VALIDATE_UTF16LE = 0, 1, 2, 3


def available() -> bool:
    """The ``detect()`` probe: a visible sm_100 device (engine.py:141-153)."""
    return torch.cuda.is_available() and bool(_LIB.lu_device_supported(torch.cuda.current_device()))


def _src(data: bytes) -> torch.Tensor:
    if not data:
        return torch.empty(0, dtype=torch.uint8, device="cuda")
    return torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(_LIB.lu_last_error().decode())


def transcode(direction: str, data: bytes, out) -> tuple[int, int, int]:
    """Returns (status_code, consumed, written); fills out[:unit*written]."""
    utf8_in = direction == UTF8_TO_UTF16
    if not utf8_in and len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")  # scalar.py:114-115
    src = _src(data)
    n = len(data) if utf8_in else len(data) // 2
    cap = n if utf8_in else 3 * n  # engine.worst_case_output_bytes / unit
    dst = torch.empty(max(cap, 1), dtype=torch.uint16 if utf8_in else torch.uint8, device="cuda")
    op = OP_UTF8_TO_UTF16LE if utf8_in else OP_UTF16LE_TO_UTF8
    ws = torch.empty(_LIB.lu_workspace_bytes(op, n) // 8 + 1, dtype=torch.int64, device="cuda")
    res = torch.empty(3, dtype=torch.int64, device="cuda")
    fn = _LIB.lu_utf8_to_utf16le if utf8_in else _LIB.lu_utf16le_to_utf8
    _check(fn(src.data_ptr() or None, n, dst.data_ptr(), cap, ws.data_ptr(), ws.numel() * 8, res.data_ptr(),
              torch.cuda.current_stream().cuda_stream))
    status, consumed, written = res.cpu().tolist()
    unit = 2 if utf8_in else 1
    if written:
        memoryview(out)[: unit * written] = dst.view(torch.uint8)[: unit * written].cpu().numpy().tobytes()
    return status & 0xFFFFFFFF, consumed, written


def validate(direction: str, data: bytes) -> tuple[int, int, int]:
    """Read-only kernels (lu_validate_utf8 / lu_validate_utf16le); written = 0."""
    utf8_in = direction == UTF8_TO_UTF16
    if not utf8_in and len(data) % 2:
        raise ValueError("UTF-16 input must be an even number of bytes")
    src = _src(data)
    n = len(data) if utf8_in else len(data) // 2
    op = OP_VALIDATE_UTF8 if utf8_in else OP_VALIDATE_UTF16LE
    ws = torch.empty(_LIB.lu_workspace_bytes(op, n) // 8 + 1, dtype=torch.int64, device="cuda")
    res = torch.empty(3, dtype=torch.int64, device="cuda")
    fn = _LIB.lu_validate_utf8 if utf8_in else _LIB.lu_validate_utf16le
    _check(fn(src.data_ptr() or None, n, ws.data_ptr(), ws.numel() * 8, res.data_ptr(),
              torch.cuda.current_stream().cuda_stream))
    status, consumed, _ = res.cpu().tolist()
    return status & 0xFFFFFFFF, consumed, 0


def transcode_to_bytes(direction: str, data: bytes) -> tuple[tuple[int, int, int], bytes]:
    """engine.transcode_to_bytes (engine.py:212-223) with the native branch."""
    out = bytearray(2 * len(data) if direction == UTF8_TO_UTF16 else 3 * (len(data) // 2))
    rec = transcode(direction, data, out)
    unit = 2 if direction == UTF8_TO_UTF16 else 1
    return rec, bytes(out[: unit * rec[2]])
