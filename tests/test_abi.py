"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/laneutf_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from paper_2212_05098_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "laneutf_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_ \*]*?\**\s*\b(lu_[a-z0-9_]+)\s*\(", text, re.M)


def test_header_declares_the_abi():
    names = declared_functions()
    assert set(names) == set(_native.SYMBOLS), names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_host_only_calls():
    lib = _native.lib()
    assert lib.lu_version().startswith(b"laneutf_b200")
    assert lib.lu_tile_bytes() == 8192
    assert _native.workspace_bytes(_native.OP_UTF8_TO_UTF16LE, 1 << 20) >= 8 * 64
    assert _native.workspace_bytes(_native.OP_VALIDATE_UTF8, 1 << 30) >= 16
    assert _native.workspace_bytes(99, 10) == 0


def test_argument_errors_need_no_gpu():
    lib = _native.lib()
    res = ctypes.create_string_buffer(32)
    # null workspace -> invalid, before any CUDA call
    rc = lib.lu_utf8_to_utf16le(None, 0, None, 0, None, 0, res, None)
    assert rc == -1 and b"null" in lib.lu_last_error()
    # capacity below worst case
    ws = ctypes.create_string_buffer(1024)
    rc = lib.lu_utf8_to_utf16le(ctypes.c_void_p(16), 100, ctypes.c_void_p(32), 50,
                                ctypes.addressof(ws), 1024, ctypes.addressof(res), None)
    assert rc == -3
    rc = lib.lu_utf16le_to_utf8(ctypes.c_void_p(17), 10, ctypes.c_void_p(32), 30,
                                ctypes.addressof(ws), 1024, ctypes.addressof(res), None)
    assert rc == -1 and b"misaligned" in lib.lu_last_error()
