"""Streaming host-buffer pipeline for the facade's host path.

The reference's callers hand the facade host memory: ``cli.cmd_transcode``
passes ``bytes`` (/root/reference/pkg/src/laneutf/cli.py:92) and
``bench.run_bench`` times ``bytes`` in / ``bytearray`` out
(/root/reference/pkg/src/laneutf/bench.py:100-106).  This module moves such
buffers through the GPU without ever holding the whole input or the whole
worst-case output on the device:

* The input is cut into chunks at character boundaries (the multi-GPU rule,
  ``shard.snap_cut``); chunk k's local outcome shifted by the chunk offset is
  the whole-buffer outcome whenever chunks 0..k-1 were valid (SURVEY.md
  App. A.4), so processing stops at the first malformed chunk.
* A reusable ring of ``slots`` fixed-size chunk buffers (device input,
  device worst-case output, workspace, outcome record; pinned host staging
  for pageable buffers) is taken from a per-device pool, so a 100 GiB host
  input streams through a few hundred MiB of HBM and pinned memory, and
  repeated calls allocate nothing.
* Three streams: H2D copies, kernels, D2H copies.  Chunk k's H2D and kernel
  are enqueued while chunk k-1's payload (exactly ``written`` units, known
  from its 24-byte outcome record) is copied back and chunk k-2's staged
  payload is copied into the caller's buffer, so PCIe transfers in both
  directions, the kernels and the host-side staging copies overlap.
* Pinned torch tensors are read / written in place (no staging copy);
  ``bytes`` / ``bytearray`` / ``memoryview`` / numpy / pageable tensors go
  through the pinned staging slots (torch's multi-threaded CPU copy).

Every phase is bracketed by an NVTX range (``lu.stage_in``, ``lu.h2d``,
``lu.kernel``, ``lu.d2h``, ``lu.stage_out``) for nsys / ncu timelines
(SURVEY.md section 5).
"""

from __future__ import annotations

import threading
import warnings
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .outcome import STATUS_BY_CODE, TranscodeOutcome
from .shard import snap_cut

__all__ = ["pipelined_transcode", "stream_transcode", "stream_validate", "DEFAULT_CHUNK", "DEFAULT_SLOTS",
           "chunk_cuts", "host_u8"]

DEFAULT_CHUNK = 32 << 20  # bytes of input per chunk (tools/e2e_chunks.py: 16 MiB -11%, 64 MiB -1%)
DEFAULT_SLOTS = 3         # chunks in flight: H2D + kernel of k, D2H of k-1, staging copy-out of k-2


def _nvtx(name: str):
    return torch.cuda.nvtx.range(name)


def host_u8(buf, *, writable: bool = False) -> np.ndarray:
    """A flat uint8 numpy view of a host buffer (no copy)."""
    if isinstance(buf, torch.Tensor):
        t = buf
        if not t.is_contiguous():
            raise ValueError("host tensor must be contiguous")
        return t.view(torch.uint8).reshape(-1).numpy() if t.numel() else np.empty(0, np.uint8)
    if isinstance(buf, np.ndarray):
        if not buf.flags.c_contiguous:
            raise ValueError("host array must be C-contiguous")
        return buf.reshape(-1).view(np.uint8)
    mv = memoryview(buf)
    if writable and mv.readonly:
        raise ValueError("output buffer is read-only")
    if not mv.c_contiguous:
        raise ValueError("host buffer must be contiguous")
    return np.frombuffer(mv.cast("B"), dtype=np.uint8)


def _t(a: np.ndarray) -> torch.Tensor:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # read-only sources are only read
        return torch.from_numpy(a)


def chunk_cuts(src: np.ndarray, utf16: bool, be: bool, chunk_bytes: int) -> list[int]:
    """Unit offsets 0 = c_0 < c_1 < ... < c_K = n of chunks of about
    ``chunk_bytes``, every interior cut on a character boundary."""
    unit = 2 if utf16 else 1
    n = src.size // unit
    if utf16:
        words = src[: 2 * n].view("<u2" if not be else ">u2")

        def unit_at(i: int) -> int:
            return int(words[i])
    else:
        def unit_at(i: int) -> int:
            return int(src[i])
    step = max(chunk_bytes // unit, 1)
    cuts = [0]
    while cuts[-1] < n:
        nxt = min(cuts[-1] + step, n)
        if nxt < n:
            nxt = max(snap_cut(unit_at, n, nxt, utf16), cuts[-1] + 1)
        cuts.append(nxt)
    if len(cuts) == 1:
        cuts.append(0)
    return cuts


class _Ring:
    """``slots`` chunk buffers on one device plus pinned host staging."""

    def __init__(self, device: torch.device, slots: int, chunk_bytes: int):
        self.device, self.slots, self.chunk = device, slots, chunk_bytes
        out_bytes = 2 * chunk_bytes  # worst case of both directions (2x words / 1.5x bytes)
        # a chunk is at most chunk_bytes + 3 (cuts snap forward to a character boundary)
        ws_words = _native.workspace_bytes(_native.OP_UTF8_TO_UTF16LE, chunk_bytes + 16) // 8 + 1
        self.d_in = [torch.empty(chunk_bytes + 16, dtype=torch.uint8, device=device) for _ in range(slots)]
        self.d_out = [torch.empty(out_bytes + 16, dtype=torch.uint8, device=device) for _ in range(slots)]
        self.ws = [torch.empty(ws_words, dtype=torch.int64, device=device) for _ in range(slots)]
        self.res_d = torch.empty((slots, 3), dtype=torch.int64, device=device)
        self.res_h = torch.empty((slots, 3), dtype=torch.int64).pin_memory()
        self._h_in: list[torch.Tensor] | None = None
        self._h_out: list[torch.Tensor] | None = None
        self.s_h2d = torch.cuda.Stream(device)
        self.s_comp = torch.cuda.Stream(device)
        self.s_d2h = torch.cuda.Stream(device)

    def h_in(self, slot: int) -> torch.Tensor:
        if self._h_in is None:
            self._h_in = [torch.empty(self.chunk + 16, dtype=torch.uint8).pin_memory() for _ in range(self.slots)]
        return self._h_in[slot]

    def h_out(self, slot: int) -> torch.Tensor:
        if self._h_out is None:
            self._h_out = [torch.empty(2 * self.chunk + 32, dtype=torch.uint8).pin_memory() for _ in range(self.slots)]
        return self._h_out[slot]


_POOL: dict[tuple[int, int, int], list[_Ring]] = {}
_POOL_LOCK = threading.Lock()


def _acquire(device: torch.device, slots: int, chunk_bytes: int) -> _Ring:
    key = (device.index, slots, chunk_bytes)
    with _POOL_LOCK:
        free = _POOL.setdefault(key, [])
        if free:
            return free.pop()
    return _Ring(device, slots, chunk_bytes)


def _release(ring: _Ring) -> None:
    with _POOL_LOCK:
        _POOL.setdefault((ring.device.index, ring.slots, ring.chunk), []).append(ring)


def _ring_chunk(nbytes: int, chunk_bytes: int) -> int:
    """Slot size: the chunk size, or the input rounded up to a power of two
    (at least 1 MiB) when the whole input fits in one chunk, so small calls
    do not pin 32 MiB slots and the pool holds few distinct sizes."""
    if nbytes >= chunk_bytes:
        return chunk_bytes
    size = 1 << 20
    while size < nbytes:
        size *= 2
    return size


@dataclass
class _Chunk:
    k: int
    slot: int
    begin: int      # first input unit
    n_units: int
    ev_res: torch.cuda.Event | None = None
    ev_kernel: torch.cuda.Event | None = None
    ev_d2h: torch.cuda.Event | None = None
    written: int = 0
    status: int = 0
    consumed: int = 0
    out_at: int = 0        # output unit offset of this chunk's payload
    stage: int = 0         # 0 kernel enqueued, 1 payload D2H enqueued


def _op(utf8_in: bool, be: bool, validate: bool) -> int:
    if validate:
        if utf8_in:
            return _native.OP_VALIDATE_UTF8
        return _native.OP_VALIDATE_UTF16BE if be else _native.OP_VALIDATE_UTF16LE
    if utf8_in:
        return _native.OP_UTF8_TO_UTF16BE if be else _native.OP_UTF8_TO_UTF16LE
    return _native.OP_UTF16BE_TO_UTF8 if be else _native.OP_UTF16LE_TO_UTF8


def _run(utf8_in: bool, src, sink, *, be: bool, validate: bool, chunk_bytes: int,
         slots: int) -> TranscodeOutcome:
    """Core loop.  ``src``: host buffer (pinned tensor read in place, anything
    else staged).  ``sink``: None (validate), a pinned uint8 tensor written in
    place, or a writable uint8 numpy array (staged)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    src_np = host_u8(src)
    src_pinned = src.view(torch.uint8).reshape(-1) if (
        isinstance(src, torch.Tensor) and src.is_pinned() and src.numel()) else None
    sink_pinned = sink if isinstance(sink, torch.Tensor) else None
    sink_np = sink if isinstance(sink, np.ndarray) else None
    unit_in, unit_out = (1, 2) if utf8_in else (2, 1)
    nbytes = src_np.size
    n = nbytes // unit_in
    cuts = chunk_cuts(src_np, not utf8_in, be, chunk_bytes)
    ring = _acquire(dev, slots, _ring_chunk(nbytes, chunk_bytes))
    op = _op(utf8_in, be, validate)
    cur = torch.cuda.current_stream(dev)
    for s in (ring.s_h2d, ring.s_comp, ring.s_d2h):
        s.wait_stream(cur)
    inflight: deque[_Chunk] = deque()
    state = {"written": 0, "outcome": None}

    def advance(c: _Chunk) -> None:
        """Kernel done -> read the outcome, enqueue the payload D2H."""
        with _nvtx("lu.wait_result"):
            c.ev_res.synchronize()
        st, consumed, wr = (int(v) for v in ring.res_h[c.slot].tolist())
        c.status, c.consumed, c.written = st & 0xFFFFFFFF, consumed, (0 if validate else wr)
        c.out_at = state["written"]
        state["written"] += c.written
        if c.status != 0 and state["outcome"] is None:
            state["outcome"] = TranscodeOutcome(STATUS_BY_CODE[c.status], c.begin + c.consumed, state["written"])
        if c.written:
            nb = c.written * unit_out
            cap = sink_pinned.numel() if sink_pinned is not None else sink_np.size
            if (c.out_at + c.written) * unit_out > cap:
                raise ValueError("output buffer smaller than the transcoded payload")
            ring.s_d2h.wait_event(c.ev_kernel)
            with torch.cuda.stream(ring.s_d2h), _nvtx("lu.d2h"):
                if sink_pinned is not None:
                    a = c.out_at * unit_out
                    sink_pinned[a: a + nb].copy_(ring.d_out[c.slot][:nb], non_blocking=True)
                else:
                    ring.h_out(c.slot)[:nb].copy_(ring.d_out[c.slot][:nb], non_blocking=True)
            c.ev_d2h = torch.cuda.Event()
            c.ev_d2h.record(ring.s_d2h)
        c.stage = 1

    def retire(c: _Chunk) -> None:
        """Payload landed -> copy it into a pageable sink."""
        if c.ev_d2h is not None:
            with _nvtx("lu.wait_d2h"):
                c.ev_d2h.synchronize()
            if sink_np is not None:
                nb = c.written * unit_out
                a = c.out_at * unit_out
                with _nvtx("lu.stage_out"):
                    _t(sink_np[a: a + nb]).copy_(ring.h_out(c.slot)[:nb])

    try:
        for k in range(len(cuts) - 1):
            if state["outcome"] is not None:
                break  # a malformed chunk ends the call (the reference stops there too)
            slot = k % ring.slots
            # the slot's previous user must be completely done
            while inflight and inflight[0].k <= k - ring.slots:
                c = inflight.popleft()
                if c.stage == 0:
                    advance(c)
                retire(c)
            if state["outcome"] is not None:
                break
            b0, b1 = cuts[k], cuts[k + 1]
            m = (b1 - b0) * unit_in
            a = b0 * unit_in
            d_in = ring.d_in[slot][:m]
            with torch.cuda.stream(ring.s_h2d):
                if src_pinned is not None:
                    with _nvtx("lu.h2d"):
                        d_in.copy_(src_pinned[a: a + m], non_blocking=True)
                elif m:
                    h = ring.h_in(slot)
                    with _nvtx("lu.stage_in"):
                        h[:m].copy_(_t(src_np[a: a + m]))
                    with _nvtx("lu.h2d"):
                        d_in.copy_(h[:m], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(ring.s_h2d)
            ring.s_comp.wait_event(ev_in)
            n_k = b1 - b0
            if validate:
                d_out, cap = None, 0
            elif utf8_in:
                d_out, cap = ring.d_out[slot][: 2 * max(n_k, 1)].view(torch.uint16), n_k
            else:
                d_out, cap = ring.d_out[slot][: 3 * max(n_k, 1)], 3 * n_k
            with _nvtx("lu.kernel"):
                _native.launch(op, d_in, n_k, d_out, cap, ring.ws[slot], ring.res_d[slot], ring.s_comp)
            c = _Chunk(k, slot, b0, n_k)
            c.ev_kernel = torch.cuda.Event()
            c.ev_kernel.record(ring.s_comp)
            with torch.cuda.stream(ring.s_comp):
                ring.res_h[slot].copy_(ring.res_d[slot], non_blocking=True)
            c.ev_res = torch.cuda.Event()
            c.ev_res.record(ring.s_comp)
            inflight.append(c)
            # software pipeline: result of k-1, staging copy-out of k-2
            if len(inflight) >= 2 and inflight[-2].stage == 0:
                advance(inflight[-2])
            if len(inflight) >= 3 and inflight[0].stage == 1:
                retire(inflight.popleft())
        while inflight:
            c = inflight.popleft()
            if c.stage == 0:
                if state["outcome"] is None:
                    advance(c)
                else:
                    c.ev_res.synchronize()  # past the error: drain, result unused
            retire(c)
    finally:
        for s in (ring.s_h2d, ring.s_comp, ring.s_d2h):
            s.synchronize()
        cur.wait_stream(ring.s_d2h)
        _release(ring)
    if state["outcome"] is not None:
        o = state["outcome"]
        return TranscodeOutcome(o.status, o.consumed, 0 if validate else o.written)
    return TranscodeOutcome(STATUS_BY_CODE[0], n, 0 if validate else state["written"])


def stream_transcode(utf8_in: bool, src, sink, *, be: bool = False, chunk_bytes: int = DEFAULT_CHUNK,
                     slots: int = DEFAULT_SLOTS) -> TranscodeOutcome:
    """Transcode host ``src`` into host ``sink`` (a pinned uint8 tensor, or a
    writable uint8 numpy array of at least the worst case).  Writes exactly
    ``sink[:unit * written]``."""
    if isinstance(sink, torch.Tensor) and sink.is_pinned():
        if not sink.is_contiguous():
            raise ValueError("output tensor must be contiguous")
        sink = sink.view(torch.uint8).reshape(-1)
    else:
        sink = host_u8(sink, writable=True)
    return _run(utf8_in, src, sink, be=be, validate=False, chunk_bytes=chunk_bytes, slots=slots)


def stream_validate(utf8_in: bool, src, *, be: bool = False, chunk_bytes: int = DEFAULT_CHUNK,
                    slots: int = DEFAULT_SLOTS) -> TranscodeOutcome:
    """Validate host ``src`` chunk by chunk; ``written`` is 0."""
    return _run(utf8_in, src, None, be=be, validate=True, chunk_bytes=chunk_bytes, slots=slots)


def pipelined_transcode(utf8_in: bool, host_in: torch.Tensor, host_out: torch.Tensor,
                        chunk_bytes: int = DEFAULT_CHUNK, be: bool = False, ramp_bytes: int = 0,
                        slots: int = DEFAULT_SLOTS) -> TranscodeOutcome:
    """Pinned uint8 ``host_in`` -> pinned uint8 ``host_out`` (round-1 name;
    ``ramp_bytes`` is accepted and ignored)."""
    del ramp_bytes
    return stream_transcode(utf8_in, host_in, host_out, be=be, chunk_bytes=chunk_bytes, slots=slots)
