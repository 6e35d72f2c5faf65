"""Chunked host-buffer pipeline for the facade's host path.

``engine.transcode`` with a pinned host input and a pinned host output (the
call ``cli.cmd_transcode`` / ``bench.run_bench`` make in the reference,
/root/reference/pkg/src/laneutf/cli.py:92, bench.py:105) would otherwise run
H2D -> kernel -> D2H back to back.  Here the input is cut into chunks at
character boundaries (the multi-GPU rule, shard.snap_cut), every H2D copy and
every kernel is enqueued up front on their own streams, and each chunk's
payload is copied back to its final host offset as soon as that chunk's
outcome is known, so host->device and device->host transfers run
concurrently (PCIe / C2C are full duplex) and the kernels hide behind them.

Exactness: a chunk boundary is a character boundary, so chunk k's local
outcome shifted by the chunk offset is the whole-buffer outcome whenever
chunks 0..k-1 were valid; processing stops at the first
malformed chunk.
"""

from __future__ import annotations

import torch

from . import _native
from .outcome import STATUS_BY_CODE, TranscodeOutcome
from .shard import snap_cut

__all__ = ["pipelined_transcode", "DEFAULT_CHUNK"]

DEFAULT_CHUNK = 32 << 20  # bytes of input per chunk (tools/e2e_chunks.py: 16 MiB -11%, 64 MiB -1%)
DEFAULT_RAMP = 0          # first / last chunk size (bytes) of a ramp doubling up to the chunk size; 0 = none


def chunk_sizes(n_bytes: int, chunk_bytes: int, ramp_bytes: int) -> list[int]:
    """Nominal chunk sizes covering n_bytes: a ramp ramp, 2*ramp, ... up to
    chunk_bytes at both ends (a short first H2D / last D2H shortens the
    pipeline's fill and drain), chunk_bytes in between."""
    if ramp_bytes <= 0 or n_bytes <= 2 * chunk_bytes:
        ramp = []
    else:
        ramp, r = [], ramp_bytes
        while r < chunk_bytes:
            ramp.append(r)
            r *= 2
    head = list(ramp)
    tail = list(reversed(ramp))
    mid = n_bytes - sum(head) - sum(tail)
    if mid <= 0:
        head, tail, mid = [], [], n_bytes
    body = [chunk_bytes] * (mid // chunk_bytes)
    if mid % chunk_bytes:
        body.append(mid % chunk_bytes)
    return head + body + tail


def pipelined_transcode(utf8_in: bool, host_in: torch.Tensor, host_out: torch.Tensor,
                        chunk_bytes: int = DEFAULT_CHUNK, be: bool = False,
                        ramp_bytes: int = DEFAULT_RAMP) -> TranscodeOutcome:
    """Transcode pinned ``host_in`` (uint8) into pinned ``host_out`` (uint8).

    Writes exactly ``host_out[:unit * written]``.  Returns the whole-buffer
    outcome.  ``be``: the UTF-16 side is big-endian.
    """
    dev = torch.device("cuda", torch.cuda.current_device())
    nbytes = host_in.numel()
    unit_in = 1 if utf8_in else 2
    unit_out = 2 if utf8_in else 1
    n = nbytes // unit_in
    units = host_in.view(torch.uint8) if utf8_in else host_in.view(torch.int16)

    def unit_at(i: int) -> int:
        u = int(units[i].item()) & 0xFFFF
        if be and not utf8_in:
            u = ((u & 0xFF) << 8) | (u >> 8)
        return u

    steps = [max(c // unit_in, 1) for c in chunk_sizes(nbytes, chunk_bytes, ramp_bytes)]
    cuts = [0]
    while cuts[-1] < n:
        step = steps[len(cuts) - 1] if len(cuts) - 1 < len(steps) else max(chunk_bytes // unit_in, 1)
        nxt = min(cuts[-1] + step, n)
        if nxt < n:
            nxt = max(snap_cut(unit_at, n, nxt, not utf8_in), cuts[-1] + 1)
        cuts.append(nxt)
    if len(cuts) == 1:
        cuts.append(0)

    d_in = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    cap_units = n if utf8_in else 3 * n  # worst case, output units
    d_out = torch.empty(max(cap_units * unit_out, 1), dtype=torch.uint8, device=dev)
    k_chunks = len(cuts) - 1
    res_dev = torch.empty((k_chunks, 3), dtype=torch.int64, device=dev)
    res_host = torch.empty((k_chunks, 3), dtype=torch.int64).pin_memory()
    if utf8_in:
        op = _native.OP_UTF8_TO_UTF16BE if be else _native.OP_UTF8_TO_UTF16LE
    else:
        op = _native.OP_UTF16BE_TO_UTF8 if be else _native.OP_UTF16LE_TO_UTF8

    s_h2d = torch.cuda.Stream(dev)
    s_comp = torch.cuda.Stream(dev)
    s_d2h = torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)
    s_h2d.wait_stream(cur)
    s_comp.wait_stream(cur)
    s_d2h.wait_stream(cur)
    ev_res = []
    ev_done = []
    # enqueue every copy-in and every kernel; nothing here waits on the host
    for k in range(k_chunks):
        a, b = cuts[k] * unit_in, cuts[k + 1] * unit_in
        ev_in = torch.cuda.Event()
        with torch.cuda.stream(s_h2d):
            d_in[a:b].copy_(host_in[a:b], non_blocking=True)
            ev_in.record(s_h2d)
        s_comp.wait_event(ev_in)
        n_k = cuts[k + 1] - cuts[k]
        out_lo = (cuts[k] if utf8_in else 3 * cuts[k]) * unit_out  # worst-case position (bytes)
        out_cap = n_k if utf8_in else 3 * n_k
        src = d_in[a:b]
        dst = d_out[out_lo : out_lo + max(out_cap, 1) * unit_out]
        dst = dst.view(torch.uint16) if utf8_in else dst
        ws = torch.empty(_native.workspace_bytes(op, n_k) // 8 + 1, dtype=torch.int64, device=dev)
        _native.launch(op, src, n_k, dst, out_cap, ws, res_dev[k], s_comp)
        ev_c = torch.cuda.Event()
        ev_c.record(s_comp)
        ev_done.append(ev_c)
        with torch.cuda.stream(s_comp):
            res_host[k].copy_(res_dev[k], non_blocking=True)
        ev_r = torch.cuda.Event()
        ev_r.record(s_comp)
        ev_res.append(ev_r)
        # keep the per-chunk workspace alive until the kernel has run
        ws.record_stream(s_comp)

    # drain results in order; copy each payload to its final host offset
    written = 0
    outcome = None
    for k in range(k_chunks):
        ev_res[k].synchronize()
        st, consumed, wr = (int(v) for v in res_host[k].tolist())
        out_lo = (cuts[k] if utf8_in else 3 * cuts[k]) * unit_out
        if wr:
            s_d2h.wait_event(ev_done[k])
            with torch.cuda.stream(s_d2h):
                host_out[written * unit_out : (written + wr) * unit_out].copy_(
                    d_out[out_lo : out_lo + wr * unit_out], non_blocking=True)
        written += wr
        status = STATUS_BY_CODE[st & 0xFFFFFFFF]
        if (st & 0xFFFFFFFF) != 0:
            outcome = TranscodeOutcome(status, cuts[k] + consumed, written)
            break
    if outcome is None:
        outcome = TranscodeOutcome(STATUS_BY_CODE[0], n, written)
    s_d2h.synchronize()
    s_comp.synchronize()
    cur.wait_stream(s_d2h)
    return outcome
