"""Host-buffer path, streams and concurrency.

* bytes / bytearray / numpy / pageable and pinned tensors through the
  streaming chunk ring (hostpipe.py), with errors at chunk cuts, canaries
  past ``written``, and ring reuse across calls;
* the reference's acceptance criterion 9 floors (native >= 1 GB/s
  UTF-8 -> UTF-16 and >= 2 GB/s UTF-16 -> UTF-8 on a 1 MiB twobyte-heavy
  corpus, timed like ``bench.run_bench``: bytes in, bytearray out;
  /root/reference/pkg/tests/test_acceptance.py:179-198);
* launches on a side stream with the default workspace, and concurrent
  calls from two threads on two streams (concurrent calls on
  disjoint buffers are safe);
* the output-tensor checks (contiguity, device).
"""

import threading
import time

import numpy as np
import pytest
import torch

import oracle
from paper_2212_05098_b200 import (
    UTF8_TO_UTF16,
    UTF16_TO_UTF8,
    corpus,
    hostpipe,
    outcome_from_tensor,
    transcode,
    transcode_device,
    transcode_to_bytes,
    validate,
    validate_device,
)

pytestmark = pytest.mark.gpu


def _ref(utf16: bool, data: bytes):
    return oracle.utf16le_to_utf8(data) if utf16 else oracle.utf8_to_utf16le(data)


def _errs(utf16: bool, n: int, chunk_units: int):
    return [None, 0, 7, chunk_units - 1, chunk_units, chunk_units + 1, 3 * chunk_units + 2, n // 2, n - 1]


@pytest.mark.parametrize("utf16", [False, True])
@pytest.mark.parametrize("kind", ["bytes", "numpy", "pageable", "pinned"])
def test_stream_transcode_host_buffers(cuda_ok, utf16, kind):
    """Many small chunks (chunk = 1 MiB), errors at and next to chunk cuts:
    outcome and payload equal the oracle's, nothing past the payload is
    touched, and validate agrees."""
    chunk = 1 << 20
    units = (5 << 20) // (2 if utf16 else 1) + 333
    base = corpus.generate("mix", units, 71, utf16=utf16).numpy()
    cu = chunk // (2 if utf16 else 1)
    for pos in _errs(utf16, units, cu):
        b = base.copy()
        if pos is not None:
            if utf16:
                b.view("<u2")[pos] = 0xDC00
            else:
                b[pos] = 0xFF
        raw = b.tobytes()
        cap = (3 * units) if utf16 else (2 * units)
        if kind == "bytes":
            src, sink = raw, bytearray(b"\xa5" * (cap + 64))
        elif kind == "numpy":
            src, sink = b, np.full(cap + 64, 0xA5, dtype=np.uint8)
        elif kind == "pageable":
            src, sink = torch.from_numpy(b), torch.full((cap + 64,), 0xA5, dtype=torch.uint8)
        else:
            src = torch.from_numpy(b).pin_memory()
            sink = torch.full((cap + 64,), 0xA5, dtype=torch.uint8).pin_memory()
        got = hostpipe.stream_transcode(not utf16, src, sink, chunk_bytes=chunk)
        ref, payload = _ref(utf16, raw)
        assert got.as_tuple() == ref, (kind, pos, got, ref)
        out = bytes(memoryview(sink.numpy() if isinstance(sink, torch.Tensor) else sink).cast("B"))
        assert out[: len(payload)] == payload
        assert set(out[len(payload):]) <= {0xA5}
        v = hostpipe.stream_validate(not utf16, src, chunk_bytes=chunk)
        vref = oracle.validate_utf16le(raw) if utf16 else oracle.validate_utf8(raw)
        assert v.as_tuple() == vref, (kind, pos, v)


@pytest.mark.parametrize("utf16", [False, True])
def test_facade_host_bytes_large(cuda_ok, utf16):
    """The facade on 80 MiB of bytes (3 chunks of the default size): the
    reference callers' call, transcode(direction, bytes, bytearray), plus
    transcode_to_bytes and validate, twice (the chunk ring is reused)."""
    units = (80 << 20) // (2 if utf16 else 1)
    raw = corpus.generate("cjk" if utf16 else "emoji", units, 5, utf16=utf16).numpy().tobytes()
    direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
    ref, payload = _ref(utf16, raw)
    for _ in range(2):
        out = bytearray(3 * units if utf16 else 2 * units)
        assert transcode(direction, raw, out).as_tuple() == ref
        assert out[: len(payload)] == payload
        o, p = transcode_to_bytes(direction, raw)
        assert o.as_tuple() == ref and p == payload
        assert validate(direction, raw).as_tuple() == (ref[0], ref[1], 0)


def test_output_too_small_raises(cuda_ok):
    raw = corpus.generate("latin", 100_000, 1).numpy().tobytes()
    with pytest.raises(ValueError):
        transcode(UTF8_TO_UTF16, raw, bytearray(1000))
    with pytest.raises(ValueError):
        transcode(UTF8_TO_UTF16, raw, bytes(2 * len(raw)))  # read-only


def test_output_tensor_checks(cuda_ok):
    dev = torch.device("cuda", 0)
    src = corpus.generate("latin", 4096, 1, device=dev)
    strided = torch.empty((4096, 2), dtype=torch.uint16, device=dev)[:, 0]
    with pytest.raises(ValueError):
        transcode_device(UTF8_TO_UTF16, src, strided)
    with pytest.raises(ValueError):
        transcode(UTF8_TO_UTF16, src, strided)
    with pytest.raises(ValueError):
        transcode(UTF8_TO_UTF16, src.cpu(), torch.empty((4096, 2), dtype=torch.uint16)[:, 0])


def _twobyte_heavy(n: int) -> bytes:
    """UTF-8 text of mostly 2-byte characters (the reference's
    ``twobyte-heavy`` script class): the cyrillic profile, 80% U+0400-04FF."""
    return corpus.generate("cyrillic", n, 77).numpy().tobytes()


def _run_bench_like(direction, data, reps=10, warmup=3):
    """bench.run_bench's timing (src/bench.py:78-129): bytes in, bytearray
    out, min over the timed repetitions."""
    out = bytearray(2 * len(data) if direction == UTF8_TO_UTF16 else 3 * (len(data) // 2))
    for _ in range(warmup):
        transcode(direction, data, out, engine="native")
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        o = transcode(direction, data, out, engine="native")
        best = min(best, time.perf_counter_ns() - t0)
    return o, len(data) / (best / 1e9)


def test_acceptance_criterion9_native_floors(cuda_ok):
    """test_acceptance.py:179-198: the native engine transcodes a 1 MiB
    twobyte-heavy corpus at >= 1 GB/s UTF-8 -> UTF-16 and >= 2 GB/s
    UTF-16 -> UTF-8 (bytes per second of input, min over 10 reps)."""
    data = _twobyte_heavy(1 << 20)
    o, bps = _run_bench_like(UTF8_TO_UTF16, data)
    assert o.ok and bps >= 1e9, bps
    words = transcode_to_bytes(UTF8_TO_UTF16, data)[1]
    o, bps16 = _run_bench_like(UTF16_TO_UTF8, words)
    assert o.ok and bps16 >= 2e9, bps16
    print(f"criterion 9: utf8->utf16 {bps / 1e9:.2f} GB/s, utf16->utf8 {bps16 / 1e9:.2f} GB/s")


def test_side_stream_default_workspace(cuda_ok):
    """a launch on a non-current stream with the default (freshly
    allocated) workspace / output / record; the current stream then reuses
    freed blocks immediately.  Results must equal the oracle."""
    dev = torch.device("cuda", 0)
    side = torch.cuda.Stream(dev)
    data = corpus.generate("cjk", 64 << 20, 3, device=dev)
    raw = data.cpu().numpy().tobytes()
    ref, payload = oracle.utf8_to_utf16le(raw)
    for _ in range(3):
        res, out = transcode_device(UTF8_TO_UTF16, data, stream=side)
        vres = validate_device(UTF8_TO_UTF16, data, stream=side)
        # churn the allocator on the current stream while the side stream runs
        junk = [torch.full((8 << 20,), 7, dtype=torch.int64, device=dev) for _ in range(6)]
        del junk
        side.synchronize()
        assert outcome_from_tensor(res.cpu()).as_tuple() == ref
        assert outcome_from_tensor(vres.cpu()).as_tuple() == oracle.validate_utf8(raw)
        assert out.view(torch.uint8)[: len(payload)].cpu().numpy().tobytes() == payload


def test_concurrent_calls_two_threads_two_streams(cuda_ok):
    """concurrent calls on disjoint buffers are safe.  Two host
    threads, each on its own stream, run K1 / K2 / K3 on different buffers
    back to back; every result equals the oracle."""
    dev = torch.device("cuda", 0)
    jobs = []
    for i, (profile, utf16) in enumerate((("latin", False), ("emoji", True))):
        d = corpus.generate(profile, 48 << 20, 40 + i, utf16=utf16, device=dev)
        raw = d.cpu().numpy().tobytes()
        jobs.append((d, utf16, _ref(utf16, raw)))
    errors = []

    def worker(job):
        d, utf16, (ref, payload) = job
        torch.cuda.set_device(0)
        s = torch.cuda.Stream(dev)
        direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
        try:
            with torch.cuda.stream(s):
                for _ in range(8):
                    res, out = transcode_device(direction, d, stream=s)
                    vres = validate_device(direction, d, stream=s)
                    s.synchronize()
                    assert outcome_from_tensor(res.cpu()).as_tuple() == ref
                    assert outcome_from_tensor(vres.cpu()).as_tuple()[:2] == ref[:2]
                    unit = 1 if utf16 else 2
                    assert out.view(torch.uint8)[: unit * ref[2]].cpu().numpy().tobytes() == payload
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(j,)) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors


def test_concurrent_transcodes_share_the_gpu(cuda_ok):
    """Two transcodes of 256 MiB launched on two streams at once (their
    persistent grids compete for the SMs): the scanner is the first CTA to
    start, so neither launch depends on a CTA that cannot become resident."""
    dev = torch.device("cuda", 0)
    a = corpus.generate("cyrillic", 256 << 20, 2, device=dev)
    b = corpus.generate("cjk", 256 << 20, 3, device=dev)
    ra = outcome_from_tensor(transcode_device(UTF8_TO_UTF16, a)[0].cpu())
    rb = outcome_from_tensor(transcode_device(UTF8_TO_UTF16, b)[0].cpu())
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s1.wait_stream(torch.cuda.current_stream(dev))
    s2.wait_stream(torch.cuda.current_stream(dev))
    outs = []
    for _ in range(5):
        outs.append((transcode_device(UTF8_TO_UTF16, a, stream=s1)[0],
                     transcode_device(UTF8_TO_UTF16, b, stream=s2)[0]))
    torch.cuda.synchronize()
    for x, y in outs:
        assert outcome_from_tensor(x.cpu()) == ra and outcome_from_tensor(y.cpu()) == rb
