"""Multi-GPU sharding logic on the CPU: character-boundary cuts, the combine
rule, and the all-gather exchange over a 2-rank gloo group.

The per-shard transcoder here is the oracle (the GPU box runs the same logic
with the native engine and NCCL); the whole-buffer oracle is the reference
result.
"""

import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2212_05098_b200 import corpus
from paper_2212_05098_b200.shard import combine_records, plan_cuts, snap_cut, transcode_sharded


def _mutants(utf16: bool, n_cases: int, seed: int):
    rng = random.Random(seed)
    base = corpus.generate("mix", 5000, seed=seed, utf16=utf16).numpy()
    yield base.copy()
    for _ in range(n_cases):
        data = base.copy()
        for _ in range(rng.randrange(1, 4)):
            p = rng.randrange(len(data))
            data[p] = rng.choice([0x80, 0xBF, 0xC0, 0xE0, 0xED, 0xF0, 0xF4, 0xF8, 0xFF, 0x41, 0xDC, 0xD8])
        yield data


def _sharded_oracle(data: np.ndarray, world: int, utf16: bool):
    units = data.view(np.uint16) if utf16 else data
    cuts = plan_cuts(len(units), world, lambda i: int(units[i]), utf16)
    recs, payloads = [], []
    for r in range(world):
        piece = units[cuts[r] : cuts[r + 1]]
        if utf16:
            (st, consumed, written), payload = oracle.utf16le_to_utf8(piece.tobytes())
        else:
            (st, consumed, written), payload = oracle.utf8_to_utf16le(piece.tobytes())
        recs.append((0 if st == "ok" else 1, consumed, written))
        payloads.append(payload)
    status, consumed, written, offsets = combine_records(recs, cuts[:-1])
    unit = 1 if utf16 else 2
    first_bad = next((i for i, rec in enumerate(recs) if rec[0] != 0), world)
    payload = b"".join(payloads[: first_bad + 1])[: unit * written]
    return ("ok" if status == 0 else "malformed-input", consumed, written), payload, offsets


@pytest.mark.parametrize("utf16", [False, True])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sharded_equals_whole_buffer(utf16, world):
    for data in _mutants(utf16, 60, seed=world + 10 * int(utf16)):
        whole = oracle.utf16le_to_utf8(data.tobytes()) if utf16 else oracle.utf8_to_utf16le(data.tobytes())
        got, payload, _ = _sharded_oracle(data, world, utf16)
        assert got == whole[0]
        assert payload == whole[1]


def test_snap_cut_rules():
    b = bytes.fromhex("41e282ac42f09f9880")
    units = lambda i: b[i]  # noqa: E731
    assert snap_cut(units, len(b), 2, False) == 4  # inside the euro sign -> after it
    assert snap_cut(units, len(b), 6, False) == 9  # F0 9F 98 80: 3 steps
    assert snap_cut(units, len(b), 0, False) == 0
    w = [0x41, 0xD83D, 0xDE00, 0x42]
    assert snap_cut(lambda i: w[i], 4, 2, True) == 3
    assert snap_cut(lambda i: w[i], 4, 1, True) == 1
    # the same rule as the C baseline runner
    for c in range(len(b) + 1):
        assert snap_cut(units, len(b), c, False) == oracle.snap_cut(False, b, c)


def test_combine_rule():
    recs = [(0, 10, 7), (1, 3, 2), (0, 9, 9)]
    st, consumed, written, offsets = combine_records(recs, [0, 10, 20])
    assert (st, consumed, written) == (1, 13, 9)
    assert offsets == [0, 7, 9]
    st, consumed, written, offsets = combine_records([(0, 10, 7), (0, 5, 5)], [0, 10])
    assert (st, consumed, written, offsets) == (0, 15, 12, [0, 7])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, utf16, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for data in _mutants(utf16, 12, seed=99 + int(utf16)):
            units = data.view(np.uint16) if utf16 else data
            cuts = plan_cuts(len(units), world, lambda i: int(units[i]), utf16)
            piece = units[cuts[rank] : cuts[rank + 1]].tobytes()
            if utf16:
                (st, consumed, written), payload = oracle.utf16le_to_utf8(piece)
            else:
                (st, consumed, written), payload = oracle.utf8_to_utf16le(piece)
            rec = torch.tensor([0 if st == "ok" else 1, consumed, written], dtype=torch.int64)
            res = transcode_sharded(rec, cuts[rank])
            unit = 1 if utf16 else 2
            results.append((res.outcome.as_tuple(), res.out_offset, payload[: unit * res.local_written]))
        queue.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("utf16", [False, True])
def test_gloo_two_ranks(utf16):
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, utf16, queue)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(queue.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, data in enumerate(_mutants(utf16, 12, seed=99 + int(utf16))):
        whole = oracle.utf16le_to_utf8(data.tobytes()) if utf16 else oracle.utf8_to_utf16le(data.tobytes())
        (o0, off0, p0), (o1, off1, p1) = got[0][k], got[1][k]
        assert o0 == o1 == whole[0]
        unit = 1 if utf16 else 2
        assert off0 == 0 and off1 * unit == len(p0)
        assert p0 + p1 == whole[1]
