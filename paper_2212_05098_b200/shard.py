"""Multi-GPU sharding of one validating transcode.

The input is cut into P contiguous shards at character boundaries: a nominal
cut at ``r * n / P`` moves forward past at most three UTF-8 continuation
bytes, or past one UTF-16 low surrogate (both encodings are
self-synchronising).  Each rank transcodes its shard in its own HBM with the
native engine; the only exchange is one all-gather of the per-shard
``(status, consumed, written)`` records (3 x int64 per rank, NCCL over
NVLink on GPUs, gloo in the CPU tests).  Output stays sharded: rank r's
payload belongs at global output offset ``sum(written[:r])``.

Why this is exact: a whole-buffer parse that is valid up
to a cut lands exactly on it, a character truncated at a shard end is invalid
in the whole buffer too and at the same position, and a cut that still sits
on a continuation byte after three steps sits on a byte that is unclaimed in
the whole buffer.  So the global outcome is the first malformed shard's local
outcome shifted by its shard offset, and ``written`` is the prefix sum.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch

from .outcome import STATUS_BY_CODE, TranscodeOutcome

__all__ = [
    "snap_cut",
    "plan_cuts",
    "combine_records",
    "ShardedOutcome",
    "transcode_sharded",
]

_OK, _MALFORMED = 0, 1


def snap_cut(unit_at: Callable[[int], int], n: int, cut: int, utf16: bool) -> int:
    """Move a nominal cut forward to a character boundary.

    ``unit_at(i)`` returns input unit i (a byte for UTF-8, a 16-bit word for
    UTF-16).  Mirrors oracle's lo_snap_cut (the CPU baseline uses the same
    rule), so CPU and GPU sharding agree.
    """
    if cut <= 0 or cut >= n:
        return max(0, min(cut, n))
    if utf16:
        w = unit_at(cut)
        return cut + 1 if 0xDC00 <= w < 0xE000 else cut
    for _ in range(3):
        if cut >= n or not (0x80 <= unit_at(cut) < 0xC0):
            break
        cut += 1
    return min(cut, n)


def plan_cuts(n: int, world: int, unit_at: Callable[[int], int], utf16: bool) -> list[int]:
    """Cut points c_0 = 0 <= c_1 <= ... <= c_P = n (units)."""
    cuts = [0]
    for r in range(1, world):
        c = snap_cut(unit_at, n, n * r // world, utf16)
        cuts.append(max(c, cuts[-1]))
    cuts.append(n)
    return cuts


def combine_records(records: Sequence[Sequence[int]], begins: Sequence[int]):
    """Global (status code, consumed, written) and per-rank output offsets.

    ``records[r] = (status, consumed, written)`` of rank r's shard, whose
    first input unit is ``begins[r]``.  The first malformed shard decides;
    ranks after it contribute nothing (their output lies past ``written``).
    """
    written = 0
    offsets = []
    for r, (status, consumed, wr) in enumerate(records):
        offsets.append(written)
        written += int(wr)
        if int(status) != _OK:
            offsets.extend([written] * (len(records) - r - 1))
            return _MALFORMED, int(begins[r]) + int(consumed), written, offsets
    total = int(begins[-1]) + int(records[-1][1]) if records else 0
    return _OK, total, written, offsets


@dataclass(frozen=True)
class ShardedOutcome:
    outcome: TranscodeOutcome  # of the whole (virtual) input
    out_offset: int  # global output unit offset of this rank's payload
    local_written: int  # units of this rank's payload that belong to the global output
    records: tuple  # all ranks' (status, consumed, written)


def transcode_sharded(
    local_record: torch.Tensor,
    begin: int,
    *,
    group=None,
) -> ShardedOutcome:
    """Exchange per-shard outcomes and combine them (the collective step).

    ``local_record`` is this rank's int64[3] lu_outcome (on the GPU for NCCL,
    on the CPU for gloo) produced by ``transcode_device`` on the shard that
    starts at global unit ``begin``.  One all-gather of 4 int64 per rank
    (record + begin) is the only data-path collective.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # NCCL gathers device tensors; gloo (CPU tests) needs host tensors
    dev = local_record.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.empty(4, dtype=torch.int64, device=dev)
    mine[:3] = local_record.view(torch.int64)[:3].to(dev)
    mine[3] = begin
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    rows = torch.stack(gathered).cpu().tolist()
    records = [(r[0] & 0xFFFFFFFF, r[1], r[2]) for r in rows]
    begins = [r[3] for r in rows]
    status, consumed, written, offsets = combine_records(records, begins)
    out_off = offsets[rank]
    # a rank past the first malformed shard contributes nothing
    first_bad = next((i for i, rec in enumerate(records) if rec[0] != _OK), world)
    local = records[rank][2] if rank <= first_bad else 0
    outcome = TranscodeOutcome(STATUS_BY_CODE[status], consumed, written)
    return ShardedOutcome(outcome, out_off, local, tuple(records))
