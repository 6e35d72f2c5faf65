"""Multi-GPU sharding with the native engine, on one B200.

The box has one GPU, so the 2-rank test runs both ranks on cuda:0 over
gloo (the ranks' kernels do not wait on each other; only the records cross
through the collective).  The NCCL path is exercised at world size 1
through ``shard.transcode_sharded`` on a device record.  Both compare the
combined result with the whole-buffer oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, outcome_from_tensor, shard, transcode_device

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _config5_style(utf16: bool, total_units: int) -> np.ndarray:
    """A small config-5 buffer: seeded 1 MiB-unit segments of profiles a-d."""
    return corpus.config5_generate(total_units, utf16=utf16, device="cpu", segment_units=1 << 20).numpy()


def _mutations(utf16: bool, n: int) -> list[list[tuple[int, int]]]:
    """Error placements at and near the nominal cut n/2 (and in both shards)."""
    h = n // 2
    if utf16:
        hi, lo, a = 0xD800, 0xDC00, 0x41
        return [[], [(h, lo)], [(h - 1, hi), (h, a)], [(h + 1, lo)], [(h - 2, hi), (h - 1, a)],
                [(n - 1, hi)], [(3, lo), (h + 5, hi)], [(h + 7, lo)]]
    return [[], [(h, 0x80)], [(h, 0x80), (h + 1, 0x80), (h + 2, 0x80)], [(h - 1, 0xE4)], [(h - 1, 0xF0)],
            [(h + 1, 0xC0)], [(n - 1, 0xE2)], [(10, 0xFF), (h + 3, 0xFF)], [(h + 100, 0xED), (h + 101, 0xA0)]]


def _apply(base: np.ndarray, utf16: bool, muts) -> bytes:
    b = base.copy()
    if utf16:
        w = b.view("<u2")
        for i, v in muts:
            w[i] = v
    else:
        for i, v in muts:
            b[i] = v
    return b.tobytes()


def _rank_main(rank: int, world: int, port: int, utf16: bool, total: int) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    base = _config5_style(utf16, total)
    direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
    unit_in, unit_out = (2, 1) if utf16 else (1, 2)
    try:
        for muts in _mutations(utf16, total):
            data = _apply(base, utf16, muts)
            arr = np.frombuffer(data, dtype="<u2" if utf16 else np.uint8)
            n = arr.size
            cuts = shard.plan_cuts(n, world, lambda i: int(arr[i]), utf16)
            a, b = cuts[rank], cuts[rank + 1]
            src = torch.frombuffer(bytearray(data[a * unit_in: b * unit_in]), dtype=torch.uint8).to(dev)
            res, out = transcode_device(direction, src)
            got = shard.transcode_sharded(res.cpu(), a)
            ref, payload = oracle.utf16le_to_utf8(data) if utf16 else oracle.utf8_to_utf16le(data)
            assert got.outcome.as_tuple() == ref, (rank, muts, cuts, got, ref)
            mine = out.view(torch.uint8)[: unit_out * got.local_written].cpu().numpy().tobytes()
            at = unit_out * got.out_offset
            assert mine == payload[at: at + len(mine)], (rank, muts)
            # the ranks' payloads tile the global payload exactly
            lens = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(lens, torch.tensor([got.local_written]))
            assert sum(int(t) for t in lens) == ref[2], (muts, lens, ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("utf16", [False, True])
def test_sharded_native_two_ranks_gloo(cuda_ok, utf16):
    """Two ranks (both on cuda:0) cut one config-5-style buffer at character
    boundaries, transcode their shards with the native engine and combine the
    records with one all_gather: global outcome and every rank's payload equal
    the whole-buffer oracle, with errors at, just before and just after the
    cut, at the ends, and in both shards."""
    total = (6 << 20) + 12345
    mp.start_processes(_rank_main, args=(2, _free_port(), utf16, total), nprocs=2, join=True,
                       start_method="spawn")


def _nccl_world1(_index: int, port: int) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        for utf16, profile in ((False, "mix"), (True, "emoji")):
            data = corpus.generate(profile, 3 << 20, 9, utf16=utf16, device=dev)
            if utf16:
                data.view(torch.int16)[777_777] = 0xDC00 - 0x10000
            else:
                data[777_777] = 0xC1
            direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
            res, out = transcode_device(direction, data)
            got = shard.transcode_sharded(res, 0)  # device record: the NCCL all_gather
            raw = data.cpu().numpy().tobytes()
            ref, payload = oracle.utf16le_to_utf8(raw) if utf16 else oracle.utf8_to_utf16le(raw)
            assert got.outcome.as_tuple() == ref == outcome_from_tensor(res.cpu()).as_tuple()
            assert got.out_offset == 0 and got.local_written == ref[2]
            unit_out = 1 if utf16 else 2
            assert out.view(torch.uint8)[: unit_out * ref[2]].cpu().numpy().tobytes() == payload
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_nccl_world_size_1(cuda_ok):
    """shard.transcode_sharded over a real NCCL communicator (world size 1:
    one GPU on this box) with the native engine's device-resident record."""
    mp.start_processes(_nccl_world1, args=(_free_port(),), nprocs=1, join=True, start_method="spawn")


@pytest.mark.timeout(900)
def test_bench_config5_sharded_one_rank(cuda_ok):
    """bench.config5_sharded (the multi-GPU bench's config-5 step) at one
    rank: the 16 GiB input is one shard; combined outcome valid and complete."""
    import bench

    dev = torch.device("cuda", 0)
    for utf16 in (False, True):
        r = bench.config5_sharded(utf16, 1, 0, dev, 6552.0, steps=1)
        assert r["ok"], r
        assert r["consumed"] == (16 << 30) // (2 if utf16 else 1)


def _bench_c5_rank(rank: int, world: int, port: int, utf16: bool, q) -> None:
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        r = bench.config5_sharded(utf16, world, rank, torch.device("cuda", 0), 6552.0, steps=1)
        if rank == 0:
            q.put(r)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("utf16", [False, True])
def test_bench_config5_sharded_two_ranks(cuda_ok, utf16):
    """The multi-GPU bench's config-5 step at world size 2 (both ranks on
    cuda:0, gloo for the records): each rank builds only its half of the
    16 GiB input, the two cuts agree, and the combined outcome equals the
    one-rank run (valid, complete, same written count)."""
    import bench

    one = bench.config5_sharded(utf16, 1, 0, torch.device("cuda", 0), 6552.0, steps=1)
    torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_bench_c5_rank, args=(2, _free_port(), utf16, q), nprocs=2, join=True, start_method="spawn")
    two = q.get(timeout=10)
    assert two["ok"] and one["ok"], (one, two)
    assert (two["status"], two["consumed"], two["written"]) == (one["status"], one["consumed"], one["written"])
    assert two["n_gpus"] == 2 and two["rank0_local_written"] < one["written"]
