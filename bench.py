"""Benchmark: validating UTF-8 -> UTF-16LE transcode on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (config 2 of BASELINE.json): four 256 MiB valid UTF-8
buffers, one per seeded profile (latin, cyrillic, cjk, emoji; seeds 1-4),
generated directly in HBM.  One step = one validating transcode of all four
buffers.  ``value`` = input GiB/s over the whole job (device-timed with CUDA
events on the launch stream, inputs resident in HBM, max over ranks).
Every buffer is larger than the 126 MB L2, so no L2 flush is needed between
steps.  ``e2e`` repeats the step through the public facade with pinned host
buffers (H2D of the input, D2H of the outcome and of the written payload
inside the timed region).  Extra keys carry config 3 (UTF-16LE -> UTF-8) and
config 4 (validate) numbers measured in the same run.

Multi-GPU (one process per GPU; ``--gpus N`` relaunches itself under
``torch.distributed.run`` when it is not already running under it): the
headline is weak scaling -- every rank transcodes its own four config-2
buffers and the per-buffer outcomes are exchanged each step with one NCCL
all_gather.  ``extras.config5_sharded`` is north_star's config 5: one 16 GiB
input per direction cut at character boundaries across the N ranks
(shard.snap_cut), each rank transcoding its shard in its own HBM and one
NCCL all_gather of the per-shard (status, consumed, written, begin) records
inside the timed step (shard.transcode_sharded); aggregate GiB/s at N.

``--impl reference`` times the reference algorithm's CPU restatement
(oracle/, C, all host threads, character-boundary sharded) on the same
workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import faulthandler
import json
import os
import signal
import statistics
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PROFILES = (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4))
BUF_BYTES = 256 << 20
METRIC = "input GiB/s transcoded+validated (device-timed) and % of HBM roofline"
GIB = float(1 << 30)
EV_EVERY = 4  # steps of the timed region that carry per-launch timing events
REF_BUDGET_S = 150.0  # --impl reference: bound on the timed CPU run
WORKLOAD = ("config2: UTF-8->UTF-16LE, 4 x 256 MiB valid buffers per GPU "
            "(latin/cyrillic/cjk/emoji, seeds 1-4 (+100*rank))")
DATA = "synthetic (seeded SplitMix64 profiles, paper_2212_05098_b200/corpus.py)"
C5_BYTES = 16 << 30  # config 5: 16 GiB per direction


def bench_config(world: int) -> dict:
    """The ``config`` object of both arms (identical, so the driver can pair them)."""
    return {
        "workload": WORKLOAD,
        "input_bytes_per_step": world * len(PROFILES) * BUF_BYTES,
        "l2": "inputs larger than L2 (256 MiB each > 126 MB), no flush",
        "parallelism": f"dp{world} (independent shards, NCCL all_gather of outcomes)" if world > 1 else "dp1",
    }


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md, 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per input byte of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle",
        0x2: "applications_clocks_setting",
        0x4: "sw_power_cap",
        0x8: "hw_slowdown",
        0x10: "sync_boost",
        0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self._nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nvml.nvmlDeviceGetClockInfo(self._h, self._nvml.NVML_CLOCK_SM))
                bits = self._nvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for b, name in self.REASONS.items():
                    if bits & b and b != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self._nvml is not None:
            self._stop.set()
            self._t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """--impl reference: the reference algorithm (C restatement of
    laneutf.scalar) on all host threads, same workload, rank 0 only."""
    import oracle

    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2212_05098_b200 import corpus

    gen_dev = "cuda" if torch.cuda.is_available() else "cpu"
    bufs = [corpus.generate(p, BUF_BYTES, s, device=gen_dev).cpu().numpy() for p, s in PROFILES]
    outs = [np.empty(BUF_BYTES, dtype=np.uint16) for _ in bufs]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    for _ in range(args.warmup):
        for b, o in zip(bufs, outs):
            oracle.run_mt(oracle.OP_U8_U16, b, threads, o)
    step_s = (time.perf_counter() - t0) / max(args.warmup, 1)
    # bound the timed run to ~REF_BUDGET_S: each step then covers the same
    # leading fraction of every buffer, cut on a character boundary
    frac = min(1.0, REF_BUDGET_S / max(step_s * args.steps, 1e-9))
    if frac < 1.0:
        cut = []
        for b in bufs:
            k = max(1, int(BUF_BYTES * frac))
            while k < BUF_BYTES and (int(b[k]) & 0xC0) == 0x80:
                k += 1
            cut.append(k)
        bufs = [b[:k] for b, k in zip(bufs, cut)]
    step_bytes = sum(len(b) for b in bufs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for b, o in zip(bufs, outs):
            res = oracle.run_mt(oracle.OP_U8_U16, b, threads, o)
            assert res[0] == "ok"
    dt = time.perf_counter() - t0
    value = args.steps * step_bytes / GIB / dt
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GiB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * dt / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": DATA,
        "config": bench_config(world),
        "cpu_baseline": {
            "value": round(value, 3),
            "unit": "GiB/s",
            "cores": threads,
            "kind": "port",
            "sample": ("full config-2 workload per step (4 x 256 MiB)" if step_bytes == len(PROFILES) * BUF_BYTES
                       else f"leading {step_bytes / len(PROFILES) / 2**20:.1f} MiB of each of the 4 config-2 "
                       f"buffers per step (run bounded to ~{REF_BUDGET_S:.0f} s)")
            + ", oracle/laneutf_oracle.c (C restatement of laneutf.scalar), character-boundary sharded over "
            "host threads",
        },
        "e2e": {"value": round(value, 3), "unit": "GiB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """Oracle on a bounded sample of the same workload (rank 0, N=1), plus
    bounded CPU figures for configs 1, 3 and 4 and the reference's own Python
    implementation when it is installed in
    baseline/_ref."""
    import oracle

    from paper_2212_05098_b200 import corpus

    sample = 64 << 20
    bufs = [corpus.generate(p, sample, s, device="cuda").cpu().numpy() for p, s in PROFILES]
    outs = [np.empty(sample, dtype=np.uint16) for _ in bufs]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    for b, o in zip(bufs, outs):
        oracle.run_mt(oracle.OP_U8_U16, b, threads, o)
    dt_mt = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.run_mt(oracle.OP_U8_U16, bufs[2][: 16 << 20], 1, outs[2])
    dt_1 = time.perf_counter() - t0
    line = {
        "value": round(len(bufs) * sample / GIB / dt_mt, 3),
        "unit": "GiB/s",
        "cores": threads,
        "kind": "port",
        "sample": f"first 64 MiB of each config-2 profile buffer (256 MiB), oracle/laneutf_oracle.c "
        f"on {threads} host threads; single-thread cjk 16 MiB = {16 / 1024 / dt_1:.3f} GiB/s",
    }
    # the other configs, same oracle, all host threads, bounded samples
    per = {}

    def timed(op, data, out=None, reps=1):
        t0 = time.perf_counter()
        for _ in range(reps):
            r = oracle.run_mt(op, data, threads, out)
        return time.perf_counter() - t0, r

    c1 = corpus.generate("mix", 4 << 20, 0, device="cuda").cpu().numpy()
    w1 = np.empty(4 << 20, dtype=np.uint16)
    t_a, r = timed(oracle.OP_U8_U16, c1, w1, reps=5)
    words = w1[: r[2]].view(np.uint8)
    t_b, _ = timed(oracle.OP_U16_U8, words, np.empty(3 * r[2], dtype=np.uint8), reps=5)
    per["config1_round_trip_4MiB"] = {"gib_s": round(5 * (4 << 20) / GIB / (t_a + t_b), 3),
                                      "sample": "4 MiB, both directions, 5 reps"}
    c3 = {}
    for (p, sd) in PROFILES:
        w = corpus.generate(p, sample // 2, sd, utf16=True, device="cuda").cpu().numpy()
        t, _ = timed(oracle.OP_U16_U8, w, np.empty(3 * (sample // 2), dtype=np.uint8))
        c3[p] = round(sample / GIB / t, 3)
    per["config3_utf16_to_utf8"] = {"gib_s": c3, "sample": "64 MiB (32 Mi words) per profile"}
    e16 = corpus.generate("emoji", sample // 2, 4, utf16=True, device="cuda").cpu().numpy()
    t_v8, _ = timed(oracle.OP_VAL_U8, bufs[2])
    t_v16, _ = timed(oracle.OP_VAL_U16, e16)
    per["config4_validate"] = {"cjk_utf8_gib_s": round(sample / GIB / t_v8, 3),
                               "emoji_utf16_gib_s": round(sample / GIB / t_v16, 3),
                               "sample": "64 MiB zero-error buffers"}
    line["per_config"] = per
    line["reference_python"] = reference_python_baseline(bufs, c1, threads)
    return line


def reference_python_baseline(bufs, c1, threads: int) -> dict:
    """The reference package itself (pure Python, baseline/_ref) timed on the
    host: (i) ``laneutf.bench.run_bench`` with the
    scalar engine, one pinned core, on a 1 MiB character-aligned sample of each
    config-2 profile; (ii) the same engine over all cores as one worker process
    per core on 1 MiB character-aligned pieces; (iii) ``emulated-64`` (the
    paper's algorithm in Python) on a 16 KiB sample of config 1."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "laneutf")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref the reference)"}
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        from laneutf import bench as lbench
    except Exception as exc:  # pragma: no cover
        return {"unavailable": repr(exc)[:200]}

    def aligned(b: np.ndarray, k: int) -> bytes:
        while k < len(b) and (int(b[k]) & 0xC0) == 0x80:
            k += 1
        return b[:k].tobytes()

    out = {"kind": "reference (laneutf 0.1.0, pure Python, baseline/_ref)"}
    single = {}
    for (p, _), b in zip(PROFILES, bufs):
        rep, _payload = lbench.run_bench("utf8-to-utf16", aligned(b, 1 << 20), engine="scalar", repetitions=1,
                                         warmup=0, label=p)
        single[p] = round(rep.bytes_per_second / 2**20, 3)
    out["scalar_1core_mib_s"] = single
    # all cores: one process per core, each a 1 MiB character-aligned piece
    import multiprocessing as mp

    pieces = []
    for b in bufs:
        pos = 0
        for _ in range(max(1, threads // len(bufs))):
            end = pos + (1 << 20)
            while end < len(b) and (int(b[end]) & 0xC0) == 0x80:
                end += 1
            pieces.append(b[pos:end].tobytes())
            pos = end
    ctx = mp.get_context("spawn")
    with ctx.Pool(threads, initializer=_ref_worker_init, initargs=(ref_dir,)) as pool:
        pool.map(_ref_worker, pieces[:threads])  # warm the workers (imports)
        t0 = time.perf_counter()
        total = sum(pool.map(_ref_worker, pieces))
        dt = time.perf_counter() - t0
    out["scalar_all_cores"] = {"mib_s": round(total / 2**20 / dt, 3), "cores": threads,
                               "sample": f"{len(pieces)} pieces of 1 MiB from the 4 profiles, one process per core"}
    rep, _payload = lbench.run_bench("utf8-to-utf16", aligned(c1, 16 << 10), engine="emulated-64", repetitions=1,
                                     warmup=0, label="config1")
    out["emulated64_config1_mib_s"] = round(rep.bytes_per_second / 2**20, 4)
    return out


def _ref_worker_init(ref_dir: str) -> None:
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)


def _ref_worker(piece: bytes) -> int:
    from laneutf import engine as lengine

    outcome, _payload = lengine.transcode_to_bytes("utf8-to-utf16", piece, engine="scalar")
    assert outcome.status.value == "ok"
    return len(piece)


def config5_sharded(utf16: bool, world: int, rank: int, dev: torch.device, peak: float, steps: int = 3) -> dict:
    """North_star config 5 on ``world`` GPUs: 16 GiB (UTF-8 bytes, or 8 Gi
    UTF-16 words) of seeded 64 MiB profile segments, cut at character
    boundaries (shard.snap_cut on the units at each nominal cut r*n/world).
    Each rank generates only its shard plus 4 units of look-ahead, transcodes
    it in its own HBM, and the timed step ends with shard.transcode_sharded:
    one NCCL all_gather of (status, consumed, written, begin) per rank and the
    global combine.  Returns the aggregate input GiB/s (max-over-ranks device
    time) and the combined outcome."""
    import torch.distributed as dist

    from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, outcome_from_tensor, transcode_device
    from paper_2212_05098_b200.shard import combine_records, snap_cut, transcode_sharded

    unit = 2 if utf16 else 1
    n = C5_BYTES // unit
    x0, x1 = n * rank // world, n * (rank + 1) // world
    log(f"config 5 {'utf16->utf8' if utf16 else 'utf8->utf16'}: rank {rank} units [{x0}, {x1})")
    win = corpus.config5_range(n, x0, min(x1 + 4, n), utf16=utf16, device=dev)
    wv = win.view(torch.int16) if utf16 else win

    def units_at(pos: int) -> list[int]:
        return [v & 0xFFFF for v in wv[pos - x0: pos - x0 + 4].cpu().tolist()]

    def snap(x: int) -> int:
        if x <= 0 or x >= n:
            return max(0, min(x, n))
        head = units_at(x)
        return snap_cut(lambda i: head[i - x] if i - x < len(head) else 0, n, x, utf16)

    begin, end = snap(x0), snap(x1)
    shard = win[unit * (begin - x0): unit * (end - x0)]
    direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
    stream = torch.cuda.current_stream(dev)
    res, out = transcode_device(direction, shard)
    if world > 1:
        bdev = dev if dist.get_backend() == "nccl" else torch.device("cpu")
        bounds = torch.tensor([begin, end], dtype=torch.int64, device=bdev)
        allb = [torch.empty_like(bounds) for _ in range(world)]
        dist.all_gather(allb, bounds)
        allb = [t.tolist() for t in allb]
        assert all(allb[r][1] == allb[r + 1][0] for r in range(world - 1)), allb

    def combine():
        if world > 1:
            return transcode_sharded(res, begin)
        rec = [int(v) for v in res.cpu().tolist()]
        st, consumed, written, _ = combine_records([(rec[0] & 0xFFFFFFFF, rec[1], rec[2])], [begin])
        from paper_2212_05098_b200.outcome import STATUS_BY_CODE, TranscodeOutcome
        return TranscodeOutcome(STATUS_BY_CODE[st], consumed, written)

    got = combine()
    outcome = got.outcome if world > 1 else got
    local = outcome_from_tensor(res.cpu())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        transcode_device(direction, shard, out, res=res)
        combine()  # the all_gather (NCCL) and the global combine, inside the timed step
    b.record(stream)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 1e3 / steps
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=bdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        dist.barrier()
    ab = C5_BYTES + (1 if utf16 else 2) * outcome.written
    result = {"aggregate_input_gib_s": round(C5_BYTES / GIB / t, 2), "ms_per_step": round(t * 1e3, 3),
              "n_gpus": world, "frac_of_measured_x_gpus": round(ab / t / 1e9 / (peak * world), 4),
              "status": outcome.status.value, "consumed": outcome.consumed, "written": outcome.written,
              "ok": outcome.ok and outcome.consumed == n,
              "rank0_shard_units": end - begin, "rank0_local_written": local.written,
              "collective": "NCCL all_gather of 4 x int64 per rank (shard.transcode_sharded)" if world > 1
              else "none (1 rank: shard.combine_records only)",
              "steps": steps}
    del win, shard, out, res
    torch.cuda.empty_cache()
    return result


def log(msg: str) -> None:
    """Progress on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def main():
    faulthandler.register(signal.SIGUSR1)  # `timeout -s USR1` dumps the stacks of a stuck run
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-extras", action="store_true", help="skip config 3/4 side measurements")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torch.distributed.run
        import socket
        import subprocess

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world_env}: launch one process per GPU")

    if args.impl == "reference":
        run_reference(args)
        return

    import torch.distributed as dist

    from paper_2212_05098_b200 import (
        UTF8_TO_UTF16,
        UTF16_TO_UTF8,
        batch_device,
        corpus,
        count_device,
        outcome_from_tensor,
        transcode,
        transcode_device,
        validate_device,
    )
    from paper_2212_05098_b200 import _native

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    reason = _native.unavailable_reason(local)
    if reason is not None:
        raise SystemExit(f"native engine unavailable: {reason}")

    log("generating config-2 inputs")
    # ---- inputs resident in HBM (each rank: its own seeded shard of profiles)
    srcs = [corpus.generate(p, BUF_BYTES, s + 100 * rank, device=dev) for p, s in PROFILES]
    outs = [torch.empty(BUF_BYTES, dtype=torch.uint16, device=dev) for _ in srcs]
    ress = [torch.empty(3, dtype=torch.int64, device=dev) for _ in srcs]
    wss = [
        torch.empty(_native.workspace_bytes(_native.OP_UTF8_TO_UTF16LE, BUF_BYTES) // 8 + 1, dtype=torch.int64,
                    device=dev)
        for _ in srcs
    ]
    gathered = [torch.empty(3 * world, dtype=torch.int64, device=dev) for _ in srcs]
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        for i, (s, o, r, w) in enumerate(zip(srcs, outs, ress, wss)):
            if ev is not None:
                ev[i][0].record(stream)
            transcode_device(UTF8_TO_UTF16, s, o, res=r, ws=w, stream=stream)
            if ev is not None:
                ev[i][1].record(stream)
        if world > 1:
            for r, g in zip(ress, gathered):
                dist.all_gather_into_tensor(g, r)

    log("warm-up")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    outcomes = [outcome_from_tensor(r.cpu()) for r in ress]
    assert all(o.ok for o in outcomes), outcomes
    in_bytes = len(srcs) * BUF_BYTES
    out_bytes = sum(2 * o.written for o in outcomes)

    log("timed region")
    # ---- timed region
    # per-launch events (the roofline's launch durations) on every EV_EVERY-th
    # step of the timed region: a timing event pair costs ~4.5 us per launch
    # (measured, tools/rot_bench.py), which would otherwise inflate the step
    # (starting at step EV_EVERY // 2, not 0: the first launch after the
    # synchronize runs while the clocks ramp up from idle -- one ~2 ms sample in
    # 50 moved the first profile's mean by 15-40 us)
    ev_steps = list(range(min(EV_EVERY // 2, max(args.steps - 1, 0)), args.steps, EV_EVERY))
    evs = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in srcs]
           for k in ev_steps}
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            step(evs.get(k))
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    per_launch = np.array([[a.elapsed_time(b) for (a, b) in evs[k]] for k in ev_steps])  # ms [sampled steps, bufs]
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    value = world * args.steps * in_bytes / GIB / (elapsed_ms / 1e3)

    # ---- roofline of the dominant kernel (k_utf8_to_utf16le)
    peak, peak_src = measured_peak()
    alg_bytes = np.array([BUF_BYTES + 2 * o.written for o in outcomes], dtype=np.float64)
    mean_launch_s = per_launch.mean(axis=0) / 1e3
    achieved = float((alg_bytes / mean_launch_s).mean() / 1e9)
    prof_detail = {}
    for (p, _), o, ab, t in zip(PROFILES, outcomes, alg_bytes, mean_launch_s):
        prof_detail[p] = {
            "input_gib_s": round(BUF_BYTES / GIB / t, 2),
            "alg_gb_s": round(ab / t / 1e9, 1),
            "frac_of_measured": round(ab / t / 1e9 / peak, 4),
            "frac_of_8tbs": round(ab / t / 1e9 / 8000.0, 4),
            "us_per_launch": round(t * 1e6, 2),
            "written_words": o.written,
        }
    ncu = ncu_traffic()
    traffic = None
    k1_key = "K1 utf8->utf16 (k_transcode<DirU8U16>)"
    if ncu and k1_key in ncu:
        # dram read+write bytes per launch, averaged over the same four
        # 256 MiB profile buffers (tools/prof_kernels.py under ncu --set full)
        traffic = round(ncu[k1_key]["dram_bytes_per_launch"])

    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GiB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": DATA,
        "config": bench_config(world),
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "kernel": "k_transcode<DirU8U16> (K1)",
            "algorithmic_bytes": "input bytes + 2 x written words, per launch",
            "alg_bytes_per_launch": round(float(alg_bytes.mean())),
            "output_bytes_per_step": out_bytes,
            "traffic_source": "profiles/ncu_summary.json (ncu --set full, dram__bytes_read+write per launch)",
            "peak_source": peak_src,
            "per_profile": prof_detail,
            "launch_timing": f"CUDA events around each launch on every {EV_EVERY}th step of the timed region, "
            f"from step {ev_steps[0] if ev_steps else 0} ({len(ev_steps)} of {args.steps} steps)",
        },
        "gpu_launches": args.steps * len(srcs),
        "clocks": clocks.summary(),
    }

    log("e2e")
    # ---- e2e through the public facade with pinned host buffers
    hosts = [s.cpu().pin_memory() for s in srcs]
    host_outs = [torch.empty(2 * BUF_BYTES, dtype=torch.uint8).pin_memory() for _ in srcs]
    expect = [(o.status, o.consumed, o.written) for o in outcomes]

    def e2e_check(got, tag):
        got = [(o.status, o.consumed, o.written) for o in got]
        assert got == expect, (tag, got, expect)

    e2e_check([transcode(UTF8_TO_UTF16, h, ho, engine="native") for h, ho in zip(hosts, host_outs)], "warm-up")
    for o, ho in zip(outs, host_outs[:1]):  # payload spot check: the whole latin output
        assert torch.equal(ho[: 2 * outcomes[0].written].to(dev), o.view(torch.uint8)[: 2 * outcomes[0].written])
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        got = [transcode(UTF8_TO_UTF16, h, ho, engine="native") for h, ho in zip(hosts, host_outs)]
    e2e_s = time.perf_counter() - t0
    e2e_check(got, "timed")
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # host copies alone: H2D of the step's inputs and
    # D2H of its payloads, each timed with CUDA events, no kernel
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_ev.record(stream)
    for h, s_ in zip(hosts, srcs):
        s_.copy_(h, non_blocking=True)
    b_ev.record(stream)
    torch.cuda.synchronize()
    h2d_s = a_ev.elapsed_time(b_ev) / 1e3
    a_ev.record(stream)
    for o, ho, oc in zip(outs, host_outs, outcomes):
        ho[: 2 * oc.written].copy_(o.view(torch.uint8)[: 2 * oc.written], non_blocking=True)
    b_ev.record(stream)
    torch.cuda.synchronize()
    d2h_s = a_ev.elapsed_time(b_ev) / 1e3
    line["e2e"] = {
        "value": round(world * args.e2e_steps * in_bytes / GIB / e2e_s, 3),
        "unit": "GiB/s",
        "h2d_bytes_per_step": in_bytes,
        "d2h_bytes_per_step": out_bytes + 24 * len(srcs),
        "steps": args.e2e_steps,
        "api": "paper_2212_05098_b200.transcode(UTF8_TO_UTF16, pinned_in, pinned_out, engine='native')",
        "outcomes_checked": True,
        "h2d_alone": {"ms": round(h2d_s * 1e3, 3), "gib_s": round(in_bytes / GIB / h2d_s, 2)},
        "d2h_alone": {"ms": round(d2h_s * 1e3, 3), "gib_s": round(out_bytes / GIB / d2h_s, 2)},
    }
    # the reference callers' types: bytes in, bytearray out (cli.py:92, bench.py:100-106)
    log("e2e bytes")
    blobs = [h.numpy().tobytes() for h in hosts]
    ba_outs = [bytearray(2 * BUF_BYTES) for _ in srcs]
    e2e_check([transcode(UTF8_TO_UTF16, bb, ba, engine="native") for bb, ba in zip(blobs, ba_outs)], "bytes")
    t0 = time.perf_counter()
    got = [transcode(UTF8_TO_UTF16, bb, ba, engine="native") for bb, ba in zip(blobs, ba_outs)]
    eb_s = time.perf_counter() - t0
    e2e_check(got, "bytes timed")
    line["e2e"]["bytes_api"] = {
        "value": round(in_bytes / GIB / eb_s, 3), "unit": "GiB/s",
        "api": "transcode(UTF8_TO_UTF16, bytes, bytearray): pinned staging ring, chunked H2D / kernel / D2H"}
    del hosts, host_outs, blobs, ba_outs

    # ---- extras: config 3 (UTF-16 -> UTF-8) and config 4 (validate), same run
    if not args.no_extras:
        extras = {}
        k_ex = max(3, min(args.steps, 50))
        src16 = [corpus.generate(p, BUF_BYTES // 2, s + 100 * rank, utf16=True, device=dev) for p, s in PROFILES]
        out8 = torch.empty(3 * BUF_BYTES // 2, dtype=torch.uint8, device=dev)
        log("extras: config 3")
        c3 = {}
        for (p, _), s16 in zip(PROFILES, src16):
            res, _ = transcode_device(UTF16_TO_UTF8, s16, out8)
            o = outcome_from_tensor(res.cpu())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(k_ex):
                transcode_device(UTF16_TO_UTF8, s16, out8, res=res)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3 / k_ex
            ab = BUF_BYTES + o.written
            c3[p] = {"input_gib_s": round(BUF_BYTES / GIB / t, 2), "frac_of_measured": round(ab / t / 1e9 / peak, 4),
                     "ok": o.ok}
        extras["config3_utf16_to_utf8"] = c3
        log("extras: config 4")
        c4 = {}
        for name, direction, buf in (("cjk_utf8", UTF8_TO_UTF16, srcs[2]), ("emoji_utf16", UTF16_TO_UTF8, src16[3])):
            res = validate_device(direction, buf)
            o = outcome_from_tensor(res.cpu())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(k_ex):
                validate_device(direction, buf, res=res)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3 / k_ex
            c4[name] = {"input_gib_s": round(BUF_BYTES / GIB / t, 2),
                        "frac_of_measured": round(BUF_BYTES / t / 1e9 / peak, 4), "ok": o.ok,
                        "control": "zero-error buffer"}
        # config 4 with errors injected at 1e-6 per unit (seeds 101/102): the
        # validators stop at the first error; the transcode writes the valid prefix
        for name, direction, utf16, prof, seed in (("cjk_utf8_errors_1e-6", UTF8_TO_UTF16, False, "cjk", 3),
                                                   ("emoji_utf16_errors_1e-6", UTF16_TO_UTF8, True, "emoji", 4)):
            units = BUF_BYTES // 2 if utf16 else BUF_BYTES
            log(f"extras: config 4 {name}")
            ebuf = corpus.generate(prof, units, seed, utf16=utf16, device=dev)
            planted = corpus.inject_errors(ebuf, utf16=utf16, rate=1e-6, seed=101 + int(utf16))
            res = validate_device(direction, ebuf)
            o = outcome_from_tensor(res.cpu())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(k_ex):
                validate_device(direction, ebuf, res=res)
            b.record(stream)
            torch.cuda.synchronize()
            tv = a.elapsed_time(b) / 1e3 / k_ex
            eout = out8 if utf16 else outs[2]
            res, _ = transcode_device(direction, ebuf, eout)
            ot = outcome_from_tensor(res.cpu())
            a.record(stream)
            for _ in range(k_ex):
                transcode_device(direction, ebuf, eout, res=res)
            b.record(stream)
            torch.cuda.synchronize()
            tt = a.elapsed_time(b) / 1e3 / k_ex
            c4[name] = {"errors_planted": len(planted), "status": o.status.value, "first_error_unit": o.consumed,
                        "validate_us": round(tv * 1e6, 1), "transcode_us": round(tt * 1e6, 1),
                        "transcode_written": ot.written, "same_offset": ot.consumed == o.consumed}
            del ebuf
        extras["config4_validate"] = c4
        # beyond the configs: plain ASCII (the paper's ASCII fast path) and mixed
        # BMP text (accented Latin + typographic punctuation: no single class per
        # chunk), 256 MiB each, all three hot kernels
        log("extras: ascii / mixed-BMP profiles")
        px = {}
        for prof, seed in (("ascii", 5), ("typo", 6)):
            u8 = corpus.generate(prof, BUF_BYTES, seed, device=dev)
            u16 = corpus.generate(prof, BUF_BYTES // 2, seed, utf16=True, device=dev)
            ent = {}
            for name, fn, extra_of in (
                    ("utf8_to_utf16", lambda r=None: transcode_device(UTF8_TO_UTF16, u8, outs[0], res=r), lambda o: 2 * o.written),
                    ("utf16_to_utf8", lambda r=None: transcode_device(UTF16_TO_UTF8, u16, out8, res=r), lambda o: o.written),
                    ("validate_utf8", lambda r=None: (validate_device(UTF8_TO_UTF16, u8, res=r), None), lambda o: 0)):
                res = fn()[0]
                o = outcome_from_tensor(res.cpu())
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(k_ex):
                    fn(res)
                b.record(stream)
                torch.cuda.synchronize()
                t = a.elapsed_time(b) / 1e3 / k_ex
                ent[name] = {"input_gib_s": round(BUF_BYTES / GIB / t, 2),
                             "frac_of_measured": round((BUF_BYTES + extra_of(o)) / t / 1e9 / peak, 4), "ok": o.ok}
            px[prof] = ent
            del u8, u16
        extras["ascii_and_mixed_bmp_profiles"] = px
        # config 1: UTF-8 -> UTF-16LE -> UTF-8 round trip of the 4 MiB mixed
        # buffer (seed 0): two launches of a latency-bound size
        log("extras: config 1")
        c1src = corpus.generate("mix", 4 << 20, 0, device=dev)
        r1, w1 = transcode_device(UTF8_TO_UTF16, c1src)
        o1 = outcome_from_tensor(r1.cpu())
        words = w1[: o1.written]
        r2, b2 = transcode_device(UTF16_TO_UTF8, words)
        o2 = outcome_from_tensor(r2.cpu())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k_ex):
            transcode_device(UTF8_TO_UTF16, c1src, w1, res=r1)
            transcode_device(UTF16_TO_UTF8, words, b2, res=r2)
        b.record(stream)
        torch.cuda.synchronize()
        t1 = a.elapsed_time(b) / 1e3 / k_ex
        extras["config1_round_trip_4MiB"] = {"us_per_round_trip": round(t1 * 1e6, 1),
                                             "input_gib_s": round((4 << 20) / GIB / t1, 2),
                                             "ok": o1.ok and o2.ok and bool(torch.equal(b2[: o2.written], c1src)),
                                             "utf16_words": o1.written}
        del c1src, w1, b2, words
        # row 8f(4): one-pass lengths (validate + count) and char counts
        log("extras: lengths / counts")
        c8 = {}
        for name, op, buf in (("utf16_length_from_utf8_cjk", _native.OP_UTF16_LENGTH_FROM_UTF8, srcs[2]),
                              ("utf8_length_from_utf16le_emoji", _native.OP_UTF8_LENGTH_FROM_UTF16LE, src16[3]),
                              ("utf8_char_count_cjk", _native.OP_UTF8_CHAR_COUNT, srcs[2]),
                              ("utf16le_char_count_emoji", _native.OP_UTF16LE_CHAR_COUNT, src16[3])):
            count_device(op, buf)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(k_ex):
                count_device(op, buf)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3 / k_ex
            c8[name] = {"input_gib_s": round(BUF_BYTES / GIB / t, 2),
                        "frac_of_measured": round(BUF_BYTES / t / 1e9 / peak, 4)}
        extras["row8f_lengths_and_char_counts"] = c8
        # row 8f(1): UTF-16BE, swap fused into K1's compaction / K2's load
        log("extras: UTF-16BE")
        c9 = {}
        emoji_be = src16[3].view(torch.uint8).view(-1, 2).flip(1).contiguous().view(-1)  # same text, BE
        for name, direction, buf, out in (("utf8_to_utf16be_latin", UTF8_TO_UTF16, srcs[0], outs[0]),
                                          ("utf16be_to_utf8_emoji", UTF16_TO_UTF8, emoji_be, out8)):
            res, _ = transcode_device(direction, buf, out, utf16_byte_order="be")
            o = outcome_from_tensor(res.cpu())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(k_ex):
                transcode_device(direction, buf, out, res=res, utf16_byte_order="be")
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3 / k_ex
            ab = BUF_BYTES + (2 if direction == UTF8_TO_UTF16 else 1) * o.written
            c9[name] = {"input_gib_s": round(BUF_BYTES / GIB / t, 2), "frac_of_measured": round(ab / t / 1e9 / peak, 4),
                        "ok": o.ok}
        extras["row8f_utf16be"] = c9
        del emoji_be
        # row 8f(3): batched independent cases -- the 2^24 byte-triple sweep
        tri = torch.arange(1 << 24, dtype=torch.int32, device=dev)
        tri_data = torch.stack([(tri >> 16) & 255, (tri >> 8) & 255, tri & 255], dim=1).to(torch.uint8).reshape(-1)
        tri_offs = 3 * torch.arange((1 << 24) + 1, dtype=torch.int64, device=dev)
        log("extras: batch")
        cb = {}
        for name, vo in (("validate_utf8_all_byte_triples", True), ("utf8_to_utf16_all_byte_triples", False)):
            batch_device(UTF8_TO_UTF16, tri_data, tri_offs, validate_only=vo)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(3):
                batch_device(UTF8_TO_UTF16, tri_data, tri_offs, validate_only=vo)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3 / 3
            cb[name] = {"cases": 1 << 24, "ms": round(t * 1e3, 2), "cases_per_s": round((1 << 24) / t)}
        extras["row8f_batch"] = cb
        del tri, tri_data, tri_offs
        # config 5: 16 GiB per direction cut at character boundaries across the
        # ranks; every rank transcodes its shard, one all_gather of records
        extras["config5_sharded"] = {
            name: config5_sharded(utf16, world, rank, dev, peak)
            for name, utf16 in (("utf8_to_utf16_16GiB", False), ("utf16_to_utf8_16GiB", True))}
        line["extras"] = extras

    if rank == 0 and world == 1:
        log("cpu baseline")
        try:
            line["cpu_baseline"] = cpu_baseline_sample()
        except Exception as exc:  # the baseline must not sink the GPU line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
