"""Hang / progress stress test for the pipelined transcoders and validators.

    python tools/stress_kernels.py [--iters N] [--mib M] [--limit-s S]

Runs K1/K2 transcodes and K3/K4 validations on many seeded buffers (valid,
and with errors injected at several rates) and watches every launch: if the
stream has not drained after --limit-s seconds the run prints the case and
exits with code 3 (the process exit tears the spinning kernel down).  Also
checks that the transcode reports the validator's first-error offset.
"""

import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, outcome_from_tensor  # noqa: E402
from paper_2212_05098_b200 import transcode_device, validate_device  # noqa: E402


def wait(stream, limit, what):
    t0 = time.time()
    while not stream.query():
        if time.time() - t0 > limit:
            print(f"HANG: {what} (> {limit} s)", flush=True)
            os._exit(3)
        time.sleep(0.0005)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--limit-s", type=float, default=10.0)
    ap.add_argument("--random-iters", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    n = args.mib << 20
    out16 = torch.empty(n, dtype=torch.uint16, device=dev)
    out8 = torch.empty(3 * n // 2, dtype=torch.uint8, device=dev)
    profiles = ("latin", "cyrillic", "cjk", "emoji", "ascii")
    rates = (0.0, 1e-7, 1e-6, 1e-5, 1e-3)
    launches = 0
    t0 = time.time()
    for it in range(args.iters):
        prof = profiles[it % len(profiles)]
        rate = rates[(it // len(profiles)) % len(rates)]
        for utf16 in (False, True):
            units = n // 2 if utf16 else n
            buf = corpus.generate(prof, units, 1000 + it, utf16=utf16, device=dev)
            if rate:
                corpus.inject_errors(buf, utf16=utf16, rate=rate, seed=5000 + it)
            direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
            what = f"iter {it} {prof} utf16={utf16} rate={rate}"
            vres = validate_device(direction, buf)
            wait(stream, args.limit_s, "validate " + what)
            vo = outcome_from_tensor(vres.cpu())
            for rep in range(3):
                tres, _ = transcode_device(direction, buf, out8 if utf16 else out16)
                wait(stream, args.limit_s, f"transcode rep {rep} " + what)
                to = outcome_from_tensor(tres.cpu())
                launches += 2
                assert to.consumed == vo.consumed and to.status == vo.status, (what, to, vo)
            del buf
    # random sizes / misalignment / a single error near a tile or window
    # boundary (8 KiB tiles, 128-tile scanner windows = 1 MiB)
    import random

    rng = random.Random(args.seed)
    bases8 = [corpus.generate(p, n + 64, 77, device=dev) for p in ("mix", "ascii")]
    bases16 = [corpus.generate(p, n // 2 + 64, 78, utf16=True, device=dev) for p in ("mix", "ascii")]
    for it in range(args.random_iters):
        utf16 = bool(it & 1)
        base8, base16 = bases8[(it >> 1) & 1], bases16[(it >> 1) & 1]
        units = rng.choice([1, 7, 100, 4096, 65536, 1 << 20, (1 << 20) + 3, rng.randrange(1, n // 2 if utf16 else n)])
        lead = rng.randrange(0, 16)
        # a view at an odd offset: misaligned input pointers (the kernels
        # address a 16-byte aligned frame with a lead offset)
        if utf16:
            buf = base16[2 * lead: 2 * (lead + units)]
        else:
            buf = base8[lead: lead + units]
        # buf itself is valid only if the cut is on character boundaries;
        # either way the kernels must finish and agree with the validator
        restore = None
        if rng.random() < 0.7 and units > 16:
            tile_units = 8192 // (2 if utf16 else 1)
            k = rng.randrange(0, max(1, units // tile_units))
            pos = min(units - 1, max(0, k * tile_units + rng.randrange(-3, 4)))
            if utf16:
                restore = (buf.view(torch.int16), pos, buf.view(torch.int16)[pos].clone())
                buf.view(torch.int16)[pos] = torch.tensor(0xDC00 - 65536, dtype=torch.int16)
            else:
                restore = (buf, pos, buf[pos].clone())
                buf[pos] = 0xFF
        direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
        what = f"random iter {it} units={units} lead={lead} utf16={utf16}"
        vres = validate_device(direction, buf)
        wait(stream, args.limit_s, "validate " + what)
        vo = outcome_from_tensor(vres.cpu())
        tres, _ = transcode_device(direction, buf)
        wait(stream, args.limit_s, "transcode " + what)
        to = outcome_from_tensor(tres.cpu())
        launches += 2
        assert to.consumed == vo.consumed and to.status == vo.status, (what, to, vo)
        if restore is not None:
            restore[0][restore[1]] = restore[2]
    print(f"stress ok: {launches} launches in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
