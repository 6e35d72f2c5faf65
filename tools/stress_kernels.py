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
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    n = args.mib << 20
    out16 = torch.empty(n, dtype=torch.uint16, device=dev)
    out8 = torch.empty(3 * n // 2, dtype=torch.uint8, device=dev)
    profiles = ("latin", "cyrillic", "cjk", "emoji")
    rates = (0.0, 1e-7, 1e-6, 1e-5, 1e-3)
    launches = 0
    t0 = time.time()
    for it in range(args.iters):
        prof = profiles[it % 4]
        rate = rates[(it // 4) % len(rates)]
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
    print(f"stress ok: {launches} launches in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
