"""Quick per-kernel throughput check (back-to-back launches, CUDA events).

    python tools/kbench.py [--reps 20] [--mib 256]

Prints one JSON object: per kernel/profile average microseconds per call and
input GiB/s, plus the algorithmic-bytes fraction of the measured HBM peak.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, _native, corpus, outcome_from_tensor  # noqa: E402
from paper_2212_05098_b200 import count_device, transcode_device, validate_device  # noqa: E402

PROFILES = (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4), ("ascii", 5), ("mix", 0), ("typo", 6))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    n = args.mib << 20
    dev = torch.device("cuda", 0)
    peak = 6554.6
    res = torch.empty(3, dtype=torch.int64, device=dev)
    out16 = torch.empty(n, dtype=torch.uint16, device=dev)
    out8 = torch.empty(3 * n // 2, dtype=torch.uint8, device=dev)
    ws = torch.empty(_native.workspace_bytes(0, n) // 8 + 1, dtype=torch.int64, device=dev)
    report = {}

    def timeit(fn):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.reps / 1e3

    for p, s in PROFILES:
        if args.only and p not in args.only:
            continue
        u8 = corpus.generate(p, n, s, device=dev)
        t = timeit(lambda: transcode_device(UTF8_TO_UTF16, u8, out16, res=res, ws=ws))
        o = outcome_from_tensor(res.cpu())
        assert o.ok, o
        report[f"k1_{p}"] = {"us": round(t * 1e6, 1), "gib_s": round(n / t / 2**30, 1),
                             "frac": round((n + 2 * o.written) / t / 1e9 / peak, 3)}
        u16 = corpus.generate(p, n // 2, s, utf16=True, device=dev)
        t = timeit(lambda: transcode_device(UTF16_TO_UTF8, u16, out8, res=res, ws=ws))
        o = outcome_from_tensor(res.cpu())
        assert o.ok, o
        report[f"k2_{p}"] = {"us": round(t * 1e6, 1), "gib_s": round(n / t / 2**30, 1),
                             "frac": round((n + o.written) / t / 1e9 / peak, 3)}
        if p in ("cjk", "emoji", "ascii", "mix", "typo"):
            t = timeit(lambda: validate_device(UTF8_TO_UTF16, u8, res=res, ws=ws))
            report[f"k3_{p}"] = {"us": round(t * 1e6, 1), "gib_s": round(n / t / 2**30, 1),
                                 "frac": round(n / t / 1e9 / peak, 3)}
            t = timeit(lambda: validate_device(UTF16_TO_UTF8, u16, res=res, ws=ws))
            report[f"k4_{p}"] = {"us": round(t * 1e6, 1), "gib_s": round(n / t / 2**30, 1),
                                 "frac": round(n / t / 1e9 / peak, 3)}
            for name, op, src in (("len_u8", _native.OP_UTF16_LENGTH_FROM_UTF8, u8),
                                  ("len_u16", _native.OP_UTF8_LENGTH_FROM_UTF16LE, u16),
                                  ("chars_u8", _native.OP_UTF8_CHAR_COUNT, u8),
                                  ("chars_u16", _native.OP_UTF16LE_CHAR_COUNT, u16)):
                t = timeit(lambda: count_device(op, src))
                report[f"{name}_{p}"] = {"us": round(t * 1e6, 1), "gib_s": round(n / t / 2**30, 1),
                                         "frac": round(n / t / 1e9 / peak, 3)}
        del u8, u16
    print(json.dumps(report))


if __name__ == "__main__":
    main()
