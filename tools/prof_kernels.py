"""Small driver for ncu captures: each kernel on each profile, few launches.

    python tools/prof_kernels.py [--reps R]

Launch order per rep: K1 (utf8->utf16) on latin, cyrillic, cjk, emoji;
K2 (utf16->utf8) on the same four; K3 (validate utf8, cjk); K4 (validate
utf16, emoji).  Prints per-launch CUDA-event times (not for reporting under
ncu).
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, outcome_from_tensor  # noqa: E402
from paper_2212_05098_b200 import transcode_device, validate_device  # noqa: E402

PROFILES = (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4))
N = 256 << 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    u8 = [corpus.generate(p, N, s, device=dev) for p, s in PROFILES]
    u16 = [corpus.generate(p, N // 2, s, utf16=True, device=dev) for p, s in PROFILES]
    out16 = torch.empty(N, dtype=torch.uint16, device=dev)
    out8 = torch.empty(3 * N // 2, dtype=torch.uint8, device=dev)
    res = torch.empty(3, dtype=torch.int64, device=dev)
    times = {}
    for rep in range(args.reps):
        for (p, _), b in zip(PROFILES, u8):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); transcode_device(UTF8_TO_UTF16, b, out16, res=res); e.record()
            torch.cuda.synchronize()
            times[f"k1_{p}"] = a.elapsed_time(e)
            assert outcome_from_tensor(res.cpu()).ok
        for (p, _), b in zip(PROFILES, u16):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); transcode_device(UTF16_TO_UTF8, b, out8, res=res); e.record()
            torch.cuda.synchronize()
            times[f"k2_{p}"] = a.elapsed_time(e)
            assert outcome_from_tensor(res.cpu()).ok
        for name, d, b in (("k3_cjk", UTF8_TO_UTF16, u8[2]), ("k4_emoji", UTF16_TO_UTF8, u16[3])):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); validate_device(d, b, res=res); e.record()
            torch.cuda.synchronize()
            times[name] = a.elapsed_time(e)
            assert outcome_from_tensor(res.cpu()).ok
    print(json.dumps({k: round(v, 4) for k, v in times.items()}))


if __name__ == "__main__":
    main()
