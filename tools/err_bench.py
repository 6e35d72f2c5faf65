"""Config-4 transcode/validate timings on error-injected 256 MiB buffers
(errors at 1e-6 per unit, seeds 101/102) and on the zero-error controls.

    python tools/err_bench.py [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, outcome_from_tensor  # noqa: E402
from paper_2212_05098_b200 import transcode_device, validate_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 256 << 20

    def timeit(fn):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return round(a.elapsed_time(b) / args.reps * 1e3, 1)

    rep = {}
    for name, direction, utf16, prof, seed in (("cjk_utf8", UTF8_TO_UTF16, False, "cjk", 3),
                                               ("emoji_utf16", UTF16_TO_UTF8, True, "emoji", 4)):
        units = n // 2 if utf16 else n
        buf = corpus.generate(prof, units, seed, utf16=utf16, device=dev)
        out = torch.empty(3 * units if utf16 else units, dtype=torch.uint8 if utf16 else torch.uint16, device=dev)
        res = torch.empty(3, dtype=torch.int64, device=dev)
        ctl_t = timeit(lambda: transcode_device(direction, buf, out, res=res))
        corpus.inject_errors(buf, utf16=utf16, rate=1e-6, seed=101 + int(utf16))
        err_t = timeit(lambda: transcode_device(direction, buf, out, res=res))
        o = outcome_from_tensor(res.cpu())
        err_v = timeit(lambda: validate_device(direction, buf, res=res))
        rep[name] = {"control_transcode_us": ctl_t, "errors_transcode_us": err_t, "errors_validate_us": err_v,
                     "first_error": o.consumed}
    print(json.dumps(rep))


if __name__ == "__main__":
    main()
