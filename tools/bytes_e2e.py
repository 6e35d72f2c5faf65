"""bytes in / bytearray out through the facade (the reference callers' types):
GiB/s of the config-2 step, best of N.  usage: python tools/bytes_e2e.py [N]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05098_b200 import UTF8_TO_UTF16, corpus, transcode  # noqa: E402

N = 256 << 20
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
blobs = [corpus.generate(p, N, s).numpy().tobytes() for p, s in (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4))]
outs = [bytearray(2 * N) for _ in blobs]
best = 1e9
for _ in range(reps + 1):
    t0 = time.perf_counter()
    got = [transcode(UTF8_TO_UTF16, b, o, engine="native") for b, o in zip(blobs, outs)]
    best = min(best, time.perf_counter() - t0)
    assert all(g.ok for g in got)
print({"bytes_api_gib_s": round(4 * N / 2**30 / best, 2), "written": [g.written for g in got]})
