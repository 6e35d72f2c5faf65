"""Small-input latency of K1/K2 (config 1 is a 4 MiB round trip): time per
launch vs size, and the config-1 round trip, CUDA events, back-to-back.
usage: python tools/latency_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, _native, corpus, outcome_from_tensor, transcode_device  # noqa

dev = torch.device("cuda", 0)
rep = {}


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps * 1e3, 2)


mix = corpus.generate("mix", 16 << 20, 0, device=dev)
out16 = torch.empty(16 << 20, dtype=torch.uint16, device=dev)
res = torch.empty(3, dtype=torch.int64, device=dev)
ws = torch.empty(_native.workspace_bytes(0, 16 << 20) // 8 + 1, dtype=torch.int64, device=dev)
for kib in (64, 256, 1024, 4096, 16384):
    n = kib << 10
    rep[f"k1_{kib}KiB_us"] = timeit(lambda: transcode_device(UTF8_TO_UTF16, mix[:n], out16, res=res, ws=ws))
c1 = corpus.generate("mix", 4 << 20, 0, device=dev)
r1, w1 = transcode_device(UTF8_TO_UTF16, c1)
o1 = outcome_from_tensor(r1.cpu())
words = w1[: o1.written]
out8 = torch.empty(3 * o1.written, dtype=torch.uint8, device=dev)
rep["k1_config1_us"] = timeit(lambda: transcode_device(UTF8_TO_UTF16, c1, w1, res=res, ws=ws))
rep["k2_config1_us"] = timeit(lambda: transcode_device(UTF16_TO_UTF8, words, out8, res=res, ws=ws))
rep["round_trip_us"] = timeit(lambda: (transcode_device(UTF8_TO_UTF16, c1, w1, res=res, ws=ws),
                                       transcode_device(UTF16_TO_UTF8, words, out8, res=res, ws=ws)))
rep["memset_ws_us"] = timeit(lambda: ws[: _native.workspace_bytes(0, 4 << 20) // 8].zero_())
rep["empty_k1_us"] = timeit(lambda: transcode_device(UTF8_TO_UTF16, c1[:0], w1, res=res, ws=ws))
print(json.dumps(rep))

# host-side cost per call (no synchronisation inside the loop)
import time  # noqa: E402

for name, fn in (("host_transcode_device_us", lambda: transcode_device(UTF8_TO_UTF16, c1, w1, res=res, ws=ws)),
                 ("host_native_launch_us", lambda: _native.launch(_native.OP_UTF8_TO_UTF16LE, c1, c1.numel(), w1,
                                                                  w1.numel(), ws, res))):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, round((t1 - t0) / 200 * 1e6, 2))
