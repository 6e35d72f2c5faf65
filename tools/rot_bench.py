"""Per-launch K1 time: same buffers repeated vs rotating buffer sets (TLB /
locality check for bench.py's config-2 step).  usage: python tools/rot_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05098_b200 import UTF8_TO_UTF16, _native, corpus, transcode_device  # noqa: E402

N = 256 << 20
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)


def mk(p, s):
    src = corpus.generate(p, N, s, device=dev)
    out = torch.empty(N, dtype=torch.uint16, device=dev)
    res = torch.empty(3, dtype=torch.int64, device=dev)
    ws = torch.empty(_native.workspace_bytes(0, N) // 8 + 1, dtype=torch.int64, device=dev)
    return src, out, res, ws


def run(sets, reps, events):
    for _ in range(3):
        for s in sets:
            transcode_device(UTF8_TO_UTF16, s[0], s[1], res=s[2], ws=s[3], stream=stream)
    torch.cuda.synchronize()
    evs = []
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        for s in sets:
            if events:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            transcode_device(UTF8_TO_UTF16, s[0], s[1], res=s[2], ws=s[3], stream=stream)
            if events:
                e1.record(stream)
                evs.append((e0, e1))
    b.record(stream)
    torch.cuda.synchronize()
    tot = a.elapsed_time(b) * 1e3 / (reps * len(sets))
    per = sum(x.elapsed_time(y) for x, y in evs) * 1e3 / len(evs) if evs else 0
    return round(tot, 1), round(per, 1)


lat = [mk("latin", 1 + 10 * k) for k in range(4)]
print("latin same x20        ", run(lat[:1], 20, False), run(lat[:1], 20, True))
print("latin rotate 4 sets   ", run(lat, 5, False), run(lat, 5, True))
del lat
torch.cuda.empty_cache()
mix = [mk(p, s) for p, s in (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4))]
print("4 profiles rotate     ", run(mix, 5, False), run(mix, 5, True))
for i, p in enumerate(("latin", "cyrillic", "cjk", "emoji")):
    print(f"{p:9s} same x20      ", run(mix[i:i + 1], 20, False))
names = ("latin", "cyrillic", "cjk", "emoji")
import itertools
for order in ((0, 1, 2, 3), (0, 2, 1, 3), (3, 2, 1, 0), (0, 3, 1, 2), (0, 1, 2), (1, 2, 3), (0, 0, 1, 1, 2, 2, 3, 3)):
    sets = [mix[i] for i in order]
    print("rotate", "/".join(names[i] for i in order), run(sets, 8, False)[0])
