"""K1 time per launch vs input size (latin, 1 MiB .. 1 GiB) and a torch
zero_ of the workspace: the fixed per-launch cost is the intercept.
usage: python tools/size_sweep.py"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2212_05098_b200 import UTF8_TO_UTF16, _native, corpus, transcode_device
dev = torch.device("cuda", 0)
big = corpus.generate("latin", 1024 << 20, 1, device=dev)
out = torch.empty(1024 << 20, dtype=torch.uint16, device=dev)
res = torch.empty(3, dtype=torch.int64, device=dev)
ws = torch.empty(_native.workspace_bytes(0, 1024 << 20) // 8 + 1, dtype=torch.int64, device=dev)
for mib in (1, 4, 16, 64, 128, 256, 512, 1024):
    n = mib << 20
    src = big[:n]
    for _ in range(3):
        transcode_device(UTF8_TO_UTF16, src, out, res=res, ws=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        transcode_device(UTF8_TO_UTF16, src, out, res=res, ws=ws)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps * 1e3
    # memset alone
    a.record()
    for _ in range(reps):
        ws[: _native.workspace_bytes(0, n) // 8].zero_()
    b.record(); torch.cuda.synchronize()
    tm = a.elapsed_time(b) / reps * 1e3
    print(f"{mib:5d} MiB  {t:8.1f} us  {n / t / 1e3 / 1.073741824:7.1f} GiB/s   zero_ {tm:5.1f} us", flush=True)
