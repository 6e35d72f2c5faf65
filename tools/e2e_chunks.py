"""e2e (pinned host in/out) throughput of the config-2 step vs host-pipeline
chunk size.  usage: python tools/e2e_chunks.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05098_b200 import corpus, hostpipe  # noqa: E402

N = 256 << 20
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
hosts = [corpus.generate(p, N, s, device=dev).cpu().pin_memory()
         for p, s in (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4))]
outs = [torch.empty(2 * N, dtype=torch.uint8).pin_memory() for _ in hosts]
for mib in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,32,48,64,96,128,256").split(",")]:
    ch = mib << 20
    for h, o in zip(hosts, outs):
        hostpipe.pipelined_transcode(True, h, o, chunk_bytes=ch)
    torch.cuda.synchronize()
    best = 0.0
    for rep in range(5):
        t0 = time.perf_counter()
        for h, o in zip(hosts, outs):
            hostpipe.pipelined_transcode(True, h, o, chunk_bytes=ch)
        dt = time.perf_counter() - t0
        best = max(best, 4 * N / dt / 2**30)
    print(f"chunk {mib:4d} MiB: {best:6.2f} GiB/s", flush=True)
