"""e2e (pinned host in/out, and bytes -> bytearray) throughput of the
config-2 step vs host-pipeline chunk size and ring depth.
usage: python tools/e2e_chunks.py [MiB list] [slots list]"""
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
blobs = [h.numpy().tobytes() for h in hosts]
bouts = [bytearray(2 * N) for _ in hosts]
mibs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,32,64").split(",")]
slots = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "3,4,6").split(",")]
for sl in slots:
    for mib in mibs:
        ch = mib << 20
        for name, srcs, dsts in (("pinned", hosts, outs), ("bytes", blobs, bouts)):
            for h, o in zip(srcs, dsts):
                hostpipe.stream_transcode(True, h, o, chunk_bytes=ch, slots=sl)
            torch.cuda.synchronize()
            best = 0.0
            for rep in range(3):
                t0 = time.perf_counter()
                for h, o in zip(srcs, dsts):
                    hostpipe.stream_transcode(True, h, o, chunk_bytes=ch, slots=sl)
                dt = time.perf_counter() - t0
                best = max(best, 4 * N / dt / 2**30)
            print(f"slots {sl} chunk {mib:4d} MiB {name:6s}: {best:6.2f} GiB/s", flush=True)
