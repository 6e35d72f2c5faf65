"""Pinned host<->device copy bandwidth on the box (bounds the e2e number).
    python tools/pcie_probe.py"""
import json
import torch

def timed(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
h_in.fill_(1)
res = {}
res["h2d_gbs"] = n / timed(lambda: d_a.copy_(h_in, non_blocking=True)) / 1e9
res["d2h_gbs"] = n / timed(lambda: h_out.copy_(d_b, non_blocking=True)) / 1e9
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
res["duplex_each_gbs"] = n / timed(both) / 1e9
# chunked (64 MiB) H2D as the host pipeline does
def chunked():
    c = 64 << 20
    for o in range(0, n, c):
        d_a[o:o + c].copy_(h_in[o:o + c], non_blocking=True)
res["h2d_64MiB_chunks_gbs"] = n / timed(chunked) / 1e9
print(json.dumps(res))
