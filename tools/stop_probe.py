import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2212_05098_b200 import UTF8_TO_UTF16, corpus, outcome_from_tensor, validate_device
dev = torch.device("cuda", 0)
n = 256 << 20
src = corpus.generate("cjk", n, 3, device=dev)
res = torch.empty(3, dtype=torch.int64, device=dev)
def timeit(buf, reps=20):
    for _ in range(3): validate_device(UTF8_TO_UTF16, buf, res=res)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): validate_device(UTF8_TO_UTF16, buf, res=res)
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps * 1e3, 1)
print("valid", timeit(src))
for frac in [float(a) for a in sys.argv[1:]] or (0.0001, 0.01, 0.1, 0.5, 0.9):
    b = src.clone()
    p = int(n * frac)
    b[p] = 0xFF
    t = timeit(b)
    o = outcome_from_tensor(res.cpu())
    print("single error at", frac, t, "us", o.consumed == p)
