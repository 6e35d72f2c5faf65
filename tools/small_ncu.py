import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2212_05098_b200 import UTF8_TO_UTF16, _native, corpus, transcode_device
dev = torch.device("cuda", 0)
c1 = corpus.generate("mix", 4 << 20, 0, device=dev)
w1 = torch.empty(4 << 20, dtype=torch.uint16, device=dev)
res = torch.empty(3, dtype=torch.int64, device=dev)
ws = torch.empty(_native.workspace_bytes(0, 4 << 20) // 8 + 1, dtype=torch.int64, device=dev)
for n in (0, 64 << 10, 4 << 20):
    for _ in range(3):
        transcode_device(UTF8_TO_UTF16, c1[:n], w1, res=res, ws=ws)
torch.cuda.synchronize()
