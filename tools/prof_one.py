"""ncu driver: one kernel on one profile.  python tools/prof_one.py k1|k2|k3|k4 PROFILE [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, outcome_from_tensor  # noqa: E402
from paper_2212_05098_b200 import transcode_device, validate_device  # noqa: E402

SEEDS = {"latin": 1, "cyrillic": 2, "cjk": 3, "emoji": 4, "ascii": 5}
N = 256 << 20
k, p = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda", 0)
utf16 = k in ("k2", "k4")
src = corpus.generate(p, N // 2 if utf16 else N, SEEDS[p], utf16=utf16, device=dev)
out = torch.empty(3 * N // 2 if utf16 else N, dtype=torch.uint8 if utf16 else torch.uint16, device=dev)
res = torch.empty(3, dtype=torch.int64, device=dev)
d = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
for _ in range(reps):
    if k in ("k1", "k2"):
        transcode_device(d, src, out, res=res)
    else:
        validate_device(d, src, res=res)
    torch.cuda.synchronize()
    assert outcome_from_tensor(res.cpu()).ok
print("ok")
