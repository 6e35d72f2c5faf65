"""Small end-to-end case for compute-sanitizer runs (one tool per call):
K1/K2/K3/K4, counts, batch and BE on ~1 MiB with errors near tile edges."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_05098_b200 as lu  # noqa: E402
from paper_2212_05098_b200 import corpus  # noqa: E402

dev = torch.device("cuda", 0)
for profile in ("latin", "emoji", "mix"):
    u8 = corpus.generate(profile, (1 << 20) + 37, 7, device=dev)
    for err_at in (None, 8191, 600_001):
        d = u8.clone()
        if err_at is not None:
            d[err_at] = 0xC0
        for lead in (0, 3):
            s = d[lead:]
            r, o = lu.transcode_device(lu.UTF8_TO_UTF16, s)
            r2 = lu.validate_device(lu.UTF8_TO_UTF16, s)
            lu.count_device(lu._native.OP_UTF16_LENGTH_FROM_UTF8, s)
            lu.count_device(lu._native.OP_UTF8_CHAR_COUNT, s)
            lu.transcode_device(lu.UTF8_TO_UTF16, s, utf16_byte_order="be")
    u16 = corpus.generate(profile, (1 << 19) + 11, 8, utf16=True, device=dev)
    for lead in (0, 2):
        s = u16[lead:]
        lu.transcode_device(lu.UTF16_TO_UTF8, s)
        lu.validate_device(lu.UTF16_TO_UTF8, s)
        lu.count_device(lu._native.OP_UTF8_LENGTH_FROM_UTF16LE, s)
        lu.count_device(lu._native.OP_UTF16LE_CHAR_COUNT, s)
# persistent pipeline + ASCII chunk paths (needs more tiles than resident groups)
if len(sys.argv) > 1 and sys.argv[1] == "ascii":
    a8 = corpus.generate("ascii", 10 << 20, 9, device=dev)
    a8[5_000_001] = 0xC3
    a8[5_000_002] = 0xA9
    lu.transcode_device(lu.UTF8_TO_UTF16, a8)
    a16 = corpus.generate("ascii", 5 << 20, 9, utf16=True, device=dev)
    lu.transcode_device(lu.UTF16_TO_UTF8, a16)
cases = [b"abc", b"\xc3\xa9", b"\xe2\x82", "🙂".encode() * 300, b""]
lu.transcode_batch(lu.UTF8_TO_UTF16, cases)
lu.validate_batch(lu.UTF8_TO_UTF16, cases)
torch.cuda.synchronize()
print("sanitize case done")
