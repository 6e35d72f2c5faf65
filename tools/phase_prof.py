"""Phase breakdown of the pipelined transcode kernels (instrumented build).

    make -C paper_2212_05098_b200 prof && python tools/phase_prof.py

Loads liblaneutf_b200_prof.so (built with -DLU_PROF) in place of the shipped
library and prints, per profile, the average SM cycles per warp-iteration
spent in each phase of k_transcode (resolve is warp 0 only, so it is shown
per group-iteration).  Instrumentation perturbs timing; use for shares.
"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2212_05098_b200 import _native  # noqa: E402

_native.LIB_PATH = os.path.join(ROOT, "paper_2212_05098_b200", "liblaneutf_b200_prof.so")
from paper_2212_05098_b200 import UTF8_TO_UTF16, UTF16_TO_UTF8, corpus, transcode_device  # noqa: E402

PHASES = ["resolve(w0)", "prefix bar", "copy-out", "claim bar", "compute", "done bar", "iters", "combine",
          "", "spins", "spun resolves"]


def main():
    L = _native.lib()
    L.lu_prof_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 48)()
    dev = torch.device("cuda", 0)
    n = 256 << 20
    for utf16 in (False, True):
        for p, seed in (("latin", 1), ("cyrillic", 2), ("cjk", 3), ("emoji", 4), ("ascii", 5)):
            src = corpus.generate(p, n // (2 if utf16 else 1), seed, utf16=utf16, device=dev)
            direction = UTF16_TO_UTF8 if utf16 else UTF8_TO_UTF16
            for _ in range(3):
                transcode_device(direction, src)
            torch.cuda.synchronize()
            L.lu_prof_read(buf, 1)
            reps = 5
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(reps):
                transcode_device(direction, src)
            ev[1].record()
            torch.cuda.synchronize()
            L.lu_prof_read(buf, 1)
            v = list(buf)
            w0, wo = v[:24], v[24:]
            line = f"{'K2' if utf16 else 'K1'} {p:9s} {ev[0].elapsed_time(ev[1]) * 1e3 / reps:7.1f} us"
            for name, c in (("warp0", w0), ("warps1-3", wo)):
                it = max(c[6], 1)
                line += f"\n   {name:8s} iters {it // reps:6d} cycles/iter: " + "  ".join(
                    f"{PHASES[k]} {c[k] / it:6.0f}" for k in (0, 1, 2, 3, 4, 5, 7))
            line += (f"\n   scanner: {w0[11] // reps} passes/launch, {w0[12] / max(w0[11], 1):.1f} tiles/pass, "
                     f"{100 * w0[13] / max(w0[11], 1):.1f}% empty, {100 * w0[14] / max(w0[11], 1):.1f}% full, "
                     f"cycles/pass: issue {w0[16] / max(w0[11], 1):.0f} load-wait {w0[17] / max(w0[11], 1):.0f} "
                     f"process {w0[18] / max(w0[11] - w0[13], 1):.0f} (per non-empty pass) empty {w0[19] / max(w0[13], 1):.0f}")
            line += f"\n   warp0 split: resolve {w0[12] / max(w0[6], 1):.0f}  ticket wait {w0[13] / max(w0[6], 1):.0f}"
            line += f"\n   resolves that spun {100 * w0[10] / max(w0[6], 1):.1f}%, {w0[9] / max(w0[10], 1):.1f} spins each"
            print(line)

if __name__ == "__main__":
    main()
