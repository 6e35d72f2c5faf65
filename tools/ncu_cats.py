"""Instructions per 512-byte warp round of one launch of an ncu report, by
source region (file + line range).  usage: python tools/ncu_cats.py REPORT LAUNCH [MiB]"""
import collections
import csv
import subprocess
import sys

rep, launch = sys.argv[1], sys.argv[2]
mib = float(sys.argv[3]) if len(sys.argv) > 3 else 256
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", launch, "--launch-count", "1"], capture_output=True, text=True).stdout
per = collections.Counter()
cur = None
for r in csv.reader(txt.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r or not r[0].isdigit():
        continue
    try:
        per[(cur, int(r[0]))] += int(r[7] or 0)
    except (ValueError, IndexError):
        pass
rounds = mib * (1 << 20) / 512
CATS = [
    ("u8 general detect", "lu_utf8.cuh", 136, 242), ("u8 fast detect", "lu_utf8.cuh", 242, 381),
    ("u8 decode", "lu_utf8.cuh", 381, 459), ("u8 round tail", "lu_utf8.cuh", 459, 624),
    ("u8u16 warp", "lu_utf8.cuh", 624, 693), ("u8 validate", "lu_utf8.cuh", 693, 9999),
    ("u8 other", "lu_utf8.cuh", 0, 136), ("utf16", "lu_utf16.cuh", 0, 9999),
    ("copy-out", "lu_kernels.cu", 30, 150), ("pipeline", "lu_kernels.cu", 150, 430),
    ("validator loop", "lu_kernels.cu", 430, 620), ("common", "lu_common.cuh", 0, 9999),
]
tot = sum(per.values())
print(f"total {tot / rounds:.1f} warp-instr per 512 B round")
seen = set()
for name, f, a, b in CATS:
    keys = [k for k in per if k[0] == f and a <= k[1] < b]
    seen.update(keys)
    print(f"  {name:20s} {sum(per[k] for k in keys) / rounds:7.1f}")
rest = {k: v for k, v in per.items() if k not in seen}
print(f"  {'other':20s} {sum(rest.values()) / rounds:7.1f}", [(k, round(v / rounds, 1)) for k, v in collections.Counter(rest).most_common(4)])
