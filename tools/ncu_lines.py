"""Summarise an ncu report's source page: instructions per 128-byte step by
source line and SASS opcode.  usage: python tools/ncu_lines.py REPORT [MiB] [top] [launch-index]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
mib = float(sys.argv[2]) if len(sys.argv) > 2 else 256
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
launch = sys.argv[4] if len(sys.argv) > 4 else None  # one launch of the report (default: all merged)
extra = ["--launch-skip", launch, "--launch-count", "1"] if launch is not None else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + extra,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur = None
out = []
ops = collections.Counter()
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Line No", "Function Name"):
        continue
    if r[0] != "":
        try:
            n = int(r[7] or 0)
            st = int(r[4] or 0)
        except (ValueError, IndexError):
            continue
        out.append((n, st, cur, r[0], r[1][:95]))
    elif len(r) > 7 and r[2].startswith("0x"):
        s = r[3].strip().split()
        if not s:
            continue
        o = s[1] if s[0].startswith("@") else s[0]
        try:
            ops[o.split(".")[0]] += int(r[7] or 0)
        except ValueError:
            pass
steps = mib * (1 << 20) / 128
tot = sum(o[0] for o in out)
print(f"total warp-instr {tot}  per 128B step {tot / steps:.1f}")
out.sort(reverse=True)
for o in out[:top]:
    print(f"{o[0] / steps:6.2f}/step st={o[1]:5d} {o[2]}:{o[3]:>4} {o[4]}")
print([(k, round(v / steps, 2)) for k, v in ops.most_common(24)])
