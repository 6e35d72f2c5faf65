"""Stall samples of one kernel in an ncu report, by SASS opcode and by
instruction.  usage: python tools/ncu_stalls.py REPORT [launch-index] [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = None
ops = collections.Counter()
inst = []
total = 0
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    d = dict(zip(hdr, r))
    s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    src = d["Source"].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    ops[op.split(".")[0]] += s
    total += s
    inst.append((s, d["Address"][-5:], src[:70]))
print("total samples", total)
for op, s in ops.most_common(top):
    print(f"  {op:10s} {100 * s / total:5.1f}%")
print("top instructions")
for s, a, src in sorted(inst, reverse=True)[:top]:
    print(f"  {100 * s / total:5.1f}%  {a}  {src}")
