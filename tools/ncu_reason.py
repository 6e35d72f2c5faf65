"""Top SASS instructions of one launch for one stall reason (with the
preceding instructions for context).
usage: python tools/ncu_reason.py REPORT LAUNCH REASON [top]   (REASON e.g. short_sb, wait, barrier)"""
import csv
import subprocess
import sys

rep, launch, reason = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 12
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", launch, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
col = hdr.index("stall_" + reason)
seen, ins = set(), []
for r in rows:
    if not r or not r[0].startswith("0x") or r[0] in seen:
        continue
    seen.add(r[0])
    ins.append(r)
tot = sum(int(r[col] or 0) for r in ins)
print(f"{reason}: {tot} samples")
order = sorted(range(len(ins)), key=lambda i: -int(ins[i][col] or 0))
for i in order[:top]:
    print(f"--- {100 * int(ins[i][col]) / max(tot, 1):5.1f}%")
    for q in ins[max(0, i - 3): i + 1]:
        print(f"   {q[0][-5:]} {q[col]:>6} {q[1][:80]}")
