"""Summarise tools/exp_run.sh output: best us per kernel/profile per variant."""
import json
import sys

cur = None
res = {}
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.split()[1]
        continue
    if line.startswith("{"):
        for k, v in json.loads(line).items():
            res.setdefault(k, {}).setdefault(cur, []).append(v["us"])
for k, v in res.items():
    print(f"{k:22s}", "  ".join(f"{n}:{min(x):7.1f}" for n, x in v.items()))
