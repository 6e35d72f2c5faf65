import sys
for l in sys.stdin:
    if l.startswith(('k1_','k2_')): print(l.rstrip())
