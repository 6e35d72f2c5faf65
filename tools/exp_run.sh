#!/bin/bash
# A/B kernel variants on the GPU box: exp/lib_<name>.so is copied over the
# package library in turn and tools/kbench.py is run for each (twice, interleaved).
# usage: bash tools/exp_run.sh name1 name2 ...
L=paper_2212_05098_b200/liblaneutf_b200.so
cp $L /tmp/lib_keep.so
for pass in 1 2; do
  for v in "$@"; do
    cp exp/lib_$v.so $L
    echo "== $v pass $pass"
    timeout 300 python tools/kbench.py --reps 20 $KB_ARGS
  done
done
cp /tmp/lib_keep.so $L
