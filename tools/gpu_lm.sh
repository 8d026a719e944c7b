#!/bin/bash
set -u
O=gpurun_out/${1:-lm}; mkdir -p $O
for mode in "" "--pairx"; do
  timeout 120 python tools/lmbench.py --rows 16384 --reps 3 $mode >> $O/lmbench.log 2>&1; echo "mode=$mode rc=$?" >> $O/lmbench.log
done
