#!/bin/bash
set -u
O=gpurun_out/${1:-vps}; mkdir -p $O
for g in 1 2 4 8; do for r in "" "--rows4"; do
  echo "groups=$g $r" >> $O/sweep.log
  timeout 120 python tools/vpbench.py --P 8 --rows 65536 --reps 10 --peer --groups $g $r 2>&1 | grep shard >> $O/sweep.log
done; done
