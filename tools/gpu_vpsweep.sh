#!/bin/bash
set -u
O=gpurun_out/${1:-vps}; mkdir -p $O
for P in 8 4; do for rs in 0 1; do for pub in 0 1 2; do
  echo "P=$P rs=$rs pub=$pub $(timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 --peer --rs $rs --pub $pub 2>&1 | grep shard)" >> $O/sweep.log
done; done; done
