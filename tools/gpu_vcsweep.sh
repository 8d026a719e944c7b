#!/bin/bash
# vp_cache_kernel at the P = 8 width: parked rows (RS) x collector groups, one GPU
set -u
O=gpurun_out/${1:-vcsweep}; mkdir -p $O
for rs in 0 1 2; do for g in 0 2; do
  echo "rs=$rs groups=$g $(timeout 120 python tools/vpbench.py --P 8 --rows 65536 --reps 10 --peer --rs $rs --groups $g 2>&1 | tail -1)" >> $O/sweep.log
done; done
cat $O/sweep.log
