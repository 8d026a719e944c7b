#!/bin/bash
# ncu --set full of vp_ring_kernel at the P = 4 and P = 2 shard widths (one rank's share, one GPU)
set -u
O=gpurun_out/${1:-ringprof}; mkdir -p $O
for P in 4 2; do
  timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 --peer --ring > $O/time$P.log 2>&1
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_ring -s 1 -c 1 -o $O/prof_ring$P \
    python tools/vpbench.py --P $P --rows 65536 --reps 2 --peer --ring > $O/ncu$P.log 2>&1; echo "ncu rc=$?" >> $O/ncu$P.log
done
