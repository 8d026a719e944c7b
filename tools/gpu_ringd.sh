#!/bin/bash
# vp_ring_kernel L2 window: D sweep at the P = 2 / 4 widths (one GPU), ncu of the default at P = 2
set -u
O=gpurun_out/${1:-ringd}; mkdir -p $O
for P in 2 4; do for dl in 0 1 2 3; do
  echo "P=$P delay=$dl $(timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 --peer --ring --delay $dl 2>&1 | tail -1)" >> $O/sweep.log
done; done
cat $O/sweep.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_ring -s 1 -c 1 -o $O/prof_ring2 \
    python tools/vpbench.py --P 2 --rows 65536 --reps 2 --peer --ring > $O/ncu2.log 2>&1; echo "ncu rc=$?"
