#!/bin/bash
# ncu --set full (with source) of vp_cache_kernel at the P = 8 / 4 widths, one GPU
set -u
O=gpurun_out/${1:-vcprof}; mkdir -p $O
for P in 8 4; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_cache -s 1 -c 1 -o $O/prof_vpcache$P \
    python tools/vpbench.py --P $P --rows 65536 --reps 2 --peer > $O/ncu$P.log 2>&1; echo "ncu $P rc=$?"
done
