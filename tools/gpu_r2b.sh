#!/bin/bash
set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for P in 8 4; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_ring -s 1 -c 1 -o $O/prof_vpring$P \
  python tools/vpbench.py --P $P --rows 65536 --reps 2 --peer > $O/ncu_vpring$P.log 2>&1; echo "ncu P=$P rc=$?" >> $O/ncu_vpring$P.log
done
