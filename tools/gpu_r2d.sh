#!/bin/bash
set -u
O=gpurun_out/r2d; mkdir -p $O
echo "== vpbench" > $O/vpbench.log
for P in 8 4; do
  for mode in "--peer" "--peer --ring"; do
    timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 $mode >> $O/vpbench.log 2>&1; echo "P=$P $mode rc=$?" >> $O/vpbench.log
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -s -k "lmhead_loss_bwd or vocab_parallel or alternate or full_chain" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_cache -s 1 -c 1 -o $O/prof_vpcache8 \
  python tools/vpbench.py --P 8 --rows 65536 --reps 2 --peer > $O/ncu8.log 2>&1; echo "ncu rc=$?" >> $O/ncu8.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_cache -s 1 -c 1 -o $O/prof_vpcache4 \
  python tools/vpbench.py --P 4 --rows 65536 --reps 2 --peer > $O/ncu4.log 2>&1; echo "ncu rc=$?" >> $O/ncu4.log
